#!/bin/bash
# Run ON the GPU box (gpurun): the bench line, the ncu launch list of a short bench run,
# and one `ncu --set full` capture of each hot kernel at its config -> gpurun_out/.
# Then, locally: python tools/make_profiles.py <tag> gpurun_out/launches.csv name=gpurun_out/<name>.ncu-rep ...
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches_bench.log 2>&1
cap() { name=$1; shift; ncu --set full --clock-control none --import-source on -s 1 -c 1 -o gpurun_out/$name -f \
        python tools/run_one.py "$@" --reps 1 > gpurun_out/$name.log 2>&1; }
cap edm edm --rho 128 --strategy lambda
cap collide collide --rho 256 --strategy lambda
cap collide_tc collide --rho 384 --strategy tc
cap collide1d collide1d --strategy lambda
cap ca ca --rho 128 --strategy lambda
cap ca_multi ca_steps --rho 224 --k 8 --strategy lambda
cap triplet triplet --rho 32 --strategy lambda
cap dummy dummy --rho 16 --strategy lambda
ls -la gpurun_out

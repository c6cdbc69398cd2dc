#!/bin/bash
# Run ON the GPU box (gpurun): the bench line, the ncu launch list of a short bench run,
# and one `ncu --set full` capture of each hot kernel at its config -> gpurun_out/.
# Then, locally: python tools/make_profiles.py <tag> gpurun_out/launches.csv name=gpurun_out/<name>.ncu-rep ...
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/launches_bench.log 2>&1
cap() { name=$1; kre=$2; shift 2; ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 1 -c 1 \
        -o gpurun_out/$name -f python tools/run_one.py "$@" --reps 2 > gpurun_out/$name.log 2>&1; }
cap edm edm_kernel edm --rho 128 --strategy lambda
cap edm_bb edm_kernel edm --rho 128 --strategy bb
cap collide collide_kernel collide --rho 256 --strategy lambda
cap collide_bb collide_kernel collide --rho 256 --strategy bb
cap collide_tc collide_tc_kernel collide --rho 768 --strategy tc
cap collide_tc_bb collide_tc_kernel collide --rho 768 --strategy bb_tc
cap collide1d collide1d_kernel collide1d --strategy lambda
cap collide1d_bb collide1d_kernel collide1d --strategy bb
cap ca ca_multi_kernel ca --rho 128 --strategy lambda
cap ca_multi ca_multi_kernel ca_steps --rho 224 --k 8 --strategy lambda
cap ca_multi_bb ca_multi_kernel ca_steps --rho 224 --k 8 --strategy bb
cap ca_packed ca_packed_kernel ca_run --rho 240 --k 8 --strategy lambda
cap ca_packed_bb ca_packed_kernel ca_run --rho 240 --k 8 --strategy bb
cap triplet triplet32_kernel triplet --rho 32 --strategy lambda
cap triplet_bb triplet32_kernel triplet --rho 32 --strategy bb
cap dummy dummy_kernel dummy --rho 16 --strategy lambda
cap dummy_bb dummy_kernel dummy --rho 16 --strategy bb
ls -la gpurun_out
# condense on the box (the .ncu-rep files exceed what gpurun copies back): summaries into
# gpurun_out/prof, keep the full reports of the two headline kernels only
mkdir -p gpurun_out/prof && cp profiles/ncu_summary.json gpurun_out/prof/ 2>/dev/null
TRI_PROF_DIR=gpurun_out/prof python tools/make_profiles.py "${TAG:-r02}" gpurun_out/launches.csv \
    $(for f in gpurun_out/*.ncu-rep; do b=$(basename $f .ncu-rep); echo "$b=$f"; done) > gpurun_out/prof/make.log 2>&1
for f in gpurun_out/*.ncu-rep; do case $(basename $f) in edm.ncu-rep|collide_tc.ncu-rep|ca_packed.ncu-rep) ;; *) rm -f $f ;; esac; done
du -sh gpurun_out

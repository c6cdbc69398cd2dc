#!/bin/bash
# Run ON the GPU box: ncu launch counters (CTAs, threads, warps, instructions, branch
# divergence) of every production kernel under the lambda grid and the BB grid, at the
# bench's configurations -> gpurun_out/lvb/<name>.csv.  Condense locally with
# python tools/lambda_vs_bb_ncu.py <tag> gpurun_out/lvb
M=gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__ctas_launched.sum,smsp__warps_launched.sum,smsp__threads_launched.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__sass_branch_targets.sum,smsp__sass_branch_targets_threads_divergent.sum,smsp__sass_thread_inst_executed_pred_on.sum
mkdir -p gpurun_out/lvb
run() { name=$1; kre=$2; shift 2; ncu --metrics $M --clock-control none -k "regex:$kre" -s 1 -c 1 --csv \
        --log-file gpurun_out/lvb/$name.csv python tools/run_one.py "$@" --reps 1 > /dev/null 2>&1; }
for s in lambda bb; do
  run dummy_$s dummy_kernel dummy --rho 16 --strategy $s
  run dummy65536_$s dummy_kernel dummy --n 65536 --rho 16 --strategy $s
  run edm_$s edm_kernel edm --rho 128 --strategy $s
  run collide_$s collide_kernel collide --rho 256 --strategy $s
  run collide1d_$s collide1d_kernel collide1d --strategy $s
  run ca_multi_$s ca_multi_kernel ca_steps --rho 224 --k 8 --strategy $s
  run ca_step_$s ca_multi_kernel ca --rho 128 --strategy $s
  run ca_packed_$s ca_packed_kernel ca_run --rho 240 --k 8 --strategy $s
  run triplet_$s triplet32_kernel triplet --rho 32 --strategy $s
done
run collide_tc_lambda collide_tc_kernel collide --rho 768 --strategy tc
run collide_tc_bb collide_tc_kernel collide --rho 768 --strategy bb_tc
ls gpurun_out/lvb

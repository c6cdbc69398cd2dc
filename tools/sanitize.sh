#!/bin/bash
# Run ON the GPU box: compute-sanitizer over the small-size GPU parity tests (the
# full-size and exhaustive ones would take hours under the tools) -> gpurun_out/sanitizer.txt
OUT=gpurun_out/sanitizer.txt; mkdir -p gpurun_out; : > $OUT
SMALL="(map_matches_enumeration or dummy_packed or dummy_ranks or edm_small or edm_dims or edm_ranks or collide_small or collide_quantized or ca_small or ca_ranks or ca_ignores or ca_steps_single or ca_steps_deep or ca_steps_ignores or ca_steps_rho224 or ca_steps_p2p_emulated or ca_steps_p2p_single or ca_run_packed or knife_edge or collide_tc_small or triplet_small or triplet_ranks or collide1d or tet_lut_map_matches or abi_rejects)"
run() { tool=$1; sel=$2; echo "== compute-sanitizer --tool $tool, pytest -k \"$sel\"" >> $OUT
  compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$sel" 2>&1 | \
    grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Hazard|error" | tail -8 >> $OUT; }
run memcheck "$SMALL and not lambda_r"
RACE="((((ca_steps_single or ca_steps_rho224) and 1000) or (ca_small and 1000) or (triplet_small and 61) or (collide_small and 1000) or (edm_small and 4097) or (ca_run_packed and 2049)) and lambda and not lambda_) or (edm_dims and 256) or (collide_knife_edge and 0.0-1.0) or (collide1d_knife_edge and 0.0-1.0)"
run racecheck "$RACE"
run synccheck "$RACE"
echo "== probe (tools/sanitizer_probe.py: tri_dummy told a 4 KB buffer holds 1 GB) -- proves the" >> $OUT
echo "== sanitizer instruments libtri.so loaded through ctypes:" >> $OUT
compute-sanitizer --tool memcheck --print-limit 2 python tools/sanitizer_probe.py 2>&1 | grep -E "Invalid|Device Frame" | head -2 >> $OUT
cat $OUT
# round 2: the tcgen05 collision kernel (TF32 operand prep, bulk copies, one MMA per block,
# early accumulator hand-back) on both grids, every tile edge, special values
echo "== compute-sanitizer on collide_tc_prep + collide_tc_kernel (TRI_LAMBDA_TC / TRI_BB_TC, rho 256..1024)" >> $OUT
for tool in memcheck racecheck synccheck; do
  if [ $tool = memcheck ]; then sel="collide_tc_small or collide_tc_knife_edge or collide_tc_special or collide_tc_dense or collide_tc_plain"
  else sel="collide_tc_small and 1000-42"; fi
  echo "== $tool: -k \"$sel\"" >> $OUT
  compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py -q -x -p no:cacheprovider -k "$sel" 2>&1 | \
    grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Hazard|error" | tail -6 >> $OUT
done
cat $OUT

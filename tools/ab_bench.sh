#!/bin/bash
# A/B the bench's headline EDM line across alternative builds of libtri.so:
# tools/ab_bench.sh <lib>... (runs python bench.py --only-edm --no-e2e --no-cpu per lib, twice)
cp paper_1609_01490_b200/libtri.so /tmp/libtri_orig.so
for rep in 1 2; do for l in "$@"; do cp "$l" paper_1609_01490_b200/libtri.so
  python bench.py --only-edm --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$l', d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['power_w_max'], d['vs_bb'].get('lambda_ms'))"
done; done
cp /tmp/libtri_orig.so paper_1609_01490_b200/libtri.so

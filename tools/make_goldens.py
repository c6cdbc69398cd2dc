#!/usr/bin/env python
"""Write tests/golden/fullsize.txt: the CPU oracle's results at the BASELINE full sizes,
on the seeded inputs bench.py times.  Calls only oracle/ (and the seeded input
generators, which hold none of the method's arithmetic) -- never the CUDA path.

    python tools/make_goldens.py            # ~2-4 min on 8 host cores

Rows (key value):
  collide_n200000_seed42_r0.01           pair count  (config 3, reading Q9)
  collide1d_n200000_seed42_r1e-5         pair count  (reading Q10)
  ca_n32768_seed42_g{G}_sha256 / _alive  state after G generations (config 4, reading Q11)
  triplet_n4096_seed42_total / _abs      sum_t e_t and sum |E| over all triplets (config 5, reading Q15)
"""
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1609_01490_b200 import inputs  # noqa: E402


def main():
    rows = []
    t0 = time.time()
    rows.append(("collide_n200000_seed42_r0.01", oracle.collide(inputs.spheres(200000, 42, 0.01))))
    rows.append(("collide1d_n200000_seed42_r1e-5", oracle.collide1d(inputs.intervals(200000, 42, 1e-5))))
    print(f"collisions {time.time() - t0:.1f} s", file=sys.stderr)
    n = 32768
    st = inputs.ca_state(n, 42)
    done = 0
    for g in (1, 8, 100):
        st = oracle.ca_run(n, st, g - done)
        done = g
        rows.append((f"ca_n32768_seed42_g{g}_sha256", hashlib.sha256(st.tobytes()).hexdigest()))
        rows.append((f"ca_n32768_seed42_g{g}_alive", int(st.sum(dtype=np.int64))))
    print(f"ca {time.time() - t0:.1f} s", file=sys.stderr)
    x = inputs.points4(4096, 42)
    e = oracle.triplet(x)
    a = oracle.triplet_abs(x)
    rows.append(("triplet_n4096_seed42_total", repr(float(e.sum()))))
    rows.append(("triplet_n4096_seed42_abs", repr(float(a.sum()))))
    print(f"triplet {time.time() - t0:.1f} s", file=sys.stderr)
    out = os.path.join(ROOT, "tests", "golden", "fullsize.txt")
    with open(out, "w") as f:
        f.write("# Oracle results at the BASELINE full sizes on the seeds bench.py times.\n"
                "# Written by tools/make_goldens.py (calls only oracle/ + the seeded generators in\n"
                "# paper_1609_01490_b200/inputs.py); never from the CUDA path.\n"
                "# collide: config 3 (P:488-491, reading Q9); collide1d: P:570-574 (reading Q10);\n"
                "# ca: config 4, Life B3/S23 on the triangle (P:79-80, reading Q11), packed Eq. 1 uint8\n"
                "#   state after g generations -- sha256 of the bytes and the live-cell count;\n"
                "# triplet: config 5, ATM energies (reading Q15) -- sum_t e_t and sum_t A_t = sum |E|.\n"
                f"# oracle threads: {oracle.num_threads()}\n")
        for k, v in rows:
            f.write(f"{k} {v}\n")
    print(out)


if __name__ == "__main__":
    main()

"""A/B tri_ca_run (n = 32768, 100 generations, rho 240) across builds of libtri.so in ONE
process, alternating: python tools/ab_ca.py lib1.so lib2.so ... [--reps R]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1609_01490_b200 import inputs, tri  # noqa: E402


def load(path):
    tri._lib = None
    tri.LIB_PATH = os.path.abspath(path)
    L = tri.lib()
    tri._lib = None
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--strategy", nargs="+", default=["lambda"])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n = 32768
    libs = [load(p) for p in a.libs]
    tri._lib = libs[0]
    m = tri.tri_map_init(n, 240)
    x = torch.from_numpy(inputs.ca_state(n, 42)).cuda()
    y = torch.empty_like(x)
    ws = torch.empty(tri.tri_ca_run_workspace_size(m), dtype=torch.uint8, device="cuda")
    runs = [(p, L, st) for p, L in zip(a.libs, libs) for st in a.strategy]
    times = {(p, st): [] for p, _, st in runs}
    ref = None
    for rep in range(a.reps + 1):
        for p, L, st in runs:
            tri._lib = L
            tri.tri_ca_run(m, st, a.steps, x, y, ws)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            tri.tri_ca_run(m, st, a.steps, x, y, ws)
            e1.record()
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
            assert torch.equal(y, ref), f"{p}: result differs from {a.libs[0]}"
            if rep:
                times[(p, st)].append(e0.elapsed_time(e1))
    for (p, st), t in times.items():
        print(f"{p} {st}: median {statistics.median(t):.4f} min {min(t):.4f} max {max(t):.4f} ms per {a.steps} generations")


if __name__ == "__main__":
    main()

"""A/B the EDM kernel across alternative builds of libtri.so in ONE process, alternating:
python tools/ab_edm.py [--launches L] [--reps R] [--dim D] lib1.so lib2.so ...
Each rep runs L back-to-back tri_edm launches (n = 65536, rho = 128, lambda) per lib;
prints the median / min ms per launch of every lib (the bench's sustained-loop shape)."""
import argparse
import ctypes
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
    ap.add_argument("--launches", type=int, default=50)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--rho", type=int, default=128)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n = 65536
    libs = [load(p) for p in a.libs]
    tri._lib = libs[0]
    m = tri.tri_map_init(n, a.rho)
    pts = torch.from_numpy(inputs.points(n, a.dim, 42)).cuda()
    out = torch.empty(m.out_cells, dtype=torch.float32, device="cuda")
    times = {p: [] for p in a.libs}
    for rep in range(a.reps + 1):
        for p, L in zip(a.libs, libs):
            tri._lib = L
            for _ in range(3):
                tri.tri_edm(m, "lambda", pts, out)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(a.launches):
                tri.tri_edm(m, "lambda", pts, out)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times[p].append(e0.elapsed_time(e1) / a.launches)
    for p in a.libs:
        t = times[p]
        print(f"{p}: median {statistics.median(t):.4f} min {min(t):.4f} max {max(t):.4f} ms/launch "
              f"({4 * m.out_cells / statistics.median(t) / 1e6:.0f} GB/s)")


if __name__ == "__main__":
    main()

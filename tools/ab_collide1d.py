"""A/B tri_collide1d (n = 200000, rho 256, lambda) across builds of libtri.so in ONE process:
python tools/ab_collide1d.py lib1.so lib2.so ... [--reps K]"""
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
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    n = 200000
    libs = [load(p) for p in a.libs]
    tri._lib = libs[0]
    m = tri.tri_map_init(n, 256)
    x = torch.from_numpy(inputs.intervals(n, 42, 1e-5)).cuda()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    times = {p: [] for p in a.libs}
    for rep in range(a.reps + 1):
        for p, L in zip(a.libs, libs):
            tri._lib = L
            tri.tri_collide1d(m, "lambda", x, cnt)
            torch.cuda.synchronize()
            assert cnt.item() == 397884, (p, cnt.item())
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                tri.tri_collide1d(m, "lambda", x, cnt)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times[p].append(e0.elapsed_time(e1) / 5)
    for p in a.libs:
        t = times[p]
        print(f"{p}: median {statistics.median(t):.4f} min {min(t):.4f} ms")


if __name__ == "__main__":
    main()

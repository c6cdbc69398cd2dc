"""Run one hot-path kernel a few times (for ncu captures and quick sweeps).

python tools/run_one.py edm|dummy|collide|collide1d|ca|ca_steps|ca_run|triplet [--rho R] [--strategy S] [--reps K] [--n N]
Prints per-launch CUDA-event times (ms).  Product path only (no oracle)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1609_01490_b200 import inputs, tri  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--rho", type=int, default=0)
    ap.add_argument("--strategy", default="persist")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--k", type=int, default=8)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    w = a.workload
    if w == "edm":
        n = a.n or 65536
        m = tri.tri_map_init(n, a.rho or 256)
        pts = torch.from_numpy(inputs.points(n, 3, 42)).cuda()
        out = torch.empty(m.out_cells, dtype=torch.float32, device="cuda")
        fn = lambda: tri.tri_edm(m, a.strategy, pts, out)
    elif w == "dummy":
        n = a.n or 2048
        m = tri.tri_map_init(n, a.rho or 16)
        out = torch.empty(m.out_cells, dtype=torch.int32, device="cuda")
        fn = lambda: tri.tri_dummy(m, a.strategy, tri.TRI_DUMMY_PACKED, out)
    elif w == "collide":
        n = a.n or 200000
        m = tri.tri_map_init(n, a.rho or 256)
        s = torch.from_numpy(inputs.spheres(n, 42)).cuda()
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        fn = lambda: tri.tri_collide(m, a.strategy, s, cnt)
    elif w == "ca":
        n = a.n or 32768
        m = tri.tri_map_init(n, a.rho or 512)
        x = torch.from_numpy(inputs.ca_state(n, 42)).cuda()
        y = torch.empty_like(x)
        fn = lambda: tri.tri_ca_step(m, a.strategy, x, y)
    elif w == "ca_steps":
        n = a.n or 32768
        m = tri.tri_map_init(n, a.rho or 128)
        x = torch.from_numpy(inputs.ca_state(n, 42)).cuda()
        y = torch.empty_like(x)
        fn = lambda: tri.tri_ca_steps(m, a.strategy, a.k, x, y)
    elif w == "ca_run":                       # tri_ca_run: --k generations on the bit-packed state
        n = a.n or 32768
        m = tri.tri_map_init(n, a.rho or 240)
        x = torch.from_numpy(inputs.ca_state(n, 42)).cuda()
        y = torch.empty_like(x)
        ws = torch.empty(tri.tri_ca_run_workspace_size(m), dtype=torch.uint8, device="cuda")
        fn = lambda: tri.tri_ca_run(m, a.strategy, a.k, x, y, ws)
    elif w == "collide1d":
        n = a.n or 200000
        m = tri.tri_map_init(n, a.rho or 256)
        x = torch.from_numpy(inputs.intervals(n, 42, 1e-5)).cuda()
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        fn = lambda: tri.tri_collide1d(m, a.strategy, x, cnt)
    elif w == "triplet":
        n = a.n or 4096
        m = tri.tet_map_init(n, a.rho or 16)
        x = torch.from_numpy(inputs.points4(n, 42)).cuda()
        e = torch.empty(n, dtype=torch.float64, device="cuda")
        fn = lambda: tri.tet_triplet(m, a.strategy, x, e)
    else:
        raise SystemExit(f"unknown workload {w}")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{w} n={n} rho={m.rho} strategy={a.strategy} ms={['%.4f' % t for t in ts]} min={min(ts):.4f}")


if __name__ == "__main__":
    main()

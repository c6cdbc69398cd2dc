"""Phase timing of the persistent tcgen05 collision kernel (an A/B build with -DTC_PROF)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1609_01490_b200 import inputs, tri
tri.LIB_PATH = os.path.join(os.getcwd(), sys.argv[1])
L = tri.lib()
rho = int(sys.argv[2]) if len(sys.argv) > 2 else 384
n = 200000
m = tri.tri_map_init(n, rho)
s = torch.from_numpy(inputs.spheres(n, 42)).cuda()
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
tri.tri_collide(m, "tc", s, cnt); torch.cuda.synchronize()
h = (ctypes.c_ulonglong * 16)()
L.tri_tc_prof_read(h)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); tri.tri_collide(m, "tc", s, cnt); e1.record(); torch.cuda.synchronize()
L.tri_tc_prof_read(h)
names = ["prologue", "wait MMA", "load", "sync", "issue", "test"] if len(sys.argv) > 3 else ["wait accf", "load", "barrier", "issue", "test+advance", "-"]
blocks = 2e10 / 16384
print(f"ms={e0.elapsed_time(e1):.3f} count={cnt.item()}")
for k in range(6):
    print(f"{names[k]:14s} leader warp {h[k] / blocks:8.1f}   other warps {h[k + 8] / (blocks * 3):8.1f} cycles per block")
print(f"recount calls {h[6]} ({h[6] / (blocks * 128 * 4) * 100:.3f}% of (row, 32-column group)s), negative values {h[7]}")

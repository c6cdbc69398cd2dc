# Smoke check of the tcgen05 collision filter vs the oracle on small n (TCR = tile edge, 256 or 512)
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1609_01490_b200 import tri, inputs
import oracle
for n, seed, rmax in [(300, 42, 0.2), (1000, 42, 0.05), (5000, 7, 0.02)]:
    s = inputs.spheres(n, seed, rmax)
    m = tri.tri_map_init(n, int(__import__("os").environ.get("TCR", "256")))
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tri.tri_collide(m, "tc", torch.from_numpy(s).cuda(), cnt)
    torch.cuda.synchronize()
    print(n, cnt.item(), oracle.collide(s), flush=True)

import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from paper_1609_01490_b200 import inputs, tri
def T(r): return r*(r+1)//2
n, seed = 2049, 7
st = inputs.ca_state(n, seed)
D = T(n)
ref = oracle.ca_step(n, st)
for fill in (0, 255, 1):
    for rho in (128, 256):
        m = tri.tri_map_init(n, rho)
        bigA = torch.full((D + 4096,), fill, dtype=torch.uint8, device="cuda")
        bigB = torch.full((D + 4096,), fill, dtype=torch.uint8, device="cuda")
        a = bigA[:D]; b = bigB[:D]
        a.copy_(torch.from_numpy(st))
        tri.tri_ca_step(m, "lambda", a, b); torch.cuda.synchronize()
        got = b.cpu().numpy()
        bad = np.nonzero(got != ref)[0]
        print("fill", fill, "rho", rho, "bad", len(bad), bad[:5], D, flush=True)
print("state rows 2046..2048 tail:", st[T(2046)+2040:T(2046)+2047], st[T(2047)+2040:T(2047)+2048], st[T(2048)+2040:T(2048)+2049])
print("ref (2047,2047)", ref[T(2047)+2047])

"""Per-phase clock64 trace of the tcgen05 collision kernel on SM 0 (probe build from
/tmp/p_trace.py: events 0 wait-start, 1 MMA done, 2 TMEM loaded, 3 after hand-back barrier,
4 next MMA issued, 5 sign test done; recorded by thread 0 of every CTA on SM 0)."""
import ctypes, os, sys, collections
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1609_01490_b200 import inputs, tri
lib = sys.argv[1]
tri.LIB_PATH = os.path.abspath(lib); tri._lib = None
L = tri.lib()
n = 200000
m = tri.tri_map_init(n, 768)
s = torch.from_numpy(inputs.spheres(n, 42)).cuda()
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
tri.tri_collide(m, "tc", s, cnt); torch.cuda.synchronize()
buf = np.zeros(1 << 20, np.uint64); nn = ctypes.c_uint(0)
L.tri_tc_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nn))      # reset
tri.tri_collide(m, "tc", s, cnt); torch.cuda.synchronize()
L.tri_tc_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nn))
k = min(nn.value, 1 << 20); b = buf[:k]
clk = (b >> np.uint64(24)).astype(np.int64); cta = ((b >> np.uint64(8)) & np.uint64(0xffff)).astype(np.int64)
ev = ((b >> np.uint64(5)) & np.uint64(7)).astype(np.int64); idx = (b & np.uint64(31)).astype(np.int64)
print("events", k)
per = collections.defaultdict(dict)
for c, e, i, t in zip(cta, ev, idx, clk): per[(c, i)][e] = t
d = collections.defaultdict(list)
for (c, i), evs in per.items():
    for a_, b_, name in ((0, 1, "wait MMA"), (1, 2, "TMEM load"), (2, 3, "barrier"), (3, 4, "issue"), (4, 5, "test"), ):
        if a_ in evs and b_ in evs: d[name].append(evs[b_] - evs[a_])
    if 5 in evs and (c, i + 1) in per and 0 in per[(c, i + 1)]: d["to next wait"].append(per[(c, i + 1)][0] - evs[5])
for name, v in d.items():
    v = np.array(v); print(f"{name:14s} n={len(v):6d} median {np.median(v):7.0f} p10 {np.percentile(v,10):7.0f} p90 {np.percentile(v,90):7.0f}")
# concurrency: timeline of the first 40 events of 4 co-resident CTAs
order = np.argsort(clk)
t0 = clk[order[len(order)//2]]
print("mid-run timeline (clk rel, cta, event, block):")
for j in order[len(order)//2: len(order)//2 + 48]:
    print(clk[j] - t0, cta[j], ev[j], idx[j])

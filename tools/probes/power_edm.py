"""Energy per launch of the EDM kernel vs pure-store patterns (run on the GPU box from the
repo root, after building _ab/libline.so from tools/probes/line_align.cu):
    python tools/probes/power_edm.py [lib.so ...]
Each pattern runs back-to-back launches for ~2 s while nvidia-smi samples power and SM
clock every 50 ms; prints ms/launch, median W, median MHz, J per launch and pJ per byte."""
import ctypes
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1609_01490_b200 import inputs, tri  # noqa: E402

n = 65536
D = n * (n + 1) // 2
out = torch.empty(D + 256, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
P = ctypes.CDLL(os.path.join(os.getcwd(), "_ab", "libline.so"))
pts = torch.from_numpy(inputs.points(n, 3, 42)).cuda()


def sample(fn, seconds=2.0):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    k = max(10, int(seconds * 1e3 / e0.elapsed_time(e1)))
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                            "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0.record()
    for _ in range(k):
        fn()
    e1.record(); torch.cuda.synchronize()
    smi.terminate()
    rows = [l.split(",") for l in smi.stdout.read().strip().splitlines() if l.strip()]
    busy = [(float(w), float(c)) for w, c in rows if float(w) > 400]
    ms = e0.elapsed_time(e1) / k
    w = statistics.median([b[0] for b in busy]) if busy else float("nan")
    c = statistics.median([b[1] for b in busy]) if busy else float("nan")
    return ms, w, c


def show(name, fn, nbytes=4 * D):
    ms, w, c = sample(fn)
    print(f"{name:40s} {ms:.4f} ms  {nbytes / ms / 1e6:6.0f} GB/s  {w:6.1f} W  {c:5.0f} MHz  "
          f"{w * ms / 1e3:.3f} J  {w * ms / 1e3 / nbytes * 1e12:5.1f} pJ/B", flush=True)


show("torch fill_ (8.59 GB)", lambda: out.fill_(1.0))
for which, name in ((0, "probe linear 16-B stores"), (2, "probe tiles, 16-B chunk ownership"),
                    (3, "probe tiles, 128-B line ownership")):
    show(name, lambda w=which: P.run_probe(w, ctypes.c_void_p(out.data_ptr()), ctypes.c_int64(n), 148 * 8,
                                            ctypes.c_void_p(st)))
for lib in sys.argv[1:] or [os.path.join("paper_1609_01490_b200", "libtri.so")]:
    tri._lib = None
    tri.LIB_PATH = os.path.abspath(lib)
    m = tri.tri_map_init(n, 128)
    show(f"tri_edm {os.path.basename(lib)}", lambda: tri.tri_edm(m, "lambda", pts, out))

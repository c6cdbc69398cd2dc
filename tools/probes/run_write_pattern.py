import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.getcwd(), "_ab", "libprobe.so"))
n = 65536
D = n * (n + 1) // 2
out = torch.empty(D + 64, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for which, name in ((0, "rows, 16-B stores"), (1, "rows, 32-B stores")):
    for grid in (148 * 4, 148 * 8, 148 * 16, 148 * 32):
        f = lambda: L.run_probe(which, ctypes.c_void_p(out.data_ptr()), ctypes.c_int64(n), grid, 256, ctypes.c_void_p(st))
        f(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{name:20s} grid={grid:5d}: {best:.4f} ms {4 * D / best / 1e6:.0f} GB/s")

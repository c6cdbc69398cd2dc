"""Runs tools/probes/line_align.cu (build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
-shared -Xcompiler -fPIC -o _ab/libline.so tools/probes/line_align.cu).  Sustained loop of
50 launches per pattern (like the bench's EDM loop), best of 3."""
import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.getcwd(), "_ab", "libline.so"))
n = 65536
D = n * (n + 1) // 2
out = torch.empty(D + 256, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
names = {0: "linear, aligned 512-B warp stores", 1: "linear, shifted 48 B",
         2: "EDM tiles, 16-B chunk ownership", 3: "EDM tiles, 128-B line ownership"}
for which in (0, 1, 2, 3, 0, 2, 3):
    for grid in ((148 * 8,) if which < 2 else (0,)):
        f = lambda: L.run_probe(which, ctypes.c_void_p(out.data_ptr()), ctypes.c_int64(n), grid, ctypes.c_void_p(st))
        f(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(50):
                f()
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 50)
        print(f"{names[which]:36s}: {best:.4f} ms/launch {4 * D / best / 1e6:.0f} GB/s (cells of the full triangle)")

"""Run tools/probes/mma_latency.cu (build: see its header) and print cycles per iteration."""
import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.getcwd(), "_ab", "libmma.so"))
out = torch.zeros(2048, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
names = {0: "1 MMA + commit + try_wait", 1: "1 MMA + commit + test_wait spin", 2: "4 MMAs (4 accs) + 4 commits",
         3: "16 MMAs + 1 commit", 4: "1 MMA + drain (tcgen05.ld) by 4 warps"}
names[5] = "TMEM re-read, 128 cols per warp"
for threads in (128, 256, 512):
    rc = L.run_probe(5, 128, 2000, 148, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st), threads)
    torch.cuda.synchronize()
    c = out[:148].float().mean().item()
    byts = threads // 32 * 32 * 128 * 4
    print(f"mode 5 threads={threads}: {c:.1f} cycles/iter -> {byts / c:.1f} B/cycle/SM")
for grid in (1,):
    for n in (64, 128, 256):
        for mode in (0, 1, 2, 3, 4):
            if n == 256 and mode in (2, 3):
                continue
            rc = L.run_probe(mode, n, 2000, grid, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st), 128)
            torch.cuda.synchronize()
            c = out[:grid].float()
            print(f"grid={grid:3d} N={n:3d} mode={mode} ({names[mode]:38s}): {c.mean().item():8.1f} cycles/iter (max {c.max().item():.0f}) rc={rc}")

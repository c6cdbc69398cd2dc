"""tcgen05.ld throughput (tools/probes/tmem_bw.cu)."""
import ctypes, os, torch
L = ctypes.CDLL(os.path.join(os.getcwd(), "_ab", "libtmembw.so"))
out = torch.zeros(2048, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for pack in (0, 1):
    for threads in (128, 256, 512):
        for inflight in (1, 2, 4):
            rc = L.run_bw(inflight, pack, threads, 2000, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st))
            torch.cuda.synchronize()
            c = out[:148].float().mean().item()
            cols = 128 * (threads // 32)
            byts = cols * 32 * 4            # TMEM bytes covered (32-bit cells)
            print(f"pack16={pack} warps={threads // 32:2d} inflight={inflight}: {c:7.1f} cyc/iter  "
                  f"{byts / c:6.1f} B/cyc/SM of 32-bit cells  ({cols * 32 / c:6.1f} values/cyc) rc={rc}")

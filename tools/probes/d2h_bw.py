"""D2H bandwidth into pinned host memory: one stream vs two / four concurrent streams
(does tri_edm_host's single copy stream leave PCIe bandwidth unused?)."""
import torch
GB = 1 << 30
src = torch.empty(4 * GB // 4, dtype=torch.float32, device="cuda")
dst = torch.empty(4 * GB // 4, dtype=torch.float32, pin_memory=True)
band = 1 << 25                                            # floats per band (tri_edm_host's)
nb = src.numel() // band
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for b in range(nb):
            with torch.cuda.stream(streams[b % ns]):
                dst[b * band:(b + 1) * band].copy_(src[b * band:(b + 1) * band], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{ns} stream(s): {4 * GB / ms / 1e6:.1f} GB/s")

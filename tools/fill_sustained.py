import torch, time
n = 2147516416  # the EDM output size (fp32 cells)
x = torch.empty(n, dtype=torch.float32, device="cuda")
for reps in (5, 50, 200):
    for _ in range(3): x.fill_(1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): x.fill_(1.0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"fill_ 8.59 GB x{reps} back-to-back: {ms:.4f} ms/launch {4*n/ms/1e6:.1f} GB/s")

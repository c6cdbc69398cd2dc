"""Write-only HBM ceiling on this GPU: torch fill_ and cudaMemset over the EDM's
output size (8.59 GB), CUDA events, best of 10.  Context for the EDM roofline
(MEASURED_PEAKS.json's hbm_gbs is a read+write copy)."""
import torch
n = 2147516416
x = torch.empty(n, dtype=torch.float32, device="cuda")
for name, fn in (("fill_", lambda: x.fill_(1.0)), ("zero_", lambda: x.zero_())):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {best:.4f} ms  {4 * n / best / 1e6:.1f} GB/s")
y = torch.empty(n // 2, dtype=torch.float32, device="cuda")
z = torch.empty(n // 2, dtype=torch.float32, device="cuda")
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); z.copy_(y); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"copy (read+write): {best:.4f} ms  {2 * 4 * (n // 2) / best / 1e6:.1f} GB/s")

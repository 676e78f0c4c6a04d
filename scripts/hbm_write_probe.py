"""Write-only vs copy HBM bandwidth on the box (context for the c4 output-write roofline):
fp32 fills with zero and non-zero values, and a read+write copy."""
import torch
x = torch.empty(4 << 30, dtype=torch.float32, device="cuda")  # 16 GiB
y = torch.empty(1 << 30, dtype=torch.float32, device="cuda")  # 4 GiB
def t(f, n=5):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(n):
        s.record(); f(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return best
for v in (0.0, 1.0, 0.3):
    ms = t(lambda: x.fill_(v)); print("fill fp32 %.1f 16 GiB: %.3f ms = %.2f TB/s (write only)" % (v, ms, (16 << 30) / ms / 1e9))
y.normal_()
ms = t(lambda: x[: 1 << 30].copy_(y)); print("copy 4 GiB: %.3f ms = %.2f TB/s (read+write)" % (ms, (8 << 30) / ms / 1e9))
z = torch.randn(1 << 28, device="cuda")
ms = t(lambda: x[: 1 << 30].view(4, 1 << 28).copy_(z.expand(4, -1))); print("broadcast-copy (L2 reads) 4 GiB write: %.3f ms = %.2f TB/s" % (ms, (4 << 30) / ms / 1e9))

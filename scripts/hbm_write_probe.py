"""Write-only and copy HBM bandwidth probe (context for the c4 output-write roofline)."""
import torch
x = torch.empty(16 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
def t(f, n=5):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(n):
        s.record(); f(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return best
ms = t(lambda: x.fill_(1)); print("fill 16 GiB: %.3f ms = %.2f TB/s (write only)" % (ms, (16 << 30) / ms / 1e9))
ms = t(lambda: x[: 8 << 30].copy_(y)); print("copy 8 GiB: %.3f ms = %.2f TB/s (read+write)" % (ms, (16 << 30) / ms / 1e9))
z = x.view(torch.float32)
ms = t(lambda: z.zero_()); print("zero_ fp32 16 GiB: %.3f ms = %.2f TB/s" % (ms, (16 << 30) / ms / 1e9))

"""L2-resident read bandwidth (context for the GEMM's operand traffic):
repeated reductions over buffers that fit in the 126 MB L2."""
import torch
for mb in (16, 32, 64):
    x = torch.randn(mb << 18, device="cuda")  # mb MiB of fp32
    y = torch.empty(1, device="cuda")
    for _ in range(3):
        y = x.sum()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    s.record()
    for _ in range(n):
        y = x.sum()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    print("sum over %d MiB (L2-resident): %.4f ms = %.2f TB/s" % (mb, ms, (mb << 20) / ms / 1e9))

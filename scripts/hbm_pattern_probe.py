"""Is the c4 output pattern (128 B row segments, rows 1 MiB apart) slow in DRAM?
fills of column slabs of a [2^14 rows][2^18 floats] fp32 matrix (16 GiB)."""
import torch
R, Cc = 1 << 14, 1 << 18
x = torch.empty(R, Cc, dtype=torch.float32, device="cuda")
def t(f, n=5):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(n):
        s.record(); f(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return best
for w in (32, 256, 2048, Cc):
    sl = x[:, :w]
    ms = t(lambda: sl.fill_(1.0))
    print("slab of %6d cols (%6d B per row, rows 1 MiB apart): %.3f ms = %.2f TB/s" % (w, 4 * w, ms, R * w * 4 / ms / 1e9))

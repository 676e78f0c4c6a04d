"""Quick tcgen05 path-sum check + timing (run on the GPU box under `timeout`)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan

def run(inst, prec, reps=1):
    P = Plan(inst.text, inst.n_low, inst.blocks)
    out = torch.empty(1 << inst.n, dtype=torch.complex64, device="cuda")
    ph = None
    for _ in range(reps):
        ph = P.run(out, precision=prec, timings=True)
    torch.cuda.synchronize()
    return out.cpu().numpy(), ph

for tw, name in [(True, "c2"), (True, "c4"), (False, "c2")]:
    inst = make_config(name, twin=tw)
    ref, ph_s = run(inst, "simt", 2)
    for prec in ("bf16x1", "bf16x3"):
        got, ph = run(inst, prec, 3)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(f"{inst.name} n={inst.n} {prec}: max|d|={np.abs(got-ref).max():.3e} rel={rel:.3e} "
              f"phase_ms={['%.3f' % x for x in ph]} simt_phase={['%.3f' % x for x in ph_s]}", flush=True)

"""hsf_run of one config, `reps` times (for ncu captures and launch lists).

  python scripts/prof_once.py <config> [precision] [reps]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
inst = make_config(name)
P = Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
cdt = torch.complex64 if inst.dtype == "c64" else torch.complex128
if inst.bitstrings is None:
    out = torch.empty(1 << inst.n, dtype=cdt, device="cuda")
    bits = None
else:
    out = torch.empty(len(inst.bitstrings), dtype=cdt, device="cuda")
    bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
for _ in range(reps):
    P.run(out, bitstrings=bits, precision=prec)
torch.cuda.synchronize()
print("ok", name, "passes", P.passes, "levels", P.levels, "ops", P.ops)

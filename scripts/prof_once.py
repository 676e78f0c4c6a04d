"""One hsf_run of a config (for ncu --set full captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = sys.argv[2] if len(sys.argv) > 2 else "auto"
inst = make_config(name)
P = Plan(inst.text, inst.n_low, inst.blocks)
if inst.bitstrings is None:
    out = torch.empty(1 << inst.n, dtype=torch.complex64, device="cuda")
    bits = None
else:
    out = torch.empty(len(inst.bitstrings), dtype=torch.complex64, device="cuda")
    bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
P.run(out, bitstrings=bits, precision=prec)
torch.cuda.synchronize()
print("ok", name, P.passes, P.levels)

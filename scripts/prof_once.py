"""hsf_run of one config, `reps` times (for ncu captures and launch lists).

  python scripts/prof_once.py <config> [precision] [reps] [row_div]

row_div > 1 evaluates only the first 1/row_div of the output rows (full-output
configs), e.g. a same-shape slice of c4 small enough for ncu's kernel replay.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
row_div = int(sys.argv[4]) if len(sys.argv) > 4 else 1
inst = make_config(name)
P = Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
cdt = torch.complex64 if inst.dtype == "c64" else torch.complex128
rr = None
if inst.bitstrings is None:
    rows = (1 << P.n_a) // row_div
    if "prefix" in (inst.meta or {}):  # Table II shapes: the first `prefix` amplitudes
        rows = -(-inst.meta["prefix"] // (1 << inst.n_low))
    rr = (0, rows)
    out = torch.empty(rows << P.n_b, dtype=cdt, device="cuda")
    bits = None
else:
    out = torch.empty(len(inst.bitstrings), dtype=cdt, device="cuda")
    bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
for _ in range(reps):
    ph = P.run(out, bitstrings=bits, precision=prec, row_range=rr, timings=True)
torch.cuda.synchronize()
print("ok", name, "passes", P.passes, "levels", P.levels, "ops", P.ops, "phase_ms", [round(x, 3) for x in ph])

"""K1 (whole state in shared memory) vs K2 (tiled) for 2^14-amplitude halves:
times a brickwork circuit with 14|14 qubits, bitstring output, both ways.

  python scripts/k1_tier.py            (HSF_SMEM_LIMIT=13 forces tiles)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan
for name, kw in [("c3", dict(n=28, n_low=14, depth=16, n_bits=1 << 20)),
                 ("c5", dict(n=28, n_low=14, layers=8, fanout=6, n_bits=1 << 20))]:
    inst = make_config(name, **kw)
    P = Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
    out = torch.empty(len(inst.bitstrings), dtype=torch.complex64, device="cuda")
    bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
    for _ in range(3):
        P.run(out, bitstrings=bits)
    torch.cuda.synchronize()
    ph = []
    for _ in range(20):
        ph.append(P.run(out, bitstrings=bits, timings=True))
    ph = np.median(np.array(ph), axis=0)
    print(name, "m=14 limit", os.environ.get("HSF_SMEM_LIMIT", "14"), "passes", P.passes, "levels", P.levels,
          "phase_ms", [round(float(x), 4) for x in ph], flush=True)

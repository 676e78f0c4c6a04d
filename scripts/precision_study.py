"""Accuracy of the full-output path-sum precision modes.

c2 at full size against its closed form (QFT without swaps of the X-prepared
basis state, DESIGN §3 reading 9) and the c2 / c4 / c5 twins against the
oracle's Schroedinger result.  Writes one JSON object to stdout.
The closed form and the oracle are test-side references (tests/, scripts/)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from hsf_inputs import make_config  # noqa: E402
from oracle import hsf_oracle as O  # noqa: E402
from paper_2502_06959_b200 import Plan  # noqa: E402

MODES = ("simt", "bf16x1", "bf16x3", "bf16x6", "tf32x3")


def run(inst, prec):
    P = Plan(inst.text, inst.n_low, inst.blocks, dtype="c64")
    out = torch.empty(1 << inst.n, dtype=torch.complex64, device="cuda")
    P.run(out, precision=prec)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.complex128)


def err(got, ref):
    return {"relL2": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)), "max_abs": float(np.abs(got - ref).max()),
            "max_rel": float(np.abs(got - ref).max() / np.abs(ref).max())}


res = {}
inst = make_config("c2")
n, x = inst.n, inst.meta["x"]
i = np.arange(1 << n, dtype=np.int64)
rev = np.zeros_like(i)
for b in range(n):
    rev |= ((i >> b) & 1) << (n - 1 - b)
ref = np.exp(2j * np.pi * ((x * rev) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
res["c2_full_vs_closed_form"] = {m: err(run(inst, m), ref) for m in MODES}
for name in ("c2", "c4", "c5"):
    inst = make_config(name, twin=True, n_bits=0) if name == "c5" else make_config(name, twin=True)
    nq, g = O.parse_circuit(inst.text)
    ref = O.schrodinger(nq, g)
    res[name + "_twin_vs_oracle"] = {m: err(run(inst, m), ref) for m in MODES}
print(json.dumps(res))

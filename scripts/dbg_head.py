"""Debug: head fold vs no head fold on small full-output runs."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from hsf_inputs import make_config
from oracle import hsf_oracle as O
from paper_2502_06959_b200 import Plan


def run(inst, env=None, **kw):
    old = dict(os.environ)
    os.environ.update(env or {})
    try:
        P = Plan(inst.text, inst.n_low, inst.blocks, **kw)
        out = torch.empty(1 << (P.n_a + P.n_b), dtype=torch.complex64, device="cuda")
        P.run(out, precision="bf16x3")
        torch.cuda.synchronize()
        return out.cpu().numpy(), P
    finally:
        os.environ.clear(); os.environ.update(old)


inst = make_config("c2", twin=True)
n, g = O.parse_circuit(inst.text)
ref = O.schrodinger(n, g)
for env in [{}, {"HSF_NO_HEAD_FOLD": "1"}, {"HSF_TC_BMN": "0"}, {"HSF_TC_BMN": "0", "HSF_NO_HEAD_FOLD": "1"}]:
    got, P = run(inst, env)
    print(env, P.head_units, P.tail_units, "rel", np.linalg.norm(got - ref) / np.linalg.norm(ref),
          "ratio", np.vdot(ref, got) / np.vdot(ref, ref))

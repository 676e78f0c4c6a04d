"""Small runs of every kernel family for compute-sanitizer (one tool per gpurun call):
c1 (c128 SIMT, whole-state tier), c2 twin (tcgen05 pair GEMM + split kernels),
c3/c5 twins at n=26 (tiled K2 tier, JIT + interpreter), bitstring gather + fold."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan

def full(inst, **kw):
    P = Plan(inst.text, inst.n_low, inst.blocks, dtype=kw.pop("dtype", inst.dtype), **kw)
    out = torch.empty(1 << inst.n, dtype=torch.complex64 if P.dtype == "c64" else torch.complex128, device="cuda")
    P.run(out, precision="auto" if P.dtype == "c64" else "simt")
    torch.cuda.synchronize()

def bits(inst, **kw):
    P = Plan(inst.text, inst.n_low, inst.blocks, **kw)
    b = torch.from_numpy(inst.bitstrings[:4096].view(np.int64)).cuda()
    out = torch.empty(4096, dtype=torch.complex64, device="cuda")
    P.run(out, bitstrings=b, path_range=(0, 8))
    torch.cuda.synchronize()

full(make_config("c1"), dtype="c128")
full(make_config("c2", twin=True, n=18, n_low=9))                # whole tier + tcgen05 pair GEMM
full(make_config("c4", twin=True, n=20, n_low=10), tile_qubits=10)  # tiled tier, full output
for jit in (True, False):
    bits(make_config("c3", twin=True, n=26, n_low=13, n_bits=4096), jit=jit, tile_qubits=11)
    bits(make_config("c5", twin=True, n=26, n_low=13, n_bits=4096), jit=jit)
print("sanitize workload ok")

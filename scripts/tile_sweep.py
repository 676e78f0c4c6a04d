"""c3 with forced tile sizes (hsf_plan_opts.tile_qubits): ms per step and phases."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
inst = make_config(name)
bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
out = torch.empty(len(inst.bitstrings), dtype=torch.complex64, device="cuda")
for tq in (0, 10, 11, 12, 13):
    P = Plan(inst.text, inst.n_low, inst.blocks, tile_qubits=tq)
    for _ in range(3):
        P.run(out, bitstrings=bits)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for s, e in ev:
        s.record(); P.run(out, bitstrings=bits); e.record()
    torch.cuda.synchronize()
    ph = [P.run(out, bitstrings=bits, timings=True) for _ in range(3)]
    print(name, "tile", tq, "passes", P.passes, "ms %.4f" % statistics.mean(s.elapsed_time(e) for s, e in ev),
          "simA %.3f simB %.3f core %.3f" % tuple(statistics.mean(p[i] for p in ph) for i in (0, 1, 3)))

"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the HSF method: it only draws random
numbers and writes circuit files (text, hex floats), block groupings (gate
index lists) and bitstring sets.  Both `oracle/` and
`paper_2502_06959_b200/` read what it writes; neither imports the other.
"""
from .circuits import (  # noqa: F401
    Instance,
    CONFIGS,
    make_config,
    make_c1,
    make_c2,
    make_c3,
    make_c4,
    make_c5,
    make_brick_block,
    make_sbm_qaoa,
    make_table2,
    TABLE2,
    random_small_circuit,
    random_folding_circuit,
    serialize,
)

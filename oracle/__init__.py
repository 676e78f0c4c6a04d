"""CPU oracle (TEST INFRASTRUCTURE ONLY; see oracle/hsf_oracle.py header).

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never by paper_2502_06959_b200.
"""
from .hsf_oracle import *  # noqa: F401,F403

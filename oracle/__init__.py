"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY).

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs.  Shares no code with paper_2604_23265_b200.
"""
from .rte import *  # noqa: F401,F403
from . import rte  # noqa: F401

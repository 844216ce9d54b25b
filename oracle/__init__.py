"""fp64 CPU oracle for the PSCWin hot path — TEST INFRASTRUCTURE ONLY (see pscwin_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
"""
from .pscwin_oracle import *  # noqa: F401,F403

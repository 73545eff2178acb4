"""CPU oracle (TEST INFRASTRUCTURE ONLY).

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Shares no code with the product.
"""
from .xc_oracle import *  # noqa: F401,F403
from .xc_oracle import build_lib  # noqa: F401

"""TEST INFRASTRUCTURE ONLY -- the fp64 CPU oracle of ENOVA's detection path.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package
paper_2407_09486_b200 never imports it.  See enova_oracle.py for what it
computes and what pins it.
"""
from .enova_oracle import *  # noqa: F401,F403

"""CPU oracle for the PIF step -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2407_00485_b200/) never imports, links or executes anything here and
shares no code with it.
"""
from .pif_oracle import *  # noqa: F401,F403

"""CPU oracle for the DOT hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1706_05586_b200``) never imports it; the two share no code.
"""
from .dot_oracle import *  # noqa: F401,F403

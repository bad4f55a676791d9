"""fp64 CPU oracle for the KRP-sketch path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2507_23207_b200``) never imports it, and this package never imports
the product path: the two share no code.  See ``oracle/krp_oracle.py``.
"""
from .krp_oracle import *  # noqa: F401,F403
from .krp_oracle import __all__  # noqa: F401

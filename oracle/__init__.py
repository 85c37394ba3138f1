"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU float64 implementation of what the B200 path
computes (one synchronous 3D-ResAttNet training step; network partitioning;
GABRA placement; brute-force placement).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / `--impl reference` leg may import it.  The
product package `paper_2104_05035_b200` never imports it, and it never imports
the product.  Shared inputs come from the separate `synthetic` module.

Every function cites the PAPER.md passage it follows; readings of silent or
garbled passages are listed in DESIGN.md ("Readings").  Pins: tests/test_oracle_*.py.
"""
from . import net, gabra  # noqa: F401

"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Restatements of the reference algorithms (each function cites the reference
file:line it follows), used by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py as the checker / the timed CPU baseline.  The
product package (paper_2601_12713_b200) never imports this.
"""

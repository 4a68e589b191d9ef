"""CPU oracle - TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, and there only as the checker or the
timed CPU baseline.  The product package (paper_2306_11665_b200) never
imports it and has no CPU fallback.
"""

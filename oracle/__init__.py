"""CPU oracles for parity checks. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this package — and only as the checker, never as the thing measured or shipped.
The product (paper_2401_09149_b200 / libseqplan_isp.so) never touches it.
"""

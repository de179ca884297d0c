"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/fj_oracle.cpp header).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package, and only as the checker /
CPU baseline; the product (paper_2301_10841_b200) never does.
"""

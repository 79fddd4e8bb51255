"""TEST INFRASTRUCTURE ONLY: CPU oracles for the FFTMatvec path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline -- never as the product path.
"""

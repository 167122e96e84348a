"""oracle -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference (zoserve) LoZO path, pinned to golden vectors
generated from the reference itself (tests/golden/make_golden.py).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package -- as the checker, never as the product path.
"""

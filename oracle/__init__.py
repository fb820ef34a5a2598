"""CPU checker for the XNOR-conv forward path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  The product package (paper_2007_14178_b200)
never imports it; tests/test_capi.py asserts that.
"""

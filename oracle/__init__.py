"""TEST INFRASTRUCTURE ONLY: CPU oracle (checker) of the decode hot path.

Import from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg
only; the product (paper_2605_10433_b200) never imports, links or calls it.
"""

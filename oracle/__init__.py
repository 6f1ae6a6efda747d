"""CPU oracle for the renewal tau-leap — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package, and only as the checker or the timed CPU
baseline; the product package never imports it (tests/test_boundary.py
asserts that).  See spreadsim_port.py for the restatement and its pinning.
"""

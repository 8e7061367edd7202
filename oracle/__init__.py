"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's primitive kernels (minml/kernels.py,
minml/rng.py) used as the parity checker for the B200 backend.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package; the product
(paper_2201_12465_b200) never does.

Pinning: every kernel here is checked against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports /root/reference's
``minml`` in the build container) in tests/test_oracle_golden.py.
"""

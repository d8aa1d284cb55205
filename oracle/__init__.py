"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the FNO hot path.

Plain numpy/scipy restatement of the reference algorithm
(/root/reference/pkg/src/distfno: fno.py, spectral.py, oracle.py, tensor.py),
written from its behaviour, with every function citing the reference lines it
follows.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or the timed CPU baseline -- never as the product path.  The product
(``paper_2211_12709_b200``) never imports this package.

Parity pinning: the oracle is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports
/root/reference/pkg/src/distfno in the build container and writes the
fixtures; ``tests/test_oracle.py`` replays them).
"""

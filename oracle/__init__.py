"""CPU oracle for the cfcent multi-RHS Laplacian solve path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(``paper_1607_02955_b200``) imports this package; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` / ``--impl reference``) may use it, and there only as the
checker or the timed CPU reference, never as the thing measured or shipped.

The oracle restates the reference algorithm (``/root/reference/pkg/src/cfcent``)
in plain numpy/scipy; each function cites the reference file:line it follows.
It is pinned against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``), see ``tests/test_oracle_golden.py``.
"""

"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference (`oocdet` 0.1.0, /root/reference/pkg) algorithm for the
north-star hot path: the blocked symmetric MEMDET drivers `memdet_cholesky` / `memdet_ldl`
(`pkg/src/oocdet/memdet.py:322-433`) and their tile kernels (`kernels/dense.py:57-116`,
`kernels/_ldl.pyx:21-61`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import anything from this package, and only as the checker or the timed CPU
baseline — never as the product path.  The product (`paper_2503_04424_b200`) must not import
it; `tests/test_boundary.py` enforces that.

Parity pin: `tests/test_oracle_golden.py` checks this restatement against golden vectors
produced by the unmodified reference (`tests/golden/make_golden.py`, run in the build
container where /root/reference is mounted).
"""

"""CPU oracle for the GOOM LMME prefix-scan hot path.

TEST INFRASTRUCTURE ONLY. Nothing in `paper_2510_03426_b200/` may import this
package; only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs use it, and there only as the checker
or the timed CPU baseline.

`gooms_port` restates, in numpy, the reference algorithm of
`/root/reference/pkg/src/gooms/{core,scan,lyapunov}.py` for the functions on
the hot path (each function cites the file:line it follows). It is pinned
against golden vectors produced by the reference itself
(`tests/golden/make_golden.py`, run in the build container where the
reference is importable) — see `tests/test_oracle_golden.py`.
"""

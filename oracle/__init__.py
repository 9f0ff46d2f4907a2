"""CPU oracle for the MGPCG hot path of voxtop (arXiv 2201.12931).

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2201_12931_b200`) imports, links or executes this package.  The only
legitimate callers are `tests/`, `__graft_entry__.smoke()` (as the checker)
and the `cpu_baseline` / `--impl reference` legs of `bench.py`.

`oracle.cpu_path` is an independent numpy/scipy restatement of the
reference algorithm (every function cites the reference file:line it
follows).  It is pinned against the real reference through the golden
fixtures under `tests/golden/`, which `oracle/make_golden.py` generates by
importing `/root/reference/pkg/src/voxtop` in the build container; see
`tests/test_oracle_golden.py`.
"""

"""CPU oracle for the IceCache decode hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the algorithm of the reference package
(`/root/reference/pkg/src/icecache`, a pure Python/NumPy model of IceCache)
with the precision contract the B200 path implements:

* key lifting in fp64 exactly as `dci.py:517-523` / `geometry.py:68-98`,
  rounded to fp32 for storage;
* exact 1-NN parents in fp64 (`dci.py:527-543`) with a fixed fused-multiply-add
  order (C helper in `oracle/c/oracle_nn.c`);
* search distances in fp32 with the device's fixed reduction tree
  (`numerics.d2_fp32`), tie-broken by token id (`dci.py:297,360,363`);
* P-DCI visit order and level draws from the reference's own NumPy PCG64
  streams (`dci.py:180-183, 268-278`).

Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may import this package, and only as
the checker or the timed CPU baseline.  The product package
(`paper_2604_10539_b200`) never imports it.

Parity pinning: the restatement is checked against golden vectors produced
by running the unmodified reference in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`, see
`tests/test_oracle_golden.py`).
"""

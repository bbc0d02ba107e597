"""The package's NumPy workload generator (paper_2604_10539_b200.workload,
restating the reference's generate_workload draw for draw) against the
reference-written trace golden and the oracle's restatement.  CPU."""

import numpy as np
import pytest

from conftest import load_golden  # noqa: F401
from oracle.workload import Spec, generate
from paper_2604_10539_b200.errors import ConfigError
from paper_2604_10539_b200.workload import WorkloadSpec, generate_workload


@pytest.mark.parametrize("kind", ["clustered", "uniform", "planted_needle"])
def test_generator_matches_oracle_restatement(kind):
    kw = dict(kind=kind, n_tokens=257, d=12, d_prime=5, clusters=4, layers=3, kv_heads=2,
              query_heads_per_group=3, seed=7)
    wl = generate_workload(WorkloadSpec(**kw))
    k, v, q, needle = generate(Spec(**kw), fp32=False)
    assert np.array_equal(wl.keys, k) and np.array_equal(wl.values, v) and np.array_equal(wl.queries, q)
    assert wl.needle_token == needle


def test_generator_matches_reference_trace():
    """trace_small.npz: the reference's generate_workload -> save_trace ->
    load_trace (f32 payload, each group's first-head query)."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "trace_small.npz"))
    L, H, G, d, dv, n = z["shape"].tolist()
    wl = generate_workload(WorkloadSpec(kind="clustered", n_tokens=n, d=d, d_prime=dv, clusters=4, layers=L,
                                        kv_heads=H, query_heads_per_group=G, seed=11))
    assert np.array_equal(wl.keys.astype(np.float32), z["keys"])
    assert np.array_equal(wl.values.astype(np.float32), z["values"])
    assert np.array_equal(wl.queries[:, :, ::G].astype(np.float32), z["queries"][:, :, ::G])


def test_spec_validation_and_views():
    with pytest.raises(ConfigError):
        WorkloadSpec(kind="nope")
    with pytest.raises(ConfigError):
        WorkloadSpec(n_tokens=0)
    wl = generate_workload(WorkloadSpec(n_tokens=20, d=4, d_prime=4, layers=2, kv_heads=1))
    k, v = wl.prefill_view(10)
    assert k.shape == (10, 2, 1, 4) and v.shape == (10, 2, 1, 4)
    st = wl.decode_step(10, 3)
    assert st.token_id == 13 and np.array_equal(st.queries, wl.queries[13])
    with pytest.raises(ConfigError):
        wl.prefill_view(21)
    with pytest.raises(ConfigError):
        wl.decode_step(10, 10)

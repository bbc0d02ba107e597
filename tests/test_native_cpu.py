"""CPU-side checks of the native library and the host logic (no GPU needed):
the C ABI loads and exports every symbol the header declares, the host
restatement of NumPy's SeedSequence/PCG64 matches NumPy, the embedded
ziggurat tables are NumPy's, and the device's stateless P-DCI visit order
(emission keys) equals the reference's heap merge."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _lib():
    from paper_2604_10539_b200 import _native as N
    return N.lib()


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "icecache_b200.h")).read()
    names = set(re.findall(r"\b(icb_[a-z0-9_]+)\s*\(", header))
    assert len(names) >= 18
    lib = _lib()
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert lib.icb_version() == 1


def test_python_binding_covers_the_header():
    from paper_2604_10539_b200 import _native as N
    header = open(os.path.join(ROOT, "include", "icecache_b200.h")).read()
    names = set(re.findall(r"\b(icb_[a-z0-9_]+)\s*\(", header))
    assert names <= set(N.EXPORTS) | {"icb_search_profile"}


@pytest.mark.parametrize("entropy,spawn", [(0, (0,)), ([3, 5, 7], (0,)), ([0, 2, 1], (1, 17)),
                                           (2**40 + 5, (0,)), ([1, 2, 3, 4, 5], (1, 3))])
def test_host_seedseq_pcg64_matches_numpy(entropy, spawn):
    from paper_2604_10539_b200.forest import entropy_words
    words = np.array(entropy_words(entropy), dtype=np.uint32)
    sp = np.array(spawn, dtype=np.uint32)
    out = np.zeros(64)
    lib = _lib()
    rc = lib.icb_host_pcg_doubles(words.ctypes.data_as(ctypes.c_void_p), len(words),
                                  sp.ctypes.data_as(ctypes.c_void_p), len(sp), len(out),
                                  out.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    ss = np.random.SeedSequence(entropy)
    g = np.random.default_rng(np.random.SeedSequence(entropy=ss.entropy, spawn_key=spawn))
    assert np.array_equal(out, g.random(64))


@pytest.mark.parametrize("skip", [0, 1, 7, 4096, 123457, 2**40 + 3])
def test_host_pcg64_jump_matches_numpy(skip):
    """The LCG jump that splits the level-draw stream across device threads
    (rng.cuh icb_pcg_jump) lands where NumPy's PCG64 does after `skip` draws."""
    from paper_2604_10539_b200.forest import entropy_words
    words = np.array(entropy_words([3, 5, 7]), dtype=np.uint32)
    sp = np.array((0,), dtype=np.uint32)
    out = np.zeros(16)
    rc = _lib().icb_host_pcg_jump_doubles(words.ctypes.data_as(ctypes.c_void_p), len(words),
                                          sp.ctypes.data_as(ctypes.c_void_p), len(sp), skip, len(out),
                                          out.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    ss = np.random.SeedSequence([3, 5, 7])
    bg = np.random.PCG64(np.random.SeedSequence(entropy=ss.entropy, spawn_key=(0,)))
    if skip < 200000:
        assert np.array_equal(out, np.random.Generator(bg).random(skip + 16)[skip:])
    else:
        bg.advance(skip)
        assert np.array_equal(out, np.random.Generator(bg).random(16))


def test_embedded_ziggurat_tables_are_numpys():
    import importlib.util
    spec = importlib.util.spec_from_file_location("gz", os.path.join(ROOT, "tools", "gen_ziggurat.py"))
    gz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gz)
    ki, wi, fi = gz.find_tables()
    inc = open(os.path.join(ROOT, "paper_2604_10539_b200", "csrc", "ziggurat_tables.inc")).read()
    blocks = re.findall(r"=\s*\{(.*?)\};", inc, re.S)
    k2 = np.array([int(x.strip().rstrip("ULL"), 16) for x in blocks[0].split(",")], dtype=np.uint64)
    w2 = np.array([float.fromhex(x.strip()) for x in blocks[1].split(",")])
    f2 = np.array([float.fromhex(x.strip()) for x in blocks[2].split(",")])
    assert np.array_equal(k2, ki) and np.array_equal(w2, wi) and np.array_equal(f2, fi)


def _emission_order(dirs, ids, vecs, q, cap):
    """The device's stateless P-DCI order (csrc/search.cuh pdci_visit)."""
    from oracle.dci import project
    proj = project(dirs, vecs)
    qp = project(dirs, q[None, :])[0]
    m = len(ids)
    keys = []
    for i in range(m):
        best = None
        for j in range(dirs.shape[0]):
            pj = proj[i, j]
            pos = sum(1 for i2 in range(m) if (proj[i2, j], ids[i2]) < (pj, ids[i]))
            start = int((proj[:, j] < qp[j]).sum())
            gap = abs(pj - qp[j])
            sec = ((1 << 23) - 1 - pos) if pos < start else ((1 << 23) + pos)
            key = (gap, (j << 24) | sec)
            best = key if best is None or key > best else best
        keys.append(best)
    order = sorted(range(m), key=lambda i: keys[i])
    return [int(ids[i]) for i in order[:cap]]


@pytest.mark.parametrize("seed", range(6))
def test_pdci_emission_keys_equal_heap_merge(seed):
    from oracle.dci import pdci_dirs, visit_order
    rng = np.random.default_rng(seed)
    m, dim1 = int(rng.integers(65, 140)), 17
    vecs = rng.normal(size=(m, dim1))
    if seed % 2:   # duplicated members: tied projections exercise the chain-order tie rule
        vecs[m // 2:m // 2 + 6] = vecs[3]
    ids = rng.permutation(10 * m)[:m]
    dirs = pdci_dirs([seed, 1], int(rng.integers(0, 50)), dim1)
    q = rng.normal(size=dim1)
    cap = int(rng.integers(8, m))
    assert _emission_order(dirs, ids, vecs, q, cap) == visit_order(dirs, ids, vecs, q, cap)


def test_engine_config_validation_mirrors_reference():
    from paper_2604_10539_b200.engine import EngineConfig
    from paper_2604_10539_b200.errors import ConfigError
    for bad in (dict(reuse_stride=1), dict(page_size=1), dict(promotion_ratio=1.0), dict(token_budget=0),
                dict(sink_pages=0), dict(skip_layers=-1), dict(kv_dtype="fp8")):
        with pytest.raises(ConfigError):
            EngineConfig(**bad)
    c = EngineConfig(token_budget=256)
    b = c.budget()
    assert (b.k, b.beam, b.visit_cap) == (256, 512, 1024) and c.n_query_heads == c.kv_heads
    # device-path options: KV offload and the fused rotation step do not combine
    assert not c.kv_offload and not c.fuse_rotation
    EngineConfig(kv_offload=True)
    EngineConfig(fuse_rotation=True)
    with pytest.raises(ConfigError):
        EngineConfig(kv_offload=True, fuse_rotation=True)


def test_forest_config_struct_matches_header():
    """icb_forest_config as ctypes sees it: field order and offsets of the C
    struct (include/icecache_b200.h), including the KV-offload fields."""
    from paper_2604_10539_b200 import _native as N
    hdr = open(os.path.join(ROOT, "include", "icecache_b200.h")).read()
    body = hdr[hdr.index("typedef struct {", hdr.index("typedef struct icb_forest icb_forest;")):]
    body = body[:body.index("} icb_forest_config;")]
    names = re.findall(r"^\s*(?:int32_t|double)\s+(\w+);", body, flags=re.M)
    assert [f for f, _ in N.icb_forest_config._fields_] == names
    assert N.icb_forest_config.kv_host.offset == 56 and ctypes.sizeof(N.icb_forest_config) == 64


def test_sequence_sharding():
    from paper_2604_10539_b200.dist import aggregate_throughput, shard_sequences
    owned = [shard_sequences(64, 8, r) for r in range(8)]
    assert sorted(sum(owned, [])) == list(range(64))
    assert all(len(o) == 8 for o in owned)
    assert aggregate_throughput(10, 4, 2.0) == 20.0

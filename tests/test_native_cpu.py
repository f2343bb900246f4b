"""CPU: the C-ABI library loads and exports every symbol include/prsp_bsc_gpu.h
declares; the host-side logic (fixtures, sharding, statistics packing,
template counts) matches the oracle. No GPU compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "prsp_bsc_gpu.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(prsp_bsc_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1908_06843_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # every declared entry point also has a ctypes signature in the binding
    assert set(syms) <= set(_native.SIGNATURES)


def test_nccl_resolved_at_run_time():
    """The statistics all-reduce uses NCCL through dlopen (nccl_link.hpp): the
    library has no link-time NCCL dependency, and the bootstrap works here."""
    from paper_1908_06843_b200 import _native
    from paper_1908_06843_b200.bsc import nccl_unique_id

    assert "libnccl" not in os.popen(f"ldd {_native.LIB_PATH}").read()
    uid = nccl_unique_id()
    assert len(uid) == 128 and any(uid)


def test_library_is_sm100a():
    from paper_1908_06843_b200 import _native

    out = os.popen(f"cuobjdump -lelf {_native.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_no_device_reports_status():
    from paper_1908_06843_b200 import _native, bsc

    if _native.lib().prsp_bsc_gpu_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_native.PrspError):
        bsc.BscGpuModel(4, 3, bsc.TruncationConfig(3, 2, 2))


def test_config_validation_before_device():
    """Truncation validation (truncation.cpp:23-30) is reported as PRSP_ERR_CONFIG."""
    from paper_1908_06843_b200 import _native, bsc

    for hp, g in [(0, 1), (4, 1), (2, 3)]:
        with pytest.raises(_native.ConfigError):
            bsc.BscGpuModel(4, 3, bsc.TruncationConfig(3, hp, g))


def test_fixtures_match_oracle(port):
    from paper_1908_06843_b200 import bsc, configs

    y, t = bsc.bars_generate(5, 300, seed=0)
    yo, to = port.make_bars(5, 300, seed=0)
    assert np.array_equal(y, yo) and np.array_equal(t, to)
    ym, _ = bsc.bars_generate(4, 50, max_mode=True, seed=3)
    assert np.array_equal(ym, port.make_bars(4, 50, max_mode=True, seed=3)[0])
    w = bsc.random_dictionary(256, 300, 2)
    assert np.array_equal(w, port.random_dictionary(256, 300, 2))
    assert np.allclose(np.linalg.norm(w, axis=0), 5.0)
    y2 = bsc.generate(bsc.BscParams(w, 5 / 300, 0.25), 400, 2)
    assert np.array_equal(y2, port.generate(w, 5 / 300, 0.25, 400, 2))
    p = bsc.baseline_init(y2, 300, 2)
    wo, pio, s2o = port.baseline_init(y2, 300, 2)
    assert np.array_equal(p.W, wo) and p.pi == pio and p.sigma2 == s2o
    ps = bsc.standard_init(y, 10, 6, 9)
    so = port.standard_init(y, 10, 6, 3, 9)
    assert np.array_equal(ps.W, so[0]) and ps.pi == so[1] and ps.sigma2 == so[2]
    # the configs module builds c1 data through the same generators
    assert np.array_equal(configs.data(configs.CONFIGS["c1"], 64), port.make_bars(10, 64, seed=1)[0])


def test_strong_scaling_data_is_sharding_invariant(port, monkeypatch):
    """c4 is drawn in fixed blocks by global point index (configs.BLOCK): any
    world size's shards concatenate to the same dataset, and the oracle-drawn
    inputs of the reference arm are the same bytes as the package's."""
    from dataclasses import replace

    from paper_1908_06843_b200 import configs
    from paper_1908_06843_b200.dist import shard_range

    monkeypatch.setattr(configs, "BLOCK", 700)
    w = replace(configs.CONFIGS["c4"], D=16, H=20, N=3000)
    full = configs.data(w)
    assert full.shape == (3000, 16)
    for world in (1, 2, 3, 8):
        parts = [configs.data(w, rows=shard_range(w.N, world, r)) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)
    assert np.array_equal(configs.data(w, gen=configs.OracleGen(port)), full)
    wc2 = configs.CONFIGS["c2"]
    assert np.array_equal(configs.data(wc2, 300, gen=configs.OracleGen(port)), configs.data(wc2, 300))


def test_shard_range_matches_shardplan():
    from paper_1908_06843_b200.dist import shard_range

    for n in [0, 1, 7, 200000, 4_000_000]:
        for world in [1, 2, 3, 8]:
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            lens = [e - b for b, e in rs]
            assert max(lens) - min(lens) <= 1 and lens == sorted(lens, reverse=True)


def test_pack_unpack_roundtrip(port):
    from paper_1908_06843_b200.dist import pack_stats, stats_count, unpack_stats

    y, _ = port.make_bars(4, 60, seed=5)
    w, pi, s2 = port.baseline_init(y, 8, 5)
    st = port.estep_stats(w, pi, s2, y, 5, 3)
    buf = pack_stats(st, 16, 8)
    assert buf.shape == (stats_count(16, 8),)
    back = unpack_stats(buf, 16, 8)
    for k in st:
        assert np.array_equal(np.asarray(back[k]), np.asarray(st[k])), k
    # multi-valued families: value_counts has one entry per non-zero value
    from oracle.oracle import Prior

    pr = Prior("dsc", 0.0, [-1.0, 0.0, 1.0, 2.0], [0.1, 0.7, 0.1, 0.1])
    st = port.ld_estep_stats(pr, w, s2, y, 5, 3)
    buf = pack_stats(st, 16, 8)
    assert buf.shape == (stats_count(16, 8, 3),)
    back = unpack_stats(buf, 16, 8, 3)
    for k in st:
        assert np.array_equal(np.asarray(back[k]), np.asarray(st[k])), k


def test_flop_convention_matches_survey():
    import bench

    # SURVEY.md §8(d) per-point totals
    assert sum(bench.flops_per_point(25, 10, 10, 10)) == 67_390
    assert sum(bench.flops_per_point(100, 20, 10, 4)) == 22_197
    assert sum(bench.flops_per_point(256, 300, 12, 4)) == 341_848
    assert sum(bench.flops_per_point(576, 1000, 14, 5)) == 2_498_969

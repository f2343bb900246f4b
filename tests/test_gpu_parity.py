"""GPU parity of the sm_100a path (through the C ABI) against the oracle.

Bar: candidate sets bit-exact (uint32, every point); sufficient statistics,
free energy and one-step W, π, σ² within the tolerances below (north star:
1e-6 relative per iteration, fp64; Frobenius-relative for
matrices). Small cases compare with the oracle directly; the full BASELINE
sizes are checked through size-independent properties.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden, rel

pytestmark = pytest.mark.gpu

TOL_STEP = 1e-6  # north-star tolerance (W Frobenius-relative, π, σ², F relative)
TOL_STATS = 1e-10  # per-field Frobenius-relative on E-step statistics


@pytest.fixture(scope="module")
def pkg():
    import paper_1908_06843_b200 as P

    assert P._native.lib().prsp_bsc_gpu_device_count() > 0, "no CUDA device: the sm_100a path cannot run"
    return P


def model_for(P, d, h, hp, g):
    return P.BscGpuModel(d, h, P.TruncationConfig(h, hp, g))


def check_stats(sg, so, tol=TOL_STATS):
    for k in ["sum_s", "sum_ssT", "sum_y_sT", "value_counts"]:
        assert rel(getattr(sg, k), so[k]) < tol, (k, rel(getattr(sg, k), so[k]))
    assert abs(sg.sum_y2 - so["sum_y2"]) <= tol * abs(so["sum_y2"])
    assert abs(sg.log_partition - so["log_partition"]) <= tol * abs(so["log_partition"])
    assert sg.points == so["points"]


def check_step(res, w, pi, s2, f, tol=TOL_STEP):
    assert rel(res.params.W, w) < tol, rel(res.params.W, w)
    assert abs(res.params.pi - pi) <= tol * pi
    assert abs(res.params.sigma2 - s2) <= tol * s2
    assert abs(res.free_energy - f) <= tol * abs(f)


# ------------------------------------------------------------ golden fixtures
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_golden(pkg, name):
    g = load_golden(name)
    y, d, h = g["y"], g["W0"].shape[0], g["W0"].shape[1]
    hp, gm, T = int(g["hprime"]), int(g["gamma"]), float(g["temperature"])
    p0 = pkg.BscParams(g["W0"], float(g["pi0"]), float(g["sigma2_0"]))
    m = model_for(pkg, d, h, hp, gm)
    m.load(y)
    assert np.array_equal(m.candidates(p0), g["candidates"])
    sg = m.estep_stats(p0, temperature=T)
    check_stats(sg, {k[6:]: g[k] for k in g if k.startswith("stats_")})
    r = m.step(p0, temperature=T)
    check_step(r, g["W1"], float(g["pi1"]), float(g["sigma2_1"]), float(g["F0"]))
    # free-running trajectory (secondary gate)
    p = p0
    for i in range(len(g["traj_F"])):
        r = m.step(p)
        check_step(r, g["traj_W"][i], float(g["traj_pi"][i]), float(g["traj_sigma2"][i]), float(g["traj_F"][i]))
        p = r.params
    inf = m.inference(p0)
    assert np.array_equal(inf.map_states, g["map_states"])
    assert rel(inf.map_mass, g["map_mass"]) < 1e-10
    assert rel(inf.expected_states, g["expected"]) < 1e-10
    m.close()


# ------------------------------------------------------ BASELINE workloads, sampled
@pytest.mark.parametrize("cfg,n", [("c0", 1000), ("c1", 3000), ("c2", 4000), ("c3", 600)])
def test_config_parity(pkg, port, cfg, n):
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS[cfg]
    y = configs.data(w, n)
    p = configs.init(w, y)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    m.load(y)
    assert np.array_equal(m.candidates(p), port.candidates(p.W, p.pi, p.sigma2, y, w.hprime))
    check_stats(m.estep_stats(p), port.estep_stats(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma))
    wo, pio, s2o, fo = port.step(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma)
    check_step(m.step(p), wo, pio, s2o, fo)
    m.close()


def test_one_step_parity_along_trajectory(pkg, port):
    """Primary gate: at every iteration, oracle params in → params out within 1e-6."""
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c1"]
    y = configs.data(w, 2000)
    p = configs.init(w, y)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    m.load(y)
    for _ in range(8):
        wo, pio, s2o, fo = port.step(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma)
        assert np.array_equal(m.candidates(p), port.candidates(p.W, p.pi, p.sigma2, y, w.hprime))
        check_step(m.step(p), wo, pio, s2o, fo)
        p = pkg.BscParams(wo, pio, s2o)
    m.close()


def test_mstep_from_oracle_stats(pkg, port):
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c2"]
    y = configs.data(w, 1500)
    p = configs.init(w, y)
    st = port.estep_stats(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    pm = m.mstep(st, p)
    wo, pio, s2o = port.mstep(st, p.W, p.pi, p.sigma2)
    assert rel(pm.W, wo) < 1e-10 and abs(pm.pi - pio) <= 1e-14 * pio and abs(pm.sigma2 - s2o) <= 1e-10 * s2o
    m.close()


# ----------------------------------------------------------------- edge cases
@pytest.mark.parametrize("d,h,hp,g,n", [
    (25, 10, 10, 10, 37),   # exact mode, odd N
    (7, 5, 1, 1, 9),        # H' = γ = 1
    (13, 11, 11, 1, 16),    # γ = 1 with H' = H (no multi-active states)
    (33, 70, 9, 2, 1),      # single point, ragged D and H (padding)
    (9, 40, 20, 3, 50),     # large H' relative to H
    (16, 33, 32, 2, 40),    # H' ≥ 31: round-based selection path
])
def test_edge_shapes(pkg, port, d, h, hp, g, n):
    wt = port.random_dictionary(d, h, 3, 2.0)
    y = port.generate(wt, 0.15, 0.3, n, 4)
    w0, pi0, s20 = port.baseline_init(np.r_[y, y + 0.1], h, 5)  # ≥ 2 rows for the init recipe
    p = pkg.BscParams(w0, pi0, s20)
    m = model_for(pkg, d, h, hp, g)
    m.load(y)
    assert np.array_equal(m.candidates(p), port.candidates(w0, pi0, s20, y, hp))
    check_stats(m.estep_stats(p), port.estep_stats(w0, pi0, s20, y, hp, g))
    wo, pio, s2o, fo = port.step(w0, pi0, s20, y, hp, g)
    check_step(m.step(p), wo, pio, s2o, fo)
    m.close()


def test_exact_ties_lowest_index_wins(pkg, port):
    """Duplicate dictionary columns and all-zero points make selection scores tie
    exactly; the lowest index must win (truncation.cpp:48-53)."""
    rng = np.random.default_rng(0)
    d, h, hp, g = 20, 16, 5, 3
    w = rng.normal(size=(d, h))
    w[:, 9] = w[:, 3]
    w[:, 12] = w[:, 3]
    w[:, 14] = w[:, 7]
    y = rng.normal(size=(64, d)) + w[:, 3]
    y[5] = 0.0
    y[17] = w[:, 7] * 2.0
    m = model_for(pkg, d, h, hp, g)
    m.load(y)
    p = pkg.BscParams(w, 0.2, 0.7)
    assert np.array_equal(m.candidates(p), port.candidates(w, 0.2, 0.7, y, hp))
    wo, pio, s2o, fo = port.step(w, 0.2, 0.7, y, hp, g)
    check_step(m.step(p), wo, pio, s2o, fo)
    m.close()


def test_near_tie_band_uses_exact_scores(pkg, port):
    """Columns that differ in the last bits put two scores within the fast-path
    error bound; the exact re-rank must reproduce the oracle's choice."""
    rng = np.random.default_rng(1)
    d, h, hp = 64, 24, 6
    w = rng.normal(size=(d, h))
    for j, k in [(2, 5), (8, 11), (13, 20)]:
        w[:, k] = w[:, j] * (1 + 1e-15 * rng.normal(size=d))
    y = rng.normal(size=(300, d)) + w[:, 2] + w[:, 8] + w[:, 13]
    m = model_for(pkg, d, h, hp, 3)
    m.load(y)
    p = pkg.BscParams(w, 0.1, 1.3)
    assert np.array_equal(m.candidates(p), port.candidates(w, 0.1, 1.3, y, hp))
    m.close()


@pytest.mark.parametrize("s2", [1e-3, 0.02, 0.3, 1.0, 40.0])
def test_posterior_weight_paths(pkg, port, s2):
    """σ² sweeps |log-joint| terms from e^±1000 (range guard fails: exp path)
    through mixed per-point paths to flat posteriors (multiplicative path)."""
    d, h, hp, g = 24, 30, 9, 4
    wt = port.random_dictionary(d, h, 11, 2.0)
    y = port.generate(wt, 0.1, 0.05, 400, 12)
    p = pkg.BscParams(wt * 1.1, 0.1, s2)
    m = model_for(pkg, d, h, hp, g)
    m.load(y)
    assert np.array_equal(m.candidates(p), port.candidates(p.W, p.pi, s2, y, hp))
    check_stats(m.estep_stats(p), port.estep_stats(p.W, p.pi, s2, y, hp, g))
    inf = m.inference(p)
    ms, mm, ex = port.inference(p.W, p.pi, s2, y, hp, g)
    assert np.array_equal(inf.map_states, ms)
    assert rel(inf.map_mass, mm) < 1e-10
    assert rel(inf.expected_states, ex) < 1e-10
    m.close()


@pytest.mark.parametrize("cfg,n", [("c1", 500), ("c2", 3000), ("c3", 400)])
def test_temperature(pkg, port, cfg, n):
    """Annealed posteriors (linear_discrete.cpp:277-286: q ∝ exp((lj − m)/T), log Z at T = 1) at the
    bars shape and at the c2 / c3 shapes, statistics and the whole step."""
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS[cfg]
    y = configs.data(w, n)
    p = configs.init(w, y)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    m.load(y)
    for T in [1.0, 1.5, 4.0]:
        check_stats(m.estep_stats(p, temperature=T),
                    port.estep_stats(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma, T))
    if n >= 4 * w.H:  # (fewer points than units leave Σ⟨ssᵀ⟩ to the ridge, which amplifies rounding differences)
        check_step(m.step(p, temperature=2.0), *port.step(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma, temperature=2.0))
    m.close()


def test_errors(pkg):
    m = model_for(pkg, 4, 6, 3, 2)
    m.load(np.ones((5, 4)))
    bad = np.ones((4, 6))
    bad[1, 2] = np.nan
    with pytest.raises(pkg.NumericError):
        m.set_params(pkg.BscParams(bad, 0.2, 1.0))
    with pytest.raises(pkg.ConfigError):
        m.set_params(pkg.BscParams(np.ones((4, 6)), 1.2, 1.0))
    with pytest.raises(pkg.ConfigError):
        m.set_params(pkg.BscParams(np.ones((4, 6)), 0.2, -1.0))
    with pytest.raises(pkg.ConfigError):  # state explosion (truncation.cpp:111-114)
        pkg.BscGpuModel(8, 40, pkg.TruncationConfig(40, 30, 20, state_cap=1000))
    with pytest.raises(pkg.ConfigError):  # non-finite selection scores (truncation.cpp:43-45)
        m.step(pkg.BscParams(np.full((4, 6), 1e308), 0.2, 1e-300))
    m.close()


# --------------------------------------------------- full-size properties
def test_full_c2_properties(pkg, port):
    """c2 at N = 200,000: all candidate sets bit-exact vs the reference,
    shard additivity of the statistics, ⟨ssᵀ⟩ symmetry, Σ⟨s⟩ = value count,
    F = Σ log Z and EM monotone over a few iterations."""
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c2"]
    y = configs.data(w)
    p = configs.init(w, y)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    m.load(y)
    cand = m.candidates(p)
    # every one of the 200,000 candidate sets, bit-exact against the reference build
    # (oracle/_ref) when present, else the C port pinned to it
    from oracle import oracle as O

    orc = O.Oracle("ref") if O.Oracle.available("ref") else port
    want = orc.candidates(p.W, p.pi, p.sigma2, y, w.hprime, threads=os.cpu_count() or 1)
    assert np.array_equal(cand, want), int(np.count_nonzero(np.any(cand != want, axis=1)))
    st = m.estep_stats(p)
    assert np.allclose(st.sum_ssT, st.sum_ssT.T, rtol=0, atol=0)
    assert abs(st.value_counts[0] - st.sum_s.sum()) <= 1e-12 * st.value_counts[0]
    assert np.allclose(np.diag(st.sum_ssT), st.sum_s, rtol=1e-14)
    assert st.points == len(y)
    # additivity over two shards (linearity of the E-step statistics)
    ma = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    ma.load(y[:77_777])
    sa = ma.estep_stats(p)
    ma.load(y[77_777:])
    sb = ma.estep_stats(p)
    for k in ["sum_s", "sum_ssT", "sum_y_sT"]:
        assert rel(getattr(sa, k) + getattr(sb, k), getattr(st, k)) < 1e-12
    assert abs(sa.log_partition + sb.log_partition - st.log_partition) <= 1e-12 * abs(st.log_partition)
    fs = []
    for _ in range(4):
        r = m.step(p)
        fs.append(r.free_energy)
        p = r.params
    assert all(b >= a - 1e-9 * abs(a) for a, b in zip(fs, fs[1:])), fs
    m.close()
    ma.close()


def test_e2e_host_step_matches_resident(pkg):
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c1"]
    y = configs.data(w, 1000)
    p = configs.init(w, y)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    a = m.step_host(p, y)
    m2 = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    m2.load(y)
    b = m2.step(p)
    assert rel(a.params.W, b.params.W) < 1e-13 and abs(a.free_energy - b.free_energy) <= 1e-13 * abs(b.free_energy)
    m.close()
    m2.close()


@pytest.mark.parametrize("cfg,n", [("c2", 60_000), ("c3", 6_000)])
def test_bitwise_reproducible(pkg, cfg, n):
    """Every reduction of the BSC E-step is order-fixed (split-K partials,
    per-CTA partials, column sums) or order-independent (the Σ⟨ssᵀ⟩ candidate
    pairs in fixed point), so repeated E-steps and steps give the same bits —
    as the reference does at a fixed shard plan (parallel.hpp:35-37)."""
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS[cfg]
    y = configs.data(w, n)
    p = configs.init(w, y)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    m.load(y)
    a, b = m.estep_stats(p), m.estep_stats(p)
    for k in ["sum_s", "sum_ssT", "sum_y_sT", "value_counts"]:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.log_partition == b.log_partition and a.sum_y2 == b.sum_y2
    r1, r2 = m.step(p), m.step(p)
    assert np.array_equal(r1.params.W, r2.params.W)
    assert r1.params.pi == r2.params.pi and r1.params.sigma2 == r2.params.sigma2
    assert r1.free_energy == r2.free_energy
    m.close()


def test_resident_step_after_chunked_host_step(pkg):
    """step_host slices Yᵀ per host chunk (one column scale per chunk); a later
    resident step() on the same handle must not reuse those slices with chunk
    0's scales (advisor finding, round 1). Chunks with different column maxima
    (rows from 16384 on scaled ×4) make any mix-up visible."""
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c2"]
    y = configs.data(w, 40_000)
    y[16_384:] *= 4.0
    p = configs.init(w, y)
    m = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    a = m.step_host(p, y)  # 3 host chunks of ≤ 16384 points
    b = m.step(p)  # resident data are the same rows
    m2 = model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    m2.load(y)
    c = m2.step(p)
    for r in (a, b):
        assert rel(r.params.W, c.params.W) < 1e-12, rel(r.params.W, c.params.W)
        assert abs(r.free_energy - c.free_energy) <= 1e-12 * abs(c.free_energy)
        assert abs(r.params.sigma2 - c.params.sigma2) <= 1e-12 * c.params.sigma2
    m.close()
    m2.close()


# ------------------------------------------------- sliced int8 vs DMMA products
@pytest.mark.parametrize("d,h,hp,g,n", [(256, 300, 12, 4, 3000), (576, 1000, 14, 5, 600), (25, 10, 10, 10, 700)])
def test_sliced_gemm_path_matches_dmma_and_oracle(pkg, port, monkeypatch, d, h, hp, g, n):
    """Y·W and Yᵀ⟨S⟩ on the int8 tensor cores (ozaki_gemm.cuh, the default for
    the binary family) against the DMMA path (BSC_GEMM=dmma) and the oracle on
    the same inputs: candidate sets identical, statistics and the step within
    fp64 rounding of each other."""
    wt = port.random_dictionary(d, h, 21, 5.0)
    y = port.generate(wt, min(0.5, 5.0 / h), 0.25, n, 22)
    p = pkg.BscParams(wt + 0.05 * np.sin(np.arange(d * h)).reshape(d, h), 1.0 / h, 0.4)
    out = {}
    for mode in ("", "dmma"):
        if mode:
            monkeypatch.setenv("BSC_GEMM", mode)
        else:
            monkeypatch.delenv("BSC_GEMM", raising=False)
        m = model_for(pkg, d, h, hp, g)
        m.load(y)
        out[mode] = (m.candidates(p), m.estep_stats(p), m.step(p))
        m.close()
    (c0, s0, r0), (c1, s1, r1) = out[""], out["dmma"]
    assert np.array_equal(c0, c1)
    assert np.array_equal(c0, port.candidates(p.W, p.pi, p.sigma2, y, hp))
    for k in ["sum_s", "sum_ssT", "sum_y_sT", "value_counts"]:
        assert rel(getattr(s0, k), getattr(s1, k)) < 1e-12, k
    assert abs(s0.log_partition - s1.log_partition) <= 1e-13 * abs(s1.log_partition)
    check_stats(s0, port.estep_stats(p.W, p.pi, p.sigma2, y, hp, g))
    # n < H leaves Σ⟨ssᵀ⟩ rank-deficient: the 1e-9·tr/H ridge (linear_discrete.cpp:349-353)
    # amplifies the ~1e-13 statistic differences, so W′ is held to the north-star bar there
    assert rel(r0.params.W, r1.params.W) < (1e-11 if n >= 4 * h else TOL_STEP)
    assert abs(r0.free_energy - r1.free_energy) <= 1e-13 * abs(r1.free_energy)


# ------------------------------------- finish pass fused with the ⟨S⟩ᵀ slicer
@pytest.mark.parametrize("d,h,hp,g,n,s2", [(256, 300, 12, 4, 5003, 0.4), (576, 1000, 14, 5, 777, 0.4),
                                          (100, 20, 10, 4, 130, 0.3), (64, 40, 8, 3, 1000, 1e-3)])
def test_fused_finish_slice_matches_unfused(pkg, port, monkeypatch, d, h, hp, g, n, s2):
    """lane_finish_slice_kernel (finish_slice_kernels.cuh: ⟨s⟩ rows cut into the
    int8 operand of Yᵀ⟨S⟩ in shared memory, never written to HBM) against the
    unfused finish + slicer launches (BSC_FUSED_FINISH=0): every statistic
    within 1e-14 relative of the unfused launches'. Shapes: c2's and c3's (the latter takes the 16-point
    sub-tiles), a ragged N below one 128-point block, and a small σ² that sends
    points outside the range guard to the fallback launch (rows read back from ⟨S⟩)."""
    wt = port.random_dictionary(d, h, 31, 5.0)
    y = port.generate(wt, min(0.5, 4.0 / h), 0.25, n, 32)
    p = pkg.BscParams(wt + 0.05 * np.cos(np.arange(d * h)).reshape(d, h), 1.0 / h, s2)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("BSC_FUSED_FINISH", mode)
        m = model_for(pkg, d, h, hp, g)
        m.load(y)
        out[mode] = (m.estep_stats(p), m.step(p))
        m.close()
    (s0, r0), (s1, r1) = out["1"], out["0"]
    # the same terms in each launch's own fixed summation order
    assert rel(s0.sum_y_sT, s1.sum_y_sT) < 1e-14
    assert rel(s0.sum_ssT, s1.sum_ssT) < 1e-14
    assert abs(s0.log_partition - s1.log_partition) <= 1e-14 * abs(s1.log_partition)
    assert rel(s0.sum_s, s1.sum_s) < 1e-14
    check_stats(s0, port.estep_stats(p.W, p.pi, p.sigma2, y, hp, g))
    assert rel(r0.params.W, r1.params.W) < (1e-11 if n >= 4 * h else TOL_STEP)
    assert abs(r0.free_energy - r1.free_energy) <= 1e-13 * abs(r1.free_energy)


@pytest.mark.parametrize("d,h,hp,g,n", [(256, 300, 12, 4, 20011), (100, 20, 10, 4, 1300), (64, 40, 8, 3, 257)])
def test_factor_overlap_is_bitwise_the_serial_mstep(pkg, port, monkeypatch, d, h, hp, g, n):
    """step() finalises the moment sums and factors Σ⟨ssᵀ⟩ + ridge·I on a side
    stream while the Yᵀ⟨S⟩ product runs (BscEngine::fork_factor); estep_stats +
    mstep, and BSC_MSTEP_OVERLAP=0, run the same launches on one stream. Same
    kernels, same order per buffer: W′, π′, σ²′ and F are identical bits over a
    few iterations, and the chunked host-data step (the fork sits before its
    last chunk's product) lands on the same parameters within rounding."""
    wt = port.random_dictionary(d, h, 61, 5.0)
    y = port.generate(wt, min(0.5, 4.0 / h), 0.25, n, 62)
    p0 = pkg.BscParams(wt + 0.05 * np.cos(np.arange(d * h)).reshape(d, h), 1.0 / h, 0.4)
    runs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("BSC_MSTEP_OVERLAP", mode)
        m = model_for(pkg, d, h, hp, g)
        m.load(y)
        p, traj = p0, []
        for _ in range(4):
            r = m.step(p)
            p = r.params
            traj.append((p.W.copy(), p.pi, p.sigma2, r.free_energy))
        runs[mode] = traj
        if mode == "1":  # the two-call path never forks
            m.estep_stats(p0)
            r2 = m.mstep(None, p0)
            assert np.array_equal(r2.W, traj[0][0]) and r2.pi == traj[0][1] and r2.sigma2 == traj[0][2]
            rh = m.step_host(p0, y)
            assert rel(rh.params.W, traj[0][0]) < 1e-9 and abs(rh.free_energy - traj[0][3]) <= 1e-12 * abs(traj[0][3])
        m.close()
    for a, b in zip(runs["1"], runs["0"]):
        assert np.array_equal(a[0], b[0])
        assert a[1:] == b[1:]


def test_dead_dictionary_element(pkg, port):
    """A unit no data point ever selects (its column points away from all the
    data): its statistics are made of singleton weights ~e^-100 and smaller. The
    reference sums them in fp64, as the finish pass does (fp64 exp for every
    unit); the sliced Yᵀ⟨S⟩ drops entries below 2^-56 of the slice scale. That
    is not visible: the statistics, and
    the step (the dead column of W′ included: both ~0 under the ridge of
    linear_discrete.cpp:349-353), match the oracle at the usual tolerances."""
    d, h, hp, g, n = 64, 40, 8, 3, 3000
    wt = port.random_dictionary(d, h, 51, 5.0)
    y = port.generate(wt, 0.08, 0.25, n, 52)
    w0 = wt + 0.05 * np.sin(np.arange(d * h)).reshape(d, h)
    dead = 7
    w0[:, dead] = -3.0 * np.abs(y).max()  # far from every data point
    p = pkg.BscParams(w0, 1.0 / h, 0.3)
    m = model_for(pkg, d, h, hp, g)
    m.load(y)
    cand = m.candidates(p)
    assert not np.any(cand == dead)
    assert np.array_equal(cand, port.candidates(p.W, p.pi, p.sigma2, y, hp))
    sg, so = m.estep_stats(p), port.estep_stats(p.W, p.pi, p.sigma2, y, hp, g)
    check_stats(sg, so)
    assert so["sum_s"][dead] < 1e-30 and abs(sg.sum_s[dead] - so["sum_s"][dead]) <= 1e-9 * so["sum_s"][dead]
    check_step(m.step(p), *port.step(p.W, p.pi, p.sigma2, y, hp, g))
    m.close()


def test_resident_steps_follow_the_stepwise_trajectory(pkg):
    """step_resident (prsp_bsc_gpu_step from the parameters the engine holds: the bench's inner
    loop) gives the same bits as step(params) fed with its own results."""
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c1"]
    y = configs.data(w, 2000)
    p = configs.init(w, y)
    a, b = model_for(pkg, w.D, w.H, w.hprime, w.gamma), model_for(pkg, w.D, w.H, w.hprime, w.gamma)
    a.load(y)
    b.load(y)
    b.set_params(p)
    for _ in range(4):
        r = a.step(p)
        p = r.params
        f = b.step_resident()
        assert f == r.free_energy
    q = b.get_params()
    assert np.array_equal(q.W, p.W) and q.pi == p.pi and q.sigma2 == p.sigma2
    a.close()
    b.close()

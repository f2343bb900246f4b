"""GPU parity of the max-causes log-joint against the
reference goldens and the C restatement: candidates bit-exact; winner
statistics within 1e-10; one step (fixed-point W/π, residual-pass σ²) within
1e-6; inference readout.
"""
import numpy as np
import pytest

from conftest import MCA_GOLDEN_CASES, MCA_MODES, load_golden, rel

pytestmark = pytest.mark.gpu

TOL_STEP = 1e-6
TOL_STATS = 1e-10


@pytest.fixture(scope="module")
def pkg():
    import paper_1908_06843_b200 as P

    assert P._native.lib().prsp_bsc_gpu_device_count() > 0, "no CUDA device: the sm_100a path cannot run"
    return P


def check_stats(sg, so, tol=TOL_STATS):
    assert rel(sg.winner_num, so["winner_num"]) < tol, rel(sg.winner_num, so["winner_num"])
    assert rel(sg.winner_den, so["winner_den"]) < tol, rel(sg.winner_den, so["winner_den"])
    assert abs(sg.sum_act - so["sum_act"]) <= tol * abs(so["sum_act"])
    assert abs(sg.log_partition - so["log_partition"]) <= tol * abs(so["log_partition"])
    assert sg.points == so["points"]


def check_step(res, w, pi, s2, f, tol=TOL_STEP):
    assert rel(res.params.W, w) < tol, rel(res.params.W, w)
    assert abs(res.params.pi - pi) <= tol * pi
    assert abs(res.params.sigma2 - s2) <= tol * s2
    assert abs(res.free_energy - f) <= tol * abs(f)


@pytest.mark.parametrize("name", MCA_GOLDEN_CASES)
def test_golden_mca(pkg, name):
    g = load_golden(name)
    mode, rho = MCA_MODES[int(g["mode"])], float(g["rho"])
    y, w0 = g["y"], g["W0"]
    d, h = w0.shape
    hp, gm, T = int(g["hprime"]), int(g["gamma"]), float(g["temperature"])
    m = pkg.McaGpuModel(mode, d, h, pkg.TruncationConfig(h, hp, gm), soft_winner_rho=rho)
    m.load(y)
    p0 = pkg.McaParams(w0, float(g["pi0"]), float(g["sigma2_0"]))
    assert np.array_equal(m.candidates(p0), g["candidates"])
    check_stats(m.estep_stats(p0, temperature=T), {k[6:]: g[k] for k in g if k.startswith("stats_")})
    check_step(m.step(p0, temperature=T), g["W1"], float(g["pi1"]), float(g["sigma2_1"]), float(g["F0"]))
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


@pytest.mark.parametrize("mode,rho,d,h,hp,g,n", [
    ("mca", 0.0, 36, 24, 8, 3, 300),
    ("mmca", 0.0, 20, 40, 6, 4, 200),
    ("mca", 1.5, 16, 12, 12, 3, 150),   # H' = H, soft winners
    ("mmca", 0.0, 7, 70, 5, 2, 41),     # ragged shapes
])
def test_mca_parity_vs_oracle(pkg, port, mode, rho, d, h, hp, g, n):
    rng = np.random.default_rng(d * h)
    wt = np.abs(rng.normal(size=(d, h))) * 2 + 0.05 if mode == "mca" else rng.normal(size=(d, h)) * 2
    y = port.mca_generate(mode, wt, 0.15, 0.3, n, 3)
    w0, pi0, s20 = port.mca_standard_init(mode, y, h, hp, 4)
    m = pkg.McaGpuModel(mode, d, h, pkg.TruncationConfig(h, hp, g), soft_winner_rho=rho)
    m.load(y)
    p0 = pkg.McaParams(w0, pi0, s20)
    assert np.array_equal(m.candidates(p0), port.mca_candidates(mode, w0, pi0, s20, y, hp))
    check_stats(m.estep_stats(p0), port.mca_estep_stats(mode, w0, pi0, s20, y, hp, g, rho=rho))
    check_stats(m.estep_stats(p0, temperature=3.0), port.mca_estep_stats(mode, w0, pi0, s20, y, hp, g, 3.0, rho=rho))
    st = port.mca_estep_stats(mode, w0, pi0, s20, y, hp, g, rho=rho)
    wf, pf = port.mca_mstep_fixedpoint(mode, st, w0, pi0, s20)
    pm = m.mstep_fixedpoint(st, p0)
    assert rel(pm.W, wf) < 1e-12 and abs(pm.pi - pf) <= 1e-14 * pf
    wo, pio, s2o, fo = port.mca_step(mode, w0, pi0, s20, y, hp, g, rho=rho)
    check_step(m.step(p0), wo, pio, s2o, fo)
    ms, mm, ex = port.mca_inference(mode, w0, pi0, s20, y, hp, g)
    inf = m.inference(p0)
    assert np.array_equal(inf.map_states, ms)
    assert rel(inf.map_mass, mm) < 1e-10 and rel(inf.expected_states, ex) < 1e-10
    m.close()


def test_mca_errors(pkg):
    P = pkg
    with pytest.raises(P.ConfigError):
        P.McaGpuModel("mmca", 4, 6, P.TruncationConfig(6, 3, 2), soft_winner_rho=1.0)
    with pytest.raises(P.ConfigError):
        P.McaGpuModel("xca", 4, 6, P.TruncationConfig(6, 3, 2))
    m = P.McaGpuModel("mca", 4, 6, P.TruncationConfig(6, 3, 2))
    m.load(np.ones((5, 4)))
    with pytest.raises(P.ConfigError):  # weight floor (max_causes.cpp:108-112)
        m.set_params(P.McaParams(-np.ones((4, 6)), 0.2, 1.0))
    with pytest.raises(P.NumericError):
        m.set_params(P.McaParams(np.full((4, 6), np.nan), 0.2, 1.0))
    m.close()


@pytest.mark.parametrize("mode,d,h,hp,g,n", [
    ("mca", 9, 7, 7, 1, 50),     # γ = 1
    ("mmca", 8, 6, 6, 6, 40),    # exact mode H' = γ = H
])
def test_mca_edges(pkg, port, mode, d, h, hp, g, n):
    rng = np.random.default_rng(h * 7 + g)
    wt = np.abs(rng.normal(size=(d, h))) + 0.1 if mode == "mca" else rng.normal(size=(d, h))
    y = port.mca_generate(mode, wt, 0.25, 0.3, n, 5)
    w0, pi0, s20 = port.mca_standard_init(mode, y, h, hp, 6)
    m = pkg.McaGpuModel(mode, d, h, pkg.TruncationConfig(h, hp, g))
    m.load(y)
    p0 = pkg.McaParams(w0, pi0, s20)
    check_stats(m.estep_stats(p0), port.mca_estep_stats(mode, w0, pi0, s20, y, hp, g))
    wo, pio, s2o, fo = port.mca_step(mode, w0, pi0, s20, y, hp, g)
    check_step(m.step(p0), wo, pio, s2o, fo)
    if hp == h == g:
        ll = port.mca_exact_log_likelihood(mode, w0, pi0, s20, y)
        assert abs(fo - ll) <= 1e-10 * abs(ll)
    m.close()

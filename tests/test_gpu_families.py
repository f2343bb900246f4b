"""GPU parity of the multi-valued linear discrete families (SURVEY.md §8(f)
row 2): TSC and DSC through the sm_100a enumerator with the value odometer,
against the reference's golden fixtures and the C restatement.

Same bar as BSC: candidate sets bit-exact; statistics within 1e-10
(Frobenius-relative per field); one-step W, π / probs, σ², F within 1e-6.
"""
import numpy as np
import pytest

from conftest import LD_GOLDEN_CASES, golden_prior, load_golden, rel

pytestmark = pytest.mark.gpu

TOL_STEP = 1e-6
TOL_STATS = 1e-10


@pytest.fixture(scope="module")
def pkg():
    import paper_1908_06843_b200 as P

    assert P._native.lib().prsp_bsc_gpu_device_count() > 0, "no CUDA device: the sm_100a path cannot run"
    return P


def gpu_model(P, prior, d, h, hp, g):
    return P.LinearDiscreteGpuModel(prior.family, d, h, P.TruncationConfig(h, hp, g),
                                    values=prior.alpha if prior.family == "dsc" else None)


def gpu_params(P, prior, w, s2):
    return P.LinearDiscreteParams(w, s2, prior.pi, prior.probs if prior.family == "dsc" else None)


def check_stats(sg, so, tol=TOL_STATS):
    for k in ["sum_s", "sum_ssT", "sum_y_sT", "value_counts"]:
        assert rel(getattr(sg, k), so[k]) < tol, (k, rel(getattr(sg, k), so[k]))
    assert abs(sg.sum_y2 - so["sum_y2"]) <= tol * abs(so["sum_y2"])
    assert abs(sg.log_partition - so["log_partition"]) <= tol * abs(so["log_partition"])
    assert sg.points == so["points"]


def check_step(prior, res, w, pi, probs, s2, f, tol=TOL_STEP):
    p = res.params
    assert rel(p.W, w) < tol, rel(p.W, w)
    assert abs(p.sigma2 - s2) <= tol * s2
    assert abs(res.free_energy - f) <= tol * abs(f)
    if prior.family == "dsc":
        assert np.max(np.abs(np.asarray(p.probs) - probs) / probs) <= tol
    else:
        assert abs(p.pi - pi) <= tol * pi


@pytest.mark.parametrize("name", LD_GOLDEN_CASES)
def test_golden_families(pkg, name):
    g = load_golden(name)
    pr = golden_prior(g)
    y, w0, s20 = g["y"], g["W0"], float(g["sigma2_0"])
    d, h = w0.shape
    hp, gm, T = int(g["hprime"]), int(g["gamma"]), float(g["temperature"])
    m = gpu_model(pkg, pr, d, h, hp, gm)
    m.load(y)
    p0 = gpu_params(pkg, pr, w0, s20)
    assert np.array_equal(m.candidates(p0), g["candidates"])
    check_stats(m.estep_stats(p0, temperature=T), {k[6:]: g[k] for k in g if k.startswith("stats_")})
    r = m.step(p0, temperature=T)
    check_step(pr, r, g["W1"], float(g["pi1"]), g["probs1"], float(g["sigma2_1"]), float(g["F0"]))
    p = p0
    for i in range(len(g["traj_F"])):
        r = m.step(p)
        check_step(pr, r, g["traj_W"][i], float(g["traj_pi"][i]), g["traj_probs"][i] if pr.family == "dsc" else None,
                   float(g["traj_sigma2"][i]), float(g["traj_F"][i]))
        p = r.params
    inf = m.inference(p0)
    assert np.array_equal(inf.map_states, g["map_states"])
    assert rel(inf.map_mass, g["map_mass"]) < 1e-10
    assert rel(inf.expected_states, g["expected"]) < 1e-10
    m.close()


@pytest.mark.parametrize("family,alpha,probs,d,h,hp,g,n", [
    ("tsc", None, None, 32, 40, 8, 3, 600),
    ("tsc", None, None, 20, 12, 12, 3, 200),            # H' = H
    ("tsc", None, None, 9, 70, 5, 2, 33),               # ragged shapes, small γ
    ("dsc", [-1.0, 0.0, 1.0, 2.0], [0.05, 0.8, 0.1, 0.05], 24, 30, 6, 3, 400),
    ("dsc", [0.0, 2.0], [0.9, 0.1], 16, 20, 6, 3, 300),  # one non-zero value ≠ 1
    ("dsc", [-2.0, -0.5, 0.0, 0.5, 1.5], [0.05, 0.1, 0.7, 0.1, 0.05], 12, 10, 5, 2, 200),
])
def test_family_parity_vs_oracle(pkg, port, family, alpha, probs, d, h, hp, g, n):
    from oracle.oracle import Prior

    pr = Prior(family, 0.15, alpha, probs)
    wt = port.random_dictionary(d, h, 21, 2.0)
    y = port.ld_generate(pr, wt, 0.3, n, 22)
    w0, _, s20 = port.baseline_init(np.r_[y, y + 0.1], h, 23)
    m = gpu_model(pkg, pr, d, h, hp, g)
    m.load(y)
    p0 = gpu_params(pkg, pr, w0, s20)
    assert np.array_equal(m.candidates(p0), port.ld_candidates(pr, w0, s20, y, hp))
    check_stats(m.estep_stats(p0), port.ld_estep_stats(pr, w0, s20, y, hp, g))
    check_stats(m.estep_stats(p0, temperature=2.5), port.ld_estep_stats(pr, w0, s20, y, hp, g, 2.5))
    wo, pio, qo, s2o, fo = port.ld_step(pr, w0, s20, y, hp, g)
    check_step(pr, m.step(p0), wo, pio, qo, s2o, fo)
    ms, mm, ex = port.ld_inference(pr, w0, s20, y, hp, g)
    inf = m.inference(p0)
    assert np.array_equal(inf.map_states, ms)
    assert rel(inf.map_mass, mm) < 1e-10 and rel(inf.expected_states, ex) < 1e-10
    m.close()


def test_family_errors(pkg):
    P = pkg
    with pytest.raises(P.ConfigError):
        P.LinearDiscreteGpuModel("gsc", 4, 6, P.TruncationConfig(6, 3, 2))
    with pytest.raises(P.ConfigError):  # dsc alphabet must contain 0 (linear_discrete.cpp:57-59)
        P.LinearDiscreteGpuModel("dsc", 4, 6, P.TruncationConfig(6, 3, 2), values=[-1.0, 1.0])
    m = P.LinearDiscreteGpuModel("dsc", 4, 6, P.TruncationConfig(6, 3, 2), values=[1.0, 0.0, -1.0])
    assert np.array_equal(m.alphabet, [-1.0, 0.0, 1.0]) and m.n_values == 2
    m.load(np.ones((5, 4)))
    with pytest.raises(P.ConfigError):  # probabilities must sum to 1
        m.set_params(P.LinearDiscreteParams(np.ones((4, 6)), 1.0, probs=[0.2, 0.6, 0.3]))
    with pytest.raises(P.ConfigError):  # one probability per alphabet value
        m.set_params(P.LinearDiscreteParams(np.ones((4, 6)), 1.0, probs=[0.5, 0.5]))
    m.close()
    t = P.LinearDiscreteGpuModel("tsc", 4, 6, P.TruncationConfig(6, 3, 2))
    with pytest.raises(P.ConfigError):
        t.set_params(P.LinearDiscreteParams(np.ones((4, 6)), 1.0, pi=1.5))
    t.close()


@pytest.mark.parametrize("family,alpha,probs,d,h,hp,g,n", [
    ("tsc", None, None, 10, 9, 9, 1, 60),                 # γ = 1: singletons only
    ("tsc", None, None, 8, 6, 6, 6, 50),                  # exact mode H' = γ = H
    ("dsc", [0.0, 0.5, 3.0], [0.8, 0.15, 0.05], 12, 20, 4, 4, 80),   # γ = H', positive alphabet
])
def test_family_edges(pkg, port, family, alpha, probs, d, h, hp, g, n):
    from oracle.oracle import Prior

    pr = Prior(family, 0.2, alpha, probs)
    wt = port.random_dictionary(d, h, 41, 2.0)
    y = port.ld_generate(pr, wt, 0.3, n, 42)
    w0, _, s20 = port.baseline_init(np.r_[y, y + 0.1], h, 43)
    m = gpu_model(pkg, pr, d, h, hp, g)
    m.load(y)
    p0 = gpu_params(pkg, pr, w0, s20)
    assert np.array_equal(m.candidates(p0), port.ld_candidates(pr, w0, s20, y, hp))
    check_stats(m.estep_stats(p0), port.ld_estep_stats(pr, w0, s20, y, hp, g))
    wo, pio, qo, s2o, fo = port.ld_step(pr, w0, s20, y, hp, g)
    check_step(pr, m.step(p0), wo, pio, qo, s2o, fo)
    if hp == h == g:  # exact mode: F is the exact log-likelihood
        ll = port.ld_exact_log_likelihood(pr, w0, s20, y)
        assert abs(fo - ll) <= 1e-10 * abs(ll)
    m.close()

"""Oracle pinning for the max-causes log-joint:
MaxCausesModel (max_causes.cpp) — per-state max-winner residual, the winner
statistics, the fixed-point M-step and the residual pass for σ² — restated in
oracle/bsc_oracle.c (mca_*) and checked bit for bit against the reference build.
"""
import numpy as np
import pytest

from conftest import MCA_GOLDEN_CASES, MCA_MODES, load_golden


@pytest.mark.parametrize("name", MCA_GOLDEN_CASES)
def test_port_matches_reference_golden_mca(port, name):
    g = load_golden(name)
    mode, rho = MCA_MODES[int(g["mode"])], float(g["rho"])
    y, w0, pi0, s20 = g["y"], g["W0"], float(g["pi0"]), float(g["sigma2_0"])
    hp, gm, T = int(g["hprime"]), int(g["gamma"]), float(g["temperature"])
    assert np.array_equal(port.mca_candidates(mode, w0, pi0, s20, y, hp), g["candidates"])
    st = port.mca_estep_stats(mode, w0, pi0, s20, y, hp, gm, T, rho=rho)
    for k in ["winner_num", "winner_den", "sum_act", "log_partition"]:
        assert np.array_equal(st[k], g["stats_" + k]), k
    w1, p1, s1, f = port.mca_step(mode, w0, pi0, s20, y, hp, gm, T, shards=3, workers=2, rho=rho)
    assert np.array_equal(w1, g["W1"]) and p1 == g["pi1"] and s1 == g["sigma2_1"] and f == g["F0"]
    w, p, s = w0, pi0, s20
    for i in range(len(g["traj_F"])):
        w, p, s, f = port.mca_step(mode, w, p, s, y, hp, gm, 1.0, rho=rho)
        assert np.array_equal(w, g["traj_W"][i]) and p == g["traj_pi"][i]
        assert s == g["traj_sigma2"][i] and f == g["traj_F"][i]
    ms, mm, ex = port.mca_inference(mode, w0, pi0, s20, y, hp, gm)
    assert np.array_equal(ms, g["map_states"]) and np.array_equal(mm, g["map_mass"])
    assert np.array_equal(ex, g["expected"])
    if "exact_ll0" in g:
        assert port.mca_exact_log_likelihood(mode, w0, pi0, s20, y) == g["exact_ll0"]


def test_mca_exact_mode_equals_exact_likelihood(port):
    """H' = γ = H: the truncated free energy is the exact log-likelihood."""
    rng = np.random.default_rng(5)
    w = np.abs(rng.normal(size=(6, 5))) + 0.2
    y = port.mca_generate("mca", w, 0.3, 0.4, 30, 6)
    st = port.mca_estep_stats("mca", w, 0.3, 0.4, y, 5, 5)
    ll = port.mca_exact_log_likelihood("mca", w, 0.3, 0.4, y)
    assert abs(st["log_partition"] - ll) <= 1e-10 * abs(ll)


def test_mca_log_joint_and_errors(port):
    from oracle.oracle import OracleError

    w = np.array([[1.0, 2.0], [3.0, 0.5]])
    y = np.array([2.5, 1.0])
    # winners: d0 → unit 1 (2.0), d1 → unit 0 (3.0); resid = 0.25 + 4 = 4.25
    lj = port.mca_log_joint("mca", w, 0.5, 1.0, y, np.array([1.0, 1.0]))
    assert abs(lj - (2 * np.log(0.5) - np.log(2 * np.pi) - 4.25 / 2)) < 1e-12
    with pytest.raises(OracleError):  # mca weights must respect the floor (max_causes.cpp:108-112)
        port.mca_estep_stats("mca", -w, 0.5, 1.0, y[None, :], 1, 1)
    with pytest.raises(OracleError):  # soft winners need the max mode (:97-98)
        port.mca_estep_stats("mmca", w, 0.5, 1.0, y[None, :], 1, 1, rho=1.0)


def test_port_matches_reference_live_mca(port, ref):
    rng = np.random.default_rng(9)
    w = np.abs(rng.normal(size=(10, 8))) + 0.1
    y = ref.mca_generate("mca", w, 0.25, 0.3, 40, 2)
    a, b = ref.mca_estep_stats("mca", w, 0.25, 0.3, y, 5, 3), port.mca_estep_stats("mca", w, 0.25, 0.3, y, 5, 3)
    assert all(np.array_equal(a[k], b[k]) for k in ["winner_num", "winner_den", "sum_act", "log_partition"])
    A, B = ref.mca_step("mmca", w - 0.5, 0.25, 0.3, y, 5, 3, 1.0, 2, 2), port.mca_step("mmca", w - 0.5, 0.25, 0.3, y,
                                                                                       5, 3, 1.0, 2, 2)
    assert np.array_equal(A[0], B[0]) and A[1:] == B[1:]

"""Oracle pinning for the other linear discrete families:
TSC (values {−1, +1}) and DSC (an alphabet with 0) run through the same
estep_impl / mstep (linear_discrete.cpp:71-97, :202-408) with the value
odometer of the state template (truncation.cpp:116-147). The C restatement
(oracle/bsc_oracle.c, ld_*) must match the reference build bit for bit.
"""
import numpy as np
import pytest

from conftest import LD_GOLDEN_CASES, golden_prior, load_golden

FIELDS = ["sum_s", "sum_ssT", "sum_y_sT", "value_counts"]


@pytest.mark.parametrize("name", LD_GOLDEN_CASES)
def test_port_matches_reference_golden_families(port, name):
    g = load_golden(name)
    pr = golden_prior(g)
    y, w0, s20 = g["y"], g["W0"], float(g["sigma2_0"])
    hp, gm, T = int(g["hprime"]), int(g["gamma"]), float(g["temperature"])
    assert np.array_equal(port.ld_candidates(pr, w0, s20, y, hp), g["candidates"])
    st = port.ld_estep_stats(pr, w0, s20, y, hp, gm, T)
    for k in FIELDS:
        assert np.array_equal(st[k], g["stats_" + k]), k
    assert st["log_partition"] == g["stats_log_partition"] and st["sum_y2"] == g["stats_sum_y2"]
    w1, p1, q1, s1, f = port.ld_step(pr, w0, s20, y, hp, gm, T, shards=3, workers=2)
    assert np.array_equal(w1, g["W1"]) and s1 == g["sigma2_1"] and f == g["F0"]
    if pr.family == "dsc":
        assert np.array_equal(q1, g["probs1"])
    else:
        assert p1 == g["pi1"]
    w, p, s = w0, pr, s20
    from oracle.oracle import Prior

    for i in range(len(g["traj_F"])):
        w, pi, q, s, f = port.ld_step(p, w, s, y, hp, gm, 1.0)
        assert np.array_equal(w, g["traj_W"][i]) and s == g["traj_sigma2"][i] and f == g["traj_F"][i]
        p = Prior(p.family, pi if pi is not None else 0.0, p.alpha, q)
    ms, mm, ex = port.ld_inference(pr, w0, s20, y, hp, gm)
    assert np.array_equal(ms, g["map_states"]) and np.array_equal(mm, g["map_mass"])
    assert np.array_equal(ex, g["expected"])
    if "exact_ll0" in g:
        assert port.ld_exact_log_likelihood(pr, w0, s20, y) == g["exact_ll0"]


def test_family_state_counts(port):
    # 1 + H·V + Σ_k C(H',k)·V^k (truncation.cpp:83-93)
    assert port.ld_state_count(10, 4, 2, 2) == 1 + 20 + 6 * 4
    assert port.ld_state_count(6, 6, 6, 2) == 3 ** 6
    assert port.ld_state_count(12, 6, 3, 3) == 1 + 36 + 15 * 9 + 20 * 27


def test_exact_mode_equals_exact_likelihood_tsc(port):
    """H' = γ = H enumerates the whole ternary state space: F = exact LL."""
    from oracle.oracle import Prior

    rng = np.random.default_rng(3)
    w = rng.normal(size=(7, 5))
    pr = Prior("tsc", 0.3)
    y = port.ld_generate(pr, w, 0.5, 40, 4)
    st = port.ld_estep_stats(pr, w, 0.5, y, 5, 5)
    ll = port.ld_exact_log_likelihood(pr, w, 0.5, y)
    assert abs(st["log_partition"] - ll) <= 1e-10 * abs(ll)


def test_dsc_validation(port):
    from oracle.oracle import OracleError, Prior

    w = np.ones((4, 3))
    y = np.ones((5, 4))
    for alpha, probs in [([-1.0, 1.0], [0.5, 0.5]),            # no zero
                         ([1.0, 0.0, -1.0], [0.2, 0.6, 0.2]),   # not ascending
                         ([-1.0, 0.0, 1.0], [0.2, 0.6, 0.3]),   # does not sum to 1
                         ([-1.0, 0.0, 1.0], [0.0, 0.8, 0.2])]:  # non-positive
        with pytest.raises(OracleError) as e:
            port.ld_estep_stats(Prior("dsc", 0.0, alpha, probs), w, 1.0, y, 2, 2)
        assert e.value.code == 2


def test_port_matches_reference_live_families(port, ref):
    from oracle.oracle import Prior

    rng = np.random.default_rng(11)
    w = rng.normal(size=(12, 9))
    for pr in [Prior("tsc", 0.2), Prior("dsc", 0.0, [-2.0, 0.0, 0.5, 1.5], [0.1, 0.6, 0.2, 0.1])]:
        y = ref.ld_generate(pr, w, 0.5, 50, 2)
        assert np.array_equal(y, port.ld_generate(pr, w, 0.5, 50, 2))
        a, b = ref.ld_estep_stats(pr, w, 0.5, y, 5, 3), port.ld_estep_stats(pr, w, 0.5, y, 5, 3)
        for k in FIELDS:
            assert np.array_equal(a[k], b[k]), k
        A, B = ref.ld_step(pr, w, 0.5, y, 5, 3, 1.0, 3, 3), port.ld_step(pr, w, 0.5, y, 5, 3, 1.0, 3, 3)
        assert np.array_equal(A[0], B[0]) and A[3] == B[3] and A[4] == B[4]

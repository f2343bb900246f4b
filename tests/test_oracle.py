"""CPU: pin the oracle (oracle/bsc_oracle.c) before trusting it.

1. SPEC.md known answers for the path (select_candidates, state counts,
   log_sum_exp, BSC log_joint, degenerate E/M-steps).
2. Bit-exact agreement with the reference's own code on the committed golden
   fixtures (tests/golden, produced by oracle/_ref = /root/reference sources).
3. Live bit-exact agreement with oracle/_ref where it is built.
4. Model properties: exact mode equals the exact log-likelihood, truncated F is
   a lower bound, exact-mode EM is monotone.
"""
import math

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden


# ----------------------------------------------------------- SPEC known answers
def test_select_candidates_spec(port):
    # SPEC.md:107-109
    assert list(port.select_candidates([0.1, 0.9, 0.5, 0.9], 2)) == [1, 3]
    assert list(port.select_candidates([0.3] * 5, 2)) == [0, 1]
    assert list(port.select_candidates([0.3, 0.1, 0.2], 3)) == [0, 1, 2]


def test_select_candidates_errors(port):
    from oracle.oracle import OracleError

    with pytest.raises(OracleError) as e:
        port.select_candidates([0.1, 0.2], 3)
    assert e.value.code == 2
    with pytest.raises(OracleError) as e:
        port.select_candidates([0.1, float("nan")], 1)
    assert e.value.code == 2


def test_state_counts_spec(port):
    assert port.state_count(10, 4, 2) == 17
    assert port.state_count(3, 3, 3) == 8  # all binary states
    assert port.state_count(7, 5, 1) == 8  # gamma = 1 → 1 + H
    # BASELINE configs under the reference's rule
    assert port.state_count(10, 10, 10) == 1024
    assert port.state_count(20, 10, 4) == 396
    assert port.state_count(300, 12, 4) == 1082
    assert port.state_count(1000, 14, 5) == 4459


def test_enumeration_order(port):
    states = port.enumerate_binary([1, 4, 6, 9], 10, 3)
    assert states.shape == (1 + 10 + 6 + 4, 10)
    assert states[0].sum() == 0
    for h in range(10):
        assert states[1 + h].sum() == 1 and states[1 + h, h] == 1
    # DFS over positions, prefixes first (truncation.cpp:116-147)
    multi = [tuple(np.flatnonzero(s)) for s in states[11:]]
    assert multi == [(1, 4), (1, 4, 6), (1, 4, 9), (1, 6), (1, 6, 9), (1, 9), (4, 6), (4, 6, 9), (4, 9), (6, 9)]


def test_log_sum_exp_spec(port):
    assert port.log_sum_exp([3.0]) == 3.0
    assert abs(port.log_sum_exp([0.0, 0.0]) - math.log(2)) < 1e-15
    assert abs(port.log_sum_exp([-1000.0, -1000.0]) - (-1000 + math.log(2))) < 1e-12


def test_log_joint_spec(port):
    # D=1, H=1, W=[[2]], sigma2=1, pi=.5, y=2, s=1 → ln .5 − ½ ln 2π
    v = port.log_joint(np.array([[2.0]]), 0.5, 1.0, np.array([2.0]), np.array([1.0]))
    assert abs(v - (math.log(0.5) - 0.5 * math.log(2 * math.pi))) < 1e-14
    assert abs(v - (-1.61209)) < 1e-5
    # log prior of s = 0 with H = 4, pi = .5
    v0 = port.log_joint(np.zeros((1, 4)), 0.5, 1.0, np.zeros(1), np.zeros(4))
    assert abs(v0 - (4 * math.log(0.5) - 0.5 * math.log(2 * math.pi))) < 1e-14


def test_mstep_degenerate_spec(port):
    # all posterior mass on s = e_1 for one point → W' column 1 = y
    y = np.array([[1.5, -2.0, 0.25]])
    st = dict(sum_s=np.array([1.0, 0.0]), sum_ssT=np.diag([1.0, 0.0]), sum_y_sT=np.c_[y.T, np.zeros(3)],
              value_counts=np.array([1.0]), sum_y2=float((y ** 2).sum()), log_partition=0.0, points=1)
    w, pi, s2 = port.mstep(st, np.ones((3, 2)), 0.5, 1.0)
    assert np.allclose(w[:, 0], y[0], rtol=1e-8)
    # all mass on the zero state → pi hits the lower clip
    st0 = dict(sum_s=np.zeros(2), sum_ssT=np.zeros((2, 2)), sum_y_sT=np.zeros((3, 2)), value_counts=np.zeros(1),
               sum_y2=1.0, log_partition=0.0, points=1)
    w0, pi0, _ = port.mstep(st0, np.ones((3, 2)), 0.5, 1.0)
    assert pi0 == 1e-6 and np.array_equal(w0, np.ones((3, 2)))


# ---------------------------------------------------- golden (reference) fixtures
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_port_matches_reference_golden(port, name):
    g = load_golden(name)
    y, w0, pi0, s20 = g["y"], g["W0"], float(g["pi0"]), float(g["sigma2_0"])
    hp, gm, T = int(g["hprime"]), int(g["gamma"]), float(g["temperature"])
    assert np.array_equal(port.candidates(w0, pi0, s20, y, hp), g["candidates"])
    st = port.estep_stats(w0, pi0, s20, y, hp, gm, T)
    for k in ["sum_s", "sum_ssT", "sum_y_sT", "value_counts", "sum_y2", "log_partition", "points"]:
        assert np.array_equal(np.asarray(st[k]), g["stats_" + k]), k
    w1, p1, s1, f = port.step(w0, pi0, s20, y, hp, gm, T, shards=3, workers=2)
    assert np.array_equal(w1, g["W1"]) and p1 == g["pi1"] and s1 == g["sigma2_1"] and f == g["F0"]
    w, p, s = w0, pi0, s20
    for i in range(len(g["traj_F"])):
        w, p, s, f = port.step(w, p, s, y, hp, gm)
        assert np.array_equal(w, g["traj_W"][i]) and p == g["traj_pi"][i] and s == g["traj_sigma2"][i]
        assert f == g["traj_F"][i]
    ms, mm, ex = port.inference(w0, pi0, s20, y, hp, gm)
    assert np.array_equal(ms, g["map_states"]) and np.array_equal(mm, g["map_mass"])
    assert np.array_equal(ex, g["expected"])
    if "exact_ll0" in g:
        assert port.exact_log_likelihood(w0, pi0, s20, y) == g["exact_ll0"]


def test_port_matches_reference_live(port, ref):
    y, _ = ref.make_bars(5, 120, seed=3)
    assert np.array_equal(y, port.make_bars(5, 120, seed=3)[0])
    w, pi, s2 = port.baseline_init(y, 10, 3)
    for hp, gm in [(10, 10), (7, 4), (3, 1), (1, 1)]:
        a = port.step(w, pi, s2, y, hp, gm, shards=4, workers=3)
        b = ref.step(w, pi, s2, y, hp, gm, shards=4, workers=3)
        assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]
    assert np.array_equal(port.rng_normals(9, 4, 1, 50), ref.rng_normals(9, 4, 1, 50))
    wt = port.random_dictionary(12, 9, 1)
    assert np.array_equal(port.generate(wt, 0.2, 0.3, 64, 8), ref.generate(wt, 0.2, 0.3, 64, 8))


# ------------------------------------------------------------------ properties
def test_exact_mode_equals_exact_likelihood(port):
    g = load_golden("spec_acc1_d9_h6_exact")
    y = g["y"]
    w, p, s = g["W0"], float(g["pi0"]), float(g["sigma2_0"])
    prev = -np.inf
    for _ in range(5):
        ll = port.exact_log_likelihood(w, p, s, y)
        w2, p2, s2, f = port.step(w, p, s, y, 6, 6)
        assert abs(f - ll) <= 1e-10 * abs(ll)  # SPEC acceptance 1
        assert f >= prev - 1e-9 * abs(f)  # EM monotonicity in exact mode
        prev, w, p, s = f, w2, p2, s2


def test_truncated_free_energy_is_lower_bound(port):
    y, _ = port.make_bars(4, 150, seed=2)
    w, p, s = port.baseline_init(y, 8, 2)
    for _ in range(3):
        ll = port.exact_log_likelihood(w, p, s, y)
        w2, p2, s2, f = port.step(w, p, s, y, 4, 3)
        assert f <= ll + 1e-9 * abs(ll)  # SPEC acceptance 4
        w, p, s = w2, p2, s2


def test_shard_boundaries_determinism(port):
    y, _ = port.make_bars(5, 211, seed=4)
    w, p, s = port.baseline_init(y, 10, 4)
    a = port.step(w, p, s, y, 6, 3, shards=4, workers=1)
    b = port.step(w, p, s, y, 6, 3, shards=4, workers=4)
    assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]  # SPEC acceptance 10
    c = port.step(w, p, s, y, 6, 3, shards=1, workers=1)
    assert abs(c[3] - a[3]) <= 1e-12 * abs(a[3])

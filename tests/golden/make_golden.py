"""Generates the golden fixtures in this directory from the REFERENCE ITSELF:
oracle/_ref/libprsp_ref.so is the prsp sources under /root/reference/proj/src
compiled unmodified (against oracle/eigen_shim) by oracle/Makefile. Run here
(where /root/reference exists):  python tests/golden/make_golden.py

Each .npz holds the inputs of one small case and the reference's outputs:
per-point candidate sets, estep_stats fields, one-step params and F, a short
free-running trajectory, and the inference readout.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle, Prior  # noqa: E402

R = Oracle("ref")


def case(name, y, w0, pi0, s20, hprime, gamma, iters=3, temperature=1.0):
    d, h = w0.shape
    out = dict(y=y, W0=w0, pi0=pi0, sigma2_0=s20, hprime=hprime, gamma=gamma, temperature=temperature)
    out["candidates"] = R.candidates(w0, pi0, s20, y, hprime)
    st = R.estep_stats(w0, pi0, s20, y, hprime, gamma, temperature)
    for k, v in st.items():
        out["stats_" + k] = np.asarray(v)
    w1, p1, s1, f = R.step(w0, pi0, s20, y, hprime, gamma, temperature, shards=3, workers=2)
    out.update(W1=w1, pi1=p1, sigma2_1=s1, F0=f)
    ws, ps, ss, fs = [], [], [], []
    w, p, s = w0, pi0, s20
    for _ in range(iters):
        w, p, s, f = R.step(w, p, s, y, hprime, gamma, 1.0)
        ws.append(w), ps.append(p), ss.append(s), fs.append(f)
    out.update(traj_W=np.array(ws), traj_pi=np.array(ps), traj_sigma2=np.array(ss), traj_F=np.array(fs))
    ms, mm, ex = R.inference(w0, pi0, s20, y, hprime, gamma)
    out.update(map_states=ms, map_mass=mm, expected=ex)
    if h <= 10:
        out["exact_ll0"] = R.exact_log_likelihood(w0, pi0, s20, y)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k: np.shape(v) for k, v in out.items()})


def ld_case(name, prior, y, w0, s20, hprime, gamma, iters=3, temperature=1.0):
    """A linear discrete family case (tsc/dsc): the prior's family code, pi,
    alphabet and probabilities are stored beside the reference outputs."""
    d, h = w0.shape
    alpha = prior.alpha if prior.alpha is not None else np.zeros(0)
    probs = prior.probs if prior.probs is not None else np.zeros(0)
    out = dict(y=y, W0=w0, family=prior.code, pi0=prior.pi, alpha=alpha, probs0=probs, sigma2_0=s20,
               hprime=hprime, gamma=gamma, temperature=temperature)
    out["candidates"] = R.ld_candidates(prior, w0, s20, y, hprime)
    st = R.ld_estep_stats(prior, w0, s20, y, hprime, gamma, temperature)
    for k, v in st.items():
        out["stats_" + k] = np.asarray(v)
    w1, p1, q1, s1, f = R.ld_step(prior, w0, s20, y, hprime, gamma, temperature, shards=3, workers=2)
    out.update(W1=w1, pi1=p1 if p1 is not None else 0.0, probs1=q1 if q1 is not None else np.zeros(0),
               sigma2_1=s1, F0=f)
    ws, ps, qs, ss, fs = [], [], [], [], []
    w, pr, s = w0, prior, s20
    for _ in range(iters):
        w, p, q, s, f = R.ld_step(pr, w, s, y, hprime, gamma, 1.0)
        pr = Prior(pr.family, p if p is not None else 0.0, pr.alpha, q)
        ws.append(w), ps.append(pr.pi), qs.append(q if q is not None else np.zeros(0)), ss.append(s), fs.append(f)
    out.update(traj_W=np.array(ws), traj_pi=np.array(ps), traj_probs=np.array(qs), traj_sigma2=np.array(ss),
               traj_F=np.array(fs))
    ms, mm, ex = R.ld_inference(prior, w0, s20, y, hprime, gamma)
    out.update(map_states=ms, map_mass=mm, expected=ex)
    if h <= 6:
        out["exact_ll0"] = R.ld_exact_log_likelihood(prior, w0, s20, y)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k: np.shape(v) for k, v in out.items()})


def mca_case(name, mode, y, w0, pi0, s20, hprime, gamma, iters=3, temperature=1.0, rho=0.0):
    """A max-causes case (max_causes.cpp): E pass stats, one step (fixed-point
    W/π then the residual pass for σ²), a trajectory and the inference readout."""
    d, h = w0.shape
    out = dict(y=y, W0=w0, mode=0 if mode == "mca" else 1, rho=rho, pi0=pi0, sigma2_0=s20, hprime=hprime,
               gamma=gamma, temperature=temperature)
    out["candidates"] = R.mca_candidates(mode, w0, pi0, s20, y, hprime)
    st = R.mca_estep_stats(mode, w0, pi0, s20, y, hprime, gamma, temperature, rho=rho)
    for k, v in st.items():
        out["stats_" + k] = np.asarray(v)
    w1, p1, s1, f = R.mca_step(mode, w0, pi0, s20, y, hprime, gamma, temperature, shards=3, workers=2, rho=rho)
    out.update(W1=w1, pi1=p1, sigma2_1=s1, F0=f)
    ws, ps, ss, fs = [], [], [], []
    w, p, s = w0, pi0, s20
    for _ in range(iters):
        w, p, s, f = R.mca_step(mode, w, p, s, y, hprime, gamma, 1.0, rho=rho)
        ws.append(w), ps.append(p), ss.append(s), fs.append(f)
    out.update(traj_W=np.array(ws), traj_pi=np.array(ps), traj_sigma2=np.array(ss), traj_F=np.array(fs))
    ms, mm, ex = R.mca_inference(mode, w0, pi0, s20, y, hprime, gamma)
    out.update(map_states=ms, map_mass=mm, expected=ex)
    if h <= 10:
        out["exact_ll0"] = R.mca_exact_log_likelihood(mode, w0, pi0, s20, y)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k: np.shape(v) for k, v in out.items()})


def baseline_init(y, h, seed):
    # BASELINE.json's init recipe is not reference code (SURVEY.md §8(d) pins
    # it); the C restatement computes it. The reference then runs from it.
    return Oracle("port").baseline_init(y, h, seed)


if __name__ == "__main__":
    # bars 5×5 (BASELINE c0 family), truncated
    y, _ = R.make_bars(5, 200, seed=0)
    w, p, s = baseline_init(y, 10, 0)
    case("bars5_h10_hp6_g3", y, w, p, s, 6, 3)
    # same data, exact mode H'=H=γ (the reference's exact_log_likelihood applies)
    case("bars5_exact_h10", y, w, p, s, 10, 10, iters=3)
    # bars 10×10 (c1 family) at T=2 (annealed posterior)
    y, _ = R.make_bars(10, 150, seed=1)
    w, p, s = baseline_init(y, 20, 1)
    case("bars10_h20_hp10_g4_T2", y, w, p, s, 10, 4, temperature=2.0)
    # random unit-norm dictionary (c2 family), reference generate()
    wt = Oracle("port").random_dictionary(32, 40, 5, 5.0)
    y = R.generate(wt, 4 / 40, 0.25, 300, 5)
    w, p, s = baseline_init(y, 40, 5)
    case("rand_d32_h40_hp8_g3", y, w, p, s, 8, 3)
    # SPEC acceptance 1 shape: D=9, H=6, N=200, H'=H=γ=6
    wt = Oracle("port").random_dictionary(9, 6, 7, 3.0)
    y = R.generate(wt, 0.3, 0.5, 200, 7)
    w, p, s = R.standard_init(y, 6, 6, 6, 11)
    case("spec_acc1_d9_h6_exact", y, w, p, s, 6, 6, iters=5)
    # linear discrete families through the same path:
    # ternary sparse coding, and a discrete alphabet with 0
    wt = Oracle("port").random_dictionary(16, 12, 9, 3.0)
    tsc = Prior("tsc", 0.2)
    y = R.ld_generate(tsc, wt, 0.3, 160, 9)
    w, _, s = baseline_init(y, 12, 9)
    ld_case("ld_tsc_d16_h12_hp6_g3", Prior("tsc", 1.0 / 12), y, w, s, 6, 3)
    ld_case("ld_tsc_d16_h12_hp6_g3_T2", Prior("tsc", 1.0 / 12), y, w, s, 6, 3, iters=2, temperature=2.0)
    wt6 = Oracle("port").random_dictionary(10, 6, 13, 3.0)
    y = R.ld_generate(tsc, wt6, 0.4, 80, 13)
    w, _, s = baseline_init(y, 6, 13)
    ld_case("ld_tsc_exact_d10_h6", Prior("tsc", 0.25), y, w, s, 6, 6, iters=2)
    dsc = Prior("dsc", alpha=[-1.0, 0.0, 1.0, 2.0], probs=[0.05, 0.8, 0.1, 0.05])
    wt = Oracle("port").random_dictionary(16, 10, 17, 3.0)
    y = R.ld_generate(dsc, wt, 0.3, 160, 17)
    w, _, s = baseline_init(y, 10, 17)
    ld_case("ld_dsc_d16_h10_hp5_g3", Prior("dsc", alpha=dsc.alpha, probs=[0.1, 0.7, 0.1, 0.1]), y, w, s, 5, 3)
    # max causes: max-superposition bars and an absmax dictionary
    y, truth = R.make_bars(4, 150, max_mode=True, noise=1.0, seed=31)
    w, p, s = R.mca_standard_init("mca", y, 8, 6, 31)
    mca_case("mca_bars4_h8_hp6_g3", "mca", y, w, p, s, 6, 3)
    mca_case("mca_bars4_h8_hp6_g3_soft", "mca", y, w, p, s, 6, 3, iters=2, rho=2.0)
    wt = Oracle("port").random_dictionary(12, 10, 33, 3.0)
    y = R.mca_generate("mmca", wt, 0.2, 0.3, 120, 33)
    w, p, s = R.mca_standard_init("mmca", y, 10, 5, 33)
    mca_case("mca_mmca_d12_h10_hp5_g3_T2", "mmca", y, w, p, s, 5, 3, iters=2, temperature=2.0)

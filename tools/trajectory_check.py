"""Full-size parity run of a BASELINE workload on one GPU
against the reference itself (oracle/_ref: the prsp sources built by
oracle/Makefile), on all host threads with ShardPlan::with_shards(N, t, t).

At every EM iteration, from the reference's parameters:
  * candidates: the GPU's candidate set of EVERY point against the reference's
    (harness restatement of estep_impl's selection over the same Eigen-shim
    operations, oracle/ref_harness.cpp ref_candidates) -- must be identical;
  * one step (primary gate): W, pi, sigma2 and F of the GPU step against the
    reference step -- within 1e-6 relative (W Frobenius);
and the free-running GPU trajectory against the reference's (secondary).

    python tools/trajectory_check.py c2 20 [--out profiles/r02_parity_full_c2.txt]

Exit status 1 if any candidate set differs or a one-step difference exceeds 1e-6.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1908_06843_b200 import BscGpuModel, BscParams, TruncationConfig, configs  # noqa: E402

TOL = 1e-6


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="c2")
    ap.add_argument("iters", nargs="?", type=int, default=20)
    ap.add_argument("--points", type=int, default=0, help="first N points (default: the workload's N)")
    ap.add_argument("--no-free", action="store_true", help="skip the free-running trajectory")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    w = configs.CONFIGS[args.workload]
    n = args.points or w.N
    lines = []

    def log(s):
        print(s, flush=True)
        lines.append(s)

    t0 = time.perf_counter()
    if w.scaling == "strong":
        y = configs.data(w, rows=(0, n))
        p = configs.init(w, configs.data(w, rows=(0, min(n, configs.BLOCK))))
    else:
        y = configs.data(w, n)
        p = configs.init(w, y)
    threads = os.cpu_count() or 1
    ref = O.Oracle("ref")
    sess = O.RefSession(y, w.H, w.hprime, w.gamma)
    m = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma))
    m.load(y)
    free = p
    worst = dict(W=0.0, pi=0.0, sigma2=0.0, F=0.0)
    bad_total = 0
    log(f"{args.workload}: N={n} D={w.D} H={w.H} H'={w.hprime} gamma={w.gamma}; reference = oracle/_ref on "
        f"{threads} host threads; data + init {time.perf_counter() - t0:.0f} s")
    log("iter  cand: differing/points  | one-step: dW      dpi       dsigma2   dF       | free-running: dW      dF"
        "        | ref step s, ref cand s")
    for it in range(args.iters):
        t = time.perf_counter()
        cref = ref.candidates(p.W, p.pi, p.sigma2, y, w.hprime, threads=threads)
        tc = time.perf_counter() - t
        cg = m.candidates(p)
        nbad = int(np.count_nonzero(np.any(cg != cref, axis=1)))
        bad_total += nbad
        t = time.perf_counter()
        wo, pio, s2o, fo = sess.step(p.W, p.pi, p.sigma2, threads, threads)
        tref = time.perf_counter() - t
        r = m.step(p)
        d = dict(W=rel(r.params.W, wo), pi=abs(r.params.pi - pio) / pio, sigma2=abs(r.params.sigma2 - s2o) / s2o,
                 F=abs(r.free_energy - fo) / abs(fo))
        for k in worst:
            worst[k] = max(worst[k], d[k])
        fr = ""
        if not args.no_free:
            rf = m.step(free)
            free = rf.params
            fr = f"{rel(free.W, wo):.2e}  {abs(rf.free_energy - fo) / abs(fo):.2e}"
        log(f"{it:4d}  {nbad:9d}/{n:<9d}      | {d['W']:.2e}  {d['pi']:.2e}  {d['sigma2']:.2e}  {d['F']:.2e} | "
            f"{fr:24s} | {tref:.1f}, {tc:.1f}")
        p = BscParams(wo, pio, s2o)
    ok = bad_total == 0 and all(v <= TOL for v in worst.values())
    log(f"differing candidate sets over {args.iters} iterations x {n} points: {bad_total}")
    log("worst one-step relative differences: " + ", ".join(f"{k} {v:.2e}" for k, v in worst.items()) +
        f" (tolerance {TOL:g}) -> {'PASS' if ok else 'FAIL'}")
    del sess
    m.close()
    if args.out:
        with open(args.out, "w") as f:
            f.write("\n".join(lines) + "\n")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

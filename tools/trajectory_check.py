"""Full-size parity run: at every EM iteration of a BASELINE
workload, the GPU step from the reference's parameters against the reference
step itself (primary gate: one-step parity), plus the free-running GPU
trajectory against the reference's (secondary).

    python tools/trajectory_check.py c2 20     # workload, iterations

The reference is oracle/_ref (the reference sources built by oracle/Makefile),
run on all host threads with ShardPlan::with_shards(N, threads, threads).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1908_06843_b200 import BscGpuModel, BscParams, TruncationConfig, configs  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    w = configs.CONFIGS[name]
    y = configs.data(w)
    p = configs.init(w, y)
    threads = os.cpu_count() or 1
    sess = O.RefSession(y, w.H, w.hprime, w.gamma)
    m = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma))
    m.load(y)
    free = p
    worst = dict(W=0.0, pi=0.0, sigma2=0.0, F=0.0)
    print(f"{name}: N={w.N} D={w.D} H={w.H} H'={w.hprime} gamma={w.gamma}, reference on {threads} threads")
    print("iter  one-step: dW        dpi       dsigma2   dF      | free-running: dW        dF")
    for it in range(iters):
        t = time.perf_counter()
        wo, pio, s2o, fo = sess.step(p.W, p.pi, p.sigma2, threads, threads)
        tref = time.perf_counter() - t
        r = m.step(p)
        d = dict(W=rel(r.params.W, wo), pi=abs(r.params.pi - pio) / pio, sigma2=abs(r.params.sigma2 - s2o) / s2o,
                 F=abs(r.free_energy - fo) / abs(fo))
        for k in worst:
            worst[k] = max(worst[k], d[k])
        rf = m.step(free)
        free = rf.params
        print(f"{it:4d}  {d['W']:.2e}  {d['pi']:.2e}  {d['sigma2']:.2e}  {d['F']:.2e} | "
              f"{rel(free.W, wo):.2e}  {abs(rf.free_energy - fo) / abs(fo):.2e}   ({tref:.1f} s reference step)")
        p = BscParams(wo, pio, s2o)
    print("worst one-step relative differences:", {k: f"{v:.2e}" for k, v in worst.items()},
          "(north-star tolerance 1e-6)")
    del sess


if __name__ == "__main__":
    main()

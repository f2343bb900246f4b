"""Developer check on a GPU box: parity of the sm_100a path against the oracle on
small cases, then a timing breakdown at c2. Prints one JSON object per line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle  # noqa: E402
from paper_1908_06843_b200 import BscGpuModel, TruncationConfig, configs  # noqa: E402

O = Oracle("port")


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def parity(name, w, n):
    y = configs.data(w, n)
    p = configs.init(w, y)
    m = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma))
    m.load(y)
    out = {"case": name, "n": n}
    t = time.time()
    cg = m.candidates(p)
    co = O.candidates(p.W, p.pi, p.sigma2, y, w.hprime)
    out["cand_equal"] = bool(np.array_equal(cg, co))
    out["cand_mismatch_rows"] = int((cg != co).any(axis=1).sum())
    sg = m.estep_stats(p)
    so = O.estep_stats(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma)
    for k in ["sum_s", "sum_ssT", "sum_y_sT", "value_counts", "sum_y2", "log_partition"]:
        out["rel_" + k] = rel(getattr(sg, k), so[k])
    out["points"] = sg.points == so["points"]
    r = m.step(p)
    wo, pio, s2o, fo = O.step(p.W, p.pi, p.sigma2, y, w.hprime, w.gamma)
    out.update(rel_W=rel(r.params.W, wo), rel_pi=abs(r.params.pi - pio) / pio, rel_s2=abs(r.params.sigma2 - s2o) / s2o,
               rel_F=abs(r.free_energy - fo) / abs(fo))
    # M-step alone from the oracle's statistics
    pm = m.mstep(so, p)
    wm, pim, s2m = O.mstep(so, p.W, p.pi, p.sigma2)
    out.update(mstep_rel_W=rel(pm.W, wm), mstep_rel_pi=abs(pm.pi - pim) / pim, mstep_rel_s2=abs(pm.sigma2 - s2m) / s2m)
    out["secs"] = round(time.time() - t, 2)
    print(json.dumps(out), flush=True)
    m.close()


def trajectory(name, w, n, iters):
    y = configs.data(w, n)
    p = configs.init(w, y)
    m = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma))
    m.load(y)
    pg, po = p.copy(), p.copy()
    worst = {}
    for it in range(iters):
        r = m.step(pg)
        wo, pio, s2o, fo = O.step(po.W, po.pi, po.sigma2, y, w.hprime, w.gamma)
        # one-step parity from the oracle's own params
        r1 = m.step(po)
        d = dict(F=abs(r.free_energy - fo) / abs(fo), W=rel(r.params.W, wo), one_W=rel(r1.params.W, wo),
                 one_F=abs(r1.free_energy - fo) / abs(fo), one_s2=abs(r1.params.sigma2 - s2o) / s2o)
        for k, v in d.items():
            worst[k] = max(worst.get(k, 0.0), v)
        pg = r.params
        from paper_1908_06843_b200.bsc import BscParams
        po = BscParams(wo, pio, s2o)
    print(json.dumps({"trajectory": name, "iters": iters, "worst": worst}), flush=True)


def timing(name, w, n, steps=5):
    y = configs.data(w, n)
    p = configs.init(w, y)
    m = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma))
    m.load(y)
    m.set_timing(True)
    m.set_params(p)
    pp = p
    for i in range(steps):
        t = time.time()
        r = m.step(pp)
        dt = time.time() - t
        pp = r.params
        print(json.dumps({"timing": name, "n": n, "step": i, "wall_ms": dt * 1e3, **m.timings(), "F": r.free_energy}),
              flush=True)


if __name__ == "__main__":
    C = configs.CONFIGS
    parity("c0", C["c0"], 1000)
    parity("c1", C["c1"], 2000)
    parity("c2", C["c2"], 3000)
    trajectory("c1", C["c1"], 2000, 5)
    timing("c2", C["c2"], 200_000)
    if len(sys.argv) > 1 and sys.argv[1] == "c3":
        parity("c3", C["c3"], 1000)
        timing("c3", C["c3"], 200_000, 3)

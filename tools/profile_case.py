"""Run a few EM steps of one workload (for ncu captures): python tools/profile_case.py c2 20000 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_06843_b200 import BscGpuModel, TruncationConfig, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = configs.CONFIGS[name]
y = configs.data(w, n)
p = configs.init(w, y)
m = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma))
m.load(y)
for _ in range(steps):
    p = m.step(p).params
print("done", name, n, steps, p.pi, p.sigma2)

import numpy as np  # noqa: E402

from paper_1908_06843_b200 import _native as N  # noqa: E402

cyc = np.zeros(8, np.uint64)
N.call("prsp_bsc_gpu_enum_phase_cycles", m.handle, cyc.ctypes.data_as(__import__("ctypes").c_void_p))
if cyc.sum():
    names = ["scores", "select", "uP", "rel", "exp", "map", "sub+gather", "out+loop"]
    tot = cyc.sum()
    print("enumerate phase cycles/point/warp:", {k: round(float(v) / n, 1) for k, v in zip(names, cyc)})
    print("shares:", {k: f"{100 * float(v) / tot:.1f}%" for k, v in zip(names, cyc)})

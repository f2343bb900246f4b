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

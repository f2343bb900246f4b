import sys
sys.path.insert(0, '.')
from paper_1908_06843_b200 import configs, BscGpuModel, TruncationConfig
w = configs.CONFIGS['c3']
y = configs.data(w, 600)
p = configs.init(w, y)
m = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma))
m.load(y)
print('loaded', flush=True)
c = m.candidates(p)
print('cands ok', flush=True)
st = m.estep_stats(p)
print('estep ok', flush=True)
r = m.step(p)
print('step ok', r.free_energy, flush=True)
r = m.step(p)
print('step2 ok', r.free_energy, flush=True)

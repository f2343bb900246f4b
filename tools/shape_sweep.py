"""Fault sweep (compute-sanitizer is closed on this pool): step, step_host and inference over ten (D, H, H', gamma)
shapes x 15-17 data sizes around the 32 / 64 / 128-point tile boundaries, under CUDA_LAUNCH_BLOCKING=1 BSC_GUARD=1:
    CUDA_LAUNCH_BLOCKING=1 BSC_GUARD=1 python tools/shape_sweep.py
prints every (shape, N) that raised; guard bytes are checked after each case."""
import sys, os, itertools
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1908_06843_b200 as P
from paper_1908_06843_b200 import _native as N
rng = np.random.default_rng(1)
shapes = [(32, 33, 2, 2), (64, 64, 16, 6), (256, 300, 12, 4), (100, 20, 10, 4), (576, 1000, 14, 5), (128, 200, 8, 3),
          (40, 72, 5, 5), (25, 10, 10, 10), (9, 1024, 3, 2), (1000, 24, 6, 4)]
ns = [1, 2, 31, 32, 33, 63, 65, 127, 128, 129, 255, 257, 4095, 4097, 33333]
bad = 0
for (d, h, hp, g) in shapes:
    wt = P.random_dictionary(d, h, 7, 5.0)
    m = P.BscGpuModel(d, h, P.TruncationConfig(h, hp, g))
    for n in ns + ([200031, 262144 + 17] if d * h <= 80000 else []):
        y = P.generate(P.BscParams(wt, min(0.5, 3.0 / h), 0.25), n, 100 + n)
        p = P.BscParams(wt + 0.05 * np.cos(np.arange(d * h)).reshape(d, h), 1.0 / h, 0.4)
        try:
            m.load(y)
            r = m.step(p)
            r2 = m.step_host(r.params, y)
            m.inference(r2.params)
            N.call("prsp_bsc_gpu_check_guards")
            assert np.isfinite(r2.free_energy)
        except Exception as e:
            bad += 1
            print("FAIL", (d, h, hp, g), n, str(e)[:200], flush=True)
            m = P.BscGpuModel(d, h, P.TruncationConfig(h, hp, g))
    print("shape done", (d, h, hp, g), flush=True)
    m.close()
print("SWEEP DONE, failures:", bad)

"""Out-of-bounds check of the device code without compute-sanitizer (closed on
this pool): a fresh process runs the engine with BSC_GUARD=1 — every device
buffer of the library then carries 256 guard bytes of 0xA5 on both sides
(csrc/engine_util.hpp) — over the BASELINE shapes, ragged sizes, the chunked
host-buffer step, inference, the multi-valued families and max causes, and
prsp_bsc_gpu_check_guards must find every guard intact."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import numpy as np
import paper_1908_06843_b200 as P
from paper_1908_06843_b200 import _native as N

def check(tag):
    N.call("prsp_bsc_gpu_check_guards")
    print("guards ok:", tag, flush=True)

rng = np.random.default_rng(0)
for (d, h, hp, g, n) in [(256, 300, 12, 4, 5003), (576, 1000, 14, 5, 777), (100, 20, 10, 4, 130),
                         (25, 10, 10, 10, 700), (7, 5, 3, 2, 33), (64, 40, 8, 3, 1), (33, 17, 16, 6, 257)]:
    wt = P.random_dictionary(d, h, 61, 5.0)
    y = P.generate(P.BscParams(wt, min(0.5, 3.0 / h), 0.25), n, 62)
    p = P.BscParams(wt + 0.05 * np.cos(np.arange(d * h)).reshape(d, h), 1.0 / h, 0.4)
    m = P.BscGpuModel(d, h, P.TruncationConfig(h, hp, g))
    m.load(y)
    m.candidates(p)
    m.estep_stats(p)
    r = m.step(p)
    m.step(r.params)
    m.inference(r.params)
    m.step_host(p, y)
    m.step(P.BscParams(p.W, p.pi, 1e-3))   # outside the range guard: the fallback launch
    check(f"bsc {d}x{h} H'={hp} gamma={g} N={n}")
    m.close()
os = __import__("os")
os.environ["BSC_HOST_CHUNK"] = "1024"
wt = P.random_dictionary(256, 300, 61, 5.0)
y = P.generate(P.BscParams(wt, 0.01, 0.25), 5003, 63)
m = P.BscGpuModel(256, 300, P.TruncationConfig(300, 12, 4))
m.step_host(P.BscParams(wt, 1 / 300, 0.4), y)   # five host chunks
m.step(P.BscParams(wt, 1 / 300, 0.4))
check("bsc chunked host step")
m.close()
for fam, vals in [("tsc", None), ("dsc", [-1.0, 0.0, 0.5, 2.0])]:
    d, h, hp, g, n = 40, 12, 6, 3, 301
    w = rng.normal(size=(d, h))
    y = rng.normal(size=(n, d))
    m = P.LinearDiscreteGpuModel(fam, d, h, P.TruncationConfig(h, hp, g), values=vals)
    probs = None if vals is None else np.array([0.1, 0.7, 0.1, 0.1])
    m.load(y)
    q = P.LinearDiscreteParams(w, 0.5, 0.2, probs)
    m.estep_stats(q)
    m.step(q)
    m.inference(q)
    check(fam)
    m.close()
for fam in ("mca", "mmca"):
    d, h, hp, g, n = 30, 9, 5, 3, 203
    w = np.abs(rng.normal(size=(d, h))) + 0.1
    y = np.abs(rng.normal(size=(n, d)))
    m = P.McaGpuModel(fam, d, h, P.TruncationConfig(h, hp, g))
    m.load(y)
    m.step(P.McaParams(w, 0.2, 0.5))
    m.inference(P.McaParams(w, 0.2, 0.5))
    check(fam)
    m.close()
print("ALL GUARDS INTACT")
"""


def test_no_kernel_writes_outside_its_buffers():
    env = dict(os.environ, BSC_GUARD="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ALL GUARDS INTACT" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])


PROBE = r"""
import sys
from paper_1908_06843_b200 import _native as N
try:
    N.call("prsp_bsc_gpu_guard_probe", 1000, int(sys.argv[1]))
    print("PROBE OK")
except N.PrspError as e:
    print("PROBE FAULT", e)
"""


def test_vmm_guard_faults_on_a_read_past_the_end():
    """BSC_GUARD=2 (buffers end-aligned in their mapping, unmapped page behind): a device read inside a
    1000-byte buffer succeeds, one 16 bytes past its (16-byte rounded) end faults. The engine runs clean
    under the same mode in the next test, so that silence means no overrun."""
    env = dict(os.environ, BSC_GUARD="2", PYTHONPATH=ROOT)
    ok = subprocess.run([sys.executable, "-c", PROBE, "999"], env=env, capture_output=True, text=True, timeout=300)
    assert "PROBE OK" in ok.stdout, (ok.stdout, ok.stderr[-2000:])
    bad = subprocess.run([sys.executable, "-c", PROBE, "1024"], env=env, capture_output=True, text=True, timeout=300)
    assert "PROBE FAULT" in bad.stdout and "PROBE OK" not in bad.stdout, (bad.stdout, bad.stderr[-2000:])


def test_no_kernel_reads_or_writes_past_a_buffer_end():
    env = dict(os.environ, BSC_GUARD="2", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace('N.call("prsp_bsc_gpu_check_guards")', "pass")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ALL GUARDS INTACT" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])

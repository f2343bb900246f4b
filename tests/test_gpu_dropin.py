"""The compiled drop-in (integration/gpu_linear_discrete.cpp): a prsp::Model
whose step() calls the engine's C ABI, built against the reference's
unmodified headers and driven by the reference's own EM loop prsp::run
(em.cpp:22-70). Its trajectory must follow the reference's CPU
LinearDiscreteModel under the same loop within the north-star tolerance.
"""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu

LIB = os.path.join(ROOT, "integration", "_build", "libprsp_dropin.so")


@pytest.fixture(scope="module")
def dropin():
    if not os.path.exists(LIB):
        pytest.skip("integration/_build/libprsp_dropin.so not built (needs /root/reference at build time)")
    lib = C.CDLL(LIB)
    lib.dropin_last_error.restype = C.c_char_p
    return lib


def run(lib, gpu, y, w0, pi0, s20, hp, g, iters, t0=1.0, shards=4):
    n, d = y.shape
    h = w0.shape[1]
    tr, w = np.empty(iters), np.empty((d, h))
    pi, s2 = C.c_double(), C.c_double()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = lib.dropin_run_bsc(C.c_int(gpu), p(y), C.c_uint64(n), C.c_uint32(d), C.c_uint32(h), C.c_uint32(hp),
                            C.c_uint32(g), p(w0), C.c_double(pi0), C.c_double(s20), C.c_uint32(iters),
                            C.c_double(t0), C.c_uint32(shards), p(tr), p(w), C.byref(pi), C.byref(s2))
    assert rc == 0, lib.dropin_last_error()
    return tr, w, pi.value, s2.value


@pytest.mark.parametrize("t0", [1.0, 3.0])
def test_reference_em_loop_drives_the_gpu_model(dropin, port, t0):
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c1"]  # 10x10 bars, D=100, H=20, H'=10, gamma=4, N=10,000
    y = np.ascontiguousarray(configs.data(w))
    p = configs.init(w, y)
    tg, wg, pig, s2g = run(dropin, 1, y, p.W, p.pi, p.sigma2, w.hprime, w.gamma, 10, t0)
    tc, wc, pic, s2c = run(dropin, 0, y, p.W, p.pi, p.sigma2, w.hprime, w.gamma, 10, t0)
    assert np.all(np.abs(tg - tc) <= 1e-6 * np.abs(tc)), np.max(np.abs(tg - tc) / np.abs(tc))
    assert rel(wg, wc) < 1e-6 and abs(pig - pic) <= 1e-6 * pic and abs(s2g - s2c) <= 1e-6 * s2c

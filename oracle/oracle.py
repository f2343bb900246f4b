"""TEST INFRASTRUCTURE ONLY — the parity oracle, never the product.

ctypes front end over the two CPU oracles of the BSC truncated-EM path:

* ``port`` — ``oracle/_build/libbsc_oracle.so``, the plain-C restatement
  (``oracle/bsc_oracle.c``), built everywhere (here and travelling to the GPU
  box as a prebuilt ``.so``);
* ``ref``  — ``oracle/_ref/libprsp_ref.so``, the reference's own sources
  (``/root/reference/proj/src``) compiled against ``oracle/eigen_shim``.
  Built only where ``/root/reference`` exists; the prebuilt ``.so`` travels.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module. Functions raise :class:`OracleError` carrying the
prsp status code (prsp.h:39-45).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libbsc_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libprsp_ref.so")
REF_SRC = "/root/reference/proj/src"

_u32, _u64, _dbl, _int, _ptr = C.c_uint32, C.c_uint64, C.c_double, C.c_int, C.c_void_p


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(quiet: bool = True) -> None:
    """Compile the C restatement (and the reference, when its sources exist)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _p(a):
    return None if a is None else a.ctypes.data_as(_ptr)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


FAMILIES = {"bsc": 0, "tsc": 1, "dsc": 2}


class Prior:
    """Value prior of a linear discrete family (linear_discrete.cpp:71-97):
    ``pi`` for bsc/tsc; the dsc alphabet (ascending, containing 0) and its
    probabilities for dsc."""

    def __init__(self, family: str, pi: float = 0.1, alpha=None, probs=None):
        self.family = family
        self.code = FAMILIES[family]
        self.pi = float(pi) if pi is not None else 0.0
        self.alpha = None if alpha is None else _f64(alpha)
        self.probs = None if probs is None else _f64(probs)

    @property
    def values(self):
        """The non-zero alphabet in kernel order."""
        if self.family == "bsc":
            return np.array([1.0])
        if self.family == "tsc":
            return np.array([-1.0, 1.0])
        return self.alpha[self.alpha != 0.0]

    @property
    def nv(self) -> int:
        return len(self.values)

    def args(self):
        n = 0 if self.alpha is None else len(self.alpha)
        return [_u32(self.code), _p(self.alpha), _p(self.probs), _u32(n), _dbl(self.pi)]


class Oracle:
    """One CPU oracle library (``kind`` = "port" or "ref")."""

    def __init__(self, kind: str = "port"):
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run oracle.build())")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pre = "bsc_" if kind == "port" else "ref_"
        getattr(self.lib, self.pre + "last_error").restype = C.c_char_p

    @staticmethod
    def available(kind: str) -> bool:
        return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)

    def _mcall(self, name, *args):
        self._call(name, *args, pre="mca_" if self.kind == "port" else "ref_mca_")

    def _lcall(self, name, *args):
        self._call(("ld_" if self.kind == "ref" else "") + name, *args, pre="ld_" if self.kind == "port" else None)

    def _call(self, name, *args, pre=None):
        fn = getattr(self.lib, (self.pre if pre is None else pre) + name)
        fn.restype = _int
        rc = fn(*args)
        if rc != 0:
            msg = getattr(self.lib, self.pre + "last_error")().decode()
            raise OracleError(rc, msg)

    # ------------------------------------------------------------ fixtures
    def rng_normals(self, base_seed, index, derived, n):
        out = np.empty(n)
        self._call("rng_normals", _u64(base_seed), _u64(index), _int(derived), _u64(n), _p(out))
        return out

    def make_bars(self, size, n, prob=0.0, amplitude=10.0, noise=2.0, max_mode=False, seed=0):
        d, hb = size * size, 2 * size
        y = np.empty((n, d))
        truth = np.empty((d, hb))
        self._call("make_bars", _u32(size), _u64(n), _dbl(prob), _dbl(amplitude), _dbl(noise),
                   _int(int(max_mode)), _u64(seed), _p(y), _p(truth))
        return y, truth

    def generate(self, w, pi, sigma2, n, seed):
        w = _f64(w)
        d, h = w.shape
        y = np.empty((n, d))
        self._call("generate", _u32(d), _u32(h), _p(w), _dbl(pi), _dbl(sigma2), _u64(n), _u64(seed), _p(y))
        return y

    def random_dictionary(self, d, h, seed, scale=5.0):
        w = np.empty((d, h))
        self._call("random_dictionary", _u32(d), _u32(h), _u64(seed), _dbl(scale), _p(w))
        return w

    def baseline_init(self, y, h, seed):
        y = _f64(y)
        n, d = y.shape
        w = np.empty((d, h))
        pi, s2 = _dbl(), _dbl()
        self._call("baseline_init", _u32(d), _u32(h), _p(y), _u64(n), _u64(seed), _p(w), C.byref(pi), C.byref(s2))
        return w, pi.value, s2.value

    def standard_init(self, y, h, hprime, gamma, seed):
        y = _f64(y)
        n, d = y.shape
        w = np.empty((d, h))
        pi, s2 = _dbl(), _dbl()
        if self.kind == "port":
            self._call("standard_init", _u32(d), _u32(h), _u32(hprime), _p(y), _u64(n), _u64(seed),
                       _p(w), C.byref(pi), C.byref(s2))
        else:
            self._call("standard_init", _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(y), _u64(n),
                       _u64(seed), _p(w), C.byref(pi), C.byref(s2))
        return w, pi.value, s2.value

    def data_mean_variance(self, y):
        y = _f64(y)
        out = _dbl()
        self._call("data_mean_variance", _p(y), _u64(y.shape[0]), _u32(y.shape[1]), C.byref(out))
        return out.value

    # ---------------------------------------------------------- truncation
    def select_candidates(self, scores, hprime):
        s = _f64(scores)
        out = np.empty(hprime, np.uint32)
        self._call("select_candidates", _p(s), _u32(len(s)), _u32(hprime), _p(out))
        return out

    def state_count(self, h, hprime, gamma):
        out = _u64()
        self._call("state_count", _u32(h), _u32(hprime), _u32(gamma), C.byref(out))
        return out.value

    def enumerate_binary(self, cand, h, gamma):
        cand = np.ascontiguousarray(cand, dtype=np.uint32)
        cnt = _u64()
        self._call("enumerate_binary", _p(cand), _u32(len(cand)), _u32(h), _u32(gamma), None, C.byref(cnt))
        out = np.empty((cnt.value, h))
        self._call("enumerate_binary", _p(cand), _u32(len(cand)), _u32(h), _u32(gamma), _p(out), C.byref(cnt))
        return out

    def log_sum_exp(self, v):
        v = _f64(v)
        out = _dbl()
        self._call("log_sum_exp", _p(v), _u64(len(v)), C.byref(out))
        return out.value

    # --------------------------------------------------------------- model
    def log_joint(self, w, pi, sigma2, y, s):
        w, y, s = _f64(w), _f64(y), _f64(s)
        out = _dbl()
        self._call("log_joint", _u32(w.shape[0]), _u32(w.shape[1]), _p(w), _dbl(pi), _dbl(sigma2), _p(y), _p(s),
                   C.byref(out))
        return out.value

    def estep_stats(self, w, pi, sigma2, y, hprime, gamma, temperature=1.0, rows=None):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        n = y.shape[0]
        b, e = (0, n) if rows is None else rows
        st = dict(sum_s=np.empty(h), sum_ssT=np.empty((h, h)), sum_y_sT=np.empty((d, h)),
                  value_counts=np.empty(1), scalars=np.empty(3))
        self._call("estep_stats", _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w), _dbl(pi), _dbl(sigma2),
                   _dbl(temperature), _p(y), _u64(n), _u64(b), _u64(e), _p(st["sum_s"]), _p(st["sum_ssT"]),
                   _p(st["sum_y_sT"]), _p(st["value_counts"]), _p(st["scalars"]))
        sc = st.pop("scalars")
        st.update(sum_y2=sc[0], log_partition=sc[1], points=int(sc[2]))
        return st

    def mstep(self, stats, w_prev, pi_prev, sigma2_prev, hprime=1, gamma=1):
        w_prev = _f64(w_prev)
        d, h = w_prev.shape
        w = np.empty((d, h))
        pi, s2 = _dbl(), _dbl()
        sc = np.array([stats["sum_y2"], stats["log_partition"], float(stats["points"])])
        vc = _f64(np.atleast_1d(stats["value_counts"]))
        args = [_p(w_prev), _dbl(pi_prev), _dbl(sigma2_prev), _p(_f64(stats["sum_s"])), _p(_f64(stats["sum_ssT"])),
                _p(_f64(stats["sum_y_sT"])), _p(vc), _p(sc), _p(w), C.byref(pi), C.byref(s2)]
        if self.kind == "port":
            self._call("mstep", _u32(d), _u32(h), *args)
        else:
            self._call("mstep", _u32(d), _u32(h), _u32(hprime), _u32(gamma), *args)
        return w, pi.value, s2.value

    def step(self, w, pi, sigma2, y, hprime, gamma, temperature=1.0, shards=1, workers=1):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        wo = np.empty((d, h))
        pio, s2o, f = _dbl(), _dbl(), _dbl()
        self._call("step", _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w), _dbl(pi), _dbl(sigma2),
                   _dbl(temperature), _p(y), _u64(y.shape[0]), _u32(shards), _u32(workers), _p(wo),
                   C.byref(pio), C.byref(s2o), C.byref(f))
        return wo, pio.value, s2o.value, f.value

    def candidates(self, w, pi, sigma2, y, hprime, threads=1):
        """Per-point candidate sets. ``threads`` > 1 splits the rows into blocks
        computed concurrently (ctypes releases the GIL; every row is independent,
        so the result is the same bytes as one call)."""
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        n = y.shape[0]
        out = np.empty((n, hprime), np.uint32)

        def block(b, e):
            if e > b:
                self._call("candidates", _u32(d), _u32(h), _u32(hprime), _p(w), _dbl(pi), _dbl(sigma2),
                           _p(y[b:e]), _u64(e - b), _p(out[b:e]))

        if threads <= 1 or n < 2 * threads:
            block(0, n)
            return out
        from concurrent.futures import ThreadPoolExecutor

        cuts = np.linspace(0, n, 4 * threads + 1).astype(int)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: block(cuts[i], cuts[i + 1]), range(len(cuts) - 1)))
        return out

    def inference(self, w, pi, sigma2, y, hprime, gamma):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        n = y.shape[0]
        ms, mm, ex = np.empty((n, h)), np.empty(n), np.empty((n, h))
        if self.kind == "port":
            self._call("inference", _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w), _dbl(pi), _dbl(sigma2),
                       _p(y), _u64(n), _p(ms), _p(mm), _p(ex))
        else:
            self._call("inference", _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w), _dbl(pi), _dbl(sigma2),
                       _p(y), _u64(n), _u32(1), _p(ms), _p(mm), _p(ex))
        return ms, mm, ex

    def exact_log_likelihood(self, w, pi, sigma2, y):
        w, y = _f64(w), _f64(y)
        out = _dbl()
        self._call("exact_log_likelihood", _u32(w.shape[0]), _u32(w.shape[1]), _p(w), _dbl(pi), _dbl(sigma2),
                   _p(y), _u64(y.shape[0]), C.byref(out))
        return out.value


    # ------------------------------------------- linear discrete families
    def ld_state_count(self, h, hprime, gamma, nv):
        out = _u64()
        self._lcall("state_count", _u32(h), _u32(hprime), _u32(gamma), _u32(nv), C.byref(out))
        return out.value

    def ld_estep_stats(self, prior: Prior, w, sigma2, y, hprime, gamma, temperature=1.0, rows=None):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        n = y.shape[0]
        b, e = (0, n) if rows is None else rows
        st = dict(sum_s=np.empty(h), sum_ssT=np.empty((h, h)), sum_y_sT=np.empty((d, h)),
                  value_counts=np.empty(prior.nv), scalars=np.empty(3))
        self._lcall("estep_stats", *prior.args(), _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w),
                    _dbl(sigma2), _dbl(temperature), _p(y), _u64(n), _u64(b), _u64(e), _p(st["sum_s"]),
                    _p(st["sum_ssT"]), _p(st["sum_y_sT"]), _p(st["value_counts"]), _p(st["scalars"]))
        sc = st.pop("scalars")
        st.update(sum_y2=sc[0], log_partition=sc[1], points=int(sc[2]))
        return st

    def ld_mstep(self, prior: Prior, stats, w_prev, sigma2_prev):
        """→ (W, pi, probs, sigma2); probs (dsc) aligned with the alphabet."""
        w_prev = _f64(w_prev)
        d, h = w_prev.shape
        w = np.empty((d, h))
        pi, s2 = _dbl(), _dbl()
        na = 0 if prior.alpha is None else len(prior.alpha)
        probs = np.empty(max(na, 1))
        sc = np.array([stats["sum_y2"], stats["log_partition"], float(stats["points"])])
        vc = _f64(np.atleast_1d(stats["value_counts"]))
        tail = [_p(_f64(stats["sum_s"])), _p(_f64(stats["sum_ssT"])), _p(_f64(stats["sum_y_sT"])), _p(vc), _p(sc),
                _p(w), C.byref(pi), _p(probs), C.byref(s2)]
        if self.kind == "port":
            self._lcall("mstep", _u32(prior.code), _p(prior.alpha), _u32(na), _u32(d), _u32(h), _p(w_prev), *tail)
        else:
            self._lcall("mstep", _u32(prior.code), _p(prior.alpha), _p(prior.probs), _u32(na), _dbl(prior.pi),
                        _u32(d), _u32(h), _u32(prior.nv), _p(w_prev), _dbl(sigma2_prev), *tail)
        return w, (None if prior.family == "dsc" else pi.value), (probs[:na] if na else None), s2.value

    def ld_step(self, prior: Prior, w, sigma2, y, hprime, gamma, temperature=1.0, shards=1, workers=1):
        """→ (W, pi, probs, sigma2, F)."""
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        wo = np.empty((d, h))
        na = 0 if prior.alpha is None else len(prior.alpha)
        probs = np.empty(max(na, 1))
        pio, s2o, f = _dbl(), _dbl(), _dbl()
        self._lcall("step", *prior.args(), _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w), _dbl(sigma2),
                    _dbl(temperature), _p(y), _u64(y.shape[0]), _u32(shards), _u32(workers), _p(wo),
                    C.byref(pio), _p(probs), C.byref(s2o), C.byref(f))
        return wo, (None if prior.family == "dsc" else pio.value), (probs[:na] if na else None), s2o.value, f.value

    def ld_candidates(self, prior: Prior, w, sigma2, y, hprime):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        out = np.empty((y.shape[0], hprime), np.uint32)
        self._lcall("candidates", *prior.args(), _u32(d), _u32(h), _u32(hprime), _p(w), _dbl(sigma2), _p(y),
                    _u64(y.shape[0]), _p(out))
        return out

    def ld_inference(self, prior: Prior, w, sigma2, y, hprime, gamma):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        n = y.shape[0]
        ms, mm, ex = np.empty((n, h)), np.empty(n), np.empty((n, h))
        extra = [] if self.kind == "port" else [_u32(1)]
        self._lcall("inference", *prior.args(), _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w), _dbl(sigma2),
                    _p(y), _u64(n), *extra, _p(ms), _p(mm), _p(ex))
        return ms, mm, ex

    def ld_generate(self, prior: Prior, w, sigma2, n, seed):
        w = _f64(w)
        d, h = w.shape
        y = np.empty((n, d))
        self._lcall("generate", *prior.args(), _u32(d), _u32(h), _p(w), _dbl(sigma2), _u64(n), _u64(seed), _p(y))
        return y

    def ld_exact_log_likelihood(self, prior: Prior, w, sigma2, y):
        w, y = _f64(w), _f64(y)
        out = _dbl()
        self._lcall("exact_log_likelihood", *prior.args(), _u32(w.shape[0]), _u32(w.shape[1]), _p(w),
                    _dbl(sigma2), _p(y), _u64(y.shape[0]), C.byref(out))
        return out.value



    # ----------------------------------------------------------- max causes
    # mode "mca" (max) or "mmca" (absmax); rho = soft winner exponent
    @staticmethod
    def _mode(mode):
        return _u32({"mca": 0, "mmca": 1}[mode])

    def mca_estep_stats(self, mode, w, pi, sigma2, y, hprime, gamma, temperature=1.0, rows=None, rho=0.0):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        n = y.shape[0]
        b, e = (0, n) if rows is None else rows
        num, den, sc = np.empty((d, h)), np.empty((d, h)), np.empty(3)
        self._mcall("estep_stats", self._mode(mode), _dbl(rho), _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w),
                    _dbl(pi), _dbl(sigma2), _dbl(temperature), _p(y), _u64(n), _u64(b), _u64(e), _p(num), _p(den),
                    _p(sc))
        return dict(winner_num=num, winner_den=den, sum_act=sc[0], log_partition=sc[1], points=int(sc[2]))

    def mca_mstep_fixedpoint(self, mode, stats, w_prev, pi_prev, sigma2_prev):
        w_prev = _f64(w_prev)
        d, h = w_prev.shape
        w, pi = np.empty((d, h)), _dbl()
        sc = np.array([stats["sum_act"], stats["log_partition"], float(stats["points"])])
        num, den = _f64(stats["winner_num"]), _f64(stats["winner_den"])
        if self.kind == "port":
            self._mcall("mstep_fixedpoint", self._mode(mode), _u32(d), _u32(h), _p(w_prev), _p(num), _p(den), _p(sc),
                        _p(w), C.byref(pi))
        else:
            self._mcall("mstep_fixedpoint", self._mode(mode), _u32(d), _u32(h), _p(w_prev), _dbl(pi_prev),
                        _dbl(sigma2_prev), _p(num), _p(den), _p(sc), _p(w), C.byref(pi))
        return w, pi.value

    def mca_step(self, mode, w, pi, sigma2, y, hprime, gamma, temperature=1.0, shards=1, workers=1, rho=0.0):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        wo = np.empty((d, h))
        pio, s2o, f = _dbl(), _dbl(), _dbl()
        self._mcall("step", self._mode(mode), _dbl(rho), _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w),
                    _dbl(pi), _dbl(sigma2), _dbl(temperature), _p(y), _u64(y.shape[0]), _u32(shards), _u32(workers),
                    _p(wo), C.byref(pio), C.byref(s2o), C.byref(f))
        return wo, pio.value, s2o.value, f.value

    def mca_candidates(self, mode, w, pi, sigma2, y, hprime):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        out = np.empty((y.shape[0], hprime), np.uint32)
        self._mcall("candidates", self._mode(mode), _u32(d), _u32(h), _u32(hprime), _p(w), _dbl(pi), _dbl(sigma2),
                    _p(y), _u64(y.shape[0]), _p(out))
        return out

    def mca_inference(self, mode, w, pi, sigma2, y, hprime, gamma):
        w, y = _f64(w), _f64(y)
        d, h = w.shape
        n = y.shape[0]
        ms, mm, ex = np.empty((n, h)), np.empty(n), np.empty((n, h))
        extra = [] if self.kind == "port" else [_u32(1)]
        self._mcall("inference", self._mode(mode), _u32(d), _u32(h), _u32(hprime), _u32(gamma), _p(w), _dbl(pi),
                    _dbl(sigma2), _p(y), _u64(n), *extra, _p(ms), _p(mm), _p(ex))
        return ms, mm, ex

    def mca_log_joint(self, mode, w, pi, sigma2, y, s):
        w, y, s = _f64(w), _f64(y), _f64(s)
        out = _dbl()
        self._mcall("log_joint", self._mode(mode), _u32(w.shape[0]), _u32(w.shape[1]), _p(w), _dbl(pi),
                    _dbl(sigma2), _p(y), _p(s), C.byref(out))
        return out.value

    def mca_exact_log_likelihood(self, mode, w, pi, sigma2, y):
        w, y = _f64(w), _f64(y)
        out = _dbl()
        self._mcall("exact_log_likelihood", self._mode(mode), _u32(w.shape[0]), _u32(w.shape[1]), _p(w), _dbl(pi),
                    _dbl(sigma2), _p(y), _u64(y.shape[0]), C.byref(out))
        return out.value

    def mca_generate(self, mode, w, pi, sigma2, n, seed):
        w = _f64(w)
        d, h = w.shape
        y = np.empty((n, d))
        self._mcall("generate", self._mode(mode), _u32(d), _u32(h), _p(w), _dbl(pi), _dbl(sigma2), _u64(n),
                    _u64(seed), _p(y))
        return y

    def mca_standard_init(self, mode, y, h, hprime, seed):
        y = _f64(y)
        n, d = y.shape
        w = np.empty((d, h))
        pi, s2 = _dbl(), _dbl()
        self._mcall("standard_init", self._mode(mode), _u32(d), _u32(h), _u32(hprime), _p(y), _u64(n), _u64(seed),
                    _p(w), C.byref(pi), C.byref(s2))
        return w, pi.value, s2.value



    # ---------------------------------------- run I/O + EM driver (ref only)
    def save_array(self, path, a):
        a = _f64(np.atleast_2d(a))
        self._call("save_array", str(path).encode(), _p(a), _u64(a.shape[0]), _u64(a.shape[1]))

    def load_dataset(self, path):
        r, c = _u64(), _u64()
        self._call("load_dataset", str(path).encode(), C.byref(r), C.byref(c), None)
        out = np.empty((r.value, c.value))
        self._call("load_dataset", str(path).encode(), C.byref(r), C.byref(c), _p(out))
        return out

    def sha256(self, data: bytes):
        buf = C.create_string_buffer(65)
        src = C.create_string_buffer(data, len(data)) if data else None
        self._call("sha256", None if src is None else C.cast(src, _ptr), _u64(len(data)), buf)
        return buf.value.decode()

    def sha256_file(self, path):
        buf = C.create_string_buffer(65)
        self._call("sha256_file", str(path).encode(), buf)
        return buf.value.decode()

    def format_double(self, v):
        buf = C.create_string_buffer(32)
        self._call("format_double", _dbl(v), buf, _u32(32))
        return buf.value.decode()

    def train(self, model, y, latents, hprime, gamma, iterations, seed, values=None, shards=1, workers=1, tol=None,
              temperature=((0.0, 1.0),), w_noise=((0.0, 0.0),)):
        """em.cpp run() after train_run's setup; → (trace, W, pi, sigma2, probs)."""
        y = _f64(y)
        n, d = y.shape
        vals = _f64(values if values is not None else np.zeros(0))
        tp, tv = (_f64(x) for x in zip(*temperature))
        npos, nval = (_f64(x) for x in zip(*w_noise))
        trace, it = np.empty(iterations), _u64()
        w, pi, s2 = np.empty((d, latents)), _dbl(), _dbl()
        probs = np.empty(max(len(vals), 1))
        self._call("train", model.encode(), _p(vals), _u32(len(vals)), _u32(d), _u32(latents), _u32(hprime),
                   _u32(gamma), _u64(iterations), _u64(seed), _u32(shards), _u32(workers), _int(tol is not None),
                   _dbl(tol or 0.0), _p(tp), _p(tv), _u32(len(tp)), _p(npos), _p(nval), _u32(len(npos)), _p(y),
                   _u64(n), _p(trace), C.byref(it), _p(w), C.byref(pi), C.byref(s2), _p(probs))
        return trace[:it.value], w, pi.value, s2.value, (probs[:len(vals)] if len(vals) else None)



class RefSession:
    """The reference's ``LinearDiscreteModel::step`` over a resident dataset,
    for timing (bench.py ``--impl reference``)."""

    def __init__(self, y, h, hprime, gamma):
        self.lib = C.CDLL(REF_LIB)
        self.lib.ref_last_error.restype = C.c_char_p
        y = _f64(y)
        self.d, self.h, self.n = y.shape[1], h, y.shape[0]
        self.handle = _ptr()
        rc = self.lib.ref_session_create(_u32(self.d), _u32(h), _u32(hprime), _u32(gamma), _p(y), _u64(self.n),
                                         C.byref(self.handle))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def step(self, w, pi, sigma2, shards, workers):
        w = _f64(w)
        wo = np.empty_like(w)
        pio, s2o, f = _dbl(), _dbl(), _dbl()
        rc = self.lib.ref_session_step(self.handle, _p(w), _dbl(pi), _dbl(sigma2), _u32(shards), _u32(workers),
                                       _p(wo), C.byref(pio), C.byref(s2o), C.byref(f))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        return wo, pio.value, s2o.value, f.value

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.ref_session_free(self.handle)
            self.handle = None

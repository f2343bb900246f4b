"""Host-side mirror of the reference max-causes model over the sm_100a engine.

Mirrors ``prsp::MaxCausesModel`` (/root/reference/proj/src/max_causes.hpp):
``McaParams{W, pi, sigma2}``, ``step`` (E pass, fixed-point M-step, residual
pass for σ²), ``estep_stats`` (winner statistics), ``mstep_fixedpoint``,
``inference``. Every compute call goes through ``include/prsp_bsc_gpu.h``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .bsc import InferenceResult, StepResult, TruncationConfig

_dbl = C.c_double


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class McaParams:
    """model.hpp:59-63."""

    W: np.ndarray
    pi: float
    sigma2: float


@dataclass
class McaStats:
    """The MaxCausesModel SuffStats fields (max_causes.cpp:187-191)."""

    winner_num: np.ndarray
    winner_den: np.ndarray
    sum_act: float
    log_partition: float
    points: int


class McaGpuModel:
    """MaxCausesModel(MaxMode, dim, latents, TruncationConfig, soft_winner_rho)
    with ``model`` "mca" (max) or "mmca" (absmax) on one B200."""

    def __init__(self, model: str, dim: int, latents: int, trunc: TruncationConfig, soft_winner_rho: float = 0.0,
                 device: int = 0):
        self.model, self.dim, self.latents = model, int(dim), int(latents)
        self.trunc = TruncationConfig(latents, trunc.hprime, trunc.gamma, trunc.state_cap)
        h = C.c_void_p()
        N.call("prsp_mca_gpu_create", model.encode(), float(soft_winner_rho), dim, latents, trunc.hprime, trunc.gamma,
               trunc.state_cap, device, C.byref(h))
        self._h = h
        self._data_key = None
        self.n = 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().prsp_mca_gpu_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def states_per_point(self) -> int:
        v = C.c_uint64()
        N.call("prsp_mca_gpu_states_per_point", self._h, C.byref(v))
        return v.value

    def load(self, y) -> None:
        y = _f64(y)
        if y.ndim != 2 or y.shape[1] != self.dim:
            raise N.DataError(3, f"{self.model}: data dimension mismatch")
        N.call("prsp_mca_gpu_load_data", self._h, _p(y), y.shape[0])
        self.n = y.shape[0]
        self._data_key = (y.__array_interface__["data"][0], y.shape)

    def _ensure(self, data) -> None:
        if data is None:
            return
        y = _f64(data)
        if (y.__array_interface__["data"][0], y.shape) != self._data_key:
            self.load(y)

    def set_params(self, p: McaParams) -> None:
        w = _f64(p.W)
        if w.shape != (self.dim, self.latents):
            raise N.ConfigError(2, f"{self.model}: dictionary shape mismatch")
        N.call("prsp_mca_gpu_set_params", self._h, _p(w), float(p.pi), float(p.sigma2))

    def get_params(self) -> McaParams:
        w = np.empty((self.dim, self.latents))
        pi, s2 = _dbl(), _dbl()
        N.call("prsp_mca_gpu_get_params", self._h, _p(w), C.byref(pi), C.byref(s2))
        return McaParams(w, pi.value, s2.value)

    def step(self, params: McaParams, data=None, temperature: float = 1.0) -> StepResult:
        """MaxCausesModel::step (max_causes.cpp:416-446)."""
        self._ensure(data)
        self.set_params(params)
        f = _dbl()
        N.call("prsp_mca_gpu_step", self._h, float(temperature), C.byref(f))
        return StepResult(self.get_params(), f.value)

    def estep_stats(self, params: McaParams, data=None, temperature: float = 1.0) -> McaStats:
        """MaxCausesModel::estep_stats (:384-391) over the resident shard."""
        self._ensure(data)
        self.set_params(params)
        N.call("prsp_mca_gpu_estep", self._h, float(temperature))
        return self.get_stats()

    def get_stats(self) -> McaStats:
        d, h = self.dim, self.latents
        num, den, sc = np.empty((d, h)), np.empty((d, h)), np.empty(3)
        N.call("prsp_mca_gpu_get_stats", self._h, _p(num), _p(den), _p(sc))
        return McaStats(num, den, float(sc[0]), float(sc[1]), int(sc[2]))

    def mstep_fixedpoint(self, stats: McaStats | dict, prev: McaParams) -> McaParams:
        """MaxCausesModel::mstep_fixedpoint (:393-414): W', π' (σ² unchanged)."""
        self.set_params(prev)
        st = stats if isinstance(stats, dict) else stats.__dict__
        sc = np.array([st["sum_act"], st["log_partition"], float(st["points"])])
        N.call("prsp_mca_gpu_set_stats", self._h, _p(_f64(st["winner_num"])), _p(_f64(st["winner_den"])), _p(sc))
        w = np.empty((self.dim, self.latents))
        pi = _dbl()
        N.call("prsp_mca_gpu_mstep_fixedpoint", self._h, _p(w), C.byref(pi))
        return McaParams(w, pi.value, float(prev.sigma2))

    def candidates(self, params: McaParams, data=None) -> np.ndarray:
        self._ensure(data)
        self.set_params(params)
        out = np.empty((self.n, self.trunc.hprime), np.uint32)
        N.call("prsp_mca_gpu_candidates", self._h, _p(out))
        return out

    def inference(self, params: McaParams, data=None) -> InferenceResult:
        """MaxCausesModel::inference (:448-468)."""
        self._ensure(data)
        self.set_params(params)
        ms, mm, ex = np.empty((self.n, self.latents)), np.empty(self.n), np.empty((self.n, self.latents))
        N.call("prsp_mca_gpu_inference", self._h, _p(ms), _p(mm), _p(ex))
        return InferenceResult(ms, mm, ex)

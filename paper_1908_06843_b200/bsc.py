"""Host-side mirror of the reference BSC model API over the sm_100a engine.

Mirrors ``prsp::LinearDiscreteModel`` for the BSC family
(/root/reference/proj/src/linear_discrete.hpp:31-87): the same parameter
names (``W``, ``pi``, ``sigma2`` — note the reference's "sigma" is the
variance), the same E/M-step entry points (``step``, ``estep_stats``,
``mstep``, ``inference``) and the same truncation settings
(``TruncationConfig{latents, hprime, gamma, state_cap}``,
truncation.hpp:29-36). Every compute call goes through the C ABI of
``include/prsp_bsc_gpu.h``; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

_dbl = C.c_double


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class TruncationConfig:
    """truncation.hpp:29-36."""

    latents: int
    hprime: int
    gamma: int
    state_cap: int = 1_000_000


@dataclass
class BscParams:
    """LinearDiscreteParams for BSC (model.hpp:41-47): W (D×H), sigma2, pi."""

    W: np.ndarray
    pi: float
    sigma2: float

    def copy(self) -> "BscParams":
        return BscParams(self.W.copy(), float(self.pi), float(self.sigma2))


@dataclass
class LinearDiscreteParams:
    """LinearDiscreteParams (model.hpp:41-47) for any linear discrete family:
    ``pi`` for bsc/tsc, ``probs`` (aligned with the model's sorted alphabet,
    including 0) for dsc."""

    W: np.ndarray
    sigma2: float
    pi: float = 0.0
    probs: np.ndarray | None = None

    def copy(self) -> "LinearDiscreteParams":
        return LinearDiscreteParams(self.W.copy(), float(self.sigma2), float(self.pi),
                                    None if self.probs is None else np.array(self.probs, float))


@dataclass
class StepResult:
    """model.hpp:78-81: params after the step, F at the incoming params (T = 1)."""

    params: BscParams
    free_energy: float


@dataclass
class SuffStats:
    """The BSC SuffStats fields in the reference's insertion order
    (linear_discrete.cpp:211-217) plus ``points``."""

    sum_s: np.ndarray
    sum_ssT: np.ndarray
    sum_y_sT: np.ndarray
    value_counts: np.ndarray
    sum_y2: float
    log_partition: float
    points: int

    def as_dict(self) -> dict:
        return dict(sum_s=self.sum_s, sum_ssT=self.sum_ssT, sum_y_sT=self.sum_y_sT, value_counts=self.value_counts,
                    sum_y2=self.sum_y2, log_partition=self.log_partition, points=self.points)


@dataclass
class InferenceResult:
    """model.hpp:83-87."""

    map_states: np.ndarray
    map_mass: np.ndarray
    expected_states: np.ndarray


class LinearDiscreteGpuModel:
    """Truncated EM of a linear discrete family on one B200: a drop-in for
    ``LinearDiscreteModel(DiscreteFamily, dim, latents, TruncationConfig,
    dsc_values)`` (linear_discrete.cpp:32-61) with ``model`` "bsc", "tsc" or
    "dsc" (``values``: the dsc alphabet, must contain 0).

    The data shard is uploaded once by :meth:`load` (or implicitly by the
    reference-shaped :meth:`step` when it is handed a different array) and
    stays resident in HBM; parameters round-trip through host memory only where
    the reference API returns them.
    """

    def __init__(self, model: str, dim: int, latents: int, trunc: TruncationConfig, values=None, device: int = 0):
        self.dim, self.latents = int(dim), int(latents)
        self.trunc = TruncationConfig(latents, trunc.hprime, trunc.gamma, trunc.state_cap)
        h = C.c_void_p()
        vals = None if values is None else _f64(values)
        N.call("prsp_bsc_gpu_create_model", model.encode(), dim, latents, trunc.hprime, trunc.gamma,
               trunc.state_cap, None if vals is None else _p(vals), 0 if vals is None else len(vals), device,
               C.byref(h))
        self._h = h
        self._data_key = None
        self.n = 0
        fam, nv, na = C.c_int(), C.c_uint32(), C.c_uint32()
        N.call("prsp_bsc_gpu_model_info", self._h, C.byref(fam), C.byref(nv), C.byref(na), None)
        self.alphabet = np.empty(na.value)
        N.call("prsp_bsc_gpu_model_info", self._h, None, None, None, _p(self.alphabet))
        self.model = model
        self.family = fam.value
        self.n_values = nv.value

    # -------------------------------------------------------------- plumbing
    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().prsp_bsc_gpu_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def handle(self):
        return self._h

    def set_stream(self, cuda_stream_ptr: int) -> None:
        N.call("prsp_bsc_gpu_set_stream", self._h, C.c_void_p(cuda_stream_ptr))

    def sync(self) -> None:
        N.call("prsp_bsc_gpu_sync", self._h)

    def states_per_point(self) -> int:
        v = C.c_uint64()
        N.call("prsp_bsc_gpu_states_per_point", self._h, C.byref(v))
        return v.value

    def load(self, y) -> None:
        """Upload a data shard (N×D host array) to HBM."""
        y = _f64(y)
        if y.ndim != 2 or y.shape[1] != self.dim:
            raise N.DataError(3, "bsc: data dimension mismatch")
        N.call("prsp_bsc_gpu_load_data", self._h, _p(y), y.shape[0])
        self.n = y.shape[0]
        self._data_key = (y.__array_interface__["data"][0], y.shape)

    def load_device(self, ptr: int, n: int) -> None:
        """Use a device-resident N×D fp64 row-major buffer (e.g. a torch tensor)."""
        N.call("prsp_bsc_gpu_load_data_device", self._h, C.c_void_p(ptr), n)
        self.n = n
        self._data_key = ("device", ptr, n)

    def set_params(self, params) -> None:
        w = _f64(params.W)
        if w.shape != (self.dim, self.latents):
            raise N.ConfigError(2, f"{self.model}: dictionary shape mismatch")
        probs = getattr(params, "probs", None)
        pr = None if probs is None else _f64(probs)
        N.call("prsp_bsc_gpu_set_params_ex", self._h, _p(w), float(getattr(params, "pi", 0.0) or 0.0),
               float(params.sigma2), None if pr is None else _p(pr), 0 if pr is None else len(pr))

    def get_params(self):
        w = np.empty((self.dim, self.latents))
        pi, s2 = _dbl(), _dbl()
        probs = np.empty(len(self.alphabet))
        N.call("prsp_bsc_gpu_get_params_ex", self._h, _p(w), C.byref(pi), C.byref(s2), _p(probs))
        if self.model == "bsc":
            return BscParams(w, pi.value, s2.value)
        if self.model == "tsc":
            return LinearDiscreteParams(w, s2.value, pi.value)
        return LinearDiscreteParams(w, s2.value, 0.0, probs)

    # ------------------------------------------------------- reference API
    def step(self, params: BscParams, data=None, temperature: float = 1.0) -> StepResult:
        """LinearDiscreteModel::step (linear_discrete.cpp:410-427) on the resident shard
        (``data`` is uploaded first when given and not already resident)."""
        if data is not None:
            self._ensure(data)
        self.set_params(params)
        f = _dbl()
        N.call("prsp_bsc_gpu_step", self._h, float(temperature), C.byref(f))
        return StepResult(self.get_params(), f.value)

    def step_resident(self, temperature: float = 1.0) -> float:
        """One EM iteration from the parameters the engine holds (those of the last
        set_params or the last step's result), nothing but F crossing the host
        boundary: the inner loop of a training run (em.cpp:36-45). Returns F."""
        f = _dbl()
        N.call("prsp_bsc_gpu_step", self._h, float(temperature), C.byref(f))
        return f.value

    def step_host(self, params: BscParams, y, temperature: float = 1.0) -> StepResult:
        """The reference call shape end to end: host Y and params in, host params and F out."""
        if self.model == "dsc":
            raise N.ConfigError(2, "dsc: step_host takes pi; use step() with LinearDiscreteParams")
        y = _f64(y)
        w = _f64(params.W)
        wo = np.empty_like(w)
        pi, s2, f = _dbl(), _dbl(), _dbl()
        N.call("prsp_bsc_gpu_step_host", self._h, _p(y), y.shape[0], _p(w), float(params.pi), float(params.sigma2),
               float(temperature), _p(wo), C.byref(pi), C.byref(s2), C.byref(f))
        self.n = y.shape[0]
        self._data_key = (y.__array_interface__["data"][0], y.shape)
        p = BscParams(wo, pi.value, s2.value) if self.model == "bsc" else LinearDiscreteParams(wo, s2.value, pi.value)
        return StepResult(p, f.value)

    # ------------------------------------------------ multi-GPU (native NCCL)
    def nccl_init(self, unique_id: bytes, nranks: int, rank: int) -> None:
        """Join the job's NCCL communicator (ncclCommInitRank on this model's device);
        ``unique_id`` is ``nccl_unique_id()`` of rank 0, sent to every rank."""
        if len(unique_id) != 128:
            raise N.ConfigError(2, "nccl: the unique id is 128 bytes")
        buf = C.create_string_buffer(bytes(unique_id), 128)
        N.call("prsp_bsc_gpu_nccl_init", self._h, C.cast(buf, C.c_void_p), int(nranks), int(rank))

    def step_allreduce(self, params: BscParams | None = None, temperature: float = 1.0) -> float:
        """LinearDiscreteModel::step over the whole job: local E-step, NCCL sum of the
        packed statistics, replicated M-step, all inside the library. Returns F."""
        if params is not None:
            self.set_params(params)
        f = _dbl()
        N.call("prsp_bsc_gpu_step_allreduce", self._h, float(temperature), C.byref(f))
        return f.value

    def estep_stats(self, params: BscParams, data=None, temperature: float = 1.0) -> SuffStats:
        """LinearDiscreteModel::estep_stats (:327-334) over the resident shard."""
        if data is not None:
            self._ensure(data)
        self.set_params(params)
        N.call("prsp_bsc_gpu_estep", self._h, float(temperature))
        return self.get_stats()

    def get_stats(self) -> SuffStats:
        d, h = self.dim, self.latents
        s, ssT, ysT, vc, sc = np.empty(h), np.empty((h, h)), np.empty((d, h)), np.empty(self.n_values), np.empty(3)
        N.call("prsp_bsc_gpu_get_stats", self._h, _p(s), _p(ssT), _p(ysT), _p(vc), _p(sc))
        return SuffStats(s, ssT, ysT, vc, float(sc[0]), float(sc[1]), int(sc[2]))

    def stats_buffer(self):
        """(device pointer, count) of the packed statistics, for an in-place all-reduce."""
        p, n = C.c_void_p(), C.c_uint64()
        N.call("prsp_bsc_gpu_stats_buffer", self._h, C.byref(p), C.byref(n))
        return p.value, n.value

    def mstep(self, stats: SuffStats | dict | None, prev: BscParams) -> BscParams:
        """LinearDiscreteModel::mstep (:336-408). ``stats=None`` uses the device statistics."""
        self.set_params(prev)
        if stats is not None:
            st = stats.as_dict() if isinstance(stats, SuffStats) else stats
            sc = np.array([st["sum_y2"], st["log_partition"], float(st["points"])])
            N.call("prsp_bsc_gpu_set_stats", self._h, _p(_f64(st["sum_s"])), _p(_f64(st["sum_ssT"])),
                   _p(_f64(st["sum_y_sT"])), _p(_f64(np.atleast_1d(st["value_counts"]))), _p(sc))
        N.call("prsp_bsc_gpu_mstep", self._h)
        return self.get_params()

    def mstep_device(self) -> float:
        """M-step from the (all-reduced) device statistics; params stay resident.
        Returns F = Σ_n log Z_n of those statistics."""
        N.call("prsp_bsc_gpu_mstep", self._h)
        f = _dbl()
        N.call("prsp_bsc_gpu_free_energy", self._h, C.byref(f))
        return f.value

    def candidates(self, params: BscParams, data=None) -> np.ndarray:
        """Per-point candidate sets (N×H', ascending) as estep_impl selects them (:240-253)."""
        if data is not None:
            self._ensure(data)
        self.set_params(params)
        out = np.empty((self.n, self.trunc.hprime), np.uint32)
        N.call("prsp_bsc_gpu_candidates", self._h, _p(out))
        return out

    def inference(self, params: BscParams, data=None) -> InferenceResult:
        """LinearDiscreteModel::inference (:429-450)."""
        if data is not None:
            self._ensure(data)
        self.set_params(params)
        ms, mm, ex = np.empty((self.n, self.latents)), np.empty(self.n), np.empty((self.n, self.latents))
        N.call("prsp_bsc_gpu_inference", self._h, _p(ms), _p(mm), _p(ex))
        return InferenceResult(ms, mm, ex)

    def set_timing(self, on: bool) -> None:
        N.call("prsp_bsc_gpu_set_timing", self._h, int(on))

    def timings(self) -> dict:
        t = np.zeros(10, np.float32)
        N.call("prsp_bsc_gpu_timings_ex", self._h, t.ctypes.data_as(C.c_void_p), 10)
        return dict(zip(["gram", "gemm_yw", "enumerate", "gemm_ytes", "finalize", "mstep",
                         "enum_front", "enum_states", "enum_fallback", "enum_finish"], map(float, t)))

    def launches(self) -> int:
        v = C.c_int()
        N.call("prsp_bsc_gpu_launches", self._h, C.byref(v))
        return v.value

    def _ensure(self, data) -> None:
        y = _f64(data)
        key = (y.__array_interface__["data"][0], y.shape)
        if key != self._data_key:
            self.load(y)


class BscGpuModel(LinearDiscreteGpuModel):
    """BSC truncated-EM on one B200: a drop-in for LinearDiscreteModel(kBsc)."""

    def __init__(self, dim: int, latents: int, trunc: TruncationConfig, device: int = 0):
        super().__init__("bsc", dim, latents, trunc, None, device)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the engine library (rank 0 of a job)."""
    buf = C.create_string_buffer(128)
    N.call("prsp_bsc_gpu_nccl_unique_id", C.cast(buf, C.c_void_p))
    return buf.raw


# ------------------------------------------------------------------ fixtures
def bars_generate(size: int, n: int, prob: float = 0.0, amplitude: float = 10.0, noise: float = 2.0,
                  max_mode: bool = False, seed: int = 0):
    """make_bars (bars.cpp:33-65): (Y n×size², ground-truth W size²×2·size)."""
    d = size * size
    y, w = np.empty((n, d)), np.empty((d, 2 * size))
    N.call("prsp_bsc_bars_generate", size, n, prob, amplitude, noise, int(max_mode), seed, _p(y), _p(w))
    return y, w


def generate(params: BscParams, n: int, seed: int) -> np.ndarray:
    """LinearDiscreteModel::generate (linear_discrete.cpp:452-479), RngStream(seed)."""
    w = _f64(params.W)
    d, h = w.shape
    y = np.empty((n, d))
    N.call("prsp_bsc_generate", d, h, _p(w), float(params.pi), float(params.sigma2), n, seed, _p(y))
    return y


def random_dictionary(dim: int, latents: int, seed: int, scale: float = 5.0) -> np.ndarray:
    w = np.empty((dim, latents))
    N.call("prsp_bsc_random_dictionary", dim, latents, seed, scale, _p(w))
    return w


def baseline_init(y, latents: int, seed: int) -> BscParams:
    y = _f64(y)
    n, d = y.shape
    w = np.empty((d, latents))
    pi, s2 = _dbl(), _dbl()
    N.call("prsp_bsc_baseline_init", d, latents, _p(y), n, seed, _p(w), C.byref(pi), C.byref(s2))
    return BscParams(w, pi.value, s2.value)


def standard_init(y, latents: int, hprime: int, seed: int) -> BscParams:
    y = _f64(y)
    n, d = y.shape
    w = np.empty((d, latents))
    pi, s2 = _dbl(), _dbl()
    N.call("prsp_bsc_standard_init", d, latents, hprime, _p(y), n, seed, _p(w), C.byref(pi), C.byref(s2))
    return BscParams(w, pi.value, s2.value)

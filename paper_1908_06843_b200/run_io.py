"""Run I/O and the training driver around the GPU path.

Mirrors the reference's array and run-directory layer (array_io.cpp,
run_io.cpp, em.cpp; prsp.h's prsp_train / prsp_result_* / prsp_run_open /
prsp_infer): PRSPAR01 arrays, headerless CSV datasets, SHA-256 data hashes,
``train`` (every EM step on the GPU engine; optional run directory with
free_energy.csv, checkpoints, final arrays and a prsp-manifest-1 manifest),
and ``Run`` (reopen a run directory, infer on new data). Everything goes
through the C ABI of ``include/prsp_bsc_gpu.h``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def save_array(path: str, a) -> None:
    """save_array (array_io.cpp:53-64): PRSPAR01 magic, rows, cols, row-major f64."""
    a = _f64(np.atleast_2d(a))
    N.call("prsp_gpu_array_save", str(path).encode(), _p(a), a.shape[0], a.shape[1])


def _load(fn: str, path: str) -> np.ndarray:
    r, c = C.c_uint64(), C.c_uint64()
    N.call(fn, str(path).encode(), C.byref(r), C.byref(c), None)
    out = np.empty((r.value, c.value))
    N.call(fn, str(path).encode(), C.byref(r), C.byref(c), _p(out))
    return out


def load_array(path: str) -> np.ndarray:
    return _load("prsp_gpu_array_load", path)


def load_dataset(path: str) -> np.ndarray:
    """load_dataset (array_io.cpp:140-153): PRSPAR01 by magic, else headerless CSV."""
    return _load("prsp_gpu_dataset_load", path)


def sha256_hex(data: bytes | np.ndarray) -> str:
    b = data.tobytes() if isinstance(data, np.ndarray) else bytes(data)
    buf = C.create_string_buffer(65)
    src = C.create_string_buffer(b, len(b)) if b else None
    N.call("prsp_gpu_sha256", None if src is None else C.cast(src, C.c_void_p), len(b), buf)
    return buf.value.decode()


def sha256_file(path: str) -> str:
    buf = C.create_string_buffer(65)
    N.call("prsp_gpu_sha256_file", str(path).encode(), buf)
    return buf.value.decode()


def format_double(v: float) -> str:
    buf = C.create_string_buffer(32)
    N.call("prsp_gpu_format_double", float(v), buf, 32)
    return buf.value.decode()


class _TrainConfig(C.Structure):
    _fields_ = [("model", C.c_char_p), ("latents", C.c_uint32), ("hprime", C.c_uint32), ("gamma", C.c_uint32),
                ("values", C.c_void_p), ("n_values", C.c_uint32), ("iterations", C.c_uint64), ("seed", C.c_uint64),
                ("workers", C.c_uint32), ("shards", C.c_uint32), ("has_tolerance", C.c_int),
                ("tolerance", C.c_double), ("temperature_pos", C.c_void_p), ("temperature_val", C.c_void_p),
                ("n_temperature", C.c_uint32), ("w_noise_pos", C.c_void_p), ("w_noise_val", C.c_void_p),
                ("n_w_noise", C.c_uint32), ("soft_winner_rho", C.c_double), ("device", C.c_int)]


@dataclass
class TrainConfig:
    """RunConfig (run_io.hpp) for the GPU models: bsc, tsc, dsc, mca, mmca."""

    model: str
    latents: int
    hprime: int = 0
    gamma: int = 0
    values: list | None = None
    iterations: int = 50
    seed: int = 0
    workers: int = 1
    shards: int = 1
    tolerance: float | None = None
    temperature: list = field(default_factory=lambda: [(0.0, 1.0)])
    w_noise: list = field(default_factory=lambda: [(0.0, 0.0)])
    soft_winner_rho: float = 0.0
    device: int = 0


@dataclass
class TrainResult:
    """prsp_result: the free-energy trace and the final parameter arrays by name."""

    free_energy: np.ndarray
    params: dict


def train(cfg: TrainConfig, y, data_file: str | None = None, out_dir: str | None = None) -> TrainResult:
    """train_run (run_io.cpp:196-230) with every EM step on the GPU."""
    y = _f64(y)
    keep = []

    def arr(v):
        a = _f64(v)
        keep.append(a)
        return _p(a)

    tp, tv = zip(*cfg.temperature)
    npos, nval = zip(*cfg.w_noise)
    c = _TrainConfig(cfg.model.encode(), cfg.latents, cfg.hprime, cfg.gamma,
                     arr(cfg.values) if cfg.values is not None else None, len(cfg.values or []), cfg.iterations,
                     cfg.seed, cfg.workers, cfg.shards, int(cfg.tolerance is not None), float(cfg.tolerance or 0.0),
                     arr(tp), arr(tv), len(tp), arr(npos), arr(nval), len(npos), float(cfg.soft_winner_rho),
                     cfg.device)
    h = C.c_void_p()
    N.call("prsp_gpu_train", C.byref(c), _p(y), y.shape[0], y.shape[1],
           None if data_file is None else str(data_file).encode(),
           None if out_dir is None else str(out_dir).encode(), C.byref(h))
    try:
        it = C.c_uint64()
        N.call("prsp_gpu_result_iterations", h, C.byref(it))
        f = np.empty(it.value)
        N.call("prsp_gpu_result_trace", h, _p(f))
        names = ["W", "sigma2"] + (["values", "probs"] if cfg.model == "dsc" else ["pi"])
        params = {}
        for nm in names:
            r, cc = C.c_uint64(), C.c_uint64()
            N.call("prsp_gpu_result_param", h, nm.encode(), C.byref(r), C.byref(cc), None)
            a = np.empty((r.value, cc.value))
            N.call("prsp_gpu_result_param", h, nm.encode(), C.byref(r), C.byref(cc), _p(a))
            params[nm] = a
        return TrainResult(f, params)
    finally:
        N.lib().prsp_gpu_result_free(h)


class Run:
    """A trained run directory (load_run, run_io.cpp:165-194) for inference."""

    def __init__(self, directory: str):
        h = C.c_void_p()
        N.call("prsp_gpu_run_open", str(directory).encode(), C.byref(h))
        self._h = h
        buf, d, l = C.create_string_buffer(16), C.c_uint32(), C.c_uint32()
        N.call("prsp_gpu_run_info", h, buf, 16, C.byref(d), C.byref(l))
        self.model, self.dim, self.latents = buf.value.decode(), d.value, l.value

    def param(self, name: str) -> np.ndarray:
        r, c = C.c_uint64(), C.c_uint64()
        N.call("prsp_gpu_run_param", self._h, name.encode(), C.byref(r), C.byref(c), None)
        a = np.empty((r.value, c.value))
        N.call("prsp_gpu_run_param", self._h, name.encode(), C.byref(r), C.byref(c), _p(a))
        return a

    def infer(self, y, device: int = 0):
        """prsp_infer: (MAP states N×H, MAP masses N, ⟨s⟩ N×H)."""
        y = _f64(y)
        ms, mm, ex = np.empty((y.shape[0], self.latents)), np.empty(y.shape[0]), np.empty((y.shape[0], self.latents))
        N.call("prsp_gpu_run_infer", self._h, _p(y), y.shape[0], y.shape[1], device, _p(ms), _p(mm), _p(ex))
        return ms, mm, ex

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().prsp_gpu_run_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

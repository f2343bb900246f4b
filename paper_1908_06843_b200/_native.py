"""ctypes binding of the C ABI in ``include/prsp_bsc_gpu.h``.

The library ``_lib/libprsp_bsc_b200.so`` is built in-tree by ``build()``
(nvcc, ``-gencode arch=compute_100a,code=sm_100a``). There is no fallback:
importing a compute entry point without the library raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# PRSP_BSC_LIB: an alternative build of the same library (A/B runs of kernel variants)
LIB_PATH = os.environ.get("PRSP_BSC_LIB") or os.path.join(HERE, "_lib", "libprsp_bsc_b200.so")

_u32, _u64, _dbl, _int, _ptr = C.c_uint32, C.c_uint64, C.c_double, C.c_int, C.c_void_p
_dp = C.POINTER(C.c_double)

# name -> (argtypes); every function returns int (prsp_status) unless listed in _RESTYPES
SIGNATURES = {
    "prsp_bsc_gpu_version": [],
    "prsp_bsc_gpu_last_error": [],
    "prsp_bsc_gpu_device_count": [],
    "prsp_bsc_gpu_create": [_u32, _u32, _u32, _u32, _u64, _int, C.POINTER(_ptr)],
    "prsp_bsc_gpu_create_model": [C.c_char_p, _u32, _u32, _u32, _u32, _u64, _ptr, _u32, _int, C.POINTER(_ptr)],
    "prsp_bsc_gpu_model_info": [_ptr, C.POINTER(_int), C.POINTER(_u32), C.POINTER(_u32), _ptr],
    "prsp_bsc_gpu_free": [_ptr],
    "prsp_bsc_gpu_set_stream": [_ptr, _ptr],
    "prsp_bsc_gpu_sync": [_ptr],
    "prsp_bsc_gpu_states_per_point": [_ptr, C.POINTER(_u64)],
    "prsp_bsc_gpu_load_data": [_ptr, _ptr, _u64],
    "prsp_bsc_gpu_load_data_device": [_ptr, _ptr, _u64],
    "prsp_bsc_gpu_set_params": [_ptr, _ptr, _dbl, _dbl],
    "prsp_bsc_gpu_get_params": [_ptr, _ptr, _dp, _dp],
    "prsp_bsc_gpu_set_params_ex": [_ptr, _ptr, _dbl, _dbl, _ptr, _u32],
    "prsp_bsc_gpu_get_params_ex": [_ptr, _ptr, _dp, _dp, _ptr],
    "prsp_bsc_gpu_estep": [_ptr, _dbl],
    "prsp_bsc_gpu_stats_buffer": [_ptr, C.POINTER(_ptr), C.POINTER(_u64)],
    "prsp_bsc_gpu_get_stats": [_ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
    "prsp_bsc_gpu_set_stats": [_ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
    "prsp_bsc_gpu_mstep": [_ptr],
    "prsp_bsc_gpu_step": [_ptr, _dbl, _dp],
    "prsp_bsc_gpu_free_energy": [_ptr, _dp],
    "prsp_bsc_gpu_nccl_unique_id": [_ptr],
    "prsp_bsc_gpu_nccl_init": [_ptr, _ptr, _int, _int],
    "prsp_bsc_gpu_nccl_attach": [_ptr, _ptr],
    "prsp_bsc_gpu_step_allreduce": [_ptr, _dbl, _dp],
    "prsp_bsc_gpu_step_host": [_ptr, _ptr, _u64, _ptr, _dbl, _dbl, _dbl, _ptr, _dp, _dp, _dp],
    "prsp_bsc_gpu_candidates": [_ptr, _ptr],
    "prsp_bsc_gpu_inference": [_ptr, _ptr, _ptr, _ptr],
    "prsp_bsc_gpu_set_timing": [_ptr, _int],
    "prsp_bsc_gpu_timings": [_ptr, _ptr],
    "prsp_bsc_gpu_timings_ex": [_ptr, _ptr, C.c_int],
    "prsp_bsc_gpu_launches": [_ptr, C.POINTER(_int)],
    "prsp_bsc_gpu_check_guards": [],
    "prsp_bsc_gpu_guard_probe": [C.c_int64, C.c_int64],
    "prsp_bsc_gpu_enum_phase_cycles": [_ptr, _ptr],
    "prsp_mca_gpu_create": [C.c_char_p, _dbl, _u32, _u32, _u32, _u32, _u64, _int, C.POINTER(_ptr)],
    "prsp_mca_gpu_free": [_ptr],
    "prsp_mca_gpu_states_per_point": [_ptr, C.POINTER(_u64)],
    "prsp_mca_gpu_load_data": [_ptr, _ptr, _u64],
    "prsp_mca_gpu_set_params": [_ptr, _ptr, _dbl, _dbl],
    "prsp_mca_gpu_get_params": [_ptr, _ptr, _dp, _dp],
    "prsp_mca_gpu_step": [_ptr, _dbl, _dp],
    "prsp_mca_gpu_estep": [_ptr, _dbl],
    "prsp_mca_gpu_stats_buffer": [_ptr, C.POINTER(_ptr), C.POINTER(_u64)],
    "prsp_mca_gpu_get_stats": [_ptr, _ptr, _ptr, _ptr],
    "prsp_mca_gpu_set_stats": [_ptr, _ptr, _ptr, _ptr],
    "prsp_mca_gpu_mstep_fixedpoint": [_ptr, _ptr, _dp],
    "prsp_mca_gpu_residual_commit": [_ptr, _dbl, _dp],
    "prsp_mca_gpu_candidates": [_ptr, _ptr],
    "prsp_mca_gpu_set_sigma2": [_ptr, _dbl],
    "prsp_mca_gpu_inference": [_ptr, _ptr, _ptr, _ptr],
    "prsp_gpu_array_save": [C.c_char_p, _ptr, _u64, _u64],
    "prsp_gpu_array_load": [C.c_char_p, C.POINTER(_u64), C.POINTER(_u64), _ptr],
    "prsp_gpu_dataset_load": [C.c_char_p, C.POINTER(_u64), C.POINTER(_u64), _ptr],
    "prsp_gpu_sha256": [_ptr, _u64, C.c_char_p],
    "prsp_gpu_sha256_file": [C.c_char_p, C.c_char_p],
    "prsp_gpu_format_double": [_dbl, C.c_char_p, _u32],
    "prsp_gpu_train": [_ptr, _ptr, _u64, _u64, C.c_char_p, C.c_char_p, C.POINTER(_ptr)],
    "prsp_gpu_result_iterations": [_ptr, C.POINTER(_u64)],
    "prsp_gpu_result_trace": [_ptr, _ptr],
    "prsp_gpu_result_param": [_ptr, C.c_char_p, C.POINTER(_u64), C.POINTER(_u64), _ptr],
    "prsp_gpu_result_free": [_ptr],
    "prsp_gpu_run_open": [C.c_char_p, C.POINTER(_ptr)],
    "prsp_gpu_run_info": [_ptr, C.c_char_p, _u32, C.POINTER(_u32), C.POINTER(_u32)],
    "prsp_gpu_run_param": [_ptr, C.c_char_p, C.POINTER(_u64), C.POINTER(_u64), _ptr],
    "prsp_gpu_run_infer": [_ptr, _ptr, _u64, _u64, _int, _ptr, _ptr, _ptr],
    "prsp_gpu_run_free": [_ptr],
    "prsp_bsc_bars_generate": [_u32, _u64, _dbl, _dbl, _dbl, _int, _u64, _ptr, _ptr],
    "prsp_bsc_generate": [_u32, _u32, _ptr, _dbl, _dbl, _u64, _u64, _ptr],
    "prsp_bsc_random_dictionary": [_u32, _u32, _u64, _dbl, _ptr],
    "prsp_bsc_baseline_init": [_u32, _u32, _ptr, _u64, _u64, _ptr, _dp, _dp],
    "prsp_bsc_standard_init": [_u32, _u32, _u32, _ptr, _u64, _u64, _ptr, _dp, _dp],
}
_RESTYPES = {
    "prsp_bsc_gpu_version": C.c_char_p,
    "prsp_bsc_gpu_last_error": C.c_char_p,
    "prsp_bsc_gpu_free": None,
    "prsp_mca_gpu_free": None,
    "prsp_gpu_result_free": None,
    "prsp_gpu_run_free": None,
}

STATUS = {0: "PRSP_OK", 2: "PRSP_ERR_CONFIG", 3: "PRSP_ERR_DATA", 4: "PRSP_ERR_NUMERIC", 5: "PRSP_ERR_INTERNAL"}


class PrspError(RuntimeError):
    """A non-zero prsp_status from the engine; ``code`` is the status."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class ConfigError(PrspError):
    pass


class DataError(PrspError):
    pass


class NumericError(PrspError):
    pass


_ERR_CLASS = {2: ConfigError, 3: DataError, 4: NumericError}


def build(quiet: bool = True) -> str:
    """Compile the CUDA engine in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    out = subprocess.run(["make", "-C", CSRC, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("engine build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if not quiet:
        print(out.stdout)
    return LIB_PATH


_lib = None


def lib() -> C.CDLL:
    """The loaded engine library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the sm_100a engine must be built (python -c 'import __graft_entry__ as g; g.build()')"
            )
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, _int)
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().prsp_bsc_gpu_last_error().decode()
        raise _ERR_CLASS.get(rc, PrspError)(rc, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))

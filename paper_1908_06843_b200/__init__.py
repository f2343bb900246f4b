"""B200-native drop-in for the BSC truncated-EM step of prsp (ProSper, arXiv:1908.06843).

Only the hot path named in BASELINE.json is built: the Expectation-Truncation
E-step of Binary Sparse Coding with its M-step sufficient statistics and the
parameter update, as hand-written sm_100a CUDA behind a C ABI
(``include/prsp_bsc_gpu.h``), and the other linear discrete families (ternary
and discrete sparse coding) through the same enumerator, and the max-causes
log-joint (mca / mmca). See DESIGN.md.
"""
from ._native import ConfigError, DataError, NumericError, PrspError, build
from .bsc import (BscGpuModel, BscParams, InferenceResult, LinearDiscreteGpuModel, LinearDiscreteParams, StepResult,
                  SuffStats, TruncationConfig, bars_generate, baseline_init, generate, random_dictionary,
                  standard_init)
from .mca import McaGpuModel, McaParams, McaStats

__all__ = [
    "BscGpuModel", "BscParams", "InferenceResult", "LinearDiscreteGpuModel", "LinearDiscreteParams", "StepResult",
    "SuffStats", "TruncationConfig", "McaGpuModel", "McaParams", "McaStats",
    "bars_generate", "baseline_init", "generate", "random_dictionary", "standard_init", "build",
    "PrspError", "ConfigError", "DataError", "NumericError",
]

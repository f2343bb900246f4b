"""Data-parallel EM over ranks: one process per GPU, contiguous row shards,
one all-reduce of the packed sufficient statistics per EM iteration, then a
replicated deterministic M-step.

The reference's only parallelism is the thread map_reduce over ShardPlan
shards (/root/reference/proj/src/parallel.cpp:27-43, :109-158); here each
rank owns one shard and the ordered fold becomes a sum all-reduce
(``torch.distributed``: NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """ShardPlan::with_shards(n, world, ·).shards[rank] (parallel.cpp:27-43):
    contiguous near-equal shards, the first n % world one row longer."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard plan: bad world/rank")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def stats_count(d: int, h: int, nv: int = 1) -> int:
    return d * h + h + h * h + nv + 3


def pack_stats(st: dict, d: int, h: int) -> np.ndarray:
    """Host copy of the device layout [sum_y_sT D·H | sum_s H | sum_ssT H·H |
    value_counts V | sum_y2 | log_partition | points] (bsc_engine.hpp StatsLayout)."""
    vc = np.atleast_1d(np.asarray(st["value_counts"], float))
    out = np.empty(stats_count(d, h, len(vc)))
    o = 0
    out[o:o + d * h] = np.asarray(st["sum_y_sT"]).ravel()
    o += d * h
    out[o:o + h] = np.asarray(st["sum_s"]).ravel()
    o += h
    out[o:o + h * h] = np.asarray(st["sum_ssT"]).ravel()
    o += h * h
    out[o:o + len(vc)] = vc
    o += len(vc)
    out[o:o + 3] = [st["sum_y2"], st["log_partition"], float(st["points"])]
    return out


def unpack_stats(buf: np.ndarray, d: int, h: int, nv: int = 1) -> dict:
    o = 0
    ysT = buf[o:o + d * h].reshape(d, h).copy()
    o += d * h
    s = buf[o:o + h].copy()
    o += h
    ssT = buf[o:o + h * h].reshape(h, h).copy()
    o += h * h
    vc = buf[o:o + nv].copy()
    t = buf[o + nv:o + nv + 3]
    return dict(sum_s=s, sum_ssT=ssT, sum_y_sT=ysT, value_counts=vc, sum_y2=float(t[0]),
                log_partition=float(t[1]), points=int(round(t[2])))


class _CudaArray:
    """__cuda_array_interface__ over an engine-owned device buffer (zero copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def stats_tensor(model):
    """A torch view of the model's device statistics buffer (for all_reduce)."""
    import torch

    ptr, count = model.stats_buffer()
    return torch.as_tensor(_CudaArray(ptr, count), device=f"cuda:{torch.cuda.current_device()}")


def distributed_step(model, stats_view, temperature: float = 1.0, group=None) -> None:
    """One EM iteration across ranks (any linear discrete family): local E-step →
    all-reduce(Σ stats) → M-step. The model must run on torch's current stream
    (``model.set_stream``)."""
    import torch.distributed as dist

    from . import _native as N

    N.call("prsp_bsc_gpu_estep", model.handle, float(temperature))
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(stats_view, op=dist.ReduceOp.SUM, group=group)
    model.mstep_device()


def init_native(model, group=None) -> None:
    """Give ``model`` the job's NCCL communicator through the engine library: rank
    0's ncclGetUniqueId is broadcast over the torch.distributed group, then every
    rank joins with ncclCommInitRank. After this, ``model.step_allreduce`` runs
    the whole iteration (E-step, statistics all-reduce, M-step) in C++/CUDA."""
    import torch.distributed as dist

    from .bsc import nccl_unique_id

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    model.nccl_init(box[0], world, rank)


def mca_distributed_step(model, temperature: float = 1.0, group=None) -> float:
    """One max-causes iteration across ranks (MaxCausesModel::step,
    max_causes.cpp:416-446): local E pass → all-reduce(Σ winner statistics) →
    replicated fixed-point M-step → local residual pass under W′ → all-reduce(Σ
    residual) → σ² = max(Σ residual / (N·D), 1e-12). Returns F."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import _native as N

    multi = dist.is_initialized() and dist.get_world_size() > 1
    N.call("prsp_mca_gpu_estep", model._h, float(temperature))
    p, n = C.c_void_p(), C.c_uint64()
    N.call("prsp_mca_gpu_stats_buffer", model._h, C.byref(p), C.byref(n))
    if multi:
        view = torch.as_tensor(_CudaArray(p.value, n.value), device=f"cuda:{torch.cuda.current_device()}")
        dist.all_reduce(view, op=dist.ReduceOp.SUM, group=group)
        torch.cuda.synchronize()
    st = model.get_stats()
    N.call("prsp_mca_gpu_mstep_fixedpoint", model._h, None, None)
    r = C.c_double()
    N.call("prsp_mca_gpu_residual_commit", model._h, float(temperature), C.byref(r))
    if multi:
        t = torch.tensor([r.value], dtype=torch.float64, device=f"cuda:{torch.cuda.current_device()}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        total = float(t.item())
        s2 = max(total / (st.points * model.dim), 1e-12)
        N.call("prsp_mca_gpu_set_sigma2", model._h, s2)
    return st.log_partition

"""Multi-rank EM on the GPU engine: row shards as
ShardPlan::with_shards (parallel.cpp:27-43), the packed statistics summed
across ranks in place of map_reduce's ordered fold (parallel.cpp:109-158), a
replicated M-step.

Only one GPU is available to the tests, so the two-rank cases run two
processes on cuda:0 over gloo (host-staged all-reduce of the engine's CUDA
statistics view: no kernel of one rank waits on the other's). The native NCCL
path (prsp_bsc_gpu_step_allreduce) is exercised with a one-rank communicator.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _c2_inputs(n):
    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS["c2"]
    y = configs.data(w, n)
    return w, y, configs.init(w, y)


def _bsc_worker(rank, world, port, out_dir, n, iters):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_1908_06843_b200 as P
    from paper_1908_06843_b200 import dist as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, y, p = _c2_inputs(n)
    b, e = D.shard_range(len(y), world, rank)
    m = P.BscGpuModel(w.D, w.H, P.TruncationConfig(w.H, w.hprime, w.gamma))
    m.set_stream(torch.cuda.current_stream().cuda_stream)
    m.load(y[b:e])
    m.set_params(p)
    view = D.stats_tensor(m)
    out = []
    for _ in range(iters):
        D.distributed_step(m, view)
        torch.cuda.synchronize()
        q = m.get_params()
        out.append(np.r_[q.W.ravel(), q.pi, q.sigma2])
    st = m.get_stats()  # the all-reduced statistics of the last E-step
    np.save(os.path.join(out_dir, f"bsc{rank}.npy"), np.array(out))
    np.save(os.path.join(out_dir, f"bsc_lp{rank}.npy"), np.array([st.log_partition, st.points]))
    m.close()
    dist.destroy_process_group()


def test_two_rank_bsc_step_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    import paper_1908_06843_b200 as P

    n, iters = 6_001, 3
    mp.start_processes(_bsc_worker, args=(2, _free_port(), str(tmp_path), n, iters), nprocs=2, start_method="spawn")
    r0, r1 = np.load(tmp_path / "bsc0.npy"), np.load(tmp_path / "bsc1.npy")
    assert np.array_equal(r0, r1)  # replicated M-step: the same bits on every rank
    w, y, p = _c2_inputs(n)
    m = P.BscGpuModel(w.D, w.H, P.TruncationConfig(w.H, w.hprime, w.gamma))
    m.load(y)
    for i in range(iters):
        r = m.step(p)
        p = r.params
        want = np.r_[p.W.ravel(), p.pi, p.sigma2]
        got = r0[i]
        assert rel(got[:-2], want[:-2]) < 1e-12, (i, rel(got[:-2], want[:-2]))
        assert abs(got[-2] - want[-2]) <= 1e-12 * want[-2] and abs(got[-1] - want[-1]) <= 1e-12 * want[-1]
    lp = np.load(tmp_path / "bsc_lp0.npy")
    assert lp[1] == n and abs(lp[0] - r.free_energy) <= 1e-12 * abs(r.free_energy)
    m.close()


def _mca_inputs(n):
    from oracle.oracle import Oracle

    port = Oracle("port")
    rng = np.random.default_rng(5)
    d, h, hp, g = 16, 12, 6, 3
    wt = np.abs(rng.normal(size=(d, h))) * 2 + 0.05
    y = port.mca_generate("mca", wt, 0.15, 0.3, n, 3)
    w0, pi0, s20 = port.mca_standard_init("mca", y, h, hp, 4)
    return (d, h, hp, g), y, (w0, pi0, s20)


def _mca_worker(rank, world, port, out_dir, n, iters):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_1908_06843_b200 as P
    from paper_1908_06843_b200 import dist as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    (d, h, hp, g), y, (w0, pi0, s20) = _mca_inputs(n)
    b, e = D.shard_range(len(y), world, rank)
    m = P.McaGpuModel("mca", d, h, P.TruncationConfig(h, hp, g))
    m.load(y[b:e])
    m.set_params(P.McaParams(w0, pi0, s20))
    out = []
    for _ in range(iters):
        f = D.mca_distributed_step(m)
        q = m.get_params()
        out.append(np.r_[q.W.ravel(), q.pi, q.sigma2, f])
    np.save(os.path.join(out_dir, f"mca{rank}.npy"), np.array(out))
    dist.destroy_process_group()


def test_two_rank_mca_step_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    import paper_1908_06843_b200 as P

    n, iters = 301, 3
    mp.start_processes(_mca_worker, args=(2, _free_port(), str(tmp_path), n, iters), nprocs=2, start_method="spawn")
    r0, r1 = np.load(tmp_path / "mca0.npy"), np.load(tmp_path / "mca1.npy")
    assert np.array_equal(r0, r1)
    (d, h, hp, g), y, (w0, pi0, s20) = _mca_inputs(n)
    m = P.McaGpuModel("mca", d, h, P.TruncationConfig(h, hp, g))
    m.load(y)
    p = P.McaParams(w0, pi0, s20)
    for i in range(iters):
        r = m.step(p)
        p = r.params
        want = np.r_[p.W.ravel(), p.pi, p.sigma2, r.free_energy]
        got = r0[i]
        assert rel(got[:-3], want[:-3]) < 1e-12, (i, rel(got[:-3], want[:-3]))
        for k in (-3, -2, -1):
            assert abs(got[k] - want[k]) <= 1e-12 * abs(want[k]), (i, k, got[k], want[k])
    m.close()


def test_native_nccl_step_one_rank():
    """prsp_bsc_gpu_step_allreduce with a one-rank communicator: the same bits
    as the single-process step (the all-reduce is the identity)."""
    import paper_1908_06843_b200 as P
    from paper_1908_06843_b200.bsc import nccl_unique_id

    w, y, p = _c2_inputs(3_000)
    a = P.BscGpuModel(w.D, w.H, P.TruncationConfig(w.H, w.hprime, w.gamma))
    a.load(y)
    a.nccl_init(nccl_unique_id(), 1, 0)
    b = P.BscGpuModel(w.D, w.H, P.TruncationConfig(w.H, w.hprime, w.gamma))
    b.load(y)
    pa = pb = p
    for _ in range(3):
        fa = a.step_allreduce(pa)
        pa = a.get_params()
        rb = b.step(pb)
        pb = rb.params
        assert np.array_equal(pa.W, pb.W) and pa.pi == pb.pi and pa.sigma2 == pb.sigma2
        assert fa == rb.free_energy
    a.close()
    b.close()

"""CPU, world_size 2 over gloo: the multi-rank EM path (contiguous shards,
packed statistics, sum all-reduce, replicated M-step) reproduces the
single-process step. Each rank's E-step here is the oracle (test
infrastructure); the sharding, packing and collective are the product's
(paper_1908_06843_b200/dist.py)."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_1908_06843_b200.dist import pack_stats, shard_range, unpack_stats

    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("port")
    y, _ = orc.make_bars(5, 301, seed=2)
    w, pi, s2 = orc.baseline_init(y, 10, 2)
    b, e = shard_range(len(y), world, rank)
    for _ in range(3):
        st = orc.estep_stats(w, pi, s2, y[b:e], 6, 3)
        t = torch.from_numpy(pack_stats(st, 25, 10))
        dist.all_reduce(t)
        tot = unpack_stats(t.numpy(), 25, 10)
        w, pi, s2 = orc.mstep(tot, w, pi, s2)
    np.save(os.path.join(out_dir, f"w{rank}.npy"), np.r_[w.ravel(), pi, s2, tot["log_partition"]])
    dist.destroy_process_group()


def test_two_rank_step_matches_single_process(tmp_path, port):
    import torch.multiprocessing as mp

    port_no = _free_port()
    mp.start_processes(_worker, args=(2, port_no, str(tmp_path)), nprocs=2, start_method="spawn")
    r0, r1 = np.load(tmp_path / "w0.npy"), np.load(tmp_path / "w1.npy")
    assert np.array_equal(r0, r1)  # replicated M-step: identical params on every rank
    y, _ = port.make_bars(5, 301, seed=2)
    w, pi, s2 = port.baseline_init(y, 10, 2)
    for _ in range(3):
        w, pi, s2, f = port.step(w, pi, s2, y, 6, 3, shards=2, workers=1)
    ref = np.r_[w.ravel(), pi, s2, f]
    assert np.allclose(r0, ref, rtol=1e-12, atol=0)

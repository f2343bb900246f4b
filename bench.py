"""Benchmark: BSC truncated-EM data points/s per EM iteration on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

One "step" = one full EM iteration (E-step over the resident shard + sufficient
statistics + all-reduce across ranks + M-step) of BASELINE.json's headline
single-GPU workload c2 (D=256, H=300, H'=12, γ=4, N=200,000 points per GPU,
fp64, synthetic seeded data — see paper_1908_06843_b200/configs.py). Prints one
JSON line (rank 0). `--impl reference` times the reference's own CPU step
(oracle/_ref: the prsp sources built against oracle/eigen_shim) on the host
cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAKS = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
TRAFFIC = os.path.join(ROOT, "profiles", "r02_traffic.json")


def measured_traffic(workload, kernel, points):
    """DRAM bytes per launch of `kernel` (dram__bytes_read.sum + dram__bytes_write.sum)
    from the committed `ncu --set full` capture of this workload, scaled to this
    run's points per launch; (null, why) when no capture matches."""
    if not os.path.exists(TRAFFIC):
        return None, "no committed capture"
    with open(TRAFFIC) as f:
        t = json.load(f)
    if t.get("workload") != workload or kernel not in t.get("per_launch_bytes", {}):
        return None, f"no committed capture of {kernel} at {workload}"
    return (int(t["per_launch_bytes"][kernel] * points / t["points_per_launch"]),
            f"{os.path.relpath(TRAFFIC, ROOT)}: committed ncu capture ({t.get('capture', '?')}), "
            f"scaled to {points} points")


def flops_per_point(D, H, hprime, gamma):
    """SURVEY.md §8(d) algorithmic flop convention (FMA = 2, exp not counted)."""
    from math import comb

    dense = 4 * D * H + 2 * D + 4 * H
    state = 0
    for k in range(0, gamma + 1):
        cnt = 1 if k == 0 else (H if k == 1 else comb(hprime, k))
        f_eval = 0 if k == 0 else 3 * k + k * (k - 1) + 4
        f_acc = 2 * k + k * (k - 1) // 2
        state += cnt * (f_eval + 2 + f_acc)
    return dense, state


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def fp64_peak():
    if os.path.exists(FP64_PEAKS):
        with open(FP64_PEAKS) as f:
            j = json.load(f)
        return j["dmma_m8n8k4_tflops"], j["dfma_tflops"], "profiles/r01_fp64_peaks.json (measured, FP64 DMMA/DFMA)"
    return 37.0, 37.0, "nominal B200 FP64 (no measurement found)"


def int8_peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            bf16 = json.load(f)["bf16_tflops"]
        return round(2.0 * bf16, 1), "2 x MEASURED_PEAKS.json bf16_tflops (B200 dense int8 = 2 x bf16)"
    except Exception:
        return 4500.0, "nominal B200 dense int8 (4.5 POPS)"


def _oracle():
    from oracle import oracle as O

    kind = "ref" if O.Oracle.available("ref") else "port"
    if not O.Oracle.available("port"):
        O.build()
    return O, kind


def oracle_inputs(w, n, rows=None):
    """The workload's inputs drawn through the oracle library (bit-identical to
    the package's fixtures), so the reference arm never maps the product .so."""
    from paper_1908_06843_b200 import configs

    O, _ = _oracle()
    gen = configs.OracleGen(O.Oracle("port"))
    if w.scaling == "strong":
        y = configs.data(w, gen=gen, rows=rows or (0, n))
        y0 = configs.data(w, gen=gen, rows=(0, min(w.N, configs.BLOCK)))
    else:
        y = configs.data(w, n, gen=gen)
        y0 = y
    wi, pi, s2 = O.Oracle("port").baseline_init(y0, w.H, w.seed)
    return y, (wi, pi, s2)


def cpu_reference_rate(y, p, w, threads):
    """The reference's CPU EM step (oracle/_ref, else the C port) over y: points/s."""
    O, kind = _oracle()
    wi, pi, s2 = p
    if kind == "ref":
        sess = O.RefSession(y, w.H, w.hprime, w.gamma)
        t = time.perf_counter()
        sess.step(wi, pi, s2, threads, threads)
        dt = time.perf_counter() - t
        del sess
    else:
        orc = O.Oracle("port")
        t = time.perf_counter()
        orc.step(wi, pi, s2, y, w.hprime, w.gamma, shards=threads, workers=threads)
        dt = time.perf_counter() - t
    return len(y) / dt, ("reference" if kind == "ref" else "port"), dt


def run_reference(args, w, rank, world):
    """The reference arm: the reference's own LinearDiscreteModel::step (oracle/_ref,
    the unmodified prsp sources) on all host threads, rank 0 only, over the same
    workload (c2: the full 200,000-point shard of one GPU per timed step)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = args.points or (w.N if w.scaling == "weak" else w.N)
    sample = min(n, args.ref_sample) if args.ref_sample else n
    y, p = oracle_inputs(w, sample)
    vals = []
    for i in range(args.warmup + args.steps):
        v, kind, dt = cpu_reference_rate(y, p, w, threads)
        if i >= args.warmup:
            vals.append((v, dt))
    value = float(np.mean([v for v, _ in vals]))
    ms = float(np.mean([dt for _, dt in vals]) * 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": w.scaling, "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": config_of(w, n, world),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": kind,
                         "sample": f"{sample} points of {w.name} per timed step (one full EM step: "
                                   f"LinearDiscreteModel::step, ShardPlan::with_shards({sample}, {threads}, "
                                   f"{threads})); inputs drawn by the oracle library"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "BSC truncated-EM data points/sec per iteration"
DATA = "synthetic (seeded BASELINE.json recipe; random init of the stated architecture)"


def config_of(w, n_per_gpu, world):
    return {**w.describe(), "points_per_gpu": n_per_gpu, "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (Y 8·N·D = %.0f MB per GPU)" % (8 * n_per_gpu * w.D / 1e6)}


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--points", type=int, default=0, help="points per GPU (default: the config's N)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="points per reference-arm step (default: the whole per-GPU workload)")
    ap.add_argument("--baseline-sample", type=int, default=0,
                    help="points in the cpu_baseline sample (default: the whole per-GPU workload)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    from paper_1908_06843_b200 import configs

    w = configs.CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        return run_reference(args, w, rank, world)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1908_06843_b200 import BscGpuModel, TruncationConfig, bsc
    from paper_1908_06843_b200 import dist as bdist

    # weak scaling (c0–c3): every rank holds its own N-point shard (seeded per
    # rank); strong scaling (c4): the job's N points are sharded as
    # ShardPlan::with_shards would (parallel.cpp:27-43), each rank drawing its
    # global rows of the blocked dataset (configs.BLOCK), so every world size
    # runs over the same points. Initial params are identical on every rank.
    strong = w.scaling == "strong"
    if strong:
        b, e = bdist.shard_range(args.points or w.N, world, rank)
        n_local = e - b
        y = configs.data(w, rows=(b, e))
        p0 = configs.init(w, configs.data(w, rows=(0, min(w.N, configs.BLOCK))))
    else:
        n_local = args.points or w.N
        y = configs.data(w, n_local, seed_offset=1000 * rank)
        p0 = configs.init(w, y if rank == 0 else configs.data(w, n_local, seed_offset=0))

    model = BscGpuModel(w.D, w.H, TruncationConfig(w.H, w.hprime, w.gamma), device=local)
    stream = torch.cuda.current_stream()
    model.set_stream(stream.cuda_stream)
    model.load(y)
    model.set_params(p0)
    if world > 1:
        # the job's NCCL communicator inside the engine library: an iteration is one
        # C call (E-step, ncclAllReduce of the packed statistics, replicated M-step)
        bdist.init_native(model)

        def one_step():
            model.step_allreduce()
    else:

        def one_step():  # E-step + M-step from the resident parameters: one C call (prsp_bsc_gpu_step)
            model.step_resident()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:  # sampled over warm-up + timed steps (≥ 0.2 s of load)
        for _ in range(args.warmup):
            one_step()
        model.set_timing(True)
        one_step()  # per-kernel breakdown of one step (engine CUDA events)
        kern = model.timings()
        launches_per_step = model.launches()
        model.set_timing(False)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            one_step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms = ms_total / args.steps
    n_total = (args.points or w.N) if strong else n_local * world
    value = n_total / (ms / 1e3)

    # ---- end to end through the reference-facing API with host buffers: every
    # step copies this rank's Y shard from pinned host memory and reads the new
    # parameters back (one GPU: prsp_bsc_gpu_step_host, whose chunked copies
    # overlap the E-step; N GPUs: load + distributed step + get_params)
    e2e = None
    if args.e2e_steps > 0:
        ypin = torch.empty((n_local, w.D), dtype=torch.float64, pin_memory=True)
        ypin.numpy()[:] = y
        p = model.get_params()

        def e2e_step(p):
            if world == 1:
                return model.step_host(p, ypin.numpy()).params
            model.load(ypin.numpy())
            model.set_params(p)
            one_step()
            return model.get_params()

        p = e2e_step(p)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            p = e2e_step(p)
        dt = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": n_total / dt, "unit": "points/s", "h2d_bytes_per_step": int(ypin.numel() * 8 + w.D * w.H * 8),
               "d2h_bytes_per_step": int(w.D * w.H * 8 + 3 * 8), "ms_per_step": dt * 1e3,
               "path": ("prsp_bsc_gpu_step_host (pinned Y + W in, W/pi/sigma2/F out)" if world == 1 else
                        "per rank: prsp_bsc_gpu_load_data (pinned Y shard) + estep + all-reduce + mstep + "
                        "get_params; max over ranks"),
               "bytes_per_rank": world > 1}

    # ---- rooflines. State evaluation (the enumerator launches) against the
    # measured FP64 peak (SURVEY.md §8(d) flop convention); the two sliced
    # products against the int8 tensor-core peak with the int8 work they issue
    # (36 slice products of 2·N·D·H ops). `roofline` is the dominant kernel's.
    dense, state = flops_per_point(w.D, w.H, w.hprime, w.gamma)
    dmma_peak, dfma_peak, peak_src = fp64_peak()
    sliced = os.environ.get("BSC_GEMM", "") != "dmma"
    i8_peak, i8_src = int8_peak()
    gemm_flops = 2.0 * n_local * w.D * w.H
    gemm_work = 36.0 * gemm_flops if sliced else gemm_flops
    gemm_peak, gemm_src = (i8_peak, i8_src) if sliced else (dmma_peak, peak_src)
    gemm_pipe = "tensor (tcgen05 kind::i8, int8 ops)" if sliced else "tensor (DMMA fp64)"
    rows = {
        "enumerate": (state * n_local, kern["enumerate"], dfma_peak, "fp64 pipe (DFMA/exp)", peak_src),
        "gemm_yw": (gemm_work, kern["gemm_yw"], gemm_peak, gemm_pipe, gemm_src),
        "gemm_ytes": (gemm_work, kern["gemm_ytes"], gemm_peak, gemm_pipe, gemm_src),
    }

    def roof(k):
        fl, tms, pk, pipe, src = rows[k]
        ach = fl / (tms / 1e3) / 1e12
        return {"kernel": k, "bound": "tensor" if k.startswith("gemm") else "fp64", "pipe": pipe,
                "achieved": round(ach, 3), "peak": pk, "unit": "TFLOP/s", "frac": round(ach / pk, 4),
                "ms": round(tms, 4), "peak_source": src}

    dom = max(rows, key=lambda k: rows[k][1])
    kernels = {k: roof(k) for k in rows}
    if sliced:
        kernels["gemm_ytes"]["includes"] = "⟨S⟩ slicing + column sums"
    kernels.update({k: {"ms": round(kern[k], 4)} for k in ("gram", "finalize", "mstep")})
    if kern.get("enum_front", 0.0) > 0.0:  # the lane path's launches inside "enumerate"
        kernels["enumerate"]["parts_ms"] = {k[5:]: round(kern[k], 4)
                                            for k in ("enum_front", "enum_states", "enum_fallback", "enum_finish")}
    traffic, traffic_src = measured_traffic(w.name, dom, n_local)
    step_flops = (dense + state) * n_total
    line = {
        "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": w.scaling, "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": config_of(w, n_local, world),
        "roofline": {**roof(dom), "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic": "SURVEY.md §8(d): F_state=%d, F_dense=%d flops/point; int8 slice products "
                                    "36·2·D·H ops/point per product" % (state, dense)},
        "state_roofline": roof("enumerate"),
        "step_rate": {"flops_per_step": step_flops, "tflops_per_gpu": round(step_flops / (ms / 1e3) / 1e12 / world, 3),
                      "note": "SURVEY.md §8(d) fp64-equivalent algorithmic flops of the whole step per second; not a "
                              "fraction of any one peak: the two products run as int8 slice products on the tensor "
                              "cores (kernels.gemm_*: int8 ops against the int8 peak), the state evaluation on the "
                              "FP64 pipe (state_roofline)"},
        "kernels": kernels,
        "clocks": clk.summary(),
        "gpu_launches": int(launches_per_step * args.steps),
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            # bounded samples: the whole c2 workload on all host threads (~5 s on 16),
            # the same CPU work for the larger dictionaries (cost per point ∝ D·H);
            # and a 1-core figure on a tenth of that
            sample = args.baseline_sample or min(n_local, max(2000, 200000 * 256 * 300 // (w.D * w.H)))
            yb, pb = oracle_inputs(w, sample)
            v, kind, dt = cpu_reference_rate(yb, pb, w, threads)
            s1 = max(500, sample // 20)
            v1, _, dt1 = cpu_reference_rate(yb[:s1], pb, w, 1)
            line["cpu_baseline"] = {"value": v, "unit": "points/s", "cores": threads, "kind": kind,
                                    "sample": f"{sample} points of {w.name}, one full EM "
                                              f"step on all host threads ({dt:.1f} s)",
                                    "value_1core": v1,
                                    "sample_1core": f"first {s1} of those points, one full EM step on 1 thread "
                                                    f"({dt1:.1f} s)"}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    model.close()


if __name__ == "__main__":
    main()

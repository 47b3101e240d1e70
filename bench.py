#!/usr/bin/env python
"""bench.py -- training samples/s and peak HBM per GPU of the index-batched DCRNN step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config pems] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU, NCCL)

A step = gather (index batching) -> DCGRU forward + BPTT -> NCCL gradient all-reduce -> Adam,
replayed as one CUDA graph per step, on synthetic seeded inputs of the named workload shape
(BASELINE.json configs; full-PeMS-shaped by default = the largest config that fits one GPU, the
north_star target).  Timing: W untimed warm-up
steps, then exactly K steps between barrier + synchronize, CUDA events on the launching stream,
max over ranks.  Prints ONE JSON line on rank 0 (contract: see DESIGN.md "Measurement").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training samples/sec and peak HBM per GPU, index-batched DCRNN, at 1/2/4/8 B200"
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # SIMT FFMA peak at max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: about 2 s of steps for the workload)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="pems",
                    help="workload (synth.CONFIGS); default: full-PeMS-shaped, the largest "
                         "BASELINE.json config that fits one GPU (the north_star target)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", type=int, default=1,
                    help="1 = bf16 tcgen05 path (default, 2e-2 parity); 0 = fp32 SIMT (1e-5 parity)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=3,
                    help="graph replays traced with CUPTI (torch.profiler) for per-kernel times")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--epoch", action="store_true",
                    help="also train one full epoch (every rank's shard) and report its time")
    ap.add_argument("--placement", default="halo", choices=["halo", "replicated"],
                    help="halo shard (BASELINE north star) or the paper's replicated copy with a "
                         "global shuffle and per-epoch validation all-reduce (P:325, P:424)")
    ap.add_argument("--model", default="stepwise", choices=["stepwise", "encdec"],
                    help="stepwise PGT-DCRNN (default) or Li et al.'s encoder-decoder (f3)")
    ap.add_argument("--cheb", action="store_true",
                    help="diffusion blocks by the Chebyshev recurrence (f3, reading c25)")
    ap.add_argument("--zero-copy", action="store_true",
                    help="read windows straight from the series by index (no x/y gather, f2)")
    ap.add_argument("--shuffle", default="window", choices=["window", "batch", "none"],
                    help="per-epoch window shuffle, batch-order shuffle (P:454), or none")
    return ap.parse_args()


def env_ranks():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------------------ clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200", "-i",
                                       str(gpu)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        sm, mx, reasons, pw = [], [], set(), []
        for line in open(self.f.name):
            c = [x.strip() for x in line.split(",")]
            if len(c) < 8:
                continue
            try:
                sm.append(float(c[1]))
                mx.append(float(c[2]))
                pw.append(float(c[3]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, c[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------ oracle legs
def host_cores() -> dict:
    """What the host offers the oracle: os.cpu_count(), the affinity mask, and the BLAS pools
    per library (threadpoolctl; numpy and scipy may each bring their own)."""
    info = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "blas": {}}
    try:
        import numpy  # noqa: F401  (loads the BLAS pools to be listed)
        import scipy.sparse  # noqa: F401
        import threadpoolctl
        for i in threadpoolctl.threadpool_info():
            if i.get("user_api") == "blas":
                key = f"{i.get('internal_api')}:{os.path.basename(i.get('filepath', ''))}"
                info["blas"][key] = i.get("num_threads")
    except Exception as e:  # pragma: no cover
        info["blas_error"] = str(e)
    # the oracle's heavy work (dense GEMMs) runs on one BLAS pool at a time, bounded by the
    # affinity mask; SciPy's CSR products are single-threaded
    info["used"] = min(info["affinity"], max(info["blas"].values() or [1]))
    return info


class OracleLeg:
    """The float64 oracle (Alg. 1 materialisation of the sampled windows + DCGRU forward/backward
    + Adam), as it stands, on a bounded sample of the workload (tests' oracle/, host cores)."""

    def __init__(self, cfg, model: str = "stepwise"):
        import numpy as np

        import synth
        from oracle import pipeline

        self.np, self.cfg, self.model = np, cfg, model
        t0 = time.perf_counter()
        # bounded setup: the oracle's cost per window does not depend on E, so huge series (full
        # PeMS: 9.4 GB of float32) are cut to their first rows for the timing sample
        self.rows = cfg.E
        if cfg.N * cfg.E > 200_000_000:
            self.rows = max(256, min(4096, 20_000_000 // cfg.N))
        self.ref = pipeline.Reference(cfg.replace(E=self.rows) if self.rows < cfg.E else cfg,
                                      materialize_all=False)
        self.setup_s = time.perf_counter() - t0
        self.theta = synth.make_params(cfg, kind="train", model=model).astype(np.float64)
        self.m = np.zeros_like(self.theta)
        self.v = np.zeros_like(self.theta)
        self.plan = self.ref.plan(1, 0)
        self.j, self.it = 0, 0

    def batch(self, n: int) -> float:
        """One training step of the oracle on the next n windows of the plan; seconds."""
        from oracle import adam, dcgru, encdec
        np = self.np
        if self.j + n > self.plan.size:
            self.j = 0
        idx = self.plan[self.j:self.j + n]
        self.j += n
        t1 = time.perf_counter()
        x, y = self.ref.batch(idx)
        f = encdec.loss_and_grad if self.model == "encdec" else dcgru.backward
        _, g, _ = f(self.theta, self.ref.d, self.ref.Pf, self.ref.Pb, x.astype(np.float64),
                    y.astype(np.float64))
        self.it += 1
        self.theta, self.m, self.v = adam.adam_step(self.theta, g, self.m, self.v, self.it, 1e-2)
        return time.perf_counter() - t1

    def details(self) -> dict:
        return dict(setup_s=round(self.setup_s, 2), series_rows=self.rows,
                    cores=host_cores())


def cpu_baseline_leg(cfg, model, budget_s: float = 20.0):
    """cpu_baseline of our arm (rank 0, N = 1): one warm-up window (also the per-window cost),
    then as many windows as fit ~budget_s (1 .. B) as one timed batch."""
    leg = OracleLeg(cfg, model)
    per = leg.batch(1)
    n = int(max(1, min(cfg.B, budget_s // max(per, 1e-9))))
    t = leg.batch(n)
    det = leg.details()
    det.update(warmup_windows=1, warmup_s=round(per, 2), windows=n, timed_s=round(t, 2))
    return {"value": round(n / t, 4), "unit": "samples/s", "cores": det["cores"]["used"],
            "kind": "oracle",
            "sample": f"one batch of {n} windows of {cfg.name} (B={cfg.B} in the GPU step) after "
                      f"a 1-window warm-up: float64 Alg. 1 materialisation + DCGRU fwd/bwd + "
                      f"Adam, series cut to {leg.rows} rows (cost per window is independent of "
                      f"E); host {det['cores']['cpu_count']} CPUs, affinity "
                      f"{det['cores']['affinity']}", "details": det}


def run_reference(args, cfg):
    """--impl reference: the oracle is this tier's reference arm (rank 0 only, host cores)."""
    rank, world, _ = env_ranks()
    if rank != 0:
        return
    K, W = args.steps or 5, args.warmup
    leg = OracleLeg(cfg, args.model)
    per = leg.batch(1)            # calibration (counts toward nothing)
    # size each step so the whole run ends in ~3 min (a step is at least one window)
    b = int(max(1, min(cfg.B, math.floor(150.0 / max(1, K + W) / max(per, 1e-9)))))
    for _ in range(W):
        leg.batch(b)
    t = sum(leg.batch(b) for _ in range(K))
    sps = K * b / t
    det = leg.details()
    det.update(windows_per_step=b, timed_s=round(t, 2), calibration_s=round(per, 2))
    line = {"metric": METRIC, "value": round(sps, 4), "unit": "samples/s", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": round(1000.0 * t / K, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, world, args, arm="reference", windows_per_step=b),
            "cpu_baseline": {"value": round(sps, 4), "unit": "samples/s",
                             "cores": det["cores"]["used"], "kind": "oracle",
                             "sample": f"{K} steps x {b} windows of the {cfg.name} workload "
                                       f"(after {W} warm-up steps), float64 oracle on the host"},
            "e2e": {"value": round(sps, 4), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "oracle": det}
    emit(line)


# The JSON line goes to the ORIGINAL stdout; everything else written to fd 1 afterwards (NCCL's
# version banner, library chatter) is redirected to stderr so stdout carries exactly one line.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict):
    _claim_stdout()
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()


def config_dict(cfg, world, args, arm="ours", windows_per_step=None):
    d = {"workload": cfg.name, "N": cfg.N, "E": cfg.E, "F": cfg.F, "T_in": cfg.T_in,
         "T_out": cfg.T_out, "layers": cfg.L, "hidden": cfg.H, "K_hops": cfg.K,
         "model": args.model, "diffusion_basis": "chebyshev" if cfg.cheb else "powers"}
    if arm == "reference":
        d.update({"precision": "fp64 (the oracle)", "windows_per_step": windows_per_step,
                  "per_gpu_batch_of_our_arm": cfg.B,
                  "parallelism": "one host process (rank 0), no GPU"})
        return d
    d.update({"per_gpu_batch": cfg.B, "global_batch": cfg.B * world,
              "parallelism": f"dp{world} ({args.placement} distributed-index-batching, "
                             f"{args.shuffle} shuffle)",
              "precision": "fp32" if args.precision == 0 else "bf16",
              "l2": "no flush: each step writes >= 1 GB of fresh activations (>> 126 MB L2)",
              "cuda_graph": not args.no_graph, "zero_copy": bool(args.zero_copy)})
    return d


# ------------------------------------------------------------------------------ kernel trace
def kernel_class(name: str) -> str:
    """libpgti kernel name (demangled) -> the accounting class of profile.cuh."""
    n = name.lower()
    if "nccl" in n:
        return "allreduce"
    if "k_gather" in n:
        return "gather"
    if "k_spmm" in n:
        return "spmm"
    if "k_tc_fwd" in n:
        import re
        m = re.search(r"k_tc_fwdp?<\s*\d+\s*,\s*([^>]+)>", name)
        mode = m.group(1) if m else ""
        return "gemm_dgrad" if ("2" in mode or "bwd" in mode.lower()) else "gemm_fwd"
    if "k_gconv_fwd" in n:
        return "gemm_fwd"
    if "k_gconv_dgrad" in n:
        return "gemm_dgrad"
    if "reduce" in n:
        return "reduce"
    if "wgrad" in n and "k_xpart" not in n:
        return "gemm_wgrad"
    if "k_loss" in n:
        return "loss"
    if "k_adam" in n or "k_incr" in n:
        return "adam"
    if "k_keys" in n or "radix" in n or "k_expand" in n:
        return "index"
    return "elementwise"


def _busy(intervals) -> float:
    """Length of the union of [start, end) intervals."""
    tot, cur_s, cur_e = 0.0, None, None
    for a, b in sorted(intervals):
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def kernel_trace(torch, replay, P: int, rank: int) -> dict:
    """Kernel durations of P replays of the captured step from CUPTI activity records
    (torch.profiler / kineto chrome trace): per kernel name and per class, ms per step (sum of
    exclusive kernel durations, PDL pre-wait removed; raw CUPTI sums alongside) and busy ms per
    step (union of the class's exclusive intervals)."""
    res = {"kernels": {}, "class_ms_per_step": {}, "class_busy_ms_per_step": {}}
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as pr:
            for j in range(P):
                replay(j)
            torch.cuda.synchronize()
        fd, path = tempfile.mkstemp(suffix=".json")
        os.close(fd)
        pr.export_chrome_trace(path)
        ev = json.load(open(path)).get("traceEvents", [])
        os.unlink(path)
    except Exception as e:  # the bench value does not depend on this
        res["error"] = f"{type(e).__name__}: {e}"
        return res
    # a kernel launched with programmatic dependent launch starts while its stream predecessor
    # drains and waits at griddepcontrol.wait: its CUPTI interval includes that wait.  The
    # exclusive interval starts at max(its start, the predecessor's end on the same stream).
    kev = [e for e in ev if e.get("cat") == "kernel" and "dur" in e]
    kev.sort(key=lambda e: float(e["ts"]))
    last_end = {}
    per_name, per_cls, per_cls_x, spans = {}, {}, {}, {}
    for e in kev:
        name = e.get("name", "?")
        a = float(e["ts"]) / 1e3
        b = a + float(e["dur"]) / 1e3                        # us -> ms
        sid = (e.get("args") or {}).get("stream", e.get("tid"))
        ax = max(a, last_end.get(sid, a))
        last_end[sid] = max(b, last_end.get(sid, b))
        c = kernel_class(name)
        k = per_name.setdefault(name, {"class": c, "ms": 0.0, "xms": 0.0, "launches": 0})
        k["ms"] += b - a
        k["xms"] += max(0.0, b - ax)
        k["launches"] += 1
        per_cls[c] = per_cls.get(c, 0.0) + (b - a)
        per_cls_x[c] = per_cls_x.get(c, 0.0) + max(0.0, b - ax)
        spans.setdefault(c, []).append((ax, max(ax, b)))
    res["kernels"] = {n: {"class": v["class"], "ms_per_step": round(v["xms"] / P, 5),
                          "raw_ms_per_step": round(v["ms"] / P, 5),
                          "launches_per_step": v["launches"] / P,
                          "us_per_launch": round(1e3 * v["xms"] / v["launches"], 3)}
                      for n, v in sorted(per_name.items(), key=lambda kv: -kv[1]["xms"])}
    res["class_ms_per_step"] = {c: v / P for c, v in per_cls_x.items()}
    res["class_raw_ms_per_step"] = {c: v / P for c, v in per_cls.items()}
    res["class_busy_ms_per_step"] = {c: _busy(sp) / P for c, sp in spans.items()}
    all_spans = [x for sp in spans.values() for x in sp]
    res["gpu_busy_ms_per_step"] = _busy(all_spans) / P
    # idle time: gaps between the merged busy intervals, by (kernel that ended last, kernel that
    # starts next), ms per step; the largest ones say where the step waits on dependencies
    named = sorted(((a, b, kernel_class(e.get("name", "?")), e.get("name", "?"))
                    for e in kev for a, b in [(float(e["ts"]) / 1e3,
                                               float(e["ts"]) / 1e3 + float(e["dur"]) / 1e3)]))
    gaps, end, end_name = {}, None, None
    for a, b, _, n in named:
        if end is not None and a > end:
            key = f"{_short(end_name)} -> {_short(n)}"
            gaps[key] = gaps.get(key, 0.0) + (a - end) / P
        if end is None or b > end:
            end, end_name = b, n
    res["idle_gaps_ms_per_step"] = {k: round(v, 4) for k, v in
                                    sorted(gaps.items(), key=lambda kv: -kv[1])[:12]}
    return res


def _short(name: str) -> str:
    """Kernel name without namespaces and parameter list (for the gap table)."""
    n = name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")
    return n.split("::")[-1]


# ------------------------------------------------------------------------------ our arm
def main():
    _claim_stdout()
    args = parse()
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.cheb:
        cfg = cfg.replace(cheb=True)
    if args.precision == 1 and cfg.H != 64:
        # the tcgen05 path is built for 64 hidden units (one 128-byte SWIZZLE_128B row per
        # diffusion block); Chickenpox's 32-unit model runs on the fp32 SIMT path
        print(f"bench: {cfg.name} has H={cfg.H}: running the fp32 path (precision 0)",
              file=sys.stderr)
        args.precision = 0
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if args.steps is None:   # about 2 s of timed steps
        args.steps = {"chickenpox": 300, "metr_la": 1000, "pems_bay": 700,
                      "pems_all_la": 100, "pems": 25}.get(cfg.name, 50)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2507_11683_b200 import pgti
    from paper_2507_11683_b200.trainer import Trainer

    rank, world, local = env_ranks()
    if world > 1:   # NCCL reports each communicator's setup (ranks, transports) on stderr
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    # libpgti's NCCL communicator (the gradient all-reduce, a8).  At world 1 it is a 1-rank
    # communicator: the step still runs the (identity) ncclAllReduce, like every rank at N > 1.
    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(pgti.comm_unique_id()), dtype=torch.uint8))
    if world > 1:
        dist.broadcast(uid, 0)
    comm = pgti.Comm(bytes(uid.cpu().numpy().tolist()), rank, world, local)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------------------------------------------------------- setup (untimed)
    graph = synth.make_graph(cfg.N, cfg.knn)
    params0 = synth.make_params(cfg, kind="train", model=args.model)
    from paper_2507_11683_b200.trainer import shard_plan, train_windows, window_count
    from paper_2507_11683_b200.trainer import replicated_plan
    S_tr = train_windows(window_count(cfg.E, cfg.T_in, cfg.T_out))
    p = (shard_plan(S_tr, world, rank, cfg.T_in, cfg.T_out) if args.placement == "halo"
         else replicated_plan(S_tr, cfg.E, cfg.T_in))
    rows = synth.make_series(cfg, row_lo=p.row_lo, row_hi=p.row_hi)
    barrier()
    t0 = time.perf_counter()
    tr = Trainer(cfg, graph, lambda a, b: rows, params0, rank, world, local, comm,
                 precision=args.precision, use_cuda_graph=not args.no_graph,
                 placement=args.placement, zero_copy=args.zero_copy,
                 model=1 if args.model == "encdec" else 0,
                 shuffle={"window": True, "batch": "batch", "none": False}[args.shuffle])
    torch.cuda.synchronize()
    load_s = time.perf_counter() - t0
    spe = tr.start_epoch(0)
    state = {"epoch": 0}

    def run(jg):
        e, j = divmod(jg, spe)
        if e != state["epoch"]:
            tr.start_epoch(e)
            state["epoch"] = e
        tr.step(j)

    for j in range(args.warmup):
        run(j)
    tr.check()
    barrier()
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed region
    clocks = Clocks(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev0.record()
    for j in range(args.warmup, args.warmup + args.steps):
        run(j)
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    t_ms = float(ms.item())
    value = world * cfg.B * args.steps / (t_ms / 1000.0)
    tr.check()
    loss_last = float(tr.loss.item())

    # ---------------------------------------------------------------- per-kernel breakdown
    # (1) ALGORITHMIC bytes / flops per kernel class: libpgti's per-launch accounting (DESIGN.md
    #     section 5 models), collected on one eager step right after the timed region -- counts
    #     only, no timing is taken from it;
    # (2) TIME per kernel class: CUPTI activity records (torch.profiler / kineto) of
    #     --profile-steps replays of the SAME captured graph the timed region replays, so the
    #     durations are those of the timed step's launches (PDL chaining and stream concurrency
    #     included).  Profiler numbers explain the step; the bench value is the event-timed one.
    use_graph = tr.use_cuda_graph
    tr.use_cuda_graph = False
    pgti.profile_read()
    pgti.profile_enable(True)
    base = args.warmup + args.steps
    run(base)
    torch.cuda.synchronize()
    prof = pgti.profile_read()
    pgti.profile_enable(False)
    tr.use_cuda_graph = use_graph
    ours = {k: v for k, v in prof.items() if k != "allreduce" and v["launches"]}
    launches_per_step = sum(v["launches"] for v in ours.values())
    P = args.profile_steps
    trace = kernel_trace(torch, lambda j: run(base + 1 + j), P, rank)
    cls_ms = trace["class_ms_per_step"]
    kernels = {k: {"ms_per_step": round(cls_ms.get(k, 0.0), 4),
                   "busy_ms_per_step": round(trace["class_busy_ms_per_step"].get(k, 0.0), 4),
                   "launches_per_step": v["launches"],
                   "GB_per_step": round(v["bytes"] / 1e9, 4),
                   "GFLOP_per_step": round(v["flops"] / 1e9, 3)}
               for k, v in prof.items() if v["launches"]}
    timed = {k: v for k, v in ours.items() if cls_ms.get(k, 0.0) > 0}
    dom = max(timed, key=lambda k: cls_ms[k]) if timed else max(ours, key=lambda k: ours[k]["ms"])
    d = prof[dom]
    dms = cls_ms.get(dom) or d["ms"]
    peaks, src = measured_peaks()
    if dom.startswith("gemm") and args.precision == 0:
        ach = d["flops"] / (dms / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": round(ach, 3), "peak": round(FP32_PEAK_TFLOPS, 1),
                "unit": "TFLOP/s", "frac": round(ach / FP32_PEAK_TFLOPS, 4), "traffic": None,
                "kernel": dom, "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz"}
    elif dom.startswith("gemm"):
        ach = d["flops"] / (dms / 1e3) / 1e12
        pk = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
        roof = {"bound": "tensor", "achieved": round(ach, 3), "peak": pk, "unit": "TFLOP/s",
                "frac": round(ach / pk, 4), "traffic": None, "kernel": dom,
                "peak_source": f"{src}, sustained (kernel timed inside a long step)"}
    else:
        ach = d["bytes"] / (dms / 1e3) / 1e9
        pk = peaks["hbm_gbs"]
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk, "unit": "GB/s",
                "frac": round(ach / pk, 4), "traffic": None, "kernel": dom, "peak_source": src}
    step_ms = t_ms / args.steps
    roof["timing"] = ("CUPTI kernel records of captured-graph replays (torch.profiler), "
                      f"{P} replays; each kernel's interval starts at max(its start, its stream "
                      "predecessor's end) so the PDL pre-wait is not counted"
                      if trace["kernels"] else "eager event brackets (no CUPTI)")
    roof["raw_cupti_ms_per_step"] = round(trace.get("class_raw_ms_per_step", {}).get(dom, 0.0), 4)
    roof["share_of_step"] = round(trace["class_busy_ms_per_step"].get(dom, dms) / step_ms, 4)
    roof["per_launch_ms"] = round(dms / d["launches"], 5)
    roof["launches_per_step"] = d["launches"]
    # whole step against the HBM roofline: the algorithmic bytes of every libpgti launch of one
    # step (the per-kernel models of DESIGN.md section 5) over the timed step time
    step_bytes = sum(v["bytes"] for k, v in ours.items())
    step_ach = step_bytes / (step_ms / 1e3) / 1e9
    step_roof = {"bytes_per_step": step_bytes, "bytes_per_sample": step_bytes / cfg.B,
                 "achieved": round(step_ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                 "frac": round(step_ach / peaks["hbm_gbs"], 4)}
    # traffic: DRAM bytes per launch of this kernel class from the committed ncu --set full
    # capture of the same workload (profiles/traffic_<config>.json, cold cache per launch)
    tpath = os.path.join(ROOT, "profiles", f"traffic_{cfg.name}.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        tk = "gemm" if dom in ("gemm_fwd", "gemm_dgrad") and "gemm" in tj else dom
        if tk in tj:
            roof["traffic"] = tj[tk]["dram_bytes_per_launch"]
            roof["traffic_source"] = f"profiles/traffic_{cfg.name}.json ({tj[tk]['source']})"
    roof["algorithmic_per_launch"] = {"bytes": d["bytes"] / d["launches"],
                                      "flops": d["flops"] / d["launches"]}
    # the gate GEMMs against the tensor-core roofline (north star: "the gate GEMMs report
    # tensor-pipe utilisation"): every tcgen05 GEMM class of the step
    gemm_roof = None
    gk = [k for k in ("gemm_fwd", "gemm_dgrad", "gemm_wgrad") if k in ours and cls_ms.get(k)]
    if gk and args.precision == 1:
        gf = sum(ours[k]["flops"] for k in gk)
        gms = sum(cls_ms[k] for k in gk)
        pk = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
        ach = gf / (gms / 1e3) / 1e12
        gemm_roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": pk, "unit": "TFLOP/s",
                     "frac": round(ach / pk, 4), "kernels": gk,
                     "per_class_tflops": {k: round(ours[k]["flops"] / (cls_ms[k] / 1e3) / 1e12, 2)
                                          for k in gk}, "peak_source": src}
    if rank == 0 and trace["kernels"]:
        out = os.path.join(ROOT, "gpurun_out")
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"kernel_trace_{cfg.name}_n{world}.json"), "w") as f:
            json.dump({"config": cfg.name, "world": world, "step_ms": step_ms,
                       "replays": P, **trace}, f, indent=1)

    # ---------------------------------------------------------------- end to end (host buffers)
    e2e = None
    if not args.no_e2e:
        B = cfg.B
        tr.start_epoch(1)
        plan_host = tr.epoch_plan().cpu().pin_memory()
        loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()
        n_e2e = min(args.steps, tr.n_used // B)
        for j in range(min(3, n_e2e)):
            tr.step_from_host(plan_host[j * B:(j + 1) * B])
        torch.cuda.synchronize()
        barrier()
        t1 = time.perf_counter()
        for j in range(n_e2e):
            tr.step_from_host(plan_host[j * B:(j + 1) * B])
            loss_host.copy_(tr.loss, non_blocking=True)
            torch.cuda.current_stream().synchronize()   # the host reads this step's loss
        barrier()
        te = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * B * n_e2e / float(te.item()), 2), "unit": "samples/s",
               "h2d_bytes_per_step": 4 * B, "d2h_bytes_per_step": 4, "steps": n_e2e,
               "what": "per step: pinned H2D of the batch's window starts, graph replay of "
                       "gather+fwd+bwd+allreduce+Adam, D2H of the loss, host sync",
               "load_s": round(load_s, 3)}

    # ---------------------------------------------------------------- one full epoch
    epoch = None
    if args.epoch:
        tr.start_epoch(2)
        barrier()
        torch.cuda.synchronize()
        ev0.record()
        for j in range(spe):
            tr.step(j)
        ev1.record()
        torch.cuda.synchronize()
        tr.check()
        barrier()
        ems = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        esec = float(ems.item()) / 1e3
        val = None
        if args.placement == "replicated":  # the paper's per-epoch validation all-reduce
            barrier()
            torch.cuda.synchronize()
            tv = time.perf_counter()
            mae = tr.validate()
            torch.cuda.synchronize()
            val = {"mae_normalised": mae, "seconds": round(time.perf_counter() - tv, 3)}
        epoch = {"steps_per_rank": spe, "samples": world * cfg.B * spe, "seconds": round(esec, 3),
                 "validation": val,
                 "samples_per_s": round(world * cfg.B * spe / esec, 2),
                 "loss_last": float(tr.loss.item()),
                 "what": "epoch 2 of this placement's plan, CUDA-graph steps, max over ranks"}

    # ---------------------------------------------------------------- memory + gather
    peak_alloc = torch.cuda.max_memory_allocated(dev) / 1e9
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        nvml_used = pynvml.nvmlDeviceGetMemoryInfo(h).used / 1e9
    except Exception:
        nvml_used = None
    mem = torch.tensor([peak_alloc, nvml_used or 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mem, op=dist.ReduceOp.MAX)
        gathered = [None] * world
        dist.all_gather_object(gathered, ck)
        reasons = sorted({r for g in gathered for r in g.get("reasons", [])})
        ck["reasons"] = reasons
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(cfg, args.model)
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "samples/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(t_ms / args.steps, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f32" if args.precision == 0 else "bf16",
                "data": "synthetic (seeded series + kNN sensor graph of the workload's shape, "
                        "random-init parameters)",
                "config": config_dict(cfg, world, args),
                "peak_hbm_gb": {"torch_max_allocated": round(float(mem[0]), 3),
                                "nvml_used": round(float(mem[1]), 3) if nvml_used else None},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps,
                "launches_per_step": launches_per_step, "clocks": ck,
                "step_roofline": step_roof, "gemm_roofline": gemm_roof,
                "kernels": kernels,
                "gpu_busy_ms_per_step": round(trace.get("gpu_busy_ms_per_step", 0.0), 4),
                "loss_last": loss_last, "steps_per_epoch": spe}
        if epoch is not None:
            line["epoch"] = epoch
        emit(line)
    # tear down: drop the captured graph (it holds NCCL kernels) before the communicator
    tr.graph = None
    torch.cuda.synchronize()
    barrier()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

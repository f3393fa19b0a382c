#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 MCR-DL collective hot path.

Metric (BASELINE.json): collective bus GB/s at 1/2/4/8 B200. One step = one
all_reduce (sum, fp32, out of place) of S = 256 MiB per rank through the
public API (Runtime.post on an nvlink backend), configs[1]'s >= 64 MB point.

  value  = whole-job bus bytes / time = N * busbw, busbw = 2(N-1)/N * S / t
           (nccl-tests definition), the same definition at every N. At N = 1
           there are no peers: the all_reduce is a local copy and its bus
           bytes are taken as S (each element delivered once); the HBM view
           of that copy (2*S read + write vs the HBM peak) is reported
           separately as config.local_copy_floor_gbs and in `roofline`.
  e2e    = the same metric through the same API with HOST (pinned) buffers:
           H2D of the input, the collective, D2H of the result, per step.
  roofline: dominant kernel (k_ar_pipe for N > 1, k_copy for N = 1),
           algorithmic bytes per launch / mean launch time (CUDA events on
           the launching stream) vs NVLink 900 GB/s/direction (N > 1) or
           the measured HBM copy peak (N = 1).
  cpu_baseline: the reference package itself (baseline/_ref, pure Python +
           numpy, thread world of N ranks, the SAME S) on a bounded number of
           steps, rank 0, at every N.

  --impl reference  times the reference's own CPU implementation on the same
           metric, config (S per rank, N thread-ranks) and --steps/--warmup
           (capped only if the estimate exceeds a few minutes, then stated);
           rank 0 runs it, other ranks exit.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
       (N > 1: launched under torch.distributed.run, one process per GPU)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MIB = 1 << 20
METRIC = "Collective bus GB/s vs message size at 2/4/8 B200 (alltoallv, allreduce)"
NVLINK_PEAK = 900.0  # GB/s per direction per GPU (north_star nominal)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("native", "reference"), default="native")
    ap.add_argument("--size-mib", type=int, default=256)
    ap.add_argument("--no-secondary", action="store_true")
    return ap.parse_args()


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:  # noqa: BLE001
        return {}


def bus_bytes(n: int, size: int) -> float:
    """Per-rank bus bytes of one all_reduce: 2(n-1)/n * S (nccl-tests busbw);
    n = 1 (no peers, a local copy): S, each element delivered once."""
    return float(size) if n == 1 else 2.0 * (n - 1) / n * size


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), line.strip()))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        rows = self.rows
        if self.window:
            inside = [r for r in rows if self.window[0] - 0.05 <= r[0] <= self.window[1] + 0.05]
            rows = inside or rows
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for _t, line in rows:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ reference arm
def reference_allreduce(p: int, size: int, steps: int, warmup: int):
    """The reference's own CPU path (baseline/_ref mcrdl, public API, thread
    world over inproc, default ring policy; tuner.py:151-214 method)."""
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import numpy as np
    from mcrdl import BackendConfig, Buffer, CommOpKind, CommRequest, DType, ReduceOp, run_thread_world

    n = size // 4

    def entry(rt, rank):
        rt.init([BackendConfig("a", transport="inproc")])
        rng = np.random.default_rng(rank)
        a = Buffer(rng.standard_normal(n).astype(np.float32))
        b = Buffer.zeros(DType.f32, n)
        z = Buffer.zeros(DType.f32, 0)
        out = []
        for it in range(warmup + steps):
            rt.post(CommRequest(CommOpKind.all_reduce, input=z, output=z, op=ReduceOp.sum,
                                backend="a"))
            t0 = time.perf_counter()
            rt.post(CommRequest(CommOpKind.all_reduce, input=a, output=b, op=ReduceOp.sum,
                                backend="a"))
            dt = time.perf_counter() - t0
            if it >= warmup:
                out.append(dt)
        d = Buffer(np.array(out, dtype=np.float64))
        if p > 1:
            rt.all_reduce("a", d, ReduceOp.max)
        rt.finalize()
        return d.array.tolist()

    res = run_thread_world(p, entry, timeout=600.0, join_timeout=3600.0)
    per_step = res[0]
    t = statistics.median(per_step)
    return t, per_step


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count(), model


def reference_line_cpu(n: int, size: int, t: float, steps: int, note: str = "") -> dict:
    cores, model = cpu_info()
    return {"value": n * bus_bytes(n, size) / t / 1e9, "unit": "GB/s", "cores": n,
            "nproc": cores, "cpu_model": model, "kind": "reference",
            "sample": f"{steps} steps of all_reduce sum f32 {size // MIB} MiB per rank x {n} "
                      f"thread-ranks of the reference (baseline/_ref mcrdl, inproc transport, "
                      f"default ring policy, tuner.py:151-214 timing; one Python process, GIL)"
                      f"{note}"}


def run_reference(args) -> int:
    rank = int(os.environ.get("RANK", "0"))
    n = args.gpus
    if rank != 0:
        return 0
    # Same config as the native arm: S per rank, N ranks, --steps/--warmup.
    size = args.size_mib * MIB
    steps, warmup = args.steps, args.warmup
    t_probe, _ = reference_allreduce(n, size, 1, 0)
    budget = float(os.environ.get("MCRDL_REF_BUDGET_S", "240"))
    note = ""
    if t_probe * (steps + warmup) > budget:  # keep the run within minutes
        steps = max(3, int(budget / t_probe) - warmup)
        note = f"; steps capped to {steps} (probe {t_probe:.2f} s/step, budget {budget:.0f} s)"
    t, _ = reference_allreduce(n, size, steps, warmup)
    value = n * bus_bytes(n, size) / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": n, "steps": steps, "warmup": warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (standard normal)",
        "same_config": True, "same_steps": steps == args.steps,
        "config": {"workload": f"all_reduce sum f32, {size // MIB} MiB per rank, world {n} "
                               f"(BASELINE configs[1] point >= 64 MB)",
                   "op": "all_reduce", "world": n, "bytes_per_rank": size,
                   "algorithm": "reference default (ring)", "l2": "host path",
                   "value_definition": "N * bus_bytes(N, S) / t (as the native arm)"},
        "cpu_baseline": reference_line_cpu(n, size, t, steps, note),
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- native arm
def run_native(args) -> int:
    import torch
    import torch.distributed as dist

    from paper_2303_08374_b200 import BackendConfig, Buffer, CommOpKind, CommRequest, ReduceOp, Runtime
    from paper_2303_08374_b200.nvl import _lib

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo")  # host control plane (barrier, max over ranks)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    clocks.start()
    rt = Runtime(rank, world)
    cfgs = [BackendConfig("nvl", workspace_bytes=2 << 30)]
    if world > 1 and not args.no_secondary:
        # cfg5's fused small-tensor all_reduces (FusionConfig B = 1 MiB, T = 5 ms)
        from paper_2303_08374_b200 import FusionConfig

        cfgs.append(BackendConfig("nvl_fused", workspace_bytes=256 << 20,
                                  fusion=FusionConfig(max_bytes=1 << 20, max_wait=0.005)))
    rt.init(cfgs)
    size = args.size_mib * MIB
    n = size // 4
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    a = torch.randn(n, device=dev, generator=g)
    b = torch.empty_like(a)
    A, B = Buffer(a), Buffer(b)

    def step():
        rt.post(CommRequest(CommOpKind.all_reduce, input=A, output=B, op=ReduceOp.sum,
                            backend="nvl"))

    # configs[1]: "algorithm chosen by tuning table" -> build it in situ for the
    # headline cell (every candidate algorithm timed on this box and world size,
    # cross-rank max), then the timed steps route through it.
    tuning = autotune(rt, size, world)
    for _ in range(args.warmup):
        step()
    barrier()
    stream = torch.cuda.current_stream()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    t_wall0 = time.monotonic()
    s.record(stream)
    for _ in range(args.steps):
        step()
    e.record(stream)
    e.synchronize()
    t_wall1 = time.monotonic()
    launches = _lib.launch_count() - l0
    barrier()
    clocks.mark(t_wall0, t_wall1)
    ms = s.elapsed_time(e) / args.steps
    ms = max_over_ranks(ms)
    t = ms * 1e-3
    rt.synchronize()  # surfaces any latched device error
    value = world * bus_bytes(world, size) / t / 1e9
    # roofline bytes: NVLink bus bytes (N > 1); HBM read + write of the local
    # copy (N = 1)
    roof_bytes = 2.0 * size if world == 1 else bus_bytes(world, size)
    per_launch_bytes = roof_bytes * args.steps / max(launches, 1)
    t_launch = t * args.steps / max(launches, 1)
    peaks = measured_peaks()
    if world == 1:
        peak, peak_src, bound = float(peaks.get("hbm_gbs", 6650.0)), \
            "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6.65 TB/s", "hbm"
    else:
        peak, peak_src, bound = NVLINK_PEAK, "NVLink 5 nominal per direction (north_star)", "nvlink"
    achieved = per_launch_bytes / t_launch / 1e9
    clk = clocks.stop()

    # ---- e2e: host (pinned) buffers through the same public API
    ha = torch.randn(n, generator=torch.Generator().manual_seed(99 + rank)).pin_memory()
    hb = torch.empty(n, dtype=torch.float32).pin_memory()
    HA, HB = Buffer(ha), Buffer(hb)

    def e2e_step():
        rt.post(CommRequest(CommOpKind.all_reduce, input=HA, output=HB, op=ReduceOp.sum,
                            backend="nvl"))

    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()  # blocking: returns after the D2H copy landed in hb
    t_e2e = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e_value = world * bus_bytes(world, size) / t_e2e / 1e9

    # ---- NCCL comparator + secondary workloads (N > 1)
    extra = {}
    if world > 1 and not args.no_secondary:
        extra = secondary(rt, world, rank, dev, size, barrier, max_over_ranks)
    # ---- CPU baseline: the reference at the same S and N (thread-ranks),
    # rank 0, a bounded number of steps
    cpu = None
    if rank == 0:
        try:
            cs = 3 if world > 2 else 5
            tc, _ = reference_allreduce(world, size, cs, 1)
            cpu = reference_line_cpu(world, size, tc, cs)
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (torch.randn, seeded per rank)",
            "config": {
                "workload": f"all_reduce sum f32 out-of-place, {args.size_mib} MiB per rank, "
                            f"world {world} (BASELINE configs[1] point >= 64 MB)",
                "op": "all_reduce", "world": world, "bytes_per_rank": size,
                "algorithm": tuning.get("winner"),
                "tuning_table_cell": tuning,
                "value_definition": "N * busbw, busbw = bus_bytes(N, S) / t with bus_bytes = "
                                    "2(N-1)/N*S (N >= 2), S (N = 1, local copy)",
                "busbw_gbs_per_rank": bus_bytes(world, size) / t / 1e9,
                "frac_of_900": (bus_bytes(world, size) / t / 1e9 / NVLINK_PEAK) if world > 1 else None,
                "local_copy_floor_gbs": (2.0 * size / t / 1e9) if world == 1 else None,
                "l2": f"inputs {args.size_mib} MiB > 126 MB L2 (no flush needed)",
                "parallelism": f"{world} ranks, one process per GPU",
            },
            "roofline": {"bound": bound,
                         "kernel": ({"nvls": "k_ar_nvls", "one_shot": "k_ar_oneshot"}.get(
                             tuning.get("winner"), "k_ar_pipe") if world > 1 else "k_copy"),
                         "achieved": achieved, "peak": peak, "peak_source": peak_src,
                         "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None,
                         "bytes_per_launch": per_launch_bytes},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": size,
                    "d2h_bytes_per_step": size, "ms_per_step": t_e2e * 1e3,
                    "path": "Runtime.post on numpy-style host Buffers (pinned torch CPU tensors)"},
            "gpu_launches": launches,
            "clocks": clk,
        }
        line.update(extra)
        traffic = _ncu_traffic(world)
        if traffic is not None:
            line["roofline"]["traffic"] = traffic.get("dram")
            line["roofline"]["traffic_over_algorithmic"] = (
                traffic["dram"] / per_launch_bytes if traffic.get("dram") else None)
            if traffic.get("nvltx") is not None:
                line["roofline"]["nvlink_tx_bytes"] = traffic["nvltx"]
            line["roofline"]["traffic_source"] = traffic.get("source")
        print(json.dumps(line), flush=True)
    rt.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def autotune(rt, size: int, world: int) -> dict:
    """Tuning-table cell for (all_reduce, world, size) built with the repo's
    tuner (CUDA-event device time, cross-rank max) and installed on the
    runtime; returns {algorithm: median_us} and the winner."""
    from paper_2303_08374_b200.core import CommOpKind, DType
    from paper_2303_08374_b200.tuner import BenchConfig, bench, build_table

    if world == 1:
        return {"winner": "local copy (p = 1)"}
    cfg = BenchConfig(ops=[CommOpKind.all_reduce], sizes=[size], dtype=DType.f32,
                      warmup_iters=2, measure_iters=3)
    samples, skipped = bench(rt, cfg, "nvl")
    rt.tuning_table = build_table(samples, skipped=skipped, system="bench.py in-situ")
    entry = rt.tuning_table.lookup_entry(CommOpKind.all_reduce, world, size)
    import statistics

    return {"candidates_us": {s.algorithm: round(statistics.median(s.durations) * 1e6, 1)
                              for s in samples},
            "winner": entry.algorithm if entry else None}


def _ncu_traffic(world: int):
    """DRAM read+write bytes (and NVLink tx bytes at N > 1) per launch of the
    dominant kernel from the committed ncu captures (profiles/ncu_traffic.json:
    `ncu --set full` of k_copy at N = 1, tools/ncu_multi.py at N = 2, 4)."""
    try:
        doc = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
    except Exception:  # noqa: BLE001
        return None
    if doc.get(str(world)) is None:
        return None
    return {"dram": doc[str(world)], "nvltx": doc.get(f"{world}_nvltx_bytes"),
            "source": doc.get(f"{world}_source", doc.get("_source"))}


def secondary(rt, world, rank, dev, size, barrier, max_over_ranks):
    """NCCL comparator at the headline size, DLRM all_to_allv (cfg4) and
    DS-MoE all_to_all_single (cfg3 shape) on the same ranks."""
    import torch
    import torch.distributed as dist

    from paper_2303_08374_b200 import Buffer

    out = {}
    iters = 10

    def dev_time(fn, reps=iters):
        for _ in range(3):
            fn()
        barrier()
        st = torch.cuda.current_stream()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(reps):
            fn()
        e.record(st)
        e.synchronize()
        return max_over_ranks(s.elapsed_time(e) / reps * 1e-3)

    # NCCL comparator (torch.distributed, same size and dtype)
    try:
        pg = dist.new_group(backend="nccl")
        x = torch.randn(size // 4, device=dev)
        t = dev_time(lambda: dist.all_reduce(x, group=pg))
        out["nccl_all_reduce"] = {"busbw_gbs": bus_bytes(world, size) / t / 1e9,
                                  "ms": t * 1e3, "bytes_per_rank": size}
    except Exception as exc:  # noqa: BLE001
        pg = None
        out["nccl_all_reduce"] = {"error": repr(exc)}

    # Same all_reduce on torch tensors allocated in the symmetric MemPool
    # (Runtime.symmetric_pool, csrc/pool.cu): the zero-copy kernels (NVLS
    # multicast at p >= 3, peer loads at p = 2) — the analogue of NCCL
    # user-buffer registration, reported beside the headline (which uses
    # tensors from torch's default allocator).
    if world > 1:
        try:
            pool = rt.symmetric_pool("nvl", 2 * size + (64 << 20))
            with torch.cuda.use_mem_pool(pool):
                a_s = torch.empty(size // 4, device=dev)
                o_s = torch.empty(size // 4, device=dev)
            a_s.normal_()
            from paper_2303_08374_b200 import CommOpKind, CommRequest, ReduceOp

            req = lambda: rt.post(CommRequest(CommOpKind.all_reduce, input=Buffer(a_s),  # noqa: E731
                                              output=Buffer(o_s), op=ReduceOp.sum, backend="nvl"))
            t = dev_time(req)
            out["all_reduce_symmetric"] = {
                "busbw_gbs": bus_bytes(world, size) / t / 1e9, "ms": t * 1e3,
                "frac_of_900": bus_bytes(world, size) / t / 1e9 / 900.0, "bytes_per_rank": size,
                "path": rt._instance("nvl").last_algorithm(CommOpKind.all_reduce),
                "tensors": "torch.empty under torch.cuda.use_mem_pool(Runtime.symmetric_pool)"}
        except Exception as exc:  # noqa: BLE001
            out["all_reduce_symmetric"] = {"error": repr(exc)}

    # DLRM cfg4: 26 tables, dim 128, f32, global batch 65536, uniform local batch
    tables = [len(x) for x in _array_split(26, world)]
    B = 65536
    b = B // world
    sc = [b * tables[rank] * 128 for _ in range(world)]
    rc = [b * tables[j] * 128 for j in range(world)]
    sd = [sum(sc[:j]) for j in range(world)]
    rdp = [sum(rc[:j]) for j in range(world)]
    inp = torch.randn(sum(sc), device=dev)
    outp = torch.empty(sum(rc), device=dev)
    I, O = Buffer(inp), Buffer(outp)
    t = dev_time(lambda: rt.all_to_allv("nvl", O, I, sc, rc, sd, rdp))
    egress = max(sum(sc) - sc[rank], sum(rc) - rc[rank]) * 4
    egress = max_over_ranks(egress)
    res = {"busbw_gbs": egress / t / 1e9, "ms": t * 1e3, "max_pair_egress_bytes": egress,
           "workload": "cfg4 DLRM 26 tables x dim 128 f32, batch 65536 (uniform)"}
    if pg is not None:
        try:
            t2 = dev_time(lambda: dist.all_to_all_single(outp, inp, rc, sc, group=pg))
            res["nccl_busbw_gbs"] = egress / t2 / 1e9
        except Exception as exc:  # noqa: BLE001
            res["nccl_error"] = repr(exc)
    out["all_to_allv_dlrm"] = res

    # DLRM cfg4, skewed variant: per-rank batch b_j from Zipf(1.1) weights
    # (w_j = (j+1)^-1.1, normalized to 65536, remainder to the last rank)
    wz = [(j + 1) ** -1.1 for j in range(world)]
    bz = [int(B * w / sum(wz)) for w in wz]
    bz[-1] += B - sum(bz)
    ssc = [bz[j] * tables[rank] * 128 for j in range(world)]
    src = [bz[rank] * tables[j] * 128 for j in range(world)]
    ssd = [sum(ssc[:j]) for j in range(world)]
    srd = [sum(src[:j]) for j in range(world)]
    sinp = torch.randn(sum(ssc), device=dev)
    sout = torch.empty(sum(src), device=dev)
    SI, SO = Buffer(sinp), Buffer(sout)
    t = dev_time(lambda: rt.all_to_allv("nvl", SO, SI, ssc, src, ssd, srd))
    egress = max_over_ranks(max(sum(ssc) - ssc[rank], sum(src) - src[rank]) * 4)
    res = {"busbw_gbs": egress / t / 1e9, "ms": t * 1e3, "max_pair_egress_bytes": egress,
           "workload": f"cfg4 DLRM skewed: local batches {bz} (Zipf 1.1 weights)"}
    if pg is not None:
        try:
            t2 = dev_time(lambda: dist.all_to_all_single(sout, sinp, src, ssc, group=pg))
            res["nccl_busbw_gbs"] = egress / t2 / 1e9
        except Exception as exc:  # noqa: BLE001
            res["nccl_error"] = repr(exc)
    out["all_to_allv_dlrm_skew"] = res

    # cfg5 mixed-collective step, REPLAYED from its LogRecord-
    # schema JSONL trace (paper_2303_08374_b200/trace.py; the p = 8 trace is
    # committed as profiles/cfg5_trace_p8.jsonl): a2av forward (cfg4), the 14
    # DLRM MLP gradient all_reduces posted async on the fusion backend
    # (B = 1 MiB, T = 5 ms), all_gatherv i64 (1000 + 137 r), gatherv f32 ->
    # root 0 (16 (r+1)), a2av backward (transposed counts). Device time per
    # step, max over ranks, host posting included (the step is what a trainer
    # sees).
    try:
        import tempfile

        from paper_2303_08374_b200 import trace as tr

        with tempfile.TemporaryDirectory() as d:
            path = f"{d}/cfg5.jsonl"
            tr.write_jsonl(tr.cfg5_trace(world), path)
            recs = tr.load_jsonl(path)
        rp = tr.Replay(rt, recs, rank, dev)
        rp.fill(5)
        log = rt.comm_log
        reps = 20
        rt.synchronize()
        n0 = len(log.records())
        t = dev_time(rp.step, reps=reps)
        rt.synchronize()
        recs_log = log.records()[n0:]
        fused = [r_ for r_ in recs_log if r_.backend == "nvl_fused" and r_.fused]
        steps_logged = reps + 3  # dev_time's warm-up steps included
        out["mixed_step_cfg5"] = {
            "step_ms": t * 1e3, "ops_posted_per_step": len(rp.ops),
            "fused_flushes_per_step": len(fused) / steps_logged,
            "fused_members_per_step": sum(r_.members for r_ in fused) / steps_logged,
            "log_records_per_step": len(recs_log) / steps_logged,
            "workload": "cfg5 trace replay (LogRecord JSONL): a2av fwd (cfg4) + 14 MLP-grad "
                        "all_reduce (fusion B=1MiB, T=5ms) + all_gatherv i64 + gatherv f32 + a2av bwd"}
    except Exception as exc:  # noqa: BLE001
        out["mixed_step_cfg5"] = {"error": repr(exc)}
    # DS-MoE cfg3 shape: 4096 tokens x 4096 hidden bf16 per rank, all_to_all_single
    x = torch.randn(4096 * 4096, device=dev).to(torch.bfloat16)
    y = torch.empty_like(x)
    X, Y = Buffer(x), Buffer(y)
    t = dev_time(lambda: rt.all_to_all_single("nvl", Y, X))
    nb = x.numel() * 2 * (world - 1) / world
    res = {"busbw_gbs": nb / t / 1e9, "ms": t * 1e3,
           "workload": "cfg3 DS-MoE a2a 4096x4096 bf16 per rank"}
    if pg is not None:
        try:
            t2 = dev_time(lambda: dist.all_to_all_single(y, x, group=pg))
            res["nccl_busbw_gbs"] = nb / t2 / 1e9
        except Exception as exc:  # noqa: BLE001
            res["nccl_error"] = repr(exc)
    out["all_to_all_moe"] = res
    return out


def _array_split(n, parts):
    q, r = divmod(n, parts)
    out, o = [], 0
    for i in range(parts):
        k = q + (1 if i < r else 0)
        out.append(list(range(o, o + k)))
        o += k
    return out


def main() -> int:
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not under torchrun: relaunch one process per GPU
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
               "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
               "--master-port", os.environ.get("MASTER_PORT", "29533"), __file__] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())

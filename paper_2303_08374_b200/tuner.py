"""Tuning suite: time every (op, message size, algorithm) cell of the NVLink
backend with CUDA events, pick the fastest algorithm per cell, and emit a
tuning table whose entries carry the algorithm.

Reference: tuner.py:1-277 (BenchConfig, bench with barrier + per-iteration
rotation + cross-rank max, winner_grid, build_table, emit). Differences:
the candidates are algorithms of one backend instead of backends, time is
device time on the lane stream (CUDA events), and the cross-rank max runs
through the backend's own all_reduce(max).

CLI (one process per GPU, e.g. under torchrun):
    python -m paper_2303_08374_b200.tuner --ops all_reduce,all_to_allv \
        --sizes 8:1G --out table.json [--nccl]
"""

from __future__ import annotations

import argparse
import json
import statistics as stats
import sys
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from .collectives import ALGORITHMS, AlgorithmPolicy, bus_factor
from .core import Buffer, CommOpKind, DType, ReduceOp
from .dispatch import NVL_SIZE_BUCKETS, TableEntry, TuningTable, save_table
from .errors import EmptySamples, ValidationError

STATISTICS = ("median", "mean", "min")
DEFAULT_OPS = (CommOpKind.all_reduce, CommOpKind.all_to_allv, CommOpKind.all_gatherv,
               CommOpKind.bcast)


@dataclass
class BenchConfig:
    ops: Sequence[CommOpKind] = DEFAULT_OPS
    sizes: Sequence[int] = NVL_SIZE_BUCKETS
    dtype: DType = DType.f32
    warmup_iters: int = 5
    measure_iters: int = 20
    statistic: str = "median"
    algorithms: Optional[Dict[CommOpKind, Sequence[str]]] = None
    symmetric: bool = False  # all_reduce buffers from Runtime.symmetric_empty (zero-copy path)

    def __post_init__(self):
        self.ops = [CommOpKind(o) if isinstance(o, str) else o for o in self.ops]
        if self.measure_iters < 3:
            raise ValidationError("measure_iters", "must be >= 3")
        if list(self.sizes) != sorted(self.sizes):
            raise ValidationError("sizes", "must be ascending")
        if self.statistic not in STATISTICS:
            raise ValidationError("statistic", f"one of {STATISTICS}")

    def candidates(self, op: CommOpKind, nvls: bool = False) -> List[str]:
        if self.algorithms and op in self.algorithms:
            return list(self.algorithms[op])
        return [a for a in ALGORITHMS[op] if a != "auto" and (nvls or a != "nvls")]


@dataclass
class BenchSample:
    op: CommOpKind
    backend: str
    world_size: int
    bytes: int
    durations: List[float]  # seconds, cross-rank max per iteration
    algorithm: Optional[str] = None

    def busbw_gbs(self, statistic: str = "median") -> float:
        t = statistic_value(self.durations, statistic)
        return bus_factor(self.op, self.world_size) * self.bytes / t / 1e9 if t > 0 else 0.0


@dataclass
class SkippedCombination:
    op: CommOpKind
    backend: str
    world_size: int
    bytes: int
    reason: str


def statistic_value(durations: Sequence[float], statistic: str) -> float:
    if statistic == "median":
        return stats.median(durations)
    if statistic == "mean":
        return stats.fmean(durations)
    if statistic == "min":
        return min(durations)
    raise ValidationError("statistic", f"one of {STATISTICS}")


_SYMM_CACHE: dict = {}  # keyed by the owning communicator: freed with it


def _comm_key(rt, backend: str):
    comm = rt._instance(backend).comm
    return (id(comm), int(comm.handle.value or 0))


def make_op(rt, backend: str, kind: CommOpKind, nbytes: int, dtype: DType,
            symmetric: bool = False):
    """Closure posting one op whose canonical message size is ~nbytes.
    symmetric=True draws the buffers from the backend's symmetric memory
    (one cached pair of blocks per size; collective on first use)."""
    import torch

    p, r = rt.world_size, rt.rank
    dev = rt._instance(backend).device
    es = dtype.size_bytes
    n = max(nbytes // es, 1)
    td = dtype.torch_dtype

    def t(count):
        return torch.ones(count, dtype=td, device=dev)

    if symmetric and kind is CommOpKind.all_reduce:
        key = (_comm_key(rt, backend), n, dtype)
        if key not in _SYMM_CACHE:
            pair = [rt.symmetric_empty(backend, n, dtype) for _ in range(2)]
            for x in pair:
                x.fill_(1)
            _SYMM_CACHE[key] = pair
        a_t, o_t = _SYMM_CACHE[key]
        a, o = Buffer(a_t), Buffer(o_t)
        from .core import CommRequest

        return lambda: rt.post(CommRequest(kind, input=a, output=o, op=ReduceOp.sum,
                                           backend=backend))

    if kind is CommOpKind.all_reduce:
        a, o = Buffer(t(n)), Buffer(t(n))
        from .core import CommRequest

        return lambda: rt.post(CommRequest(kind, input=a, output=o, op=ReduceOp.sum,
                                           backend=backend))
    if kind is CommOpKind.bcast:
        b = Buffer(t(n))
        return lambda: rt.bcast(backend, b, 0)
    def out_t(count):  # symmetric output (zero-copy exchange) when asked
        if not symmetric:
            return t(count)
        key = (_comm_key(rt, backend), "out", count, dtype)
        if key not in _SYMM_CACHE:
            _SYMM_CACHE[key] = rt.symmetric_empty(backend, count, dtype)
        return _SYMM_CACHE[key]

    if kind is CommOpKind.all_to_all_single:
        m = max(n // p, 1)
        i, o = Buffer(t(m * p)), Buffer(out_t(m * p))
        return lambda: rt.all_to_all_single(backend, o, i)
    if kind in (CommOpKind.all_gatherv, CommOpKind.all_gather):
        m = max(n // p, 1)
        i, o = Buffer(t(m)), Buffer(out_t(m * p))
        counts, displs = [m] * p, [k * m for k in range(p)]
        return lambda: rt.all_gatherv(backend, o, i, counts, displs)
    if kind in (CommOpKind.all_to_allv, CommOpKind.all_to_all_single):
        m = max(n // p, 1)
        i, o = Buffer(t(m * p)), Buffer(t(m * p))
        c, d = [m] * p, [k * m for k in range(p)]
        return lambda: rt.all_to_allv(backend, o, i, c, c, d, d)
    if kind in (CommOpKind.gatherv, CommOpKind.gather):
        m = max(n // p, 1)
        i = Buffer(t(m))
        o = Buffer(t(m * p)) if r == 0 else None
        counts, displs = [m] * p, [k * m for k in range(p)]
        return lambda: rt.gatherv(backend, o, i, 0, counts, displs)
    if kind in (CommOpKind.send, CommOpKind.recv):
        # the reference's rank 0 <-> 1 ping-pong, other ranks sit out
        # (tuner.py:128-145); the receiver posts first so messages above the
        # mailbox stream (rendezvous) without deadlock
        if p == 1:
            raise ValidationError("op", "send/recv ping-pong needs two ranks")
        a, b = Buffer(t(n)), Buffer(t(n))

        def pingpong():
            if r == 0:
                rt.send(backend, a, 1)
                rt.recv(backend, b, 1)
            elif r == 1:
                rt.recv(backend, b, 0)
                rt.send(backend, a, 0)
        return pingpong
    raise ValidationError("op", f"{kind.name} is not benchmarkable")


SLEEP_CYCLES = 4_000_000  # ~2 ms at 1.9 GHz: the stream stays blocked while the host enqueues


def batch_for(nbytes: int) -> int:
    """Back-to-back ops per timed sample (nccl-tests style) so small-message
    numbers are device time, not host enqueue time."""
    return max(1, min(20, (64 << 20) // max(nbytes, 1)))


def time_op(rt, backend: str, fn, warmup: int, iters: int, *, batch: int = 1,
            barrier: bool = True, cross_rank: bool = True) -> List[float]:
    """Per-op device time (s) on the caller's stream, cross-rank max per
    sample. With batch > 1 the stream is held by a sleep kernel while the host
    enqueues `batch` ops back to back, so host launch overhead is hidden."""
    import torch

    inst = rt._instance(backend)
    stream = torch.cuda.current_stream(inst.device)
    for _ in range(warmup):
        fn()
    out = []
    for _ in range(iters):
        if barrier:
            rt.barrier(backend)
        if batch > 1:
            torch.cuda._sleep(SLEEP_CYCLES * batch // 8)  # >= 250 us of host time per op
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(batch):
            fn()
        e.record(stream)
        e.synchronize()
        out.append(s.elapsed_time(e) * 1e-3 / batch)
    if cross_rank and rt.world_size > 1:
        v = torch.tensor(out, dtype=torch.float64, device=inst.device)
        rt.all_reduce(backend, Buffer(v), ReduceOp.max)
        torch.cuda.synchronize(inst.device)
        out = v.cpu().tolist()
    rt.synchronize([backend])
    return out


def bench(rt, config: BenchConfig, backend: Optional[str] = None
          ) -> Tuple[List[BenchSample], List[SkippedCombination]]:
    """Run the sweep on every rank (identical config on all ranks)."""
    backend = backend or rt.get_backends()[0]
    inst = rt._instance(backend)
    saved = inst.policy
    samples: List[BenchSample] = []
    skipped: List[SkippedCombination] = []
    p = rt.world_size
    for _ in range(4):
        rt.barrier(backend)
    try:
        for op in config.ops:
            for nbytes in config.sizes:
                nvls = bool(inst.comm.caps.nvls_supported) and config.dtype in (DType.f32,
                                                                                 DType.bf16)
                for algo in config.candidates(op, nvls):
                    if algo == "one_shot" and nbytes > inst.comm.caps.max_oneshot_bytes:
                        continue  # the library would run two_shot: not a distinct cell
                    inst.policy = AlgorithmPolicy({op: algo})
                    try:
                        fn = make_op(rt, backend, op, nbytes, config.dtype, config.symmetric)
                        d = time_op(rt, backend, fn, config.warmup_iters, config.measure_iters,
                                    batch=batch_for(nbytes))
                    except ValidationError as exc:
                        skipped.append(SkippedCombination(op, backend, p, nbytes, str(exc)))
                        continue
                    samples.append(BenchSample(op, backend, p, nbytes, d, algo))
    finally:
        inst.policy = saved
    return samples, skipped


def winner_grid(samples: Sequence[BenchSample], statistic: str = "median",
                skipped: Sequence[SkippedCombination] = ()) -> Dict[tuple, Tuple[str, str]]:
    """(op, world, size) -> (backend, algorithm) with the minimum statistic;
    ties break lexicographically (tuner.py:221-254)."""
    if not samples:
        raise EmptySamples("no benchmark samples")
    cells: Dict[tuple, List[BenchSample]] = {}
    for s in samples:
        cells.setdefault((s.op, s.world_size, s.bytes), []).append(s)
    skip = {(s.op, s.world_size, s.bytes) for s in skipped}
    ops = sorted({s.op for s in samples} | {s.op for s in skipped}, key=lambda k: k.value)
    worlds = sorted({s.world_size for s in samples} | {s.world_size for s in skipped})
    sizes = sorted({s.bytes for s in samples} | {s.bytes for s in skipped})
    grid = {}
    for op in ops:
        for w in worlds:
            for size in sizes:
                key = (op, w, size)
                if key not in cells:
                    if key in skip:
                        continue
                    raise EmptySamples(f"missing combination {op.value}/{w}/{size}B")
                best = min(cells[key], key=lambda s: (statistic_value(s.durations, statistic),
                                                      s.backend, s.algorithm or ""))
                grid[key] = (best.backend, best.algorithm)
    return grid


def build_table(samples: Sequence[BenchSample], statistic: str = "median", *,
                skipped: Sequence[SkippedCombination] = (), system: str = "b200-nvl",
                base: Optional[TuningTable] = None) -> TuningTable:
    grid = winner_grid(samples, statistic, skipped)
    by_key: Dict[tuple, List[tuple]] = {}
    for (op, w, size), (be, algo) in grid.items():
        by_key.setdefault((op, w), []).append((size, be, algo))
    tables = {k: dict(v) for k, v in base.tables.items()} if base is not None else {}
    for (op, w), cells in by_key.items():
        cells.sort()
        tables.setdefault(op, {})[w] = TuningTable.merge_runs(
            [TableEntry(size, be, algo) for size, be, algo in cells])
    return TuningTable(tables, system=system)


def emit(table: TuningTable, path: str) -> None:
    save_table(table, path)


def parse_size(tok: str) -> int:
    tok = tok.strip().upper()
    mult = 1
    for suf, m in (("K", 1 << 10), ("M", 1 << 20), ("G", 1 << 30)):
        if tok.endswith(suf):
            tok, mult = tok[:-1], m
    return int(float(tok) * mult)


def parse_sizes(spec: str) -> List[int]:
    if ":" in spec:
        lo, hi = (parse_size(x) for x in spec.split(":"))
        out, s = [], 1
        while s < lo:
            s <<= 1
        while s <= hi:
            out.append(s)
            s <<= 1
        return out
    return sorted(parse_size(x) for x in spec.split(","))


def nccl_times(sizes: Sequence[int], op: CommOpKind, dtype: DType, warmup: int, iters: int,
               device: int) -> Dict[int, List[float]]:
    """torch.distributed (NCCL) comparator on the same sizes."""
    import torch
    import torch.distributed as dist

    out = {}
    p = dist.get_world_size()
    stream = torch.cuda.current_stream(device)
    for nbytes in sizes:
        n = max(nbytes // dtype.size_bytes, 1)
        rank = dist.get_rank()
        if op is CommOpKind.all_reduce:
            x = torch.ones(n, dtype=dtype.torch_dtype, device=device)
            fn = lambda: dist.all_reduce(x)  # noqa: E731
        elif op is CommOpKind.bcast:
            x = torch.ones(n, dtype=dtype.torch_dtype, device=device)
            fn = lambda: dist.broadcast(x, 0)  # noqa: E731
        elif op in (CommOpKind.all_gatherv, CommOpKind.all_gather):
            m = max(n // p, 1)
            x = torch.ones(m, dtype=dtype.torch_dtype, device=device)
            y = torch.empty(m * p, dtype=dtype.torch_dtype, device=device)
            fn = lambda: dist.all_gather_into_tensor(y, x)  # noqa: E731
        elif op in (CommOpKind.send, CommOpKind.recv):
            x = torch.ones(n, dtype=dtype.torch_dtype, device=device)
            y = torch.empty_like(x)

            def fn():
                if rank == 0:
                    dist.send(x, 1)
                    dist.recv(y, 1)
                elif rank == 1:
                    dist.recv(y, 0)
                    dist.send(x, 0)
        else:
            m = max(n // p, 1)
            x = torch.ones(m * p, dtype=dtype.torch_dtype, device=device)
            y = torch.empty_like(x)
            fn = lambda: dist.all_to_all_single(y, x)  # noqa: E731
        for _ in range(warmup):
            fn()
        ts = []
        batch = batch_for(nbytes)
        for _ in range(iters):
            dist.barrier()
            if batch > 1:
                torch.cuda._sleep(SLEEP_CYCLES * batch // 8)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            for _ in range(batch):
                fn()
            e.record(stream)
            e.synchronize()
            ts.append(s.elapsed_time(e) * 1e-3 / batch)
        t = torch.tensor(ts, dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[nbytes] = t.cpu().tolist()
    return out


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2303_08374_b200.tuner")
    ap.add_argument("--ops", default="all_reduce,all_to_allv")
    ap.add_argument("--sizes", default="8:1G")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--statistic", choices=STATISTICS, default="median")
    ap.add_argument("--out", default=None, help="write the tuning table here (rank 0)")
    ap.add_argument("--csv", default=None, help="write per-cell busbw CSV here (rank 0)")
    ap.add_argument("--nccl", action="store_true", help="also time torch.distributed NCCL")
    ap.add_argument("--codec", action="store_true",
                    help="backend with CompressionConfig (trunc16 fused in the exchange kernel);"
                         " busbw counts the user (f32) bytes")
    ap.add_argument("--symm", action="store_true",
                    help="all_reduce on symmetric-memory tensors (zero-copy kernels)")
    ap.add_argument("--algorithms", default=None,
                    help="comma list restricting the candidates (e.g. two_shot,nvls)")
    ap.add_argument("--api", action="store_true",
                    help="API latency: one op per sample on an idle GPU (host enqueue included)")
    args = ap.parse_args(argv)
    if args.api:
        global batch_for
        batch_for = lambda nbytes: 1  # noqa: E731
    import torch

    from .runtime import BackendConfig, Runtime

    rt = Runtime()
    torch.cuda.set_device(rt.local_device if rt.local_device is not None else rt.rank)
    from .middleware import CompressionConfig

    rt.init([BackendConfig("nvl", workspace_bytes=2 << 30,
                           compression=CompressionConfig() if args.codec else None)])
    cfg = BenchConfig(ops=args.ops.split(","), sizes=parse_sizes(args.sizes),
                      dtype=DType.from_name(args.dtype), warmup_iters=args.warmup,
                      measure_iters=args.iters, statistic=args.statistic, symmetric=args.symm)
    if args.algorithms:
        wanted = args.algorithms.split(",")
        cfg.algorithms = {op: [a for a in ALGORITHMS[op] if a in wanted] or ["auto"]
                          for op in cfg.ops}
    samples, skipped = bench(rt, cfg)
    nccl = {}
    if args.nccl and rt.world_size > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", rt._instance("nvl").device))
        for op in cfg.ops:
            if op in (CommOpKind.all_reduce, CommOpKind.all_to_allv, CommOpKind.bcast,
                      CommOpKind.all_gatherv, CommOpKind.send):
                nccl[op] = nccl_times(cfg.sizes, op, cfg.dtype, args.warmup, args.iters,
                                      rt._instance("nvl").device)
    if rt.rank == 0:
        rows = ["op,world,bytes,algorithm,median_us,min_us,busbw_gbs,frac_900"]
        for s in samples:
            med = statistic_value(s.durations, "median")
            bw = s.busbw_gbs("median")
            rows.append(f"{s.op.value},{s.world_size},{s.bytes},{s.algorithm},{med*1e6:.2f},"
                        f"{min(s.durations)*1e6:.2f},{bw:.2f},{bw/900:.3f}")
        for op, cells in nccl.items():
            for nb, d in cells.items():
                med = stats.median(d)
                bw = bus_factor(op, rt.world_size) * nb / med / 1e9
                rows.append(f"{op.value},{rt.world_size},{nb},nccl,{med*1e6:.2f},"
                            f"{min(d)*1e6:.2f},{bw:.2f},{bw/900:.3f}")
        text = "\n".join(rows)
        print(text)
        if args.csv:
            with open(args.csv, "w") as fh:
                fh.write(text + "\n")
        if args.out:
            emit(build_table(samples, args.statistic, skipped=skipped), args.out)
    rt.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Ranks of a multi-rank parity run (launched by tests/test_gpu_parity.py
and __graft_entry__.smoke via tests/gpu_launch.py). Runs every scenario
through the public Runtime API on the nvlink backend and checks each rank's
result against the CPU oracle (oracle/seqref.py) on identically seeded
inputs. Writes a JSON report {rank, failures, checked, launches} per rank.

Two layouts:
* one process per GPU (the production layout):
    RANK=r WORLD_SIZE=p LOCAL_RANK=r MCRDL_MASTER_PORT=... \
        python tests/gpu_worker.py <report.json> [scenario,...]
* co-located ranks: p threads of ONE process sharing one GPU, each with its
  own Runtime, communicator and CUDA stream — the reference's own
  thread-world test layout (run_thread_world) on the device. The
  same kernels and flag protocol run; the communicator detects the shared
  device (UUIDs), drops NVLS and splits the SMs so that every rank's grids
  are resident at once:
    MCRDL_MASTER_PORT=... python tests/gpu_worker.py --threads p <report_dir> [scenario,...]
"""

from __future__ import annotations

import contextlib
import json
import os
import sys
import threading
import traceback
import zlib
from collections import OrderedDict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

if "--threads" in sys.argv:  # co-located ranks share one context: no lazy kernel loads
    os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2303_08374_b200 as mc  # noqa: E402
from paper_2303_08374_b200 import (AlgorithmPolicy, BackendConfig, Buffer, CommOpKind,  # noqa: E402
                                   CommRequest, CompressionConfig, DType, FusionConfig, ReduceOp,
                                   Runtime)
from paper_2303_08374_b200.errors import OrderMismatch  # noqa: E402
from paper_2303_08374_b200.nvl import _lib  # noqa: E402
from oracle import seqref  # noqa: E402

NP = {DType.f32: np.float32, DType.f64: np.float64, DType.i32: np.int32, DType.i64: np.int64,
      DType.u8: np.uint8, DType.bf16: np.uint16}


def seed_of(*parts) -> int:
    return zlib.crc32("|".join(str(p) for p in parts).encode())


class _Memo:
    """Co-located ranks generate the same seeded inputs: share them (bounded
    LRU of read-only arrays, so no rank can mutate another rank's view)."""

    def __init__(self, max_bytes: int = 6 << 30):
        self.max_bytes = max_bytes
        self.items: "OrderedDict" = OrderedDict()
        self.bytes = 0
        self.lock = threading.Lock()

    def get(self, key, make):
        with self.lock:
            if key in self.items:
                self.items.move_to_end(key)
                return self.items[key]
        arr = make()
        arr.flags.writeable = False
        with self.lock:
            if key not in self.items:
                self.items[key] = arr
                self.bytes += arr.nbytes
                while self.bytes > self.max_bytes and len(self.items) > 1:
                    _, old = self.items.popitem(last=False)
                    self.bytes -= old.nbytes
            return self.items[key]


_MEMO = None  # set in thread mode


def values(dtype: DType, n: int, *seed) -> np.ndarray:
    if _MEMO is not None:
        return _MEMO.get(("v", dtype, n, seed), lambda: _values(dtype, n, *seed))
    return _values(dtype, n, *seed)


def _values(dtype: DType, n: int, *seed) -> np.ndarray:
    """Seeded inputs (tests/cases.py:32-37): floats normal, ints [-1000,1000),
    u8 [0,256); bf16 as RNE-rounded normals (uint16 bits)."""
    rng = np.random.default_rng(seed_of(*seed))
    if dtype is DType.bf16:
        return seqref.f32_to_bf16_bits(rng.standard_normal(n).astype(np.float32))
    if dtype.is_float:
        return rng.standard_normal(n).astype(NP[dtype])
    if dtype is DType.u8:
        return rng.integers(0, 256, size=n).astype(np.uint8)
    return rng.integers(-1000, 1000, size=n).astype(NP[dtype])


def small_prod_values(dtype, n, *seed):
    rng = np.random.default_rng(seed_of(*seed))
    if dtype is DType.bf16:
        return seqref.f32_to_bf16_bits(rng.uniform(0.5, 1.5, n).astype(np.float32))
    if dtype.is_float:
        return rng.uniform(0.5, 1.5, n).astype(NP[dtype])
    return rng.integers(1, 4, size=n).astype(NP[dtype])


def to_dev(arr: np.ndarray, dtype: DType, dev) -> torch.Tensor:
    if not arr.flags.writeable:
        arr = arr.copy()
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if dtype is DType.bf16:
        t = t.view(torch.bfloat16)
    return t.to(dev)


def from_dev(t: torch.Tensor, dtype: DType) -> np.ndarray:
    t = t.detach().cpu()
    if dtype is DType.bf16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def _raw_stream(device: int):
    """A non-blocking stream created directly with the driver (not from
    torch's round-robin pool, which hands one stream to several callers)."""
    from cuda.bindings import driver as drv

    err, s = drv.cuStreamCreate(drv.CUstream_flags.CU_STREAM_NON_BLOCKING)
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"cuStreamCreate: {err}")
    return torch.cuda.ExternalStream(int(s), device=device)


class Shared:
    """State of a co-located (thread) world."""

    def __init__(self, world: int, timeout: float = 600.0):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.lock = threading.Lock()
        self.timeout = timeout
        self._rv: dict = {}
        self._rv_lock = threading.Lock()
        self.rv_timeout = 60.0
        self.broken = False

    def rendezvous(self, key) -> None:
        """Runtime.launch_hook: every rank reaches the launch of op `key`
        before any rank launches it (so a device-synchronizing host call in
        one rank only ever waits on kernels whose peers are launched)."""
        with self._rv_lock:
            ent = self._rv.get(key)
            if ent is None:
                ent = self._rv[key] = [0, threading.Event()]
            ent[0] += 1
            if ent[0] == self.world:
                ent[1].set()
                del self._rv[key]
        if self.broken:
            return
        if not ent[1].wait(self.rv_timeout):
            # a rank skipped this launch (it failed earlier): stop lock-stepping
            # so the remaining ops fail fast instead of each waiting here
            self.broken = True
            raise TimeoutError(f"co-located rendezvous {key} timed out")


class Ctx:
    def __init__(self, rt: Runtime, backend: str, shared: "Shared" = None):
        self.rt = rt
        self.b = backend
        self.p = rt.world_size
        self.r = rt.rank
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.failures = []
        self.checked = 0
        self.shared = shared

    def sync(self):
        """Host-wait for this rank's work. Co-located ranks wait on their own
        stream only: a device-wide sync would also wait for a peer rank's
        kernel that spins on an op this rank has not launched yet."""
        if self.shared is None:
            torch.cuda.synchronize()
        else:
            torch.cuda.current_stream().synchronize()

    @contextlib.contextmanager
    def exclusive(self):
        """A section that may synchronize the whole device (CUDA graph
        capture): co-located ranks first drain and meet, then enter one at a
        time, and meet again before anyone launches collectives."""
        if self.shared is None:
            torch.cuda.synchronize()
            yield
            return
        sh = self.shared
        torch.cuda.current_stream().synchronize()
        sh.barrier.wait(sh.timeout)
        with sh.lock:
            yield
        sh.barrier.wait(sh.timeout)

    def upload(self, g):
        """Co-located ranks: upload an instantiated graph while the device is
        idle (inside exclusive()). A first replay would otherwise upload it
        then, and the upload can wait for the context to idle while a peer
        rank's replayed kernel spins on this rank's."""
        if self.shared is None:
            return
        from cuda.bindings import driver as drv

        st = torch.cuda.current_stream()
        err, = drv.cuGraphUpload(drv.CUgraphExec(init_value=g.raw_cuda_graph_exec()),
                                 drv.CUstream(init_value=st.cuda_stream))
        if err != drv.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"cuGraphUpload: {err}")
        st.synchronize()

    def lockstep(self, key):
        """Co-located ranks: meet before launching work outside the Runtime
        (CUDA graph replays)."""
        if self.shared is not None:
            self.shared.rendezvous(("lockstep",) + tuple(key))

    def graph(self, g):
        """torch.cuda.graph capture; thread-local capture mode for co-located
        ranks (peer threads stay idle in exclusive())."""
        if self.shared is None:
            return torch.cuda.graph(g)
        return torch.cuda.graph(g, capture_error_mode="thread_local")

    def check(self, name, got, want, float_reduction=False, rtol=1e-5):
        self.checked += 1
        try:
            seqref.assert_matches(got, want, float_reduction=float_reduction, rtol=rtol, where=name)
        except AssertionError as exc:
            msg = str(exc)
            self.failures.append(f"{name}: {msg[:600]}")


# ---------------------------------------------------------------- scenarios

def sc_all_reduce(cx: Ctx):
    p, r = cx.p, cx.r
    sizes = [1, 7, 64, 1000, 4097, 65536 + 3, 1 << 20]
    for algo in ("one_shot", "two_shot"):
        for dtype in (DType.f32, DType.bf16, DType.i64, DType.i32, DType.f64, DType.u8):
            for op in ("sum", "prod", "min", "max"):
                for n in sizes:
                    if op == "prod" and n > 4097:
                        continue
                    gen = small_prod_values if op == "prod" else values
                    ins = [gen(dtype, n, "ar", algo, dtype.name, op, n, q) for q in range(p)]
                    if dtype is DType.bf16:
                        want = seqref.fold_bf16(ins, op)
                    else:
                        want = seqref.fold(ins, op)
                    t = to_dev(ins[r], dtype, cx.dev)
                    req = CommRequest(CommOpKind.all_reduce, input=Buffer(t), output=Buffer(t),
                                      op=ReduceOp(op), backend=cx.b)
                    cx.rt._instance(cx.b).policy = AlgorithmPolicy({CommOpKind.all_reduce: algo})
                    cx.rt.post(req)
                    cx.check(f"all_reduce/{algo}/{dtype.name}/{op}/{n}", from_dev(t, dtype), want)
    cx.rt._instance(cx.b).policy = AlgorithmPolicy()
    # NVLS (switch reduction): f32/bf16 sums within the north_star tolerance
    # (rtol 1e-5 f32, 1e-2 bf16, atol = rtol * max(1, max|want|)).
    inst = cx.rt._instance(cx.b)
    cx.nvls = bool(inst.comm.caps.nvls_supported)
    if cx.nvls:
        inst.policy = AlgorithmPolicy({CommOpKind.all_reduce: "nvls"})
        for dtype, rtol in ((DType.f32, 1e-5), (DType.bf16, 1e-2)):
            for n in (1, 7, 4097, 65536 + 3, 1 << 20, (3 << 20) + 5):
                ins = [values(dtype, n, "nvls", dtype.name, n, q) for q in range(p)]
                t = to_dev(ins[r], dtype, cx.dev)
                o = torch.empty_like(t)
                cx.rt.post(CommRequest(CommOpKind.all_reduce, input=Buffer(t), output=Buffer(o),
                                       op=ReduceOp.sum, backend=cx.b))
                if dtype is DType.bf16:
                    got = seqref.bf16_bits_to_f32(from_dev(o, dtype))
                    want = seqref.bf16_bits_to_f32(seqref.fold_bf16(ins, "sum"))
                else:
                    got, want = from_dev(o, dtype), seqref.fold(ins, "sum")
                cx.check(f"all_reduce/nvls/{dtype.name}/{n}", got, want, float_reduction=True,
                         rtol=rtol)
        # integer / non-sum requests fall back to two-shot: still bit-exact
        ins = [values(DType.i64, 5000, "nvls-i64", q) for q in range(p)]
        t = to_dev(ins[r], DType.i64, cx.dev)
        cx.rt.all_reduce(cx.b, Buffer(t))
        cx.check("all_reduce/nvls-fallback/i64", from_dev(t, DType.i64), seqref.fold(ins, "sum"))
        inst.policy = AlgorithmPolicy()
    # out-of-place + misaligned (element offset 1 -> scalar path)
    for dtype in (DType.f32, DType.bf16):
        n = 10001
        ins = [values(dtype, n + 1, "arm", dtype.name, q) for q in range(p)]
        want = (seqref.fold_bf16 if dtype is DType.bf16 else seqref.fold)([x[1:] for x in ins], "sum")
        src = to_dev(ins[r], dtype, cx.dev)[1:]
        dst = torch.empty(n + 1, dtype=src.dtype, device=cx.dev)[1:]
        cx.rt.post(CommRequest(CommOpKind.all_reduce, input=Buffer(src), output=Buffer(dst),
                               op=ReduceOp.sum, backend=cx.b))
        cx.check(f"all_reduce/misaligned/{dtype.name}", from_dev(dst, dtype), want)
    # large two-shot that spans several workspace chunks
    n = (96 << 20) // 4 + 5
    ins = [values(DType.f32, n, "arbig", q) for q in range(p)]
    want = seqref.fold(ins, "sum")
    t = to_dev(ins[r], DType.f32, cx.dev)
    cx.rt.all_reduce(cx.b, Buffer(t))
    # AUTO may take NVLS for large f32 sums (tuning table): the switch's
    # summation order is within the tolerance, every other kernel bit-exact
    cx.check("all_reduce/f32/96MiB", from_dev(t, DType.f32), want, float_reduction=ran_nvls(cx),
             rtol=1e-5)


def ran_nvls(cx) -> bool:
    """Did the last AUTO all_reduce of cx.b run the NVLS (switch) kernel?"""
    return cx.rt._instance(cx.b).last_algorithm(CommOpKind.all_reduce) == "nvls"


def counts_matrix(p, count, *seed):
    rng = np.random.default_rng(seed_of(*seed))
    return [[int(rng.integers(0, count + 1)) for _ in range(p)] for _ in range(p)]


def packed(c):
    out, o = [], 0
    for x in c:
        out.append(o)
        o += x
    return out


def sc_all_to_allv(cx: Ctx):
    p, r = cx.p, cx.r
    for dtype in (DType.f32, DType.bf16, DType.i64, DType.u8):
        for count in (0, 1, 7, 64, 1000, 50000):
            sc = counts_matrix(p, count, "a2av", dtype.name, count)
            sd = [packed(row) for row in sc]
            rd = [packed([sc[j][q] for j in range(p)]) for q in range(p)]
            ins = [values(dtype, sum(sc[q]), "a2avin", dtype.name, count, q) for q in range(p)]
            want = seqref.all_to_allv(ins, sc, sd, rd,
                                      out_counts=[sum(sc[j][q] for j in range(p)) for q in range(p)])
            rcounts = [sc[j][r] for j in range(p)]
            i = to_dev(ins[r], dtype, cx.dev)
            o = torch.zeros(sum(rcounts), dtype=i.dtype, device=cx.dev)
            cx.rt.all_to_allv(cx.b, Buffer(o), Buffer(i), sc[r], rcounts, sd[r], rd[r])
            cx.check(f"a2av/{dtype.name}/{count}", from_dev(o, dtype), want[r])
            # device-resident counts
            o2 = torch.zeros_like(o)
            dc = [torch.tensor(v, dtype=torch.int64, device=cx.dev)
                  for v in (sc[r], rcounts, sd[r], rd[r])]
            cx.rt.all_to_allv(cx.b, Buffer(o2), Buffer(i), dc[0], dc[1], dc[2], dc[3])
            cx.check(f"a2av-devcounts/{dtype.name}/{count}", from_dev(o2, dtype), want[r])
    # cfg1: 1 MiB f32 per rank, skew weights 1:2..p
    n = 262144
    w = np.arange(1, p + 1, dtype=np.float64)
    row = [int(x) for x in np.floor(w / w.sum() * n)]
    row[-1] += n - sum(row)
    sc = [list(row) for _ in range(p)]
    sd = [packed(x) for x in sc]
    rd = [packed([sc[j][q] for j in range(p)]) for q in range(p)]
    ins = [values(DType.f32, n, "cfg1", q) for q in range(p)]
    want = seqref.all_to_allv(ins, sc, sd, rd)
    rc = [sc[j][r] for j in range(p)]
    i = to_dev(ins[r], DType.f32, cx.dev)
    o = torch.zeros(sum(rc), dtype=torch.float32, device=cx.dev)
    cx.rt.all_to_allv(cx.b, Buffer(o), Buffer(i), sc[r], rc, sd[r], rd[r])
    cx.check("a2av/cfg1", from_dev(o, DType.f32), want[r])
    # pairs larger than a workspace slot: acknowledged rounds with a short last
    # round (backend "small": 16 MiB workspace)
    for count in (1_500_000, 3_000_001):
        sc = counts_matrix(p, count, "a2av-rounds", count)
        sd = [packed(row) for row in sc]
        rd = [packed([sc[j][q] for j in range(p)]) for q in range(p)]
        ins = [values(DType.f32, sum(sc[q]), "a2av-rounds-in", count, q) for q in range(p)]
        want = seqref.all_to_allv(ins, sc, sd, rd,
                                  out_counts=[sum(sc[j][q] for j in range(p)) for q in range(p)])
        rc = [sc[j][r] for j in range(p)]
        o = torch.zeros(sum(rc), dtype=torch.float32, device=cx.dev)
        cx.rt.all_to_allv("small", Buffer(o), Buffer(to_dev(ins[r], DType.f32, cx.dev)), sc[r], rc,
                          sd[r], rd[r])
        cx.check(f"a2av/rounds/{count}", from_dev(o, DType.f32), want[r])


def sc_all_to_all(cx: Ctx):
    p, r = cx.p, cx.r
    for m in (0, 1, 5, 4096, 100003):
        ins = [values(DType.i64, p * m, "a2as", m, q) for q in range(p)]
        want = seqref.all_to_all_single(ins)
        i = to_dev(ins[r], DType.i64, cx.dev)
        o = torch.zeros_like(i)
        cx.rt.all_to_all_single(cx.b, Buffer(o), Buffer(i))
        cx.check(f"a2a_single/{m}", from_dev(o, DType.i64), want[r])
        # in place (the reference snapshots, collectives.py:662-663)
        io = to_dev(ins[r], DType.i64, cx.dev)
        bb = Buffer(io)
        cx.rt.post(CommRequest(CommOpKind.all_to_all_single, input=bb, output=bb, backend=cx.b))
        cx.check(f"a2a_single/inplace/{m}", from_dev(io, DType.i64), want[r])
    # list form
    blocks = [[values(DType.f32, 3 + q + j, "a2al", q, j) for j in range(p)] for q in range(p)]
    want = seqref.all_to_all(blocks)
    ins = [Buffer(to_dev(blocks[r][j], DType.f32, cx.dev)) for j in range(p)]
    outs = [Buffer(torch.zeros(3 + j + r, dtype=torch.float32, device=cx.dev)) for j in range(p)]
    cx.rt.all_to_all(cx.b, outs, ins)
    for j in range(p):
        cx.check(f"a2a_list[{j}]", from_dev(outs[j].array, DType.f32), want[r][j])


def sc_gathers(cx: Ctx):
    p, r = cx.p, cx.r
    for dtype in (DType.i64, DType.f32, DType.u8):
        for count in (0, 1, 5, 1000, 70001):
            rng = np.random.default_rng(seed_of("agv", dtype.name, count))
            counts = [int(rng.integers(0, count + 1)) for _ in range(p)]
            if p > 2:
                counts[1] = 0  # zero-length middle segment (test_collectives.py:84-94)
            displs = packed(counts)
            ins = [values(dtype, counts[q], "agvin", dtype.name, count, q) for q in range(p)]
            want = seqref.all_gatherv(ins, counts, displs)
            i = to_dev(ins[r], dtype, cx.dev)
            o = torch.zeros(sum(counts), dtype=i.dtype, device=cx.dev)
            cx.rt.all_gatherv(cx.b, Buffer(o), Buffer(i), counts, displs)
            cx.check(f"allgatherv/{dtype.name}/{count}", from_dev(o, dtype), want[r])
            for root in range(p):
                o = torch.zeros(sum(counts), dtype=i.dtype, device=cx.dev) if r == root else None
                cx.rt.gatherv(cx.b, Buffer(o) if o is not None else None, Buffer(i), root, counts,
                              displs)
                if r == root:
                    cx.check(f"gatherv/{dtype.name}/{count}/root{root}", from_dev(o, dtype),
                             seqref.gatherv(ins, root, counts, displs)[root])
            # GPU-resident rcounts / displs (mcrdl_all_gatherv_dev / mcrdl_gatherv_dev),
            # segments packed in reverse rank order (displs not ascending)
            gdispls, off = [0] * p, 0
            for q in reversed(range(p)):
                gdispls[q] = off
                off += counts[q]
            dcnt = torch.tensor(counts, dtype=torch.int64, device=cx.dev)
            ddsp = torch.tensor(gdispls, dtype=torch.int64, device=cx.dev)
            o = torch.zeros(off, dtype=i.dtype, device=cx.dev)
            cx.rt.all_gatherv(cx.b, Buffer(o), Buffer(i), dcnt, ddsp)
            cx.check(f"allgatherv_dev/{dtype.name}/{count}", from_dev(o, dtype),
                     seqref.all_gatherv(ins, counts, gdispls)[r])
            for root in (0, p - 1):
                o = torch.zeros(off, dtype=i.dtype, device=cx.dev) if r == root else None
                cx.rt.gatherv(cx.b, Buffer(o) if o is not None else None, Buffer(i), root, dcnt,
                              ddsp)
                if r == root:
                    cx.check(f"gatherv_dev/{dtype.name}/{count}/root{root}", from_dev(o, dtype),
                             seqref.gatherv(ins, root, counts, gdispls)[root])
        n = 333
        ins = [values(dtype, n, "ag", dtype.name, q) for q in range(p)]
        i = to_dev(ins[r], dtype, cx.dev)
        o = torch.zeros(p * n, dtype=i.dtype, device=cx.dev)
        cx.rt.all_gather(cx.b, Buffer(o), Buffer(i))
        cx.check(f"allgather/{dtype.name}", from_dev(o, dtype), seqref.all_gather(ins)[r])
        root = p - 1
        o = torch.zeros(p * n, dtype=i.dtype, device=cx.dev) if r == root else None
        cx.rt.gather(cx.b, Buffer(o) if o is not None else None, Buffer(i), root)
        if r == root:
            cx.check(f"gather/{dtype.name}", from_dev(o, dtype), seqref.gather(ins, root)[root])


def sc_bcast_scatter(cx: Ctx):
    p, r = cx.p, cx.r
    for dtype, n in ((DType.u8, 65536), (DType.f32, 1), (DType.i32, 12345), (DType.bf16, 4096)):
        for root in range(p):
            ins = [values(dtype, n, "bc", dtype.name, root, q) for q in range(p)]
            t = to_dev(ins[r], dtype, cx.dev)
            cx.rt.bcast(cx.b, Buffer(t), root)
            cx.check(f"bcast/{dtype.name}/root{root}", from_dev(t, dtype), ins[root])
    # NVLS multicast bcast (explicit, and AUTO at >= 1 MiB): partial final
    # packs, a buffer misaligned on one rank only, multi-chunk sizes
    inst = cx.rt._instance(cx.b)
    if bool(inst.comm.caps.nvls_supported) and p > 1:
        for algo in ("nvls", "auto"):
            inst.policy = AlgorithmPolicy({CommOpKind.bcast: algo})
            for dtype, n in ((DType.u8, 1), (DType.u8, 17), (DType.f32, 1000), (DType.u8, (1 << 20) + 3),
                             (DType.f32, (5 << 20) + 1), (DType.bf16, 3 << 20)):
                for root in (0, p - 1):
                    ins = [values(dtype, n, "bcnv", algo, dtype.name, n, root, q) for q in range(p)]
                    t = to_dev(ins[r], dtype, cx.dev)
                    cx.rt.bcast(cx.b, Buffer(t), root)
                    cx.check(f"bcast/{algo}/{dtype.name}/{n}/root{root}", from_dev(t, dtype),
                             ins[root])
            # rank 1's buffer starts one byte into its allocation
            n = (2 << 20) + 5
            ins = [values(DType.u8, n, "bcnvmis", algo, q) for q in range(p)]
            base = to_dev(np.concatenate([np.zeros(1, np.uint8), ins[r]]), DType.u8, cx.dev)
            t = base[1:] if r == 1 else base[1:].clone()
            cx.rt.bcast(cx.b, Buffer(t), 0)
            cx.check(f"bcast/{algo}/misaligned", from_dev(t, DType.u8), ins[0])
        inst.policy = AlgorithmPolicy()
    # pipelined chain bcast: partial chunks, odd sizes, a buffer misaligned on
    # one rank, and (on the 8 MiB-workspace backend) messages spanning several
    # launches
    if p > 1:
        for be, cases in ((cx.b, ((DType.u8, 1), (DType.u8, 100003), (DType.f32, (3 << 20) + 7),
                                  (DType.bf16, 5 << 20))),
                          ("bsmall", ((DType.f32, (5 << 20) + 3), (DType.u8, 9 << 20)))):
            binst = cx.rt._instance(be)
            binst.policy = AlgorithmPolicy({CommOpKind.bcast: "chain"})
            for dtype, n in cases:
                for root in (0, p - 1, p // 2):
                    ins = [values(dtype, n, "bcch", be, dtype.name, n, root, q) for q in range(p)]
                    t = to_dev(ins[r], dtype, cx.dev)
                    cx.rt.bcast(be, Buffer(t), root)
                    cx.check(f"bcast/chain/{be}/{dtype.name}/{n}/root{root}", from_dev(t, dtype),
                             ins[root])
            n = (2 << 20) + 5
            ins = [values(DType.u8, n, "bcchmis", be, q) for q in range(p)]
            base = to_dev(np.concatenate([np.zeros(1, np.uint8), ins[r]]), DType.u8, cx.dev)
            t = base[1:] if r == 1 else base[1:].clone()
            cx.rt.bcast(be, Buffer(t), 0)
            cx.check(f"bcast/chain/{be}/misaligned", from_dev(t, DType.u8), ins[0])
            binst.policy = AlgorithmPolicy()
    for root in range(p):
        m = 777
        src = values(DType.f32, p * m, "sc", root)
        o = torch.zeros(m, dtype=torch.float32, device=cx.dev)
        i = Buffer(to_dev(src, DType.f32, cx.dev)) if r == root else None
        cx.rt.scatter(cx.b, Buffer(o), i, root)
        cx.check(f"scatter/root{root}", from_dev(o, DType.f32), seqref.scatter(src, p)[r])
        counts = [(q * 7 + 3) % 11 for q in range(p)]
        displs = packed(counts)
        src = values(DType.i64, sum(counts), "scv", root)
        o = torch.zeros(counts[r], dtype=torch.int64, device=cx.dev)
        i = Buffer(to_dev(src, DType.i64, cx.dev)) if r == root else None
        cx.rt.scatterv(cx.b, Buffer(o), i, root, counts, displs)
        cx.check(f"scatterv/root{root}", from_dev(o, DType.i64),
                 seqref.scatterv(src, counts, displs)[r])


def sc_reduce_family(cx: Ctx):
    p, r = cx.p, cx.r
    n = 5000
    for root in range(p):
        ins = [values(DType.f32, n, "red", root, q) for q in range(p)]
        t = to_dev(ins[r], DType.f32, cx.dev)
        cx.rt.reduce(cx.b, Buffer(t), root, ReduceOp.sum)
        if r == root:
            cx.check(f"reduce/root{root}", from_dev(t, DType.f32), seqref.fold(ins, "sum"))
        else:
            cx.check(f"reduce/nonroot-untouched/{root}", from_dev(t, DType.f32), ins[r])
    # native root mode (mcrdl_reduce: RS + gather to the root): large messages
    # and explicit two_shot, every dtype/op, in place and out of place,
    # misaligned, multi-chunk; non-roots untouched
    inst = cx.rt._instance(cx.b)
    cases = [(DType.f32, "sum", (3 << 20) + 5, "auto"), (DType.bf16, "sum", 5 << 20, "auto"),
             (DType.i64, "max", 40_001, "two_shot"), (DType.i32, "min", 99_999, "two_shot"),
             (DType.u8, "sum", 3_000_003, "auto"), (DType.f64, "prod", 4097, "two_shot"),
             (DType.f32, "sum", (160 << 20) // 4 + 3, "auto")]
    for dtype, op, n, algo in cases:
        inst.policy = AlgorithmPolicy({CommOpKind.reduce: algo})
        root = (n + 1) % p
        gen = small_prod_values if op == "prod" else values
        ins = [gen(dtype, n, "rednat", dtype.name, op, n, q) for q in range(p)]
        want = (seqref.fold_bf16 if dtype is DType.bf16 else seqref.fold)(ins, op)
        src = to_dev(ins[r], dtype, cx.dev)
        if n % 2:  # out of place into a misaligned view (every rank passes one,
            # as the reference's validate requires; only the root's is written)
            out = torch.zeros(n + 1, dtype=src.dtype, device=cx.dev)[1:]
            cx.rt.post(CommRequest(CommOpKind.reduce, input=Buffer(src), output=Buffer(out),
                                   root=root, op=ReduceOp(op), backend=cx.b))
            got = out if r == root else None
        else:
            cx.rt.reduce(cx.b, Buffer(src), root, ReduceOp(op))
            got = src
        if r == root:
            cx.check(f"reduce/native/{dtype.name}/{op}/{n}", from_dev(got, dtype), want)
        elif got is not None:
            cx.check(f"reduce/native-untouched/{dtype.name}/{n}", from_dev(got, dtype), ins[r])
    inst.policy = AlgorithmPolicy()
    # composed path (m*8 % 16 != 0) and the native RS kernel (aligned segments)
    for dtype, m, op in ((DType.i64, 1001, "sum"), (DType.f32, 1 << 16, "sum"),
                         (DType.bf16, 4096, "sum"), (DType.i32, 12288, "max"),
                         (DType.f32, (3 << 20) + 4, "sum")):
        ins = [values(dtype, p * m, "rs", dtype.name, m, q) for q in range(p)]
        o = torch.zeros(m, dtype=dtype.torch_dtype, device=cx.dev)
        cx.rt.reduce_scatter(cx.b, Buffer(o), Buffer(to_dev(ins[r], dtype, cx.dev)), ReduceOp(op))
        if dtype is DType.bf16:
            want = seqref.fold_bf16([x[r * m:(r + 1) * m] for x in ins], op)
        else:
            want = seqref.reduce_scatter(ins, op)[r]
        cx.check(f"reduce_scatter/{dtype.name}/{m}/{op}", from_dev(o, dtype), want)


def sc_host_buffers(cx: Ctx):
    """Reference-style numpy Buffers through the device backend (staged)."""
    p, r = cx.p, cx.r
    ins = [values(DType.f32, 4099, "host", q) for q in range(p)]
    b = Buffer(ins[r].copy())
    cx.rt.all_reduce(cx.b, b)
    cx.check("host/all_reduce", b.array, seqref.fold(ins, "sum"))
    # partner.py known answers (p=2 world, frontend/test/helpers/partner.py:60-159)
    if p == 2:
        buf = Buffer.from_values(DType.i64, [r + 1, 10 * (r + 1)])
        cx.rt.all_reduce(cx.b, buf)
        cx.check("known/allreduce_i64", buf.array, np.array([3, 30], dtype=np.int64))
        buf = Buffer.from_values(DType.f32, [0.5 + r, 2.5 * (r + 1)])
        cx.rt.all_reduce(cx.b, buf)
        cx.check("known/allreduce_f32", buf.array, np.array([2.0, 7.5], dtype=np.float32))
        sc = [[1, 2], [2, 1]]
        inp = Buffer.from_values(DType.i64, [[1, 2, 3], [4, 5, 6]][r])
        rc = [sc[j][r] for j in range(p)]
        out = Buffer.zeros(DType.i64, sum(rc))
        cx.rt.all_to_allv(cx.b, out, inp, sc[r], rc, [0, sc[r][0]], [0, rc[0]])
        cx.check("known/alltoallv", out.array, np.array([[1, 4, 5], [2, 3, 6]][r], dtype=np.int64))
        inp = Buffer.from_values(DType.i64, [[1, 2], [3, 4]][r])
        out = Buffer.zeros(DType.i64, 2)
        cx.rt.all_to_all_single(cx.b, out, inp)
        cx.check("known/a2a_single", out.array, np.array([[1, 3], [2, 4]][r], dtype=np.int64))
        inp = Buffer.from_values(DType.i64, [11, 12] if r == 0 else [21])
        gout = Buffer.zeros(DType.i64, 3) if r == 1 else None
        cx.rt.gatherv(cx.b, gout, inp, 1, [2, 1], [0, 2])
        if r == 1:
            cx.check("known/gatherv", gout.array, np.array([11, 12, 21], dtype=np.int64))
        buf = Buffer.from_values(DType.f32, [3.25, -1.5]) if r == 0 else Buffer.zeros(DType.f32, 2)
        cx.rt.bcast(cx.b, buf, 0)
        cx.check("known/bcast", buf.array, np.array([3.25, -1.5], dtype=np.float32))


def sc_async_and_fusion(cx: Ctx):
    p, r = cx.p, cx.r
    # 14 DLRM MLP gradients through fusion, posted async
    shapes = [6656, 512, 262144, 512, 65536, 128, 490496, 1024, 1048576, 1024, 1048576, 1024,
              1024, 1]
    ins = [[values(DType.f32, n, "fus", k, q) for q in range(p)] for k, n in enumerate(shapes)]
    ts = [to_dev(ins[k][r], DType.f32, cx.dev) for k in range(len(shapes))]
    hs = [cx.rt.all_reduce("fused", Buffer(t), ReduceOp.sum, async_op=True) for t in ts]
    for h in hs:
        cx.rt.wait(h)
    cx.sync()
    for k, t in enumerate(ts):
        cx.check(f"fusion/{k}/{shapes[k]}", from_dev(t, DType.f32), seqref.fold(ins[k], "sum"))
    # a fusion group whose one-shot slots exceed the workspace half of its
    # backend ("fused_big": 4 MiB workspace, B = 2 MiB): pack kernel ->
    # all_reduce on the packed buffer -> unpack kernel
    shapes = [100_000, 200_000, 150_000, 7]
    ins = [[values(DType.f32, n, "fusbig", k, q) for q in range(p)] for k, n in enumerate(shapes)]
    ts = [to_dev(ins[k][r], DType.f32, cx.dev) for k in range(len(shapes))]
    hs = [cx.rt.all_reduce("fused_big", Buffer(t), ReduceOp.sum, async_op=True) for t in ts]
    for h in hs:
        cx.rt.wait(h)
    cx.sync()
    for k, t in enumerate(ts):
        cx.check(f"fusion-packed/{k}/{shapes[k]}", from_dev(t, DType.f32), seqref.fold(ins[k], "sum"))
    # async handles on the plain backend + synchronize
    xs = [values(DType.i32, 10000 + k, "async", k, q) for k in range(6) for q in range(p)]
    ts = [to_dev(xs[k * p + r], DType.i32, cx.dev) for k in range(6)]
    hs = [cx.rt.all_reduce(cx.b, Buffer(t), async_op=True) for t in ts]
    cx.rt.synchronize([cx.b])
    for k, h in enumerate(hs):
        assert h.test()
        cx.check(f"async/{k}", from_dev(ts[k], DType.i32),
                 seqref.fold([xs[k * p + q] for q in range(p)], "sum"))


def sc_order_mismatch(cx: Ctx):
    """Ranks post different ops at the same seq -> OrderMismatch everywhere
    (test_acceptance.py:214-243, collectives.py:283-285)."""
    if cx.p < 2:
        return
    n = 1000 + (7 if cx.r == 0 else 0)
    t = torch.ones(n, dtype=torch.float32, device=cx.dev)
    cx.rt.all_reduce("mism", Buffer(t), async_op=True)
    raised = None
    try:
        cx.rt.synchronize(["mism"])
    except OrderMismatch as exc:
        raised = exc
    except Exception as exc:  # noqa: BLE001
        raised = exc
    cx.checked += 1
    if not isinstance(raised, OrderMismatch):
        cx.failures.append(f"order_mismatch: expected OrderMismatch, got {raised!r}")


def sc_graphs(cx: Ctx):
    """Collectives captured into one CUDA graph and replayed with fresh inputs,
    eager ops interleaved between replays. Works because the op epoch lives
    on the device (common.cuh epoch_enter/epoch_exit): a replayed launch has
    no host-baked per-op state. Covers the LL, one-shot, two-shot (and NVLS
    when present) all_reduce kernels and the exchange kernel."""
    p, r, dev = cx.p, cx.r, cx.dev
    inst = cx.rt._instance(cx.b)
    sizes = {"ll": 1000, "one_shot": 300_003, "two_shot": (24 << 20) // 4 + 3}
    xs = {k: torch.empty(n, dtype=torch.float32, device=dev) for k, n in sizes.items()}
    outs = {k: torch.empty_like(v) for k, v in xs.items()}
    nv = bool(inst.comm.caps.nvls_supported) and p > 1
    nv_x = torch.empty(1 << 18, dtype=torch.float32, device=dev)
    m = 4099
    a_in = torch.empty(p * m, dtype=torch.int64, device=dev)
    a_out = torch.empty_like(a_in)

    def run_ops():
        for k in xs:
            inst.policy = AlgorithmPolicy({CommOpKind.all_reduce: k if k != "ll" else "auto"})
            cx.rt.post(CommRequest(CommOpKind.all_reduce, input=Buffer(xs[k]),
                                   output=Buffer(outs[k]), op=ReduceOp.sum, backend=cx.b))
        if nv:
            inst.policy = AlgorithmPolicy({CommOpKind.all_reduce: "nvls"})
            cx.rt.all_reduce(cx.b, Buffer(nv_x))
        inst.policy = AlgorithmPolicy()
        cx.rt.all_to_all_single(cx.b, Buffer(a_out), Buffer(a_in))

    def fill(it):
        ins = {k: [values(DType.f32, n, "graph", k, it, q) for q in range(p)]
               for k, n in sizes.items()}
        nvi = [values(DType.f32, nv_x.numel(), "graph-nv", it, q) for q in range(p)]
        a = [values(DType.i64, p * m, "graph-a2a", it, q) for q in range(p)]
        for k in xs:
            xs[k].copy_(torch.from_numpy(ins[k][r]))
        nv_x.copy_(torch.from_numpy(nvi[r]))
        a_in.copy_(torch.from_numpy(a[r]))
        return ins, nvi, a

    def verify(tag, ins, nvi, a):
        for k in xs:
            cx.check(f"graph/{tag}/{k}", from_dev(outs[k], DType.f32), seqref.fold(ins[k], "sum"))
        if nv:
            cx.check(f"graph/{tag}/nvls", from_dev(nv_x, DType.f32), seqref.fold(nvi, "sum"),
                     float_reduction=True, rtol=1e-5)
        cx.check(f"graph/{tag}/a2a", from_dev(a_out, DType.i64), seqref.all_to_all_single(a)[r])

    state = fill(0)
    run_ops()  # eager warm-up outside the capture
    cx.sync()
    verify("eager", *state)
    g = torch.cuda.CUDAGraph()
    with cx.exclusive():
        with cx.graph(g):
            run_ops()
        cx.upload(g)
    for it in range(1, 5):
        state = fill(it)
        cx.lockstep(("graph", it))
        g.replay()
        cx.lockstep(("graph-enqueued", it))
        # an eager op between replays keeps the device epoch in step
        e = [values(DType.i32, 777, "graph-eager", it, q) for q in range(p)]
        t = to_dev(e[r], DType.i32, dev)
        cx.rt.all_reduce(cx.b, Buffer(t))
        cx.sync()
        verify(f"replay{it}", *state)
        cx.check(f"graph/eager{it}", from_dev(t, DType.i32), seqref.fold(e, "sum"))
    del g


def sc_p2p(cx: Ctx):
    """send/recv (runtime.py:498-508, executed at runtime.py:244-262): ring
    shifts over the chunk boundaries, 40 queued eager sends, a rendezvous
    message larger than the 32 MiB mailbox (recv posted first, async), the
    tuner's rank 0<->1 ping-pong (tuner.py:128-145), self-send, staged numpy
    buffers, CUDA-graph replay, and LengthMismatch (runtime.py:256-260) on a
    dedicated backend.

    send/recv do not go through the collective launch rendezvous, so for
    co-located ranks every step allocates its buffers first and then meets
    the peers (cx.lockstep) before launching: no rank is inside a
    device-synchronizing allocation while a peer's kernel waits on it."""
    p, r, dev = cx.p, cx.r, cx.dev
    nxt, prv = (r + 1) % p, (r - 1) % p
    only = os.environ.get("MCRDL_P2P_PARTS")  # debugging: run a subset of the parts
    parts = set(only.split(",")) if only else {"ring", "queued", "rendezvous", "pingpong", "self",
                                                "host", "graph", "lenm"}
    for n in ((0, 1, 1000, 131072, 131073, 3_000_001) if "ring" in parts else ()):
        x = [values(DType.f32, n, "p2p", n, q) for q in range(p)]
        dst = torch.full((n,), -1.0, device=dev)
        src = to_dev(x[r], DType.f32, dev)
        cx.lockstep(("ring", n))
        cx.rt.send(cx.b, Buffer(src), nxt)
        cx.rt.recv(cx.b, Buffer(dst), prv)
        cx.lockstep(("ring-enqueued", n))
        cx.check(f"p2p/ring/{n}", from_dev(dst, DType.f32), x[prv])
    # 40 sends queued before their receives (eager: headers and slots free)
    if "queued" in parts:
        _p2p_queued(cx, nxt, prv)
    if "rendezvous" in parts:
        _p2p_rendezvous(cx, nxt, prv)
    if "pingpong" in parts:
        _p2p_pingpong(cx)
    if "self" in parts:
        _p2p_self(cx)
    if "host" in parts:
        _p2p_host(cx, nxt, prv)
    if "graph" in parts:
        _p2p_graph(cx, nxt, prv)
    if "lenm" in parts:
        _p2p_lenm(cx)


def _p2p_queued(cx, nxt, prv):
    p, r, dev = cx.p, cx.r, cx.dev
    xs = [[values(DType.i64, 100 + k, "p2pq", k, q) for q in range(p)] for k in range(40)]
    srcs = [to_dev(xs[k][r], DType.i64, dev) for k in range(40)]
    outs = [torch.zeros(100 + k, dtype=torch.int64, device=dev) for k in range(40)]
    cx.lockstep(("queued",))
    for k in range(40):
        cx.rt.send(cx.b, Buffer(srcs[k]), nxt)
    for k in range(40):
        cx.rt.recv(cx.b, Buffer(outs[k]), prv)
    cx.lockstep(("queued-enqueued",))
    for k in range(40):
        cx.check(f"p2p/queued/{k}", from_dev(outs[k], DType.i64), xs[k][prv])


def _p2p_rendezvous(cx, nxt, prv):
    """40 MiB + 12 B > mailbox; the recv runs on the lane stream."""
    p, r, dev = cx.p, cx.r, cx.dev
    n = (10 << 20) + 3
    x = [values(DType.f32, n, "p2pbig", q) for q in range(p)]
    dst = torch.zeros(n, device=dev)
    src = to_dev(x[r], DType.f32, dev)
    cx.lockstep(("rendezvous",))
    h = cx.rt.recv(cx.b, Buffer(dst), prv, async_op=True)
    cx.rt.send(cx.b, Buffer(src), nxt)
    cx.lockstep(("rendezvous-enqueued",))
    h.wait()
    torch.cuda.current_stream().wait_stream(cx.rt._instance(cx.b).stream)
    cx.check("p2p/rendezvous", from_dev(dst, DType.f32), x[prv])


def _p2p_pingpong(cx):
    """Ping-pong between ranks 0 and 1, bf16 payload."""
    p, r, dev = cx.p, cx.r, cx.dev
    y = [values(DType.bf16, 70000, "pp", q) for q in range(2)]
    mine = to_dev(y[min(r, 1)], DType.bf16, dev)
    got = torch.zeros_like(mine)
    cx.lockstep(("pingpong",))
    if p >= 2 and r < 2:
        if r == 0:
            cx.rt.send(cx.b, Buffer(mine), 1)
            cx.rt.recv(cx.b, Buffer(got), 1)
        else:
            cx.rt.recv(cx.b, Buffer(got), 0)
            cx.rt.send(cx.b, Buffer(mine), 0)
    cx.lockstep(("pingpong-enqueued",))
    if p >= 2 and r < 2:
        cx.check("p2p/pingpong", from_dev(got, DType.bf16), y[1 - r])


def _p2p_self(cx):
    p, r, dev = cx.p, cx.r, cx.dev
    z = values(DType.u8, 9999, "self", r)
    zd = torch.zeros(9999, dtype=torch.uint8, device=dev)
    zs = to_dev(z, DType.u8, dev)
    cx.lockstep(("self",))
    cx.rt.send(cx.b, Buffer(zs), r)
    cx.rt.recv(cx.b, Buffer(zd), r)
    cx.lockstep(("self-enqueued",))
    cx.check("p2p/self", from_dev(zd, DType.u8), z)


def _p2p_host(cx, nxt, prv):
    """Staged numpy buffers (reference-style host Buffers)."""
    p, r, dev = cx.p, cx.r, cx.dev
    hx = [values(DType.i32, 5000, "p2phost", q) for q in range(p)]
    hout = np.zeros(5000, dtype=np.int32)
    cx.lockstep(("host",))
    cx.rt.send(cx.b, Buffer(hx[r].copy()), nxt)
    cx.rt.recv(cx.b, Buffer(hout), prv)
    cx.check("p2p/host", hout, hx[prv])


def _p2p_graph(cx, nxt, prv):
    """CUDA graph: one captured ring shift, replayed with fresh inputs."""
    p, r, dev = cx.p, cx.r, cx.dev
    gi = torch.zeros(777_777, device=dev)
    go = torch.zeros_like(gi)
    cx.lockstep(("graph-warmup",))
    cx.rt.send(cx.b, Buffer(gi), nxt)  # warm-up outside the capture
    cx.rt.recv(cx.b, Buffer(go), prv)
    cx.lockstep(("graph-warmup-enqueued",))
    cx.sync()
    g = torch.cuda.CUDAGraph()
    with cx.exclusive():
        with cx.graph(g):
            cx.rt.send(cx.b, Buffer(gi), nxt)
            cx.rt.recv(cx.b, Buffer(go), prv)
        cx.upload(g)
    for it in range(3):
        x = [values(DType.f32, gi.numel(), "p2pgraph", it, q) for q in range(p)]
        gi.copy_(torch.from_numpy(x[r]))
        cx.lockstep(("p2pgraph", it))
        g.replay()
        cx.lockstep(("p2pgraph-enqueued", it))
        cx.sync()
        cx.check(f"p2p/graph{it}", from_dev(go, DType.f32), x[prv])
    del g


def _p2p_lenm(cx):
    """LengthMismatch: rank 1 posts one element more than rank 0 sends."""
    p, r, dev = cx.p, cx.r, cx.dev
    lm = torch.ones(100, device=dev) if r == 0 else torch.zeros(101, device=dev)
    cx.lockstep(("lenm",))
    if p >= 2 and r < 2:
        if r == 0:
            cx.rt.send("lenm", Buffer(lm), 1)
            cx.sync()
        else:
            raised = None
            try:
                cx.rt.recv("lenm", Buffer(lm), 0, async_op=True)
                cx.rt.synchronize(["lenm"])
            except Exception as exc:  # noqa: BLE001
                raised = exc
            cx.checked += 1
            if type(raised).__name__ != "LengthMismatch":
                cx.failures.append(f"p2p/length_mismatch: expected LengthMismatch, got {raised!r}")


def sc_symm(cx: Ctx):
    """all_reduce on symmetric tensors (Runtime.symmetric_empty): the zero-copy
    kernels (csrc/allreduce.cu k_ar_symm) — NVLS multicast for aligned f32/bf16
    sums (tolerance), peer loads + ascending fold otherwise (bit-exact) — in
    place, out of place, misaligned slices, and a symmetric input with a plain
    output (standard path)."""
    p, r, dev = cx.p, cx.r, cx.dev
    inst = cx.rt._instance(cx.b)
    A = cx.rt.symmetric_empty(cx.b, 64 << 20, "u8")
    B = cx.rt.symmetric_empty(cx.b, 64 << 20, "u8")
    nv = bool(inst.comm.caps.nvls_supported) and p > 1

    def view(blk, dtype, n, off=0):
        es = dtype.size_bytes
        return blk[off * es:(off + n) * es].view(dtype.torch_dtype)

    cases = [(DType.f32, "sum", "auto"), (DType.bf16, "sum", "auto"), (DType.f32, "sum", "two_shot"),
             (DType.i64, "sum", "auto"), (DType.i32, "max", "auto"), (DType.u8, "min", "auto"),
             (DType.f64, "prod", "auto")]
    for dtype, op, algo in cases:
        inst.policy = AlgorithmPolicy({CommOpKind.all_reduce: algo})
        sizes = (1, 7, 4097, 65536 + 3) if op == "prod" else (1, 7, 4097, 65536 + 3, 1 << 20,
                                                                (12 << 20) // dtype.size_bytes + 5)
        for n in sizes:
            for off in (0, 1):
                for inplace in (True, False):
                    gen = small_prod_values if op == "prod" else values
                    ins = [gen(dtype, n, "symm", dtype.name, op, algo, n, off, q) for q in range(p)]
                    want = (seqref.fold_bf16 if dtype is DType.bf16 else seqref.fold)(ins, op)
                    src = view(A, dtype, n, off)
                    src.copy_(to_dev(ins[r], dtype, dev))
                    dst = src if inplace else view(B, dtype, n, off)
                    cx.rt.post(CommRequest(CommOpKind.all_reduce, input=Buffer(src),
                                           output=Buffer(dst), op=ReduceOp(op), backend=cx.b))
                    zero_copy_nvls = (nv and op == "sum" and algo == "auto" and off == 0
                                      and dtype in (DType.f32, DType.bf16)
                                      and (n * dtype.size_bytes) % 16 == 0)
                    tag = f"symm/{dtype.name}/{op}/{algo}/{n}/off{off}/{'in' if inplace else 'out'}"
                    if zero_copy_nvls and dtype is DType.bf16:
                        cx.check(tag, seqref.bf16_bits_to_f32(from_dev(dst, dtype)),
                                 seqref.bf16_bits_to_f32(want), float_reduction=True, rtol=1e-2)
                    elif zero_copy_nvls:
                        cx.check(tag, from_dev(dst, dtype), want, float_reduction=True, rtol=1e-5)
                    else:
                        cx.check(tag, from_dev(dst, dtype), want)
    inst.policy = AlgorithmPolicy()
    # exchanges into symmetric outputs (csrc/symm_x.cu: senders store straight
    # into every peer's output above the LL pair size; LL below)
    for dtype, m, off in ((DType.f32, (5 << 20) // 4 + 3, 0), (DType.i64, (5 << 20) // 8 + 1, 1),
                          (DType.bf16, 3 << 20, 0), (DType.f32, 100_003, 0), (DType.f32, 1000, 0)):
        ins = [values(dtype, p * m, "symm-a2a", dtype.name, m, q) for q in range(p)]
        src = to_dev(ins[r], dtype, dev)
        dst = view(B, dtype, p * m, off)
        dst.zero_()
        cx.rt.all_to_all_single(cx.b, Buffer(dst), Buffer(src))
        cx.check(f"symm/a2a_single/{dtype.name}/{m}/off{off}", from_dev(dst, dtype),
                 seqref.all_to_all_single(ins)[r])
    # in place on a symmetric buffer (the input is snapshotted, the output is symmetric)
    m = (5 << 20) // 4 + 7
    ins = [values(DType.f32, p * m, "symm-a2a-ip", q) for q in range(p)]
    io = view(A, DType.f32, p * m)
    io.copy_(to_dev(ins[r], DType.f32, dev))
    bb = Buffer(io)
    cx.rt.post(CommRequest(CommOpKind.all_to_all_single, input=bb, output=bb, backend=cx.b))
    cx.check("symm/a2a_single/inplace", from_dev(io, DType.f32), seqref.all_to_all_single(ins)[r])
    counts = [(5 << 20) // 4 + 1013 * q for q in range(p)]
    displs = packed(counts)
    ins = [values(DType.f32, counts[q], "symm-agv", q) for q in range(p)]
    dst = view(B, DType.f32, sum(counts), 3)
    cx.rt.all_gatherv(cx.b, Buffer(dst), Buffer(to_dev(ins[r], DType.f32, dev)), counts, displs)
    cx.check("symm/all_gatherv", from_dev(dst, DType.f32), seqref.all_gatherv(ins, counts, displs)[r])
    # symmetric input, ordinary output: the standard (staged) path
    n = 100_003
    ins = [values(DType.i64, n, "symm-mixed", q) for q in range(p)]
    src = view(A, DType.i64, n)
    src.copy_(to_dev(ins[r], DType.i64, dev))
    dst = torch.zeros(n, dtype=torch.int64, device=dev)
    cx.rt.post(CommRequest(CommOpKind.all_reduce, input=Buffer(src), output=Buffer(dst),
                           op=ReduceOp.sum, backend=cx.b))
    cx.check("symm/mixed", from_dev(dst, DType.i64), seqref.fold(ins, "sum"))


def sc_codec(cx: Ctx):
    """Trunc16 codec fused into the exchange kernel (CompressionConfig,
    middleware.py:43-95): every compressible kind on backend "cmp" against the
    oracle with peers' data truncated (seqref.trunc16) and the own segment
    exact; non-f32 payloads bypass; misaligned f32; numpy Buffers; and ranks
    that disagree on the codec -> CodecMismatch (collectives.py:226-228)."""
    p, r, dev, b = cx.p, cx.r, cx.dev, "cmp"
    T = seqref.trunc16

    def mine(xs, src_rank_of=None):
        return [x if q == r else T(x) for q, x in enumerate(xs)]

    # all_to_allv: random counts (zeros included), pairs past one workspace round
    for count in (0, 5, 1000, 70_000, 3_000_000):
        sc = counts_matrix(p, count, "cdc-a2av", count)
        sd = [packed(row) for row in sc]
        rd = [packed([sc[j][q] for j in range(p)]) for q in range(p)]
        ins = [values(DType.f32, sum(sc[q]), "cdc-a2av-in", count, q) for q in range(p)]
        want = seqref.all_to_allv(mine(ins), sc, sd, rd,
                                  out_counts=[sum(sc[j][q] for j in range(p)) for q in range(p)])
        rc = [sc[j][r] for j in range(p)]
        o = torch.zeros(sum(rc), device=dev)
        cx.rt.all_to_allv(b, Buffer(o), Buffer(to_dev(ins[r], DType.f32, dev)), sc[r], rc, sd[r], rd[r])
        cx.check(f"codec/a2av/{count}", from_dev(o, DType.f32), want[r])
    # all_to_all_single, misaligned by one element on every rank
    m = 40_001
    ins = [values(DType.f32, p * m + 1, "cdc-a2as", q) for q in range(p)]
    want = seqref.all_to_all_single(mine([x[1:] for x in ins]))
    src = to_dev(ins[r], DType.f32, dev)[1:]
    o = torch.zeros(p * m + 1, device=dev)[1:]
    cx.rt.all_to_all_single(b, Buffer(o), Buffer(src))
    cx.check("codec/a2a_single/misaligned", from_dev(o, DType.f32), want[r])
    # list form
    blocks = [[values(DType.f32, 300 + q + j, "cdc-a2al", q, j) for j in range(p)] for q in range(p)]
    tb = [[blk if q == r else T(blk) for blk in row] for q, row in enumerate(blocks)]
    want = seqref.all_to_all(tb)
    outs = [Buffer(torch.zeros(300 + j + r, device=dev)) for j in range(p)]
    cx.rt.all_to_all(b, outs, [Buffer(to_dev(x, DType.f32, dev)) for x in blocks[r]])
    for j in range(p):
        cx.check(f"codec/a2a_list[{j}]", from_dev(outs[j].array, DType.f32), want[r][j])
    # all_gatherv / gatherv / scatterv / bcast
    counts = [5000 * (q + 1) + 3 for q in range(p)]
    displs = packed(counts)
    ins = [values(DType.f32, counts[q], "cdc-agv", q) for q in range(p)]
    o = torch.zeros(sum(counts), device=dev)
    cx.rt.all_gatherv(b, Buffer(o), Buffer(to_dev(ins[r], DType.f32, dev)), counts, displs)
    cx.check("codec/all_gatherv", from_dev(o, DType.f32),
             seqref.all_gatherv(mine(ins), counts, displs)[r])
    root = p - 1
    o = torch.zeros(sum(counts), device=dev) if r == root else None
    cx.rt.gatherv(b, Buffer(o) if o is not None else None, Buffer(to_dev(ins[r], DType.f32, dev)),
                  root, counts, displs)
    if r == root:
        cx.check("codec/gatherv", from_dev(o, DType.f32),
                 seqref.gatherv(mine(ins), root, counts, displs)[root])
    src = values(DType.f32, sum(counts), "cdc-scv")
    o = torch.zeros(counts[r], device=dev)
    cx.rt.scatterv(b, Buffer(o), Buffer(to_dev(src, DType.f32, dev)) if r == 0 else None, 0,
                   counts, displs)
    cx.check("codec/scatterv", from_dev(o, DType.f32),
             seqref.scatterv(src if r == 0 else T(src), counts, displs)[r])
    for n in (1, 777, (3 << 20) + 1):
        ins = [values(DType.f32, n, "cdc-bc", n, q) for q in range(p)]
        t = to_dev(ins[r], DType.f32, dev)
        cx.rt.bcast(b, Buffer(t), 0)
        cx.check(f"codec/bcast/{n}", from_dev(t, DType.f32), ins[0] if r == 0 else T(ins[0]))
    # non-f32 payloads bypass the codec (exact)
    ins = [values(DType.i64, p * 999, "cdc-i64", q) for q in range(p)]
    o = torch.zeros(p * 999, dtype=torch.int64, device=dev)
    cx.rt.all_to_all_single(b, Buffer(o), Buffer(to_dev(ins[r], DType.i64, dev)))
    cx.check("codec/i64-bypass", from_dev(o, DType.i64), seqref.all_to_all_single(ins)[r])
    # reference-style numpy Buffers (staged) through the compressed kernel
    ins = [values(DType.f32, p * 4096, "cdc-np", q) for q in range(p)]
    hout = np.zeros(p * 4096, dtype=np.float32)
    cx.rt.all_to_all_single(b, Buffer(hout), Buffer(ins[r].copy()))
    cx.check("codec/numpy", hout, seqref.all_to_all_single(mine(ins))[r])
    # ranks disagreeing on the codec (rank 0 compresses on "cm"): CodecMismatch
    # with bulk-sized pairs (flag signatures) and, on a fresh backend, with
    # LL-sized pairs (LL header signatures)
    if p >= 2:
        for be, n in (("cm", p * 100_000), ("cm_ll", p * 1000)):
            x = torch.ones(n, device=dev)
            y = torch.zeros(n, device=dev)
            raised = None
            try:
                cx.rt.all_to_all_single(be, Buffer(y), Buffer(x), async_op=True)
                cx.rt.synchronize([be])
            except Exception as exc:  # noqa: BLE001
                raised = exc
            cx.checked += 1
            if type(raised).__name__ != "CodecMismatch":
                cx.failures.append(f"codec/mismatch/{n // p}: expected CodecMismatch, got {raised!r}")


def sc_commlog(cx: Ctx):
    """Every completed op appends one CommLog record with a DEVICE duration, as
    the reference logs every op (runtime.py:209-230): blocking device ops via
    deferred CUDA events on the caller's stream, async ops when their handle
    settles; report() aggregates the flushed per-rank log (middleware.py:
    174-215)."""
    import tempfile

    from paper_2303_08374_b200.middleware import report

    p, r, dev = cx.p, cx.r, cx.dev
    log = cx.rt.comm_log
    cx.rt.synchronize([cx.b])
    n0 = len(log.records())
    t = torch.ones(1 << 20, device=dev)
    cx.rt.all_reduce(cx.b, Buffer(t))                      # inline
    x = torch.ones(p * 4096, device=dev)
    y = torch.zeros_like(x)
    cx.rt.all_to_all_single(cx.b, Buffer(y), Buffer(x))    # inline
    h = cx.rt.all_reduce(cx.b, Buffer(torch.ones(4096, device=dev)), async_op=True)
    h.wait()
    cx.rt.synchronize([cx.b])
    recs = log.records()[n0:]
    cx.checked += 1
    ops = sorted(rec.op for rec in recs)
    if ops != sorted(["all_reduce", "all_to_all_single", "all_reduce"]):
        cx.failures.append(f"commlog: records {ops}")
    for rec in recs:
        # at p >= 2 every op runs a kernel that stamps its own device time:
        # the 0.001 us "no stamps" placeholder is a failure there
        floor = 0.0011 if p > 1 else 0.0
        if not (rec.dur_us > floor and rec.backend == cx.b and rec.rank == r):
            cx.failures.append(f"commlog: bad record {rec}")
        want_bytes = {"all_reduce": None, "all_to_all_single": p * 4096 * 4}.get(rec.op)
        if want_bytes is not None and rec.bytes != want_bytes:
            cx.failures.append(f"commlog: bytes {rec.bytes} != {want_bytes} for {rec.op}")
    with tempfile.TemporaryDirectory() as d:
        path = f"{d}/rank{r}.jsonl"
        log.flush(path)
        bd = report([path])
        cx.checked += 1
        rows = {(row.op, row.backend): row for row in bd.rows}
        if ("all_reduce", cx.b) not in rows or rows[("all_reduce", cx.b)].count < 2:
            cx.failures.append(f"commlog: report rows {bd.rows}")


# ------------------------------------------------------- BASELINE configs

def bits(dtype: DType, n: int, *seed) -> np.ndarray:
    """Seeded random BIT PATTERNS of `dtype` (movement parity: every pattern,
    NaN payloads included, must arrive unchanged)."""
    def make():
        rng = np.random.default_rng(seed_of("bits", *seed))
        w = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[dtype.size_bytes]
        return rng.integers(0, np.iinfo(w).max, size=n, dtype=w, endpoint=True).view(NP[dtype])
    if _MEMO is not None:
        return _MEMO.get(("b", dtype, n, seed), make)
    return make()


def dlrm_counts(p: int, skew: bool):
    """cfg4: 26 tables of dim 128 split over ranks like
    np.array_split, global batch 65536; uniform local batch B/p or Zipf(1.1)
    weights normalized to 65536 (remainder to the last rank).
    sc[i][j] = b_j * T_i * 128 elements rank i sends to rank j."""
    tables = [len(x) for x in np.array_split(np.arange(26), p)]
    B = 65536
    if skew:
        wz = [(j + 1) ** -1.1 for j in range(p)]
        b = [int(B * w / sum(wz)) for w in wz]
        b[-1] += B - sum(b)
    else:
        b = [B // p] * p
    return [[b[j] * tables[i] * 128 for j in range(p)] for i in range(p)], b


def _a2av_case(cx, name, dtype, sc, backend=None, devcounts=True):
    """all_to_allv with counts matrix sc (sc[i][j]: i -> j), packed displs;
    host counts and (optionally) device-resident counts, vs the oracle."""
    p, r = cx.p, cx.r
    b = backend or cx.b
    sd = [packed(row) for row in sc]
    rd = [packed([sc[j][q] for j in range(p)]) for q in range(p)]
    ins = [bits(dtype, sum(sc[q]), name, q) for q in range(p)]
    rc = [sc[j][r] for j in range(p)]
    want = seqref.all_to_allv_rank(ins, sc, sd, rd, r, sum(rc))
    i = to_dev(ins[r], dtype, cx.dev)
    o = torch.zeros(sum(rc), dtype=i.dtype, device=cx.dev)
    cx.rt.all_to_allv(b, Buffer(o), Buffer(i), sc[r], rc, sd[r], rd[r])
    cx.check(f"{name}/host-counts", from_dev(o, dtype), want)
    if devcounts:
        o.zero_()
        dc = [torch.tensor(v, dtype=torch.int64, device=cx.dev) for v in (sc[r], rc, sd[r], rd[r])]
        cx.rt.all_to_allv(b, Buffer(o), Buffer(i), dc[0], dc[1], dc[2], dc[3])
        cx.check(f"{name}/device-counts", from_dev(o, dtype), want)
    return i, o


def sc_baseline(cx: Ctx):
    """BASELINE.json configs 3-5 at full size through the public API, every
    output against the oracle: cfg3 DS-MoE token all_to_all,
    cfg4 DLRM all_to_allv (uniform + Zipf-skewed, host and device counts),
    cfg5 one mixed step incl. the fusion grouping of the 14 MLP gradients
    against the reference FusionManager's own grouping (tests/golden/
    cfg5_fusion.json, oracle/make_golden.py cfg5)."""
    p, r, dev = cx.p, cx.r, cx.dev
    # cfg3: 4096 tokens x 4096 hidden bf16 per rank, one expert per rank
    n = 4096 * 4096
    ins = [bits(DType.bf16, n, "cfg3", q) for q in range(p)]
    m = n // p
    want = np.concatenate([ins[j][r * m:(r + 1) * m] for j in range(p)])
    x = to_dev(ins[r], DType.bf16, dev)
    y = torch.zeros_like(x)
    cx.rt.all_to_all_single(cx.b, Buffer(y), Buffer(x))
    cx.check("cfg3/all_to_all_single", from_dev(y, DType.bf16), want)
    del x, y
    _a2av_case(cx, "cfg3/a2av-uniform", DType.bf16, [[m] * p for _ in range(p)])
    # cfg4: DLRM embedding all_to_allv, f32
    for skew in (False, True):
        sc, _b = dlrm_counts(p, skew)
        _a2av_case(cx, f"cfg4/{'skew' if skew else 'uniform'}", DType.f32, sc)
    # cfg5: one mixed step, replayed from its LogRecord-schema JSONL trace
    # (paper_2303_08374_b200.trace: written, read back, replayed through
    # Runtime), every output checked, and the fusion flush grouping compared
    # with the reference FusionManager's on the same posting order
    import tempfile

    from paper_2303_08374_b200 import trace as tr

    golden = json.loads((ROOT / "tests" / "golden" / "cfg5_fusion.json").read_text())
    with tempfile.TemporaryDirectory() as d:
        path = f"{d}/cfg5.jsonl"
        tr.write_jsonl(tr.cfg5_trace(p), path)
        recs = tr.load_jsonl(path)
    rp = tr.Replay(cx.rt, recs, r, dev, backend_map={"nvl": cx.b, "nvl_fused": "fused"})
    by_rank = {}
    for rec in recs:
        by_rank.setdefault(rec["rank"], []).append(rec)
    for v in by_rank.values():
        v.sort(key=lambda x: x["seq"])
    wants = []
    for i, ent in enumerate(rp.ops):
        dt = ent["dtype"]
        peers = [by_rank[q][i] for q in range(p)]
        if ent["op"] == "all_to_allv":
            scm = [[int(x) for x in pr["scounts"]] for pr in peers]
            ins = [bits(dt, sum(scm[q]), "cfg5", i, q) for q in range(p)]
            want = seqref.all_to_allv_rank(ins, scm, [packed(x) for x in scm],
                                           [packed([scm[j][q] for j in range(p)]) for q in range(p)],
                                           r, sum(ent["rc"]))
            ent["inp"].copy_(to_dev(ins[r], dt, dev))
            wants.append((ent["out"], want, False))
        elif ent["op"] == "all_reduce":
            ins = [values(dt, ent["buf"].numel(), "cfg5", i, q) for q in range(p)]
            ent["buf"].copy_(to_dev(ins[r], dt, dev))
            wants.append((ent["buf"], seqref.fold(ins, "sum"), False))
        else:
            rc = ent["rc"]
            ins = [values(dt, rc[q], "cfg5", i, q) for q in range(p)]
            ent["inp"].copy_(to_dev(ins[r], dt, dev))
            if ent["op"] == "all_gatherv":
                wants.append((ent["out"], seqref.all_gatherv(ins, rc, ent["dp"])[r], False))
            elif r == ent["root"]:
                wants.append((ent["out"], seqref.gatherv(ins, ent["root"], rc, ent["dp"])[r], False))
    cx.sync()
    cx.rt.synchronize([cx.b, "fused"])
    n0 = len(cx.rt.comm_log.records())
    rp.step()
    cx.rt.synchronize([cx.b, "fused"])
    for k, (got, want, _) in enumerate(wants):
        dt = DType.i64 if got.dtype == torch.int64 else DType.f32
        cx.check(f"cfg5/trace-replay/{k}", from_dev(got, dt), want)
    recs_log = sorted((x for x in cx.rt.comm_log.records()[n0:] if x.backend == "fused"),
                      key=lambda x: x.seq)
    got = [x.members for x in recs_log if x.fused]
    unfused = sum(1 for x in recs_log if not x.fused)
    cx.checked += 1
    if got != golden["flush_members"] or unfused != golden["unfused_records"]:
        cx.failures.append(f"cfg5/fusion grouping: flushes {got} (+{unfused} unfused) vs reference "
                           f"{golden['flush_members']} (+{golden['unfused_records']})")


def _ints_f32(n: int, q: int) -> np.ndarray:
    """Small-integer f32 values: every partial sum is exact, so any summation
    order (ascending fold, NVLS switch order) gives the same bits."""
    i = np.arange(n, dtype=np.int64)
    return (((i * 31 + q * 17) % 29) - 14).astype(np.float32)


def sc_large(cx: Ctx):
    """all_reduce at the sizes AUTO sends to the large-message kernels:
    256 MiB f32 / bf16 (two-shot with TMA bulk senders for aligned buffers,
    NVLS at p >= 4 where the switch exists) and 1 GiB f32 (several launches
    through the workspace / NVLS halves), against the oracle. 1 GiB uses
    exactly-summable integer values (any reduction order is bit-exact)."""
    p, r, dev = cx.p, cx.r, cx.dev
    inst = cx.rt._instance(cx.b)
    nvls = bool(inst.comm.caps.nvls_supported)
    n = (256 << 20) // 4
    ins = [values(DType.f32, n, "large-f32", q) for q in range(p)]
    t = to_dev(ins[r], DType.f32, dev)
    cx.rt.all_reduce(cx.b, Buffer(t))
    cx.check("large/f32/256MiB", from_dev(t, DType.f32), seqref.fold(ins, "sum"),
             float_reduction=ran_nvls(cx), rtol=1e-5)
    del t
    # misaligned by one element: the same share geometry, LD/ST senders
    base = torch.zeros(n + 1, device=dev)
    t = base[1:]
    t.copy_(torch.from_numpy(ins[r].copy()))
    cx.rt.all_reduce(cx.b, Buffer(t))
    cx.check("large/f32/256MiB-misaligned", from_dev(t, DType.f32), seqref.fold(ins, "sum"),
             float_reduction=ran_nvls(cx), rtol=1e-5)
    del t, base, ins
    nb = (256 << 20) // 2
    ins = [values(DType.bf16, nb, "large-bf16", q) for q in range(p)]
    t = to_dev(ins[r], DType.bf16, dev)
    cx.rt.all_reduce(cx.b, Buffer(t))
    if ran_nvls(cx):
        cx.check("large/bf16/256MiB", seqref.bf16_bits_to_f32(from_dev(t, DType.bf16)),
                 seqref.bf16_bits_to_f32(seqref.fold_bf16(ins, "sum")), float_reduction=True,
                 rtol=1e-2)
    else:
        cx.check("large/bf16/256MiB", from_dev(t, DType.bf16), seqref.fold_bf16(ins, "sum"))
    del t, ins
    if p <= 4:
        n = (1 << 30) // 4
        t = torch.from_numpy(_ints_f32(n, r)).to(dev)
        cx.rt.all_reduce(cx.b, Buffer(t))
        acc = _ints_f32(n, 0)
        for q in range(1, p):
            acc += _ints_f32(n, q)
        cx.check("large/f32/1GiB", from_dev(t, DType.f32), acc)
        del t, acc


def sc_tuning(cx: Ctx):
    """The tuning table drives AUTO (mcrdl_comm_set_tuning): editing the
    table's all_reduce cell changes the kernel the C layer launches, results
    stay bit-exact, and restoring the shipped table restores its choice."""
    from paper_2303_08374_b200.dispatch import TuningTable

    p, r, dev = cx.p, cx.r, cx.dev
    inst = cx.rt._instance(cx.b)
    if p < 2:
        return
    for algo in ("two_shot", "one_shot", "two_shot"):
        t = TuningTable.from_dict({"tables": {"all_reduce": {str(p): [
            {"max_bytes": 1 << 40, "backend": "nvl", "algorithm": algo}]}}})
        inst.install_tuning(t)
        for n in (1000, 300_001):
            ins = [values(DType.f32, n, "tune", algo, n, q) for q in range(p)]
            x = to_dev(ins[r], DType.f32, dev)
            cx.rt.all_reduce(cx.b, Buffer(x))
            cx.check(f"tuning/{algo}/{n}", from_dev(x, DType.f32), seqref.fold(ins, "sum"))
            got = inst.last_algorithm(CommOpKind.all_reduce)
            cx.checked += 1
            if got != algo:
                cx.failures.append(f"tuning: table says {algo} for {n} f32, C layer ran {got}")
    inst.install_tuning(cx.rt.algorithm_table)
    rows = inst.tuning_rows[CommOpKind.all_reduce]
    if rows:
        x = torch.ones(1000, device=dev)
        cx.rt.all_reduce(cx.b, Buffer(x))
        cx.checked += 1
        if inst.last_algorithm(CommOpKind.all_reduce) != rows[0][1]:
            cx.failures.append(f"tuning: shipped table row {rows[0]} not applied")


A3_KINDS = ("all_reduce", "all_gather", "bcast", "all_to_all_single", "reduce_scatter")


def sc_a3(cx: Ctx):
    """Reference acceptance A3 (test_acceptance.py:160-243) on the device:
    seeded mixed programs of 3-8 ASYNC collectives spread over two backends,
    waited for in a shuffled order, then synchronize; every result checked
    against the oracle and every program bounded in time (no deadlock). Then
    injected order mismatches: one rank posts bcast where the others post
    all_reduce at the same sequence number -> every rank raises OrderMismatch
    (the device restatement of the header agreement, collectives.py:178-285),
    none hangs."""
    import random
    import time

    p, r, dev = cx.p, cx.r, cx.dev
    n_programs = int(os.environ.get("MCRDL_A3_PROGRAMS", "200"))
    slow = []
    for seed in range(n_programs):
        rng = random.Random(seed)
        ops = [(rng.choice(A3_KINDS), rng.choice(["a3a", "a3b"]), rng.choice([1, 4, 32]),
                seed * 1000 + i) for i in range(rng.randint(3, 8))]
        order = list(range(len(ops)))
        rng.shuffle(order)
        t0 = time.monotonic()
        hs, checks = [], []
        for kind, be, c, sd in ops:
            if kind == "all_reduce":
                ins = [values(DType.i64, c, "a3", sd, q) for q in range(p)]
                t = to_dev(ins[r], DType.i64, dev)
                hs.append(cx.rt.all_reduce(be, Buffer(t), async_op=True))
                checks.append((t, seqref.fold(ins, "sum")))
            elif kind == "all_gather":
                ins = [values(DType.i64, c, "a3", sd, q) for q in range(p)]
                o = torch.zeros(p * c, dtype=torch.int64, device=dev)
                hs.append(cx.rt.all_gather(be, Buffer(o), Buffer(to_dev(ins[r], DType.i64, dev)),
                                           async_op=True))
                checks.append((o, seqref.all_gather(ins)[r]))
            elif kind == "bcast":
                root = sd % p
                ins = [values(DType.i64, c, "a3", sd, q) for q in range(p)]
                t = to_dev(ins[r], DType.i64, dev)
                hs.append(cx.rt.bcast(be, Buffer(t), root, async_op=True))
                checks.append((t, ins[root]))
            elif kind == "all_to_all_single":
                ins = [values(DType.i64, p * c, "a3", sd, q) for q in range(p)]
                o = torch.zeros(p * c, dtype=torch.int64, device=dev)
                hs.append(cx.rt.all_to_all_single(be, Buffer(o), Buffer(to_dev(ins[r], DType.i64, dev)),
                                                  async_op=True))
                checks.append((o, seqref.all_to_all_single(ins)[r]))
            else:
                ins = [values(DType.i64, p * c, "a3", sd, q) for q in range(p)]
                o = torch.zeros(c, dtype=torch.int64, device=dev)
                hs.append(cx.rt.reduce_scatter(be, Buffer(o), Buffer(to_dev(ins[r], DType.i64, dev)),
                                               async_op=True))
                checks.append((o, seqref.reduce_scatter(ins, "sum")[r]))
        for idx in order:
            cx.rt.wait(hs[idx])
        cx.rt.synchronize(["a3a", "a3b"])
        if time.monotonic() - t0 > 10.0:
            slow.append(seed)
        for k, (got, want) in enumerate(checks):
            cx.check(f"a3/program{seed}/op{k}/{ops[k][0]}", from_dev(got, DType.i64), want)
    cx.checked += 1
    if slow:
        cx.failures.append(f"a3: programs over the 10 s budget: {slow[:10]}")
    if p < 2:
        return
    for trial in range(5):  # injected mismatches, one fresh backend per trial
        be = f"inj{trial}"
        victim = trial % p
        buf = torch.ones(1, device=dev)
        raised = None
        t0 = time.monotonic()
        try:
            if r == victim:
                cx.rt.bcast(be, Buffer(buf), victim, async_op=True)
            else:
                cx.rt.all_reduce(be, Buffer(buf), async_op=True)
            cx.rt.synchronize([be])
        except Exception as exc:  # noqa: BLE001
            raised = exc
        cx.checked += 1
        if type(raised).__name__ != "OrderMismatch":
            cx.failures.append(f"a3/injection{trial}: expected OrderMismatch, got {raised!r}")
        elif time.monotonic() - t0 > 30.0:
            cx.failures.append(f"a3/injection{trial}: verdict took {time.monotonic() - t0:.1f} s")


def sc_pool(cx: Ctx):
    """Runtime.symmetric_pool: ordinary torch tensors allocated in the
    symmetric MemPool (csrc/pool.cu via torch's pluggable allocator) take the
    zero-copy kernels — all_reduce in and out of place (k_ar_symm: NVLS
    multimem where a switch exists, else peer loads), all_to_all_single into a
    pool output (k_x_symm direct writes) — checked against the oracle."""
    p, r, dev = cx.p, cx.r, cx.dev
    pool = cx.rt.symmetric_pool(cx.b, 256 << 20)
    inst = cx.rt._instance(cx.b)
    n = (12 << 20) // 4 + 7  # above the zero-copy threshold (8 MiB at p = 2)
    ins = [values(DType.f32, n, "pool", q) for q in range(p)]
    m = (6 << 20) // 4  # 6 MiB per pair: inside the direct-write window
    a2a = [values(DType.i64, p * m // 2, "pool-a2a", q) for q in range(p)]
    with torch.cuda.use_mem_pool(pool):
        x = torch.empty(n, device=dev)
        y = torch.empty(n, device=dev)
        ai = torch.empty(p * m // 2, dtype=torch.int64, device=dev)
        ao = torch.empty_like(ai)
    x.copy_(torch.from_numpy(ins[r].copy()))
    ai.copy_(torch.from_numpy(a2a[r].copy()))
    cx.rt.post(CommRequest(CommOpKind.all_reduce, input=Buffer(x), output=Buffer(y),
                           op=ReduceOp.sum, backend=cx.b))
    algo = inst.last_algorithm(CommOpKind.all_reduce)
    cx.check("pool/all_reduce/out", from_dev(y, DType.f32), seqref.fold(ins, "sum"),
             float_reduction=algo == "nvls", rtol=1e-5)
    cx.checked += 1
    if p > 1 and algo not in ("nvls", "direct_write"):
        cx.failures.append(f"pool: all_reduce on pool tensors ran {algo}, not the zero-copy kernel")
    cx.rt.all_reduce(cx.b, Buffer(x))
    cx.check("pool/all_reduce/in", from_dev(x, DType.f32), seqref.fold(ins, "sum"),
             float_reduction=inst.last_algorithm(CommOpKind.all_reduce) == "nvls", rtol=1e-5)
    cx.rt.all_to_all_single(cx.b, Buffer(ao), Buffer(ai))
    cx.check("pool/a2a_single", from_dev(ao, DType.i64), seqref.all_to_all_single(a2a)[r])
    del x, y, ai, ao


def sc_smoke(cx: Ctx):
    """One small invocation of each hot-path family (smoke()): LL, one-shot
    and two-shot all_reduce (explicit algorithms: at p = 1 too they run their
    real kernels), all_to_allv with host and with device-resident counts, and
    (p > 1) the chain bcast and all_gatherv with device-resident counts."""
    p, r = cx.p, cx.r
    inst = cx.rt._instance(cx.b)
    for algo, n in (("one_shot", 1000), ("one_shot", 70001), ("two_shot", 70001)):
        ins = [values(DType.f32, n, "smoke", algo, n, q) for q in range(p)]
        t = to_dev(ins[r], DType.f32, cx.dev)
        inst.policy = AlgorithmPolicy({CommOpKind.all_reduce: algo})
        cx.rt.all_reduce(cx.b, Buffer(t))
        cx.check(f"smoke/all_reduce/{algo}/{n}", from_dev(t, DType.f32), seqref.fold(ins, "sum"))
    inst.policy = AlgorithmPolicy()
    sc = counts_matrix(p, 5000, "smoke-a2av")
    _a2av_case(cx, "smoke/all_to_allv", DType.bf16, sc)
    if p > 1:
        # pipelined chain bcast and all_gatherv with GPU-resident counts
        n = 300007
        ins = [values(DType.u8, n, "smoke-chain", q) for q in range(p)]
        t = to_dev(ins[r], DType.u8, cx.dev)
        inst.policy = AlgorithmPolicy({CommOpKind.bcast: "chain"})
        cx.rt.bcast(cx.b, Buffer(t), p - 1)
        inst.policy = AlgorithmPolicy()
        cx.check("smoke/bcast/chain", from_dev(t, DType.u8), ins[p - 1])
        counts = [1000 + 37 * q for q in range(p)]
        displs = packed(counts)
        ins = [values(DType.i64, counts[q], "smoke-agv", q) for q in range(p)]
        o = torch.zeros(sum(counts), dtype=torch.int64, device=cx.dev)
        cx.rt.all_gatherv(cx.b, Buffer(o), Buffer(to_dev(ins[r], DType.i64, cx.dev)),
                          torch.tensor(counts, dtype=torch.int64, device=cx.dev),
                          torch.tensor(displs, dtype=torch.int64, device=cx.dev))
        cx.check("smoke/all_gatherv_dev", from_dev(o, DType.i64),
                 seqref.all_gatherv(ins, counts, displs)[r])


def sc_golden(cx: Ctx):
    """Replay the reference's own selftest parity dump (tests/golden/
    selftest_p{p}.json, produced by `mcrdl launch -n p selftest --out`) and
    the live-algorithm fixtures for this world size through the nvlink
    backend; outputs must equal the reference's recorded outputs bit-exactly."""
    import golden_cases as gc

    p, r = cx.p, cx.r
    dev = cx.dev

    def T(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    for case in gc.load_selftest(p):
        op, dt = case["op"], gc.NPD[case["dtype"]]
        root, count = case["root"], case["count"]
        want = case["expected"][r]
        name = f"golden/p{p}/{op}/{case['dtype']}/{count}"
        ins = gc.selftest_arrays(case, "inputs") if "inputs" in case else None
        got = None
        if op == "all_reduce":
            t = T(ins[r])
            cx.rt.all_reduce(cx.b, Buffer(t))
            got = t
        elif op == "reduce":
            t = T(ins[r])
            cx.rt.reduce(cx.b, Buffer(t), root)
            got = t if r == root else None
        elif op == "bcast":
            t = T(ins[r])
            cx.rt.bcast(cx.b, Buffer(t), root)
            got = t
        elif op == "all_gather":
            o = torch.zeros(p * count, dtype=T(ins[r]).dtype, device=dev)
            cx.rt.all_gather(cx.b, Buffer(o), Buffer(T(ins[r])))
            got = o
        elif op == "gather":
            i = T(ins[r])
            o = torch.zeros(p * count, dtype=i.dtype, device=dev) if r == root else None
            cx.rt.gather(cx.b, Buffer(o) if o is not None else None, Buffer(i), root)
            got = o
        elif op == "scatter":
            src = T(np.asarray(case["root_input"], dtype=dt))
            o = torch.zeros(count, dtype=src.dtype, device=dev)
            cx.rt.scatter(cx.b, Buffer(o), Buffer(src) if r == root else None, root)
            got = o
        elif op == "reduce_scatter":
            i = T(ins[r])
            o = torch.zeros(count, dtype=i.dtype, device=dev)
            cx.rt.reduce_scatter(cx.b, Buffer(o), Buffer(i))
            got = o
        elif op == "all_to_all_single":
            i = T(ins[r])
            o = torch.zeros_like(i)
            cx.rt.all_to_all_single(cx.b, Buffer(o), Buffer(i))
            got = o
        elif op == "all_to_all":
            x = ins[r]
            inb = [Buffer(T(x[j * count:(j + 1) * count])) for j in range(p)]
            outb = [Buffer(torch.zeros(count, dtype=inb[0].array.dtype, device=dev))
                    for _ in range(p)]
            cx.rt.all_to_all(cx.b, outb, inb)
            got = torch.cat([b.array for b in outb]) if count else torch.zeros(0, device=dev)
        elif op in ("gatherv", "all_gatherv"):
            rc, dp = case["rcounts"], case["displs"]
            i = T(ins[r])
            if op == "all_gatherv":
                o = torch.zeros(sum(rc), dtype=i.dtype, device=dev)
                cx.rt.all_gatherv(cx.b, Buffer(o), Buffer(i), rc, dp)
                got = o
            else:
                o = torch.zeros(sum(rc), dtype=i.dtype, device=dev) if r == root else None
                cx.rt.gatherv(cx.b, Buffer(o) if o is not None else None, Buffer(i), root, rc, dp)
                got = o
        elif op == "scatterv":
            sc, dp = case["scounts"], case["displs"]
            src = T(np.asarray(case["root_input"], dtype=dt))
            o = torch.zeros(sc[r], dtype=src.dtype, device=dev)
            cx.rt.scatterv(cx.b, Buffer(o), Buffer(src) if r == root else None, root, sc, dp)
            got = o
        elif op == "all_to_allv":
            sc, sd, rd = case["scounts"], case["sdispls"], case["rdispls"]
            rc = [sc[j][r] for j in range(p)]
            i = T(ins[r])
            o = torch.zeros(sum(rc), dtype=i.dtype, device=dev)
            cx.rt.all_to_allv(cx.b, Buffer(o), Buffer(i), sc[r], rc, sd[r], rd[r])
            got = o
        if got is None:
            continue
        # the selftest dump holds the reference's DEFAULT (ring) results: float
        # reductions agree to the reference tolerance (cases.py:232-236), the
        # ascending fold is pinned bit-exactly by the live naive cases
        fred = op in ("all_reduce", "reduce", "reduce_scatter") and np.dtype(dt).kind == "f"
        cx.check(name, got.cpu().numpy().astype(dt), np.asarray(want, dtype=dt),
                 float_reduction=fred, rtol=1e-5)


SCENARIOS = {
    "golden": sc_golden,
    "smoke": sc_smoke,
    "all_reduce": sc_all_reduce,
    "all_to_allv": sc_all_to_allv,
    "all_to_all": sc_all_to_all,
    "gathers": sc_gathers,
    "bcast_scatter": sc_bcast_scatter,
    "reduce_family": sc_reduce_family,
    "host_buffers": sc_host_buffers,
    "async_fusion": sc_async_and_fusion,
    "graphs": sc_graphs,
    "p2p": sc_p2p,
    "symm": sc_symm,
    "codec": sc_codec,
    "commlog": sc_commlog,
    "order_mismatch": sc_order_mismatch,
    "baseline": sc_baseline,
    "large": sc_large,
    "tuning": sc_tuning,
    "a3": sc_a3,
    "pool": sc_pool,
}


def run_rank(rank: int, world: int, device: int, report: str, names, shared=None) -> int:
    torch.cuda.set_device(device)
    out = {"rank": rank, "failures": [], "checked": 0}
    rt = Runtime(rank=rank, world_size=world)
    rt.local_device = device
    if shared is not None:
        # Co-located rank: exactly two streams (issue + lane), made up front
        # in rank order so the ranks' streams land on distinct hardware queues
        # (a stream sharing a queue with a peer's blocked stream can stall
        # behind it); the legacy default stream would serialize the ranks.
        issue, lane = shared.streams[rank]
        torch.cuda.set_stream(issue)
        rt.lane_stream = lane
        rt.launch_hook = shared.rendezvous
    cx = None
    try:
        cfgs = [BackendConfig("nvl"), BackendConfig("fused", fusion=FusionConfig(max_bytes=1 << 20,
                                                                               max_wait=5.0))]
        if "order_mismatch" in names:
            cfgs.append(BackendConfig("mism", workspace_bytes=8 << 20))
        if "async_fusion" in names:
            cfgs.append(BackendConfig("fused_big", workspace_bytes=4 << 20,
                                      fusion=FusionConfig(max_bytes=2 << 20, max_wait=5.0)))
        if "a3" in names:
            cfgs += [BackendConfig("a3a", workspace_bytes=8 << 20),
                     BackendConfig("a3b", workspace_bytes=8 << 20)]
            cfgs += [BackendConfig(f"inj{k}", workspace_bytes=4 << 20) for k in range(5)]
        if "all_to_allv" in names:
            cfgs.append(BackendConfig("small", workspace_bytes=16 << 20))
        if "bcast_scatter" in names:
            cfgs.append(BackendConfig("bsmall", workspace_bytes=8 << 20))
        if "p2p" in names:
            cfgs.append(BackendConfig("lenm", workspace_bytes=8 << 20))
        if "codec" in names:
            # small workspace: large pairs move in several acknowledged rounds
            cfgs.append(BackendConfig("cmp", workspace_bytes=16 << 20,
                                      compression=CompressionConfig()))
            # "cm": only rank 0 compresses -> CodecMismatch on every rank
            cfgs.append(BackendConfig("cm", workspace_bytes=64 << 20,
                                      compression=CompressionConfig() if rank == 0 else None))
            cfgs.append(BackendConfig("cm_ll", workspace_bytes=16 << 20,
                                      compression=CompressionConfig() if rank == 0 else None))
        rt.init(cfgs)
        cx = Ctx(rt, "nvl", shared)
        out["colocated"] = int(rt._instance("nvl").comm.caps.ranks_per_device)
        out["num_sms"] = int(rt._instance("nvl").comm.caps.num_sms)
        for name in names:
            try:
                SCENARIOS[name](cx)
            except Exception:  # noqa: BLE001
                cx.failures.append(f"{name}: exception\n{traceback.format_exc()[-3000:]}")
        cx.sync()
        try:
            rt.synchronize([b for b in ("nvl", "fused", "fused_big") if b in rt.get_backends()])
        except Exception as exc:  # noqa: BLE001
            cx.failures.append(f"synchronize: {exc!r}")
        out["failures"] = cx.failures
        out["checked"] = cx.checked
        if cx.failures:  # what each rank ran last (compare ranks on a failure)
            out["log_tail"] = [[x.backend, x.op, x.bytes, x.seq, x.algorithm]
                               for x in rt.comm_log.records()[-40:]]
        out["nvls"] = getattr(cx, "nvls", None)
        out["launches"] = _lib.launch_count()
    except Exception:  # noqa: BLE001
        out["failures"].append("init/run: " + traceback.format_exc()[-3000:])
    finally:
        Path(report).write_text(json.dumps(out))
        if shared is not None:
            try:  # every rank done before any communicator is torn down
                shared.barrier.wait(shared.timeout)
            except threading.BrokenBarrierError:
                pass
        try:
            rt.close()
        except Exception:  # noqa: BLE001
            pass
    return 0 if not out["failures"] else 1


def main() -> int:
    global _MEMO
    if sys.argv[1] == "--threads":
        world = int(sys.argv[2])
        rdir = Path(sys.argv[3])
        names = sys.argv[4].split(",") if len(sys.argv) > 4 else [s for s in SCENARIOS if s != "smoke"]
        device = int(os.environ.get("MCRDL_COLOCATED_DEVICE", "0"))
        dump = float(os.environ.get("MCRDL_WORKER_DUMP_SECS", "0"))
        if dump > 0:  # periodic all-thread stack dumps (hang diagnosis)
            import faulthandler

            faulthandler.dump_traceback_later(dump, repeat=True)
        _MEMO = _Memo()
        shared = Shared(world, timeout=float(os.environ.get("MCRDL_THREAD_TIMEOUT", "600")))
        torch.cuda.set_device(device)
        torch.empty(1, device=f"cuda:{device}")  # primary context current in this thread
        shared.streams = [(_raw_stream(device), _raw_stream(device)) for _ in range(world)]
        rcs = [1] * world

        def body(r):
            rcs[r] = run_rank(r, world, device, str(rdir / f"r{r}.json"), names, shared)

        threads = [threading.Thread(target=body, args=(r,), name=f"rank{r}") for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        return 0 if not any(rcs) else 1
    report = sys.argv[1]
    names = sys.argv[2].split(",") if len(sys.argv) > 2 else [s for s in SCENARIOS if s != "smoke"]
    rank = int(os.environ["RANK"])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return run_rank(rank, world, int(os.environ.get("LOCAL_RANK", rank)), report, names)


if __name__ == "__main__":
    sys.exit(main())

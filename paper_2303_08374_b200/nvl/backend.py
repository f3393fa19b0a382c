"""The NVLink/NVSwitch backend: one communicator per backend id, one lane
CUDA stream, and a C-ABI call per collective.

Reference seam: ``BackendConfig.transport`` ->
``Runtime._build_transport`` (runtime.py:359-383) and
``BackendInstance.post/_process/execute`` (runtime.py:142-277). The
reference's lane THREAD becomes a lane STREAM ("records a CUDA
event e onto the communication stream"); its inline fast path (runtime.py:
150-168) is the default here because a post only enqueues device work.

Buffers that are CUDA tensors run zero-copy. Host buffers (numpy, as in the
reference) are staged through pinned memory on the lane stream and copied
back when the handle settles. There is no host/CPU execution path: if the
native library or a CUDA device is missing, init raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
from ctypes import byref, c_void_p
from typing import List, Optional, Sequence

import numpy as np

from ..collectives import ALGO_CODES, AlgorithmPolicy, canonical
from ..core import (P2P_KINDS, Buffer, CommOpKind, CommRequest, CompletionEvent, DType, HandleState,
                    WorkHandle)
from ..dispatch import message_bytes
from ..errors import (BackendFinalized, CommError, NativeBackendMissing, PendingAfterTimeout,
                      UnsupportedOperation, ValidationError)
from . import _lib
from .bootstrap import StoreBootstrap, make_store

try:
    import torch
except Exception:  # pragma: no cover
    torch = None  # type: ignore[assignment]


class NvlComm:
    """Owner of one native communicator (symmetric workspace + signal pads)."""

    def __init__(self, rank: int, world: int, device: int, bootstrap: Optional[StoreBootstrap],
                 workspace_bytes: int, timeout: float):
        self.lib = _lib.load()
        self.rank, self.world, self.device = rank, world, device
        self._bootstrap = bootstrap  # keeps the ctypes callback alive
        handle = c_void_p()
        cb = bootstrap.c_callback if bootstrap is not None else ctypes.cast(None, _lib.ALLGATHER_FN)
        _lib.check(self.lib.mcrdl_comm_init(byref(handle), rank, world, device, cb, None,
                                            int(workspace_bytes), float(timeout)))
        self.handle = handle
        caps = _lib.Caps()
        _lib.check(self.lib.mcrdl_comm_caps(handle, byref(caps)))
        self.caps = caps

    def status(self) -> None:
        _lib.check(self.lib.mcrdl_comm_status(self.handle))

    def stream(self, which: int):
        """One of the communicator's own CUDA streams as a torch stream
        (0: lane, 1: H2D staging, 2: D2H staging)."""
        raw = c_void_p()
        _lib.check(self.lib.mcrdl_comm_stream(self.handle, int(which), byref(raw)))
        return torch.cuda.ExternalStream(int(raw.value), device=self.device)

    def symm_alloc(self, nbytes: int) -> int:
        """Collective: a peer-mapped (and, with NVLS, multicast-bound) device
        allocation of `nbytes` on every rank; returns this rank's pointer."""
        ptr = c_void_p()
        _lib.check(self.lib.mcrdl_symm_alloc(self.handle, int(nbytes), byref(ptr)))
        return int(ptr.value)

    def destroy(self) -> None:
        if self.handle:
            self.lib.mcrdl_comm_destroy(self.handle)
            self.handle = c_void_p()


class _CudaBlock:
    """__cuda_array_interface__ view of raw device bytes (zero-copy torch wrap)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class _PinnedPool:
    """Reusable pinned host staging buffers (cudaHostAlloc is milliseconds per
    call at hundreds of MiB; allocating per op would dominate host-buffer ops)."""

    def __init__(self):
        self._free: dict = {}
        self._lock = threading.Lock()

    def get(self, numel: int, dtype):
        key = (numel, dtype)
        with self._lock:
            lst = self._free.get(key)
            if lst:
                return lst.pop()
        return torch.empty(numel, dtype=dtype, pin_memory=True)

    def put(self, t) -> None:
        with self._lock:
            self._free.setdefault((t.numel(), t.dtype), []).append(t)


class _Staging:
    """Maps request Buffers to device tensors for one op on the lane stream.
    Host buffers: pinned torch tensors are copied directly (H2D/D2H, async);
    numpy arrays go through pooled pinned staging and are copied back when the
    handle settles."""

    def __init__(self, device, stream, pool: _PinnedPool):
        self.device = device
        self.stream = stream
        self.pool = pool
        self.keep: list = []
        self.copy_back: list = []  # (Buffer, pinned staging or None, device tensor)
        self._staged: list = []    # pooled pinned tensors to return at finish
        self._cache = {}

    def dev(self, buf: Optional[Buffer], *, upload: bool = True, download: bool = False):
        if buf is None:
            return None
        key = id(buf)
        if key in self._cache:
            t = self._cache[key]
            if download and not any(entry[0] is buf for entry in self.copy_back):
                self._download(buf, t)
            return t
        if buf.is_device:
            t = buf.array
            if t.device.index != self.device:
                raise ValidationError("buffer", f"tensor on cuda:{t.device.index}, backend uses "
                                      f"cuda:{self.device}")
            t.record_stream(self.stream)
        else:
            host = buf.array if buf.is_tensor else torch.from_numpy(buf.array)
            t = torch.empty(host.shape[0], dtype=host.dtype, device=self.device)
            if upload and host.shape[0]:
                if host.is_pinned():
                    src = host
                else:
                    src = self.pool.get(host.shape[0], host.dtype)
                    src.copy_(host)
                    self._staged.append(src)
                t.copy_(src, non_blocking=True)
                self.keep.append(host)
            if download:
                self._download(buf, t)
        self._cache[key] = t
        return t

    def _download(self, buf: Buffer, t) -> None:
        if buf.is_device:
            return
        if buf.is_tensor and buf.array.is_pinned():
            self.copy_back.append((buf, None, t))  # D2H straight into the caller's pinned tensor
        else:
            pinned = self.pool.get(t.shape[0], t.dtype)
            self._staged.append(pinned)
            self.copy_back.append((buf, pinned, t))

    def issue_downloads(self) -> None:
        for buf, pinned, t in self.copy_back:
            if t.shape[0]:
                (buf.array if pinned is None else pinned).copy_(t, non_blocking=True)

    def scratch(self, count: int, dtype: DType):
        return torch.empty(max(count, 0), dtype=dtype.torch_dtype, device=self.device)

    def finish(self) -> None:
        for buf, pinned, _t in self.copy_back:
            if pinned is None:
                continue
            if buf.is_tensor:
                buf.array.copy_(pinned)
            else:
                np.copyto(buf.array, pinned.numpy())
        self.copy_back.clear()
        self.keep.clear()
        for p in self._staged:
            self.pool.put(p)
        self._staged.clear()


class _Direct:
    """Staging for the inline path: device tensors used in place on the
    caller's stream (no record_stream, no copies)."""

    __slots__ = ("device", "keep")

    def __init__(self, device):
        self.device = device
        self.keep: list = []

    def dev(self, buf: Optional[Buffer], *, upload: bool = True, download: bool = False):
        if buf is None:
            return None
        t = buf.array
        if t.device.index != self.device:
            raise ValidationError("buffer", f"tensor on cuda:{t.device.index}, backend uses "
                                  f"cuda:{self.device}")
        return t

    def scratch(self, count: int, dtype: DType):
        return torch.empty(max(count, 0), dtype=dtype.torch_dtype, device=self.device)


def _raw_stream(device: int) -> int:
    return int(torch._C._cuda_getCurrentRawStream(device))


def _ptr(t) -> Optional[int]:
    return None if t is None else (int(t.data_ptr()) or None)


class NvlBackendInstance:
    """A registered ``transport="nvlink"`` backend."""

    transport_name = "nvlink"

    def __init__(self, config, runtime):
        if torch is None or not torch.cuda.is_available():
            raise NativeBackendMissing(
                "the nvlink transport needs a CUDA device (B200); no CPU fallback exists")
        _lib.load()
        # CompressionConfig (middleware.py:78-95): the trunc16 codec runs inside
        # the exchange kernel (MCRDL_CODEC_TRUNC16), halving NVLink bytes for f32.
        self.compression = getattr(config, "compression", None)
        self.config = config
        self.name = config.name
        self.runtime = runtime
        self.policy: AlgorithmPolicy = config.policy or AlgorithmPolicy()
        self.state = "initialized"
        self.collectives_executed = 0
        self._seq = 0
        self._lock = threading.RLock()  # one host thread at a time per communicator
        self._pending: List[WorkHandle] = []
        self._errors: List[BaseException] = []
        self._last_raw: Optional[int] = None  # stream of the most recent op
        self._pool = _PinnedPool()
        self._symm_keep: list = []  # symmetric allocations (freed with the communicator)
        self._pools: list = []  # (mcrdl_pool handle, torch MemPool)
        self._log_pending: list = []  # (request, first log id, last log id) of inline ops
        n_dev = torch.cuda.device_count()
        dev = config.device if config.device is not None else runtime.local_device
        if dev is None:
            dev = runtime.rank % max(n_dev, 1)
        self.device = int(dev)
        torch.cuda.set_device(self.device)
        boot = None
        if runtime.world_size > 1:
            store = runtime._control_store(config)
            boot = StoreBootstrap(runtime.rank, runtime.world_size, store,
                                  prefix=f"mcrdl-nvl/{self.name}/{runtime._init_generation}")
        ws = config.workspace_bytes or runtime.default_workspace_bytes
        self.comm = NvlComm(runtime.rank, runtime.world_size, self.device, boot, ws,
                            runtime.timeout)
        # Lane = the communicator's own stream (not one from torch's
        # round-robin pool, which hands the same stream to several callers).
        self._lane = None  # created on first async post (see the stream property)
        self.tuning_rows = {}
        self.install_tuning(runtime.algorithm_table)

    @property
    def stream(self):
        """The progress lane (reference: the backend's lane thread,
        runtime.py:117-126): Runtime.lane_stream when the host set one (one
        lane for all of a rank's backends, e.g. co-located ranks), else the
        communicator's own stream, created on first use."""
        if self._lane is None:
            self._lane = self.runtime.lane_stream or self.comm.stream(0)
        return self._lane

    # ------------------------------------------------------------ tuning
    TUNE_KINDS = {CommOpKind.all_reduce: 0, CommOpKind.bcast: 1}  # MCRDL_TUNE_*

    def install_tuning(self, table) -> None:
        """Push the table's per-size algorithm rows for this world into the
        communicator: AUTO then resolves in the C layer (mcrdl_comm_set_tuning).
        No table / no cell: the library's built-in crossovers. Every rank
        loads the same table, so every rank resolves AUTO alike."""
        from ..dispatch import algorithm_rows

        lib, c = self.comm.lib, self.comm.handle
        for kind, code in self.TUNE_KINDS.items():
            rows = algorithm_rows(table, kind, self.world_size, self.name)
            self.tuning_rows[kind] = rows
            mb = (ctypes.c_uint64 * max(len(rows), 1))(*[r[0] for r in rows])
            al = (ctypes.c_int * max(len(rows), 1))(*[ALGO_CODES[canonical(kind, r[1])] for r in rows])
            _lib.check(lib.mcrdl_comm_set_tuning(c, code, len(rows), mb, al))

    def last_algorithm(self, kind: CommOpKind) -> Optional[str]:
        """Algorithm the last AUTO-resolved launch of `kind` ran (C layer)."""
        code = self.comm.lib.mcrdl_comm_last_algo(self.comm.handle, self.TUNE_KINDS[kind])
        return _ALGO_NAMES.get(code)

    # ------------------------------------------------------------ properties
    @property
    def rank(self) -> int:
        return self.runtime.rank

    @property
    def world_size(self) -> int:
        return self.runtime.world_size

    def next_seq(self) -> int:
        with self._lock:
            s = self._seq
            self._seq += 1
            return s

    def pending_count(self) -> int:
        with self._lock:
            self._reap()
            return sum(1 for h in self._pending if not h.test())

    def drain_errors(self) -> List[BaseException]:
        with self._lock:
            errs, self._errors = self._errors, []
            return errs

    # ---------------------------------------------------------------- posting
    def _algo_code(self, kind: CommOpKind, nbytes: int) -> int:
        name = self.policy.algorithm(kind)
        if name == "auto" and self.runtime.tuning_table is not None:
            t = self.runtime.tuning_table.algorithm_for(kind, self.world_size, nbytes, self.name)
            if t is not None:
                name = canonical(kind, t)
        return ALGO_CODES.get(name, 0)

    def inline_ok(self, request: CommRequest) -> bool:
        """Blocking op on device tensors: run on the caller's current stream
        with no lane hop, no events and no staging (the reference's inline
        fast path, runtime.py:150-168). The C layer orders it after the
        communicator's previous op even across streams."""
        for b in request.buffers():
            if not b.is_device:
                return False
        return True

    def _assign_seq(self, request: CommRequest) -> None:
        """Collectives take the next backend sequence number (runtime.py:
        147-149), which the kernels fold into the flag signature. send/recv
        involve two ranks only: they are matched per (sender, receiver) pair
        on the device and must not advance the world-wide sequence."""
        if request.kind in P2P_KINDS:
            request.seq = 0
            return
        request.seq = self._seq
        self._seq += 1

    def post_inline(self, request: CommRequest) -> WorkHandle:
        if self.state != "initialized":
            raise BackendFinalized(f"backend {self.name!r} is {self.state}")
        with self._lock:
            self._assign_seq(request)
            self._pre_launch(request)
            lib, c = self.comm.lib, self.comm.handle
            log = self.runtime.log_ops
            if log:
                self._drain_log(block=False)
                first = lib.mcrdl_comm_log_id(c) + 1
            self._launch(request, _Direct(self.device), _raw_stream(self.device))
            if log:
                self._log_pending.append((request, first, lib.mcrdl_comm_log_id(c)))
            self.collectives_executed += 1
        return WorkHandle.completed(self.name, request)

    # -------------------------------------------- device-timed CommLog records
    def _drain_log(self, block: bool) -> None:
        """Emit the CommLog records of finished inline ops in issue order. The
        durations are the kernels' own %globaltimer stamps (mcrdl_comm_op_time:
        no events on the stream). block=True (the device has drained) emits
        everything; an op without stamps (p = 1 local copy, or a ring that
        wrapped) is logged with a 0.001 us placeholder duration."""
        from ..dispatch import message_bytes
        from ..middleware import LogRecord

        log = self.runtime.comm_log
        lib, c = self.comm.lib, self.comm.handle
        ns = ctypes.c_int64()
        if block and self._log_pending:  # the device drained: mirror every stamp now
            _lib.check(lib.mcrdl_comm_log_flush(c))
        while self._log_pending:
            req, first, last = self._log_pending[0]
            dur = None
            if last >= first:
                lib.mcrdl_comm_op_time(c, first, last, ctypes.byref(ns))
                if ns.value >= 0:
                    dur = ns.value * 1e-3
                elif ns.value == -1 and not block:
                    break
            self._log_pending.pop(0)
            members = getattr(req, "_fused_members", 0)
            log.emit(LogRecord(ts_us=log.now_us(), rank=self.rank, op=req.kind.value,
                               backend=self.name, bytes=message_bytes(req, self.world_size),
                               dur_us=max(dur or 0.0, 0.001), seq=req.seq or 0,
                               fused=members > 0, members=members or 1,
                               algorithm=getattr(req, "_algorithm", None)))

    def post(self, request: CommRequest) -> WorkHandle:
        if self.state != "initialized":
            raise BackendFinalized(f"backend {self.name!r} is {self.state}")
        handle = WorkHandle(self.name, request)
        with self._lock:
            self._assign_seq(request)
            self._pre_launch(request)  # before any stream work of this op
            handle.mark_in_progress()
            self._reap()
            if self._pipelined_ok(request):
                self._post_pipelined(request, handle)
                return handle
            caller = torch.cuda.current_stream(self.device)
            lane = self.stream
            lane.wait_stream(caller)
            st = _Staging(self.device, lane, self._pool)
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(lane):
                t0.record(lane)
                try:
                    self._launch(request, st, int(lane.cuda_stream))
                except BaseException as exc:
                    self._fail_now(handle, request, exc)
                    raise
                st.issue_downloads()
                t1.record(lane)
            self._arm(handle, request, st, t0, t1)
        return handle

    # ------------------------------------------- pipelined host staging
    PIPE_MIN_BYTES = 16 << 20
    # H2D -> collective -> D2H chunk: pipeline fill + drain cost one chunk of
    # PCIe each way (MCRDL_PIPE_CHUNK_MB overrides)
    PIPE_CHUNK_BYTES = int(os.environ.get("MCRDL_PIPE_CHUNK_MB", "32")) << 20

    def _pipelined_ok(self, req: CommRequest) -> bool:
        """Large all_reduce on pinned host tensors: overlap H2D, the collective
        and D2H chunk by chunk (PCIe is full duplex)."""
        if req.kind is not CommOpKind.all_reduce:
            return False
        for b in (req.input, req.output):
            if not (b.is_tensor and not b.is_device and b.array.is_pinned()):
                return False
        return req.input.nbytes >= self.PIPE_MIN_BYTES

    def _post_pipelined(self, req: CommRequest, handle: WorkHandle) -> None:
        dt = req.input.dtype
        n = req.input.count
        k = max(2, min(64, req.input.nbytes // self.PIPE_CHUNK_BYTES))
        step = ((n + k - 1) // k + 63) // 64 * 64
        h_in, h_out = req.input.array, req.output.array
        lane = self.stream
        # the first H2D chunk reads h_in: order it after the caller's work
        # (e.g. a non_blocking D2H that fills the pinned tensor)
        lane.wait_stream(torch.cuda.current_stream(self.device))
        if getattr(self, "_up", None) is None:
            self._up = self.comm.stream(1)
            self._down = self.comm.stream(2)
        up, down = self._up, self._down
        with torch.cuda.stream(lane):
            d = torch.empty(n, dtype=dt.torch_dtype, device=self.device)
        d.record_stream(up)
        d.record_stream(down)
        up.wait_stream(lane)  # d's memory is ready for reuse in lane order
        lib, c = self.comm.lib, self.comm.handle
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(up)
        algo = self._algo_code(CommOpKind.all_reduce, min(n, step) * dt.size_bytes)
        req._algorithm = _ALGO_NAMES.get(algo, "auto")
        for j, lo in enumerate(range(0, n, step)):
            hi = min(n, lo + step)
            with torch.cuda.stream(up):
                d[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            e_up = torch.cuda.Event()
            e_up.record(up)
            lane.wait_event(e_up)
            try:
                _lib.check(lib.mcrdl_all_reduce(c, int(d[lo:hi].data_ptr()), int(d[lo:hi].data_ptr()),
                                                hi - lo, dt.code, req.op.code, algo,
                                                (req.seq << 8) | (j & 0xFF), int(lane.cuda_stream)))
            except BaseException as exc:
                self._fail_now(handle, req, exc)
                raise
            e_ar = torch.cuda.Event()
            e_ar.record(lane)
            down.wait_event(e_ar)
            with torch.cuda.stream(down):
                h_out[lo:hi].copy_(d[lo:hi], non_blocking=True)
        self._last_raw = int(lane.cuda_stream)
        t1.record(down)
        lane.wait_stream(down)  # later ops of this backend see the host copy finished
        st = _Staging(self.device, lane, self._pool)
        st.keep.extend([d, h_in, h_out])
        self._arm(handle, req, st, t0, t1)

    def post_fused(self, members: Sequence[CommRequest], ready_events: Sequence,
                   flush_request: CommRequest) -> WorkHandle:
        """One launch: pack -> all_reduce -> unpack for fusion members
        (middleware FusionManager flush, middleware.py:311-344)."""
        handle = WorkHandle(self.name, flush_request)
        with self._lock:
            flush_request.seq = self._seq
            self._seq += 1
            self._pre_launch(flush_request)  # before any stream work of this op
            handle.mark_in_progress()
            lane = self.stream
            for ev in ready_events:
                if ev is not None:
                    lane.wait_event(ev)
            st = _Staging(self.device, lane, self._pool)
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(self.device), torch.cuda.stream(lane):
                t0.record(lane)
                dtype = members[0].input.dtype
                esz = dtype.size_bytes
                align = max(1, 16 // esz)
                ins, outs, counts, offs = [], [], [], []
                off = 0
                for m in members:
                    i = st.dev(m.input)
                    o = st.dev(m.output, upload=m.output is m.input, download=True)
                    ins.append(_ptr(i) or 0)
                    outs.append(_ptr(o) or 0)
                    counts.append(m.input.count)
                    offs.append(off)
                    off += (m.input.count + align - 1) // align * align
                nbytes = [c * esz for c in counts]
                offb = [o * esz for o in offs]
                table = torch.tensor([ins, outs, counts, offs, nbytes, offb],
                                     dtype=torch.int64).pin_memory()
                dtable = table.to(self.device, non_blocking=True)
                st.keep.extend([table, dtable])
                n = len(members)
                base = int(dtable.data_ptr())
                lib, c, ls = self.comm.lib, self.comm.handle, int(lane.cuda_stream)
                algo = self._algo_code(CommOpKind.all_reduce, off * esz)
                # one launch (k_ar_fused: members -> peers' slots, fold, members)
                # while the group's one-shot slots fit a workspace half; larger
                # groups: pack kernel -> all_reduce (two-shot / NVLS by AUTO) on
                # the packed buffer -> unpack kernel (middleware.py:311-344)
                slot = ((off * esz + 15) // 16 * 16 + 255) // 256 * 256
                one_launch = slot * self.world_size <= self.comm.caps.workspace_bytes // 2
                try:
                    if one_launch:
                        _lib.check(lib.mcrdl_all_reduce_fused(
                            c, base, base + 8 * n, base + 16 * n, base + 24 * n, n, off,
                            dtype.code, flush_request.op.code, algo, flush_request.seq, ls))
                    else:
                        packed = st.scratch(off, dtype)
                        st.keep.append(packed)
                        pk = _ptr(packed)
                        _lib.check(lib.mcrdl_fusion_pack(base, base + 32 * n, base + 40 * n, n, pk,
                                                         ls))
                        _lib.check(lib.mcrdl_all_reduce(c, pk, pk, off, dtype.code,
                                                        flush_request.op.code, algo,
                                                        flush_request.seq, ls))
                        _lib.check(lib.mcrdl_fusion_unpack(pk, base + 8 * n, base + 32 * n,
                                                           base + 40 * n, n, ls))
                    self._post_launch(flush_request)
                except BaseException as exc:
                    self._fail_now(handle, flush_request, exc)
                    raise
                st.issue_downloads()
                t1.record(lane)
            self._arm(handle, flush_request, st, t0, t1)
        return handle

    def _fail_now(self, handle: WorkHandle, request: CommRequest, exc: BaseException) -> None:
        self._errors.append(exc)
        for b in request.unique_buffers():
            b._checkin()
        handle.fail(exc)

    def _arm(self, handle: WorkHandle, request: CommRequest, st: _Staging, t0, t1) -> None:
        handle.event = t1
        log = self.runtime.comm_log

        def finalizer() -> None:
            try:
                st.finish()
                self.comm.status()
            except BaseException as exc:
                with self._lock:
                    self._errors.append(exc)
                raise
            finally:
                for b in request.unique_buffers():
                    b._checkin()
            self.collectives_executed += 1
            members = getattr(request, "_fused_members", 0)
            from ..dispatch import message_bytes
            from ..middleware import LogRecord

            log.emit(LogRecord(ts_us=log.now_us(), rank=self.rank, op=request.kind.value,
                               backend=self.name,
                               bytes=message_bytes(request, self.world_size),
                               dur_us=max(t0.elapsed_time(t1) * 1e3, 0.001),
                               seq=request.seq or 0, fused=members > 0,
                               members=members or 1,
                               algorithm=getattr(request, "_algorithm", None)))

        handle._finalizer = finalizer
        self._pending.append(handle)

    def _reap(self) -> None:
        keep = []
        for h in self._pending:
            if not h.test():
                keep.append(h)
        self._pending = keep

    def record_event(self) -> CompletionEvent:
        with self._lock:
            ev = torch.cuda.Event()
            # Ops of one communicator execute in issue order (the C layer
            # chains streams), so an event after the last op covers them all.
            last = self._last_raw
            if self._lane is None:  # no async work yet: the last inline op's stream
                ev.record(torch.cuda.ExternalStream(last, device=self.device) if last is not None
                          else torch.cuda.current_stream(self.device))
            elif last is not None and last != int(self._lane.cuda_stream):
                ev.record(torch.cuda.ExternalStream(last, device=self.device))
            else:
                ev.record(self._lane)
            pending = list(self._pending)
        ce = CompletionEvent(self.name, cuda_event=ev)
        ce._pending = pending  # type: ignore[attr-defined]
        return ce

    def settle(self, event: CompletionEvent) -> None:
        """After `event` fired: settle every handle it covers and emit the
        CommLog records of the inline ops before it."""
        for h in getattr(event, "_pending", []):
            if not h.test():
                h._settle()
        with self._lock:
            self._reap()
            self._drain_log(block=True)

    def symmetric_empty(self, count: int, dtype: DType):
        """Collective (same count/dtype on every rank, same order): a device
        tensor in symmetric memory. all_reduce whose input and output both
        live there runs zero-copy (csrc/allreduce.cu k_ar_symm: NVLS multicast
        for f32/bf16 sums, peer loads + stores otherwise). Freed at finalize."""
        dtype = DType.from_name(dtype) if isinstance(dtype, str) else dtype
        nbytes = max(int(count) * dtype.size_bytes, 16)
        ptr = self.comm.symm_alloc(nbytes)
        raw = torch.as_tensor(_CudaBlock(ptr, nbytes), device=torch.device("cuda", self.device))
        self._symm_keep.append(raw)
        return raw[:int(count) * dtype.size_bytes].view(dtype.torch_dtype)

    def symmetric_pool(self, nbytes: int):
        """Collective (same size, same order on every rank): a torch MemPool
        whose allocations come from one symmetric arena (csrc/pool.cu). Tensors
        allocated under `torch.cuda.use_mem_pool(pool)` are ordinary torch
        tensors that all_reduce / all_to_all take zero-copy (NVLS multimem or
        peer loads; sender-side direct writes) when every rank allocates them
        in the same order. The pool serves the calling thread (one rank per
        thread when ranks are co-located)."""
        global _POOL_ALLOCATOR
        h = c_void_p()
        _lib.check(self.comm.lib.mcrdl_pool_create(self.comm.handle, int(nbytes), byref(h)))
        _lib.check(self.comm.lib.mcrdl_pool_activate(h))
        if _POOL_ALLOCATOR is None:
            _POOL_ALLOCATOR = torch.cuda.memory.CUDAPluggableAllocator(
                str(_lib.LIB_PATH), "mcrdl_pool_malloc", "mcrdl_pool_free")
        pool = torch.cuda.MemPool(_POOL_ALLOCATOR.allocator())
        self._pools.append((h, pool))
        return pool

    def finalize(self, timeout: float) -> None:
        if self.state == "finalized":
            return
        ev = self.record_event()
        if not ev.wait(timeout):
            raise PendingAfterTimeout(f"backend {self.name!r} still has pending work after "
                                      f"{timeout}s")
        self.settle(ev)
        self.state = "finalized"
        self.comm.destroy()

    # ---------------------------------------------------------------- launch
    def _pre_launch(self, req: CommRequest, sub: int = 0) -> None:
        """Runtime.launch_hook (tests): called with (backend, seq, sub) right
        before a collective's C-ABI call. Co-located thread-rank tests use it
        to launch every rank's kernel of one op together, so that a device-
        synchronizing host call (cudaMalloc/cudaHostAlloc in torch's
        allocators, lazy module loads) in one rank never waits on a peer
        kernel that spins for an op this rank has not launched yet."""
        hook = self.runtime.launch_hook
        if (hook is not None and req.kind not in P2P_KINDS and self.world_size > 1
                and not torch.cuda.is_current_stream_capturing()):  # captures launch nothing
            hook((self.name, req.seq, sub))

    def _post_launch(self, req: CommRequest) -> None:
        """Runtime.launch_hook again once this op's kernel is enqueued: every
        rank's kernel of the op sits in the device's queues before any rank
        enqueues work that waits on it (a stream's next item waits for its
        kernel and can block a hardware queue the ranks' streams share)."""
        self._pre_launch(req, sub=-1)

    def _launch(self, req: CommRequest, st: _Staging, s: int) -> None:
        lib, c = self.comm.lib, self.comm.handle
        kind, p, rank, seq = req.kind, self.world_size, self.rank, req.seq
        name = self.policy.algorithm(kind)
        if name == "auto" and self.runtime.tuning_table is not None:
            algo = self._algo_code(kind, message_bytes(req, p))
        else:
            algo = ALGO_CODES.get(name, 0)
        req._algorithm = _ALGO_NAMES.get(algo, "auto")
        if self.compression is not None and self.compression.active_for(req) is not None:
            algo |= CODEC_TRUNC16
            req._algorithm += "+trunc16"
        posted = []

        def chk(rc):
            _lib.check(rc)
            if not posted:  # the op's (first) kernel is enqueued
                posted.append(True)
                self._post_launch(req)

        self._last_raw = s

        if kind in (CommOpKind.all_reduce, CommOpKind.reduce, CommOpKind.reduce_scatter):
            i = st.dev(req.input)
            dt, op = req.input.dtype, req.op.code
            if kind is CommOpKind.all_reduce:
                o = st.dev(req.output, upload=req.output is req.input, download=True)
                chk(lib.mcrdl_all_reduce(c, _ptr(i), _ptr(o), req.input.count, dt.code, op, algo,
                                         seq, s))
                if algo & 0xFF == 0 and p > 1:  # AUTO: log what the C layer resolved
                    req._algorithm = self.last_algorithm(kind)
            elif kind is CommOpKind.reduce:
                o = (st.dev(req.output, upload=req.output is req.input, download=True)
                     if rank == req.root else None)
                # native root mode of the two-shot pipeline where all_reduce would
                # run two-shot anyway; small messages: one-shot / LL all_reduce
                big = req.input.nbytes > ((8 << 20) if p == 2 else (2 << 20))
                if p > 1 and (big or name == "two_shot"):
                    chk(lib.mcrdl_reduce(c, _ptr(i), _ptr(o) if o is not None else None,
                                         req.input.count, dt.code, op, req.root, algo, seq, s))
                else:
                    if o is None:
                        o = st.scratch(req.input.count, dt)
                    chk(lib.mcrdl_all_reduce(c, _ptr(i), _ptr(o), req.input.count, dt.code, op,
                                             algo, seq, s))
            else:
                m = req.output.count
                o = st.dev(req.output, upload=False, download=True)
                rc = lib.mcrdl_reduce_scatter(c, _ptr(i), _ptr(o), m, dt.code, op, algo, seq, s)
                if rc == 4:  # kernel declined (alignment / size): compose on the device
                    full = st.scratch(p * m, dt)
                    chk(lib.mcrdl_all_reduce(c, _ptr(i), _ptr(full), p * m, dt.code, op, algo, seq,
                                             s))
                    o.copy_(full[rank * m:(rank + 1) * m])
                else:
                    chk(rc)
            return

        if kind is CommOpKind.send:
            b = st.dev(req.input)
            chk(lib.mcrdl_send(c, _ptr(b), req.input.nbytes, req.root, s))
            return
        if kind is CommOpKind.recv:
            b = st.dev(req.output, upload=False, download=True)
            chk(lib.mcrdl_recv(c, _ptr(b), req.output.nbytes, req.root, s))
            return

        if kind is CommOpKind.bcast:
            b = st.dev(req.output, upload=True, download=True)
            chk(lib.mcrdl_bcast(c, _ptr(b), req.output.count, req.output.dtype.code, req.root,
                                algo, seq, s))
            if algo & 0xFF == 0 and p > 1:
                req._algorithm = self.last_algorithm(kind)
            return

        if kind in (CommOpKind.all_gather, CommOpKind.all_gatherv):
            i = st.dev(req.input)
            o = st.dev(req.output, upload=False, download=True)
            dt = req.input.dtype
            if kind is CommOpKind.all_gather:
                n = req.input.count
                counts, displs = [n] * p, [r * n for r in range(p)]
            else:
                counts, displs = req.rcounts, req.rdispls
            if _is_dev(counts) or _is_dev(displs):
                # GPU-resident rcounts / displs: the kernel reads them
                dcnt, ddsp = _dev_vec(st, counts), _dev_vec(st, displs)
                chk(lib.mcrdl_all_gatherv_dev(c, _ptr(i), i.numel(), _ptr(o), o.numel(),
                                              _ptr(dcnt), _ptr(ddsp), dt.code, algo, seq, s))
            else:
                chk(lib.mcrdl_all_gatherv(c, _ptr(i), _ptr(o), _lib.i64_array(counts),
                                          _lib.i64_array(displs), dt.code, algo, seq, s))
            return

        if kind in (CommOpKind.gather, CommOpKind.gatherv):
            i = st.dev(req.input)
            o = st.dev(req.output, upload=False, download=True) if req.output is not None else None
            dt = req.input.dtype
            if kind is CommOpKind.gather:
                n = req.input.count
                counts, displs = [n] * p, [r * n for r in range(p)]
            else:
                counts, displs = req.rcounts, req.rdispls
            if _is_dev(counts) or _is_dev(displs):
                # GPU-resident rcounts / displs: no D2H sync, the kernel reads them
                dcnt, ddsp = _dev_vec(st, counts), _dev_vec(st, displs)
                chk(lib.mcrdl_gatherv_dev(c, _ptr(i), i.numel(), _ptr(o),
                                          o.numel() if o is not None else 0, _ptr(dcnt),
                                          _ptr(ddsp), req.root, dt.code, algo, seq, s))
            else:
                chk(lib.mcrdl_gatherv(c, _ptr(i), _ptr(o), _lib.i64_array(_host_list(counts)),
                                      _lib.i64_array(_host_list(displs)), req.root, dt.code,
                                      algo, seq, s))
            return

        if kind in (CommOpKind.scatter, CommOpKind.scatterv):
            o = st.dev(req.output, upload=False, download=True)
            i = st.dev(req.input) if req.input is not None else None
            dt = req.output.dtype
            if kind is CommOpKind.scatter:
                n = req.output.count
                counts, displs = [n] * p, [r * n for r in range(p)]
            else:
                counts, displs = _host_list(req.scounts), _host_list(req.sdispls)
            root = req.root
            if rank == root:
                sc, sd = list(counts), list(displs)
            else:
                sc, sd = [0] * p, [0] * p
            rc, rd = [0] * p, [0] * p
            rc[root] = counts[rank]
            chk(lib.mcrdl_all_to_allv(c, _ptr(i), _ptr(o), _lib.i64_array(sc), _lib.i64_array(sd),
                                      _lib.i64_array(rc), _lib.i64_array(rd), dt.code, algo, seq, s))
            return

        if kind is CommOpKind.all_to_all_single:
            same = req.input is req.output
            i = st.dev(req.input)
            o = i if same else st.dev(req.output, upload=False, download=True)
            if same:
                st.dev(req.output, download=True)
            if o.numel() and i.data_ptr() == o.data_ptr() and p > 1:
                i = i.clone()  # the reference snapshots aliased input (collectives.py:662-663)
                st.keep.append(i)
            chk(lib.mcrdl_all_to_all_single(c, _ptr(i), _ptr(o), req.input.count,
                                            req.input.dtype.code, algo, seq, s))
            return

        if kind is CommOpKind.all_to_all:
            ins = [st.dev(b) for b in req.input]
            outs = [st.dev(b, upload=False, download=True) for b in req.output]
            chk(lib.mcrdl_all_to_all_ptrs(
                c, _lib.ptr_array([_ptr(t) for t in ins]),
                _lib.i64_array([b.count for b in req.input]),
                _lib.ptr_array([_ptr(t) for t in outs]),
                _lib.i64_array([b.count for b in req.output]),
                req.input[0].dtype.code, algo, seq, s))
            return

        if kind is CommOpKind.all_to_allv:
            dt = req.input.dtype
            i = st.dev(req.input)
            o = st.dev(req.output, upload=False, download=True)
            vecs = (req.scounts, req.sdispls, req.rcounts, req.rdispls)
            if any(_is_dev(v) for v in vecs):
                if i.data_ptr() == o.data_ptr():
                    i = i.clone()
                dc = _dev_counts(st, *vecs)
                chk(lib.mcrdl_all_to_allv_dev(c, _ptr(i), i.numel(), _ptr(o), o.numel(), _ptr(dc),
                                              dt.code, algo, seq, s))
                return
            sc, sd, rc, rd = (list(map(int, v)) for v in vecs)
            if o.numel() and i.data_ptr() == o.data_ptr() and p > 1:
                i = i.clone()  # the reference snapshots aliased input (collectives.py:662-663)
            chk(lib.mcrdl_all_to_allv(c, _ptr(i), _ptr(o), _lib.i64_array(sc), _lib.i64_array(sd),
                                      _lib.i64_array(rc), _lib.i64_array(rd), dt.code, algo, seq, s))
            return

        raise UnsupportedOperation(f"{kind.name} is not supported by the nvlink backend")


_ALGO_NAMES = {v: k for k, v in ALGO_CODES.items()}
_POOL_ALLOCATOR = None  # torch CUDAPluggableAllocator over mcrdl_pool_malloc/free (one per process)
CODEC_TRUNC16 = 0x100  # include/mcrdl_nvl.h MCRDL_CODEC_TRUNC16


def _is_dev(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _host_list(x) -> list:
    if _is_dev(x):
        return [int(v) for v in x.tolist()]
    return [int(v) for v in x]


def _dev_vec(st: _Staging, v):
    """int64 device vector of counts (a host list is uploaded)."""
    if _is_dev(v):
        t = v.to(device=st.device, dtype=torch.int64).reshape(-1).contiguous()
    else:
        t = torch.tensor([int(x) for x in v], dtype=torch.int64).to(st.device)
    st.keep.append(t)
    return t


def _dev_counts(st: _Staging, sc, sd, rc, rd):
    parts = []
    for v in (sc, sd, rc, rd):
        if _is_dev(v):
            parts.append(v.to(device=st.device, dtype=torch.int64).reshape(-1))
        else:
            parts.append(torch.tensor([int(x) for x in v], dtype=torch.int64).to(
                st.device, non_blocking=False))
    dc = torch.cat(parts).contiguous()
    st.keep.append(dc)
    return dc

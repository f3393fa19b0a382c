"""User-facing runtime: backend registry and lifecycle, posting, handles,
waits and deadlock-free synchronize — the reference's Listing-1 surface
(runtime.py:293-626) over the B200 NVLink backend.

Plumbing differences from the reference, all B200-specific:

* ``BackendConfig(transport="nvlink")`` builds a native communicator
  (nvl/backend.py). The reference's host transports ``inproc``/``tcp`` carry
  bytes through host memory and are out of scope for this build
  (SURVEY.md §2); naming them raises UnknownTransport.
* A backend's progress lane is a CUDA stream; a blocking post on device
  tensors returns once the work is enqueued and the caller's current stream
  is ordered after it (wait() synchronises with the
  default stream). Host (numpy) buffers keep the reference's host-blocking
  behaviour. Device-detected errors surface at ``WorkHandle.wait``,
  ``Runtime.synchronize`` or the next post on the same backend.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass
from typing import Dict, Optional, Sequence, Union

from . import dispatch
from .collectives import AlgorithmPolicy
from .core import (AUTO_BACKEND, Buffer, CommOpKind, CommRequest, ReduceOp, WorkHandle,
                   check_backend_id, validate)
from .errors import (BackendFinalized, CommError, DuplicateBackend, NotInitialized,
                     PendingAfterTimeout, UnknownBackend, UnknownTransport, UnsupportedOperation,
                     ValidationError)
from .middleware import CommLog, CompressionConfig, FusionConfig, FusionManager

DEFAULT_TIMEOUT_SECS = 30.0
DEFAULT_WORKSPACE_BYTES = 2 << 30  # two 1 GiB halves: a 512 MiB two-shot chunk per launch

ENV_RANK = "MCRDL_RANK"
ENV_WORLD_SIZE = "MCRDL_WORLD_SIZE"
ENV_MASTER_ADDR = "MCRDL_MASTER_ADDR"
ENV_MASTER_PORT = "MCRDL_MASTER_PORT"
ENV_TIMEOUT = "MCRDL_TIMEOUT_SECS"
ENV_TUNING_TABLE = "MCRDL_TUNING_TABLE"
ENV_WORKSPACE = "MCRDL_NVL_WORKSPACE_BYTES"

TRANSPORTS = ("nvlink",)


@dataclass
class BackendConfig:
    """One backend = transport x algorithm policy (+ middleware). ``device``,
    ``workspace_bytes`` configure the nvlink communicator (defaults: LOCAL_RANK
    and 1 GiB of symmetric workspace)."""

    name: str
    transport: str = "nvlink"
    shape: Optional[object] = None  # reference CostShape (host transports only)
    policy: Optional[AlgorithmPolicy] = None
    fusion: Optional[FusionConfig] = None
    compression: Optional[CompressionConfig] = None
    master_addr: Optional[str] = None
    master_port: Optional[int] = None
    listen_host: str = "127.0.0.1"
    device: Optional[int] = None
    workspace_bytes: Optional[int] = None


def _env_int(*names: str, default: Optional[int] = None) -> Optional[int]:
    for n in names:
        v = os.environ.get(n)
        if v not in (None, ""):
            return int(v)
    return default


class Runtime:
    """One rank's view of the communication world. Rank/world default to
    MCRDL_RANK/MCRDL_WORLD_SIZE, else torchrun's RANK/WORLD_SIZE."""

    def __init__(self, rank: Optional[int] = None, world_size: Optional[int] = None, *,
                 fabric=None, master_addr: Optional[str] = None,
                 master_port: Optional[int] = None, timeout: Optional[float] = None):
        if fabric is not None:
            raise UnknownTransport("InprocFabric belongs to the reference's host transports; "
                                   "this build provides the nvlink transport")
        self.rank = rank if rank is not None else _env_int(ENV_RANK, "RANK", default=0)
        self.world_size = (world_size if world_size is not None
                           else _env_int(ENV_WORLD_SIZE, "WORLD_SIZE", default=1))
        self.local_device = _env_int("LOCAL_RANK")
        if timeout is None:
            timeout = float(os.environ.get(ENV_TIMEOUT, DEFAULT_TIMEOUT_SECS))
        self.timeout = timeout
        self.master_addr = (master_addr or os.environ.get(ENV_MASTER_ADDR)
                            or os.environ.get("MASTER_ADDR") or "127.0.0.1")
        self.master_port = master_port or _env_int(ENV_MASTER_PORT, default=0) or 0
        self.default_workspace_bytes = _env_int(ENV_WORKSPACE, default=DEFAULT_WORKSPACE_BYTES)
        self.comm_log = CommLog(self.rank)
        # Every completed op appends one CommLog record, as in the reference
        # (runtime.py:209-230). Durations are DEVICE times: CUDA events around
        # the op on its stream (inline ops: the caller's stream, finished
        # lazily, no host sync). MCRDL_LOG=0 turns record keeping off for
        # the lowest per-op host cost.
        self.log_ops = os.environ.get("MCRDL_LOG", "1") not in ("", "0")
        self.log_timing = self.log_ops  # (legacy name)
        self.tuning_table: Optional[dispatch.TuningTable] = None
        self._registry: Dict[str, object] = {}
        self._registry_lock = threading.Lock()
        self._registered_ids: tuple = ()
        self._fusion: Optional[FusionManager] = None
        self._store = None
        self._init_generation = 0
        # Test hook: callable((backend, seq, sub)) run right before every
        # collective's native launch (co-located thread-rank tests launch each
        # op's kernels together; tests/gpu_worker.py). None in production.
        self.launch_hook = None
        # Optional torch stream used as the progress lane by every nvlink
        # backend of this runtime (None: one communicator-owned stream each).
        self.lane_stream = None
        path = os.environ.get(ENV_TUNING_TABLE)
        if path:
            self.tuning_table = dispatch.load_table(path)
        # Algorithm table behind AUTO on nvlink backends (per op, per size):
        # MCRDL_TUNING_TABLE when set (runtime.py:330-332), else the measured
        # table shipped with the package; MCRDL_ALGO_TABLE=off keeps the
        # library's built-in crossovers.
        self.algorithm_table: Optional[dispatch.TuningTable] = None
        if os.environ.get("MCRDL_ALGO_TABLE", "") not in ("off", "0"):
            self.algorithm_table = self.tuning_table or dispatch.default_algorithm_table()

    # -------------------------------------------------------------- lifecycle
    def init(self, backends: Sequence[Union[BackendConfig, str]]) -> None:
        configs = [BackendConfig(name=b) if isinstance(b, str) else b for b in backends]
        names = [check_backend_id(c.name) for c in configs]
        if len(set(names)) != len(names):
            raise DuplicateBackend(f"duplicate backend ids in {names}")
        for cfg in configs:
            if cfg.name == AUTO_BACKEND:
                raise ValidationError("backend", '"auto" is reserved')
            with self._registry_lock:
                if cfg.name in self._registry:
                    continue  # idempotent per id
            instance = self._build_backend(cfg)
            if cfg.fusion is not None and self._fusion is None:
                self._fusion = FusionManager(self)
            with self._registry_lock:
                self._registry[cfg.name] = instance
                self._registered_ids = tuple(self._registry)

    def _build_backend(self, cfg: BackendConfig):
        if cfg.transport == "nvlink":
            from .nvl.backend import NvlBackendInstance

            self._init_generation += 1
            return NvlBackendInstance(cfg, self)
        raise UnknownTransport(f"unknown transport {cfg.transport!r} (this build provides "
                               f"{', '.join(TRANSPORTS)})")

    def _control_store(self, cfg: BackendConfig):
        """Host rendezvous store shared by this runtime's nvlink backends."""
        if self._store is None:
            from .nvl.bootstrap import make_store

            port = cfg.master_port or self.master_port or _env_int("MASTER_PORT", default=0)
            if port and not cfg.master_port and not self.master_port:
                port += 1  # MASTER_PORT belongs to torch.distributed's own store
            self._store = make_store(self.rank, self.world_size,
                                     cfg.master_addr or self.master_addr, port, self.timeout)
        return self._store

    def finalize(self, backends: Optional[Sequence[str]] = None) -> None:
        names = list(backends) if backends is not None else self.get_backends()
        for name in names:
            inst = self._instance(name)
            if self._fusion is not None:
                self._fusion.flush_backend(name)
            inst.finalize(self.timeout)
        if self._fusion is not None and not any(
                i.state == "initialized" for i in self._registry.values()):
            self._fusion.close()

    def close(self) -> None:
        try:
            self.finalize()
        except CommError:
            pass

    def __enter__(self) -> "Runtime":
        return self

    def __exit__(self, *_exc) -> None:
        self.close()

    # ---------------------------------------------------------- introspection
    def get_backends(self) -> list:
        return list(self._registered_ids)

    def _instance(self, name: str):
        inst = self._registry.get(name)
        if inst is None:
            raise UnknownBackend(f"backend {name!r} is not registered")
        return inst

    def symmetric_empty(self, backend: str, count: int, dtype="f32"):
        """Collective: a device tensor of `count` elements in `backend`'s
        symmetric memory (every rank calls it with the same arguments, in the
        same order). Collectives on such tensors skip the staging workspace
        (B200 extension; the reference has no device memory)."""
        inst = self._instance(backend)
        if not hasattr(inst, "symmetric_empty"):
            raise UnsupportedOperation(f"backend {backend!r} has no symmetric memory")
        return inst.symmetric_empty(count, dtype)

    def symmetric_pool(self, backend: str, nbytes: int):
        """Collective: a torch.cuda.MemPool over `nbytes` of `backend`'s
        symmetric memory; tensors allocated under torch.cuda.use_mem_pool(pool)
        in the same order on every rank take the zero-copy kernels (B200
        extension)."""
        inst = self._instance(backend)
        if not hasattr(inst, "symmetric_pool"):
            raise UnsupportedOperation(f"backend {backend!r} has no symmetric memory")
        return inst.symmetric_pool(nbytes)

    def get_size(self, backend: str) -> int:
        return self._instance(backend).world_size

    def get_rank(self, backend: str) -> int:
        return self._instance(backend).rank

    # ---------------------------------------------------------------- posting
    def post(self, request: CommRequest) -> WorkHandle:
        if not self._registry:
            raise NotInitialized("call init() before posting operations")
        validate(request, self.world_size, self.rank)
        if request.backend == AUTO_BACKEND:
            request.backend = dispatch.route(self.tuning_table, request.kind, self.world_size,
                                             dispatch.message_bytes(request, self.world_size),
                                             self._registered_ids)
        inst = self._instance(request.backend)
        if inst.state != "initialized":
            raise BackendFinalized(f"backend {request.backend!r} is finalized")
        cfg = inst.config
        fused = cfg.fusion is not None and self._fusion is not None and \
            self._fusion.eligible(cfg.fusion, request)
        if not fused and not request.async_op and inst.inline_ok(request):
            # Blocking device op: stream-ordered, complete when enqueued.
            return inst.post_inline(request)
        bufs = request.unique_buffers()
        for b in bufs:
            b._checkout()
        try:
            if fused:
                handle = self._fusion.post(inst, cfg.fusion, request)
            else:
                handle = inst.post(request)
        except BaseException:
            for b in bufs:
                b._checkin()
            raise
        if not request.async_op:
            if handle.error is not None:
                raise handle.error
            self.wait(handle)
        return handle

    def wait(self, handle: WorkHandle) -> None:
        """Order the caller after `handle`. Device work: the current CUDA
        stream waits on the op's event and the buffers are released for
        stream-ordered reuse. Host buffers: block the host
        (core.py:312-319)."""
        if handle.error is not None:
            raise handle.error
        if handle.event is None and handle._flush_hook is not None and not handle.test():
            handle._flush_hook()
        req = handle.request
        host = req is not None and any(not b.is_device for b in req.buffers())
        if handle.event is None or host:
            handle.wait(self.timeout * 2 + 5.0)
            return
        import torch

        torch.cuda.current_stream().wait_event(handle.event)
        if req is not None:
            for b in req.unique_buffers():
                b._checkin()

    @staticmethod
    def test(handle: WorkHandle) -> bool:
        return handle.test()

    def synchronize(self, backends: Optional[Sequence[str]] = None) -> None:
        """Drain the listed backends in registry order (runtime.py:470-494):
        flush fusion, record a completion event per lane, host-wait each,
        settle every handle, raise the first error (all attached as
        ``.aggregated``)."""
        order = self.get_backends()
        wanted = set(backends) if backends is not None else set(order)
        for name in wanted:
            self._instance(name)
        if self._fusion is not None:
            for name in order:
                if name in wanted:
                    self._fusion.flush_backend(name)
        events = [(n, self._instance(n).record_event()) for n in order if n in wanted]
        errors = []
        for name, ev in events:
            inst = self._instance(name)
            if not ev.wait(self.timeout * 2 + 5.0):
                errors.append(PendingAfterTimeout(f"backend {name!r} did not drain in time"))
                continue
            inst.settle(ev)
            errors.extend(inst.drain_errors())
            try:
                inst.comm.status()
            except CommError as exc:
                if not any(type(e) is type(exc) for e in errors):
                    errors.append(exc)
        if errors:
            first = errors[0]
            first.aggregated = errors  # type: ignore[attr-defined]
            raise first

    # ------------------------------------------------------- Listing-1 surface
    def send(self, backend: str, buffer: Buffer, peer: int, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.send, input=buffer, root=peer, backend=backend,
                                     async_op=async_op))

    def recv(self, backend: str, buffer: Buffer, peer: int, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.recv, output=buffer, root=peer, backend=backend,
                                     async_op=async_op))

    def all_reduce(self, backend: str, buffer: Buffer, op: ReduceOp = ReduceOp.sum,
                   async_op: bool = False):
        return self.post(CommRequest(CommOpKind.all_reduce, input=buffer, output=buffer, op=op,
                                     backend=backend, async_op=async_op))

    def reduce(self, backend: str, buffer: Buffer, root: int, op: ReduceOp = ReduceOp.sum,
               async_op: bool = False):
        return self.post(CommRequest(CommOpKind.reduce, input=buffer, output=buffer, root=root,
                                     op=op, backend=backend, async_op=async_op))

    def bcast(self, backend: str, buffer: Buffer, root: int, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.bcast, output=buffer, root=root, backend=backend,
                                     async_op=async_op))

    def all_gather(self, backend: str, output: Buffer, input: Buffer, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.all_gather, input=input, output=output,
                                     backend=backend, async_op=async_op))

    def all_gatherv(self, backend: str, output: Buffer, input: Buffer, rcounts, displs,
                    async_op: bool = False):
        return self.post(CommRequest(CommOpKind.all_gatherv, input=input, output=output,
                                     rcounts=rcounts, rdispls=displs, backend=backend,
                                     async_op=async_op))

    def gather(self, backend: str, output: Optional[Buffer], input: Buffer, root: int,
               async_op: bool = False):
        return self.post(CommRequest(CommOpKind.gather, input=input, output=output, root=root,
                                     backend=backend, async_op=async_op))

    def gatherv(self, backend: str, output: Optional[Buffer], input: Buffer, root: int,
                rcounts, displs, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.gatherv, input=input, output=output, root=root,
                                     rcounts=rcounts, rdispls=displs, backend=backend,
                                     async_op=async_op))

    def scatter(self, backend: str, output: Buffer, input: Optional[Buffer], root: int,
                async_op: bool = False):
        return self.post(CommRequest(CommOpKind.scatter, input=input, output=output, root=root,
                                     backend=backend, async_op=async_op))

    def scatterv(self, backend: str, output: Buffer, input: Optional[Buffer], root: int,
                 scounts, displs, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.scatterv, input=input, output=output, root=root,
                                     scounts=scounts, sdispls=displs, backend=backend,
                                     async_op=async_op))

    def reduce_scatter(self, backend: str, output: Buffer, input: Buffer,
                       op: ReduceOp = ReduceOp.sum, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.reduce_scatter, input=input, output=output, op=op,
                                     backend=backend, async_op=async_op))

    def all_to_all_single(self, backend: str, output: Buffer, input: Buffer,
                          async_op: bool = False):
        return self.post(CommRequest(CommOpKind.all_to_all_single, input=input, output=output,
                                     backend=backend, async_op=async_op))

    def all_to_all(self, backend: str, outputs: Sequence[Buffer], inputs: Sequence[Buffer],
                   async_op: bool = False):
        return self.post(CommRequest(CommOpKind.all_to_all, input=list(inputs),
                                     output=list(outputs), backend=backend, async_op=async_op))

    def all_to_allv(self, backend: str, output: Buffer, input: Buffer, scounts, rcounts,
                    sdispls, rdispls, async_op: bool = False):
        return self.post(CommRequest(CommOpKind.all_to_allv, input=input, output=output,
                                     scounts=scounts, rcounts=rcounts, sdispls=sdispls,
                                     rdispls=rdispls, backend=backend, async_op=async_op))

    # ---------------------------------------------------------- B200 extras
    def barrier(self, backend: str) -> None:
        """0-byte collective (the tuner's barrier, tuner.py:151-159)."""
        import torch

        inst = self._instance(backend)
        b = Buffer(torch.zeros(0, dtype=torch.float32, device=inst.device))
        self.all_reduce(backend, b, ReduceOp.sum)

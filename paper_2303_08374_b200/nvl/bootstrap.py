"""Host control plane for communicator setup: an all-gather over a
key-value store, handed to the C ABI as its bootstrap callback.

Reference counterpart: the TCP star bootstrap in which every rank dials rank
0 and receives the address book back (transport.py:279-376). Here the store
(torch.distributed's TCPStore, or the default store of an initialised process
group) carries only a job id and barriers; memory handles travel between the
rank processes as file descriptors over a unix socket (csrc/comm.cu).
"""

from __future__ import annotations

import ctypes
import datetime
import os
from typing import List, Optional

from ..errors import BootstrapTimeout
from ._lib import ALLGATHER_FN


class StoreBootstrap:
    def __init__(self, rank: int, world: int, store, prefix: str):
        self.rank = rank
        self.world = world
        self.store = store
        self.prefix = prefix
        self._round = 0
        self._cfn = ALLGATHER_FN(self._callback)  # keep alive for the comm's lifetime

    def allgather(self, data: bytes) -> List[bytes]:
        self._round += 1
        base = f"{self.prefix}/ag{self._round}/"
        self.store.set(base + str(self.rank), data)
        return [self.store.get(base + str(r)) for r in range(self.world)]

    def barrier(self) -> None:
        self.allgather(b"")

    def _callback(self, _ctx, send, recv, nbytes) -> int:
        try:
            mine = ctypes.string_at(send, nbytes)
            parts = self.allgather(mine)
            for r, part in enumerate(parts):
                if len(part) != nbytes:
                    return 1
                ctypes.memmove(recv + r * nbytes, part, nbytes)
            return 0
        except Exception:  # noqa: BLE001 - reported as a status code
            return 1

    @property
    def c_callback(self):
        return self._cfn


def make_store(rank: int, world: int, addr: str, port: int, timeout: float):
    """Default store of an initialised torch.distributed group, else a TCPStore
    hosted by rank 0 at addr:port."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        try:
            from torch.distributed.distributed_c10d import _get_default_store

            return _get_default_store()
        except Exception:  # pragma: no cover - private API moved
            pass
    if world > 1 and not port:
        raise BootstrapTimeout(
            "world > 1 needs a rendezvous port: set MCRDL_MASTER_PORT (or MASTER_PORT) or "
            "pass master_port to Runtime/BackendConfig")
    # MCRDL_STORE_EXTERNAL=1: another process (a launcher) hosts the store and
    # every rank is a client (e.g. rank 0 runs under a profiler)
    external = os.environ.get("MCRDL_STORE_EXTERNAL", "0") not in ("", "0")
    return dist.TCPStore(addr, int(port), world, rank == 0 and not external,
                         timeout=datetime.timedelta(seconds=max(timeout, 1.0)),
                         wait_for_workers=False)

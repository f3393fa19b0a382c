"""World-size-2 host control plane on CPU (gloo + TCPStore): the bootstrap
all-gather the C ABI calls during communicator init, invoked through its
ctypes C function pointer exactly as libmcrdl_nvl.so calls it, and the
cross-rank max the bench and tuner take (bench.py max_over_ranks)."""

import ctypes
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        from paper_2303_08374_b200.nvl.bootstrap import StoreBootstrap, make_store

        store = make_store(rank, world, "127.0.0.1", port, 30.0)
        boot = StoreBootstrap(rank, world, store, prefix="t")
        # 1) Python-level allgather
        parts = boot.allgather(f"r{rank}".encode())
        # 2) through the C function pointer (as comm.cu host_allgather does)
        n = 8
        send = (ctypes.c_uint8 * n)(*([rank + 1] * n))
        recv = (ctypes.c_uint8 * (n * world))()
        fptr = ctypes.cast(boot.c_callback, ctypes.c_void_p).value
        cfn = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_size_t)(fptr)
        rc = cfn(None, ctypes.addressof(send), ctypes.addressof(recv), n)
        # 3) gloo group: cross-rank max (host control plane of bench/tuner)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port + 1))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        t = torch.tensor([float(rank) * 2.5])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
        q.put((rank, [p.decode() for p in parts], rc, list(recv), float(t.item())))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc), -1, [], 0.0))


def test_bootstrap_allgather_two_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(30)
    for rank, parts, rc, recv, mx in res:
        assert parts == ["r0", "r1"], parts
        assert rc == 0
        assert recv == [1] * 8 + [2] * 8
        assert mx == 2.5


def test_world_one_needs_no_store():
    from paper_2303_08374_b200.nvl.bootstrap import make_store
    from paper_2303_08374_b200.errors import BootstrapTimeout

    with pytest.raises(BootstrapTimeout):
        make_store(0, 2, "127.0.0.1", 0, 1.0)

"""Timeline of one direct-write exchange (all_to_all_single) — developer tool;
needs the trace build (`python -m paper_2303_08374_b200.build --trace`, run with
MCRDL_TRACE_LIB=1). Thread 0 of each CTA stamps %globaltimer: slot 0 at start;
senders 1+r after publishing row r; receivers 1 after the local copy, 2+2r
after the row-r flag wait, 3+2r after landing row r; slot 255 at exit.
Prints per-role percentiles (us) relative to the earliest start on the rank.
usage: torchrun ... tools/trace_x.py MiB_total_per_rank
"""

import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08374_b200 import BackendConfig, Buffer, Runtime  # noqa: E402
from paper_2303_08374_b200.nvl import _lib  # noqa: E402


def pct(x):
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        return "-"
    return " ".join(f"{np.percentile(x, q):7.1f}" for q in (0, 10, 50, 90, 100))


def main():
    size = int(float(sys.argv[1]) * (1 << 20)) if len(sys.argv) > 1 else 16 << 20
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    rt = Runtime(rank, world)
    rt.init([BackendConfig("nvl")])
    n = size // 4 // world * world
    a, b = Buffer(torch.randn(n, device="cuda")), Buffer(torch.empty(n, device="cuda"))
    for _ in range(5):
        rt.all_to_all_single("nvl", b, a)
    torch.cuda.synchronize()
    ptr, slots = ctypes.POINTER(ctypes.c_uint64)(), ctypes.c_uint64()
    _lib.load().mcrdl_debug_trace(rt._instance("nvl").comm.handle, ctypes.byref(ptr),
                                  ctypes.byref(slots))
    if not ptr:
        print("not a trace build")
        return
    ns = int(slots.value)
    buf = np.ctypeslib.as_array(ptr, shape=(512 * ns,))
    rt.barrier("nvl")
    torch.cuda.synchronize()
    buf[:] = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    rt.all_to_all_single("nvl", b, a)
    e.record()
    torch.cuda.synchronize()
    tr = buf.reshape(512, ns).astype(np.int64).copy()
    used = np.nonzero(tr[:, 0])[0]
    g = len(used) // 2
    t0 = tr[used, 0].min()
    rel = lambda v: (v - t0) / 1e3  # noqa: E731
    snd, rcv = used[:g], used[g:]
    lines = [f"rank {rank}: {size >> 20} MiB/rank, CTAs/role {g}, event {s.elapsed_time(e) * 1e3:.1f} us",
             "                      p0      p10     p50     p90     p100 (us)",
             f"sender start      {pct(rel(tr[snd, 0]))}",
             f"sender row0 pub   {pct(rel(tr[snd, 1]))}",
             f"sender end        {pct(rel(tr[snd, ns - 1]))}",
             f"recv start        {pct(rel(tr[rcv, 0]))}",
             f"recv local done   {pct(rel(tr[rcv, 1]))}",
             f"recv row0 flags   {pct(rel(tr[rcv, 2]))}",
             f"recv row0 landed  {pct(rel(tr[rcv, 3]))}",
             f"recv end          {pct(rel(tr[rcv, ns - 1]))}"]
    print("\n".join(lines), flush=True)
    rt.close()


if __name__ == "__main__":
    main()

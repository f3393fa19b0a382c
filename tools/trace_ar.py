"""Timeline of one two-shot all_reduce (developer tool; needs the trace build:
`python -m paper_2303_08374_b200.build --trace`, run with MCRDL_TRACE_LIB=1).

Each CTA's thread 0 stamps %globaltimer: slot 0 at start, per-row events
(sender: 1+r after publishing row r; reducer/gatherer: 1+2r after the wait,
2+2r after the work of row r), slot 255 at exit. Prints per-role percentiles
relative to the earliest start on this rank.
"""

import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_08374_b200 import BackendConfig, Buffer, CommOpKind, CommRequest, ReduceOp, Runtime  # noqa: E402
from paper_2303_08374_b200.collectives import AlgorithmPolicy  # noqa: E402
from paper_2303_08374_b200.nvl import _lib  # noqa: E402


def main():
    size = int(float(sys.argv[1]) * (1 << 20)) if len(sys.argv) > 1 else 256 << 20
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    rt = Runtime(rank, world)
    rt.init([BackendConfig("nvl", policy=AlgorithmPolicy({CommOpKind.all_reduce: "two_shot"}))])
    a = Buffer(torch.randn(size // 4, device="cuda"))
    b = Buffer(torch.empty(size // 4, device="cuda"))
    for _ in range(5):
        rt.post(CommRequest(CommOpKind.all_reduce, input=a, output=b, op=ReduceOp.sum, backend="nvl"))
    torch.cuda.synchronize()
    inst = rt._instance("nvl")
    ptr = ctypes.POINTER(ctypes.c_uint64)()
    slots = ctypes.c_uint64()
    _lib.load().mcrdl_debug_trace(inst.comm.handle, ctypes.byref(ptr), ctypes.byref(slots))
    if not ptr:
        print("not a trace build (MCRDL_TRACE_LIB=1 and build --trace)")
        return
    ns = int(slots.value)
    buf = np.ctypeslib.as_array(ptr, shape=(512 * ns,))
    buf[:] = 0
    rt.barrier("nvl")
    torch.cuda.synchronize()
    buf[:] = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    rt.post(CommRequest(CommOpKind.all_reduce, input=a, output=b, op=ReduceOp.sum, backend="nvl"))
    e.record()
    torch.cuda.synchronize()
    tr = buf.reshape(512, ns).astype(np.int64).copy()
    used = np.nonzero(tr[:, 0])[0]
    ncta = len(used)
    t0 = tr[used, 0].min()
    gs = int(os.environ.get("TRACE_GS", "0")) or ncta // 3
    gp = (ncta - gs) // 2
    roles = {"sender": range(0, gs), "reducer": range(gs, gs + gp), "gatherer": range(gs + gp, ncta)}
    if rank == 0:
        print(f"rank {rank} world {world} size {size >> 20} MiB  op {s.elapsed_time(e) * 1e3:.1f} us"
              f"  ctas {ncta} (gs {gs}, gp {gp})")
        for name, rng in roles.items():
            idx = list(rng)
            st = (tr[idx, 0] - t0) / 1e3
            en = (tr[idx, ns - 1] - t0) / 1e3
            print(f"  {name:9s} start p0/50/100 {np.percentile(st, 0):7.1f} {np.percentile(st, 50):7.1f} "
                  f"{np.percentile(st, 100):7.1f} us | end {np.percentile(en, 0):7.1f} "
                  f"{np.percentile(en, 50):7.1f} {np.percentile(en, 100):7.1f} us")
            ev = tr[idx, 1:ns - 1]
            for k in range(min(ev.shape[1], 24)):
                col = ev[:, k]
                col = col[col > 0]
                if len(col) == 0:
                    continue
                col = (col - t0) / 1e3
                print(f"      ev{k + 1:3d} n={len(col):3d} p10 {np.percentile(col, 10):7.1f} "
                      f"p50 {np.percentile(col, 50):7.1f} p90 {np.percentile(col, 90):7.1f} us")
    rt.close()


if __name__ == "__main__":
    main()

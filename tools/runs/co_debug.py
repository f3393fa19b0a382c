"""Co-located (thread-rank) debug driver: p ranks on cuda:0 run a list of
all_reduce sizes / algorithms and report time and correctness per op."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2303_08374_b200 import AlgorithmPolicy, BackendConfig, Buffer, CommOpKind, Runtime  # noqa

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
SIZES = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else
                          ["1048576", "4194304", "16777216", "25165829"])]
ALGO = sys.argv[3] if len(sys.argv) > 3 else "two_shot"
bar = threading.Barrier(P)
lines = []


def body(r):
    torch.cuda.set_device(0)
    torch.cuda.set_stream(torch.cuda.Stream(0))
    rt = Runtime(rank=r, world_size=P)
    rt.local_device = 0
    rt.init([BackendConfig("nvl")])
    inst = rt._instance("nvl")
    inst.policy = AlgorithmPolicy({CommOpKind.all_reduce: ALGO})
    for n in SIZES:
        x = torch.full((n,), float(r + 1), device="cuda")
        torch.cuda.current_stream().synchronize()
        bar.wait()
        t0 = time.time()
        err = None
        try:
            rt.all_reduce("nvl", Buffer(x))
            torch.cuda.current_stream().synchronize()
            inst.comm.status()
        except Exception as e:  # noqa
            err = repr(e)[:200]
        dt = time.time() - t0
        ok = bool(torch.all(x == P * (P + 1) / 2).item())
        lines.append(f"r{r} n={n} algo={ALGO} t={dt*1e3:.1f}ms ok={ok} err={err}")
    bar.wait()
    rt.close()


ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
[t.start() for t in ts]
[t.join() for t in ts]
print("\n".join(sorted(lines)))

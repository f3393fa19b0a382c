"""Host overhead per API call (developer tool): time N blocking posts of a
small all_reduce / all_to_allv on device tensors with the GPU idle-bound
excluded (host wall time per call), then cProfile the hot path."""

import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_08374_b200 import BackendConfig, Buffer, Runtime  # noqa: E402


def main():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    rt = Runtime(rank, world)
    rt.init([BackendConfig("nvl")])
    x = Buffer(torch.ones(256, device="cuda"))
    o = Buffer(torch.empty(256 * world, device="cuda"))
    i = Buffer(torch.ones(256 * world, device="cuda"))
    c = [256] * world
    d = [k * 256 for k in range(world)]
    ops = {
        "all_reduce": lambda: rt.all_reduce("nvl", x),
        "all_to_allv": lambda: rt.all_to_allv("nvl", o, i, c, c, d, d),
        "all_to_all_single": lambda: rt.all_to_all_single("nvl", o, i),
    }
    n = 2000
    for name, fn in ops.items():
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        if rank == 0:
            print(f"{name}: {1e6 * (t1 - t0) / n:.2f} us host per call")
    # every rank must post the same sequence (collectives); rank 0 reports
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(n):
        ops["all_to_allv"]()
    pr.disable()
    if rank == 0:
        pstats.Stats(pr).sort_stats("tottime").print_stats(18)
    torch.cuda.synchronize()
    rt.close()


if __name__ == "__main__":
    main()

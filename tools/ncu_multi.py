"""Per-kernel ncu evidence for the multi-rank kernels (p >= 2).

Launch p ranks of this script; rank 0 alone runs under ncu with a
SINGLE-PASS metric set (no kernel replay: a replayed multi-rank kernel would
wait for peer flags that were consumed by the first pass), the others run
normally. Each rank runs the same op list; rank 0's capture yields, per
kernel launch: duration, DRAM read/write bytes and NVLink rx/tx bytes.

    python tools/ncu_multi.py --world 4 --out gpurun_out/ncu_p4 [--metrics m1,m2,...]

Writes <out>.csv (ncu --csv --page raw) and <out>.json (kernel -> per-launch
metrics, algorithmic bytes of the op that launched it).
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

MIB = 1 << 20
# (tag, op, bytes per rank, algorithm policy)
OPS = [
    ("ar_ll_64k", "all_reduce", 64 << 10, "auto"),
    ("ar_oneshot_1m", "all_reduce", 1 << 20, "one_shot"),
    ("ar_twoshot_64m", "all_reduce", 64 * MIB, "two_shot"),
    ("ar_twoshot_tma_256m", "all_reduce", 256 * MIB, "two_shot"),
    ("ar_nvls_256m", "all_reduce", 256 * MIB, "nvls"),
    ("a2a_64m", "all_to_all_single", 64 * MIB, "auto"),
    ("a2a_ll_64k", "all_to_all_single", 64 << 10, "auto"),
    ("bcast_nvls_64m", "bcast", 64 * MIB, "nvls"),
    ("bcast_chain_256m", "bcast", 256 * MIB, "chain"),
]


def rank_main(reps: int, rnd: int) -> None:
    import torch

    from paper_2303_08374_b200 import AlgorithmPolicy, BackendConfig, Buffer, CommOpKind, Runtime

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    rt = Runtime(rank, world)
    be = f"nvl{rnd}"
    rt.init([BackendConfig(be)])
    print(f"rank {rank}/{world} round {rnd}: comm up (pid {os.getpid()})", flush=True)
    inst = rt._instance(be)
    kinds = {"all_reduce": CommOpKind.all_reduce, "all_to_all_single": CommOpKind.all_to_all_single,
             "bcast": CommOpKind.bcast}
    for tag, op, nbytes, algo in OPS:
        n = nbytes // 4
        n -= n % world
        x = torch.randn(n, device="cuda")
        y = torch.empty_like(x)
        inst.policy = AlgorithmPolicy({kinds[op]: algo}) if algo != "auto" else AlgorithmPolicy()
        for _ in range(reps):
            if op == "all_reduce":
                rt.all_reduce(be, Buffer(x))
            elif op == "all_to_all_single":
                rt.all_to_all_single(be, Buffer(y), Buffer(x))
            else:
                rt.bcast(be, Buffer(x), 0)
        torch.cuda.synchronize()
        if rank == 0:
            print(f"OPDONE {tag}", flush=True)
    rt.synchronize()
    print(f"rank {rank}: all ops done", flush=True)
    rt.close()


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/ncu_multi")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--metrics", default="gpu__time_duration.sum,dram__bytes_read.sum,"
                                          "dram__bytes_write.sum")
    ap.add_argument("--rank-main", action="store_true")
    ap.add_argument("--profiled", action="store_true")
    a = ap.parse_args()
    if a.rank_main:
        # ncu starts the profiled program twice (an unprofiled first run, then
        # the profiled one): the profiled rank learns its round from a store
        # counter, every other rank plays both rounds on fresh backends
        if a.profiled:
            import datetime

            import torch.distributed as dist

            st = dist.TCPStore("127.0.0.1", int(os.environ["MCRDL_MASTER_PORT"]), is_master=False,
                               timeout=datetime.timedelta(seconds=300))
            rank_main(a.reps, int(st.add("ncu-multi-profiled-run", 1)))
        else:
            for rnd in (1, 2):
                rank_main(a.reps, rnd)
        return 0
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    import datetime

    import torch.distributed as dist

    # the launcher hosts the rendezvous store: rank 0 runs under ncu, whose
    # start-up would otherwise stall the store every rank connects to
    store = dist.TCPStore("127.0.0.1", port, a.world + 1, True,
                          timeout=datetime.timedelta(seconds=300), wait_for_workers=False)
    procs = []
    out = Path(a.out)
    for r in range(a.world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(a.world), LOCAL_RANK=str(r),
                   MCRDL_MASTER_ADDR="127.0.0.1", MCRDL_MASTER_PORT=str(port),
                   MCRDL_STORE_EXTERNAL="1", MCRDL_TIMEOUT_SECS="120", MCRDL_DEBUG="1")
        cmd = [sys.executable, __file__, "--rank-main", "--reps", str(a.reps)]
        if r == int(os.environ.get("NCU_MULTI_RANK", "0")) and not os.environ.get("NCU_MULTI_NO_NCU"):
            cmd.append("--profiled")
            cmd = ["ncu", "--target-processes", "application-only", "--metrics", a.metrics,
                   "--clock-control", "none",
                   "--kernel-name", "regex:^k_", "--csv", "--page", "raw",
                   "--log-file", str(out) + ".csv"] + cmd
        log = open(f"{out}.rank{r}.log", "w")
        procs.append(subprocess.Popen(cmd, env=env, stdout=log, stderr=subprocess.STDOUT))
    rcs = [p.wait() for p in procs]
    del store
    print("rcs", rcs)
    if not Path(str(out) + ".csv").exists():
        return 0 if all(rc == 0 for rc in rcs) else 1
    lines = open(str(out) + ".csv").read().splitlines()
    start = next((i for i, ln in enumerate(lines) if ln.startswith('"ID"')), len(lines))
    rows = list(csv.DictReader(lines[start:]))
    summary: dict = {}
    for row in rows[1:] if rows and rows[0].get("ID") == "" else rows:  # raw page: units row
        name = row.get("Kernel Name", "?").split("(")[0]
        rec = {k: row[k] for k in row if any(m.split(".")[0] in k for m in a.metrics.split(","))}
        summary.setdefault(name, []).append(rec)
    Path(str(out) + ".json").write_text(json.dumps({"world": a.world, "ops": OPS,
                                                    "kernels": summary}, indent=1))
    return 0 if all(rc == 0 for rc in rcs) else 1


if __name__ == "__main__":
    sys.exit(main())

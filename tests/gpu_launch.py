"""Launch a world of tests/gpu_worker.py ranks and collect their JSON
reports: one process per GPU, or (colocated=True) `world` thread-ranks in ONE
process sharing one GPU. Used by the GPU parity tests and smoke()."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_colocated(world: int, scenarios=None, timeout: float = 600.0, extra_env=None,
                  device: int = 0) -> list:
    """`world` ranks as threads of one process on one GPU (gpu_worker --threads)."""
    port = free_port()
    tmp = Path(tempfile.mkdtemp(prefix="mcrdl-gpu-"))
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    env.update({"MCRDL_MASTER_ADDR": "127.0.0.1", "MCRDL_MASTER_PORT": str(port),
                "MCRDL_TIMEOUT_SECS": env.get("MCRDL_TIMEOUT_SECS", "20"),
                "MCRDL_COLOCATED_DEVICE": str(device),
                "MCRDL_THREAD_TIMEOUT": str(min(120.0, max(30.0, timeout - 30.0))),
                # Lazy loading of a kernel waits for the context to go idle:
                # a rank's first launch of a kernel variant would wait for a
                # peer rank's kernel that spins on that very launch (the
                # anti-pattern the CUDA lazy-loading notes describe). One
                # context hosts every co-located rank, so load eagerly.
                "CUDA_MODULE_LOADING": "EAGER",
                # every rank's streams map onto the device's hardware queues;
                # more queues = fewer streams of different ranks sharing one
                "CUDA_DEVICE_MAX_CONNECTIONS": "32"})
    if scenarios and "p2p" not in scenarios:
        # no send/recv in this run: no point-to-point mailboxes (every rank's
        # communicators share this GPU's memory)
        env.setdefault("MCRDL_P2P_BYTES", "0")
    env.update(extra_env or {})
    cmd = [sys.executable, str(ROOT / "tests" / "gpu_worker.py"), "--threads", str(world), str(tmp)]
    if scenarios:
        cmd.append(",".join(scenarios))
    # output straight to a file: a partial log survives a hang
    log = Path(os.environ.get("MCRDL_COLOCATED_LOG") or (tmp / "worker.log"))
    with open(log, "w") as fh:
        proc = subprocess.Popen(cmd, env=env, stdout=fh, stderr=subprocess.STDOUT, text=True)
        try:
            proc.wait(timeout=timeout)
        except subprocess.TimeoutExpired:
            proc.kill()
            proc.wait()
    out = log.read_text(errors="replace")
    if proc.returncode != 0 and proc.returncode < 0:
        out = f"killed (signal {-proc.returncode}) after {timeout:.0f} s\n" + out
    reports = []
    for r in range(world):
        f = tmp / f"r{r}.json"
        if f.exists():
            rep = json.loads(f.read_text())
        else:
            rep = {"rank": r, "failures": [f"no report; output:\n{out[-4000:]}"], "checked": 0}
        rep["exit"] = proc.returncode
        rep["output_tail"] = out[-2000:]
        reports.append(rep)
    return reports


def run_world(world: int, scenarios=None, timeout: float = 600.0, extra_env=None,
              colocated: bool = False) -> list:
    if colocated:
        return run_colocated(world, scenarios, timeout, extra_env)
    port = free_port()
    tmp = Path(tempfile.mkdtemp(prefix="mcrdl-gpu-"))
    procs = []
    for r in range(world):
        env = dict(os.environ)
        env.update({"RANK": str(r), "WORLD_SIZE": str(world), "LOCAL_RANK": str(r),
                    "MCRDL_MASTER_ADDR": "127.0.0.1", "MCRDL_MASTER_PORT": str(port),
                    "MCRDL_TIMEOUT_SECS": env.get("MCRDL_TIMEOUT_SECS", "20")})
        env.update(extra_env or {})
        cmd = [sys.executable, str(ROOT / "tests" / "gpu_worker.py"), str(tmp / f"r{r}.json")]
        if scenarios:
            cmd.append(",".join(scenarios))
        procs.append(subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outputs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            out = "TIMEOUT"
        outputs.append(out)
    reports = []
    for r in range(world):
        f = tmp / f"r{r}.json"
        if f.exists():
            rep = json.loads(f.read_text())
        else:
            rep = {"rank": r, "failures": [f"no report; output:\n{outputs[r][-4000:]}"],
                   "checked": 0}
        rep["exit"] = procs[r].returncode
        rep["output_tail"] = outputs[r][-2000:]
        reports.append(rep)
    return reports


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--colocated"]
    w = int(args[0]) if args else 2
    sc = args[1].split(",") if len(args) > 1 else None
    reps = run_world(w, sc, colocated="--colocated" in sys.argv,
                     timeout=float(os.environ.get("MCRDL_LAUNCH_TIMEOUT", "1200")))
    bad = 0
    for rep in reps:
        print(f"rank {rep['rank']}: exit={rep['exit']} checked={rep['checked']} nvls={rep.get('nvls')} "
              f"colocated={rep.get('colocated')} sms={rep.get('num_sms')} "
              f"launches={rep.get('launches')} failures={len(rep['failures'])}")
        for f in rep["failures"][:20]:
            print("   ", f)
        for x in rep.get("log_tail", []):
            print("     log", x)
        bad += len(rep["failures"]) + (rep["exit"] != 0)
    sys.exit(1 if bad else 0)

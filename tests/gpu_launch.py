"""Launch `world` rank processes of tests/gpu_worker.py (one per GPU) and
collect their JSON reports. Used by the GPU parity tests and smoke()."""

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


def run_world(world: int, scenarios=None, timeout: float = 600.0, extra_env=None) -> list:
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
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    sc = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    reps = run_world(w, sc)
    bad = 0
    for rep in reps:
        print(f"rank {rep['rank']}: exit={rep['exit']} checked={rep['checked']} nvls={rep.get('nvls')} "
              f"launches={rep.get('launches')} failures={len(rep['failures'])}")
        for f in rep["failures"][:20]:
            print("   ", f)
        bad += len(rep["failures"]) + (rep["exit"] != 0)
    sys.exit(1 if bad else 0)

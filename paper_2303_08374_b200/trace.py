"""Collective step traces in the CommLog JSONL schema, and their replay.

SURVEY §8d cfg5: one training step = a fixed posting order of collectives,
stored as LogRecord-schema JSONL (reference middleware.py:100-124) and
replayed through the public Runtime API. Every line is a valid reference
LogRecord (ts_us, rank, op, backend, bytes, dur_us, seq, fused[, members]),
so the reference's CommLog loader and `report` read it unchanged
(middleware.py:120-124 ignores extra keys). The extra keys make the record
replayable: `dtype`, `async` and the per-rank counts the collective needs
(`scounts` for all_to_allv, `rcounts` for all_gatherv / gatherv), `root`.

One JSONL holds the records of every rank (field `rank`); a rank replays its
own lines in `seq` order, taking peer counts from the peers' lines.
"""

from __future__ import annotations

import json
from typing import Dict, List, Optional

import numpy as np

from .middleware import LOG_FIELDS

CFG5_MLP = [6656, 512, 262144, 512, 65536, 128, 490496, 1024, 1048576, 1024, 1048576, 1024,
            1024, 1]


def dlrm_counts(p: int, skew: bool = False):
    """cfg4: sc[i][j] = b_j * T_i * 128 f32 elements i -> j."""
    tables = [len(x) for x in np.array_split(np.arange(26), p)]
    B = 65536
    if skew:
        wz = [(j + 1) ** -1.1 for j in range(p)]
        b = [int(B * w / sum(wz)) for w in wz]
        b[-1] += B - sum(b)
    else:
        b = [B // p] * p
    return [[b[j] * tables[i] * 128 for j in range(p)] for i in range(p)]


def cfg5_trace(p: int, dense_backend: str = "nvl", fused_backend: str = "nvl_fused") -> List[dict]:
    """The cfg5 step's posting order for every rank: a2av forward (cfg4
    uniform), the 14 DLRM MLP gradients posted async on the fusion backend,
    all_gatherv i64 (1000 + 137 r), gatherv f32 to root 0 (16 (r + 1)), a2av
    backward (transposed counts)."""
    sc = dlrm_counts(p)
    agc = [1000 + 137 * q for q in range(p)]
    gvc = [16 * (q + 1) for q in range(p)]
    recs = []
    for r in range(p):
        seq = 0

        def add(op, backend, nbytes, **extra):
            nonlocal seq
            rec = {"ts_us": 0, "rank": r, "op": op, "backend": backend, "bytes": int(nbytes),
                   "dur_us": 0.0, "seq": seq, "fused": False, "members": 1}
            rec.update(extra)
            recs.append(rec)
            seq += 1

        add("all_to_allv", dense_backend, sum(sc[r]) * 4, dtype="f32", scounts=sc[r])
        for k, n in enumerate(CFG5_MLP):
            add("all_reduce", fused_backend, n * 4, dtype="f32", count=n, **{"async": True},
                tensor=f"grad{k}")
        add("all_gatherv", dense_backend, sum(agc) * 8, dtype="i64", rcounts=agc)
        add("gatherv", dense_backend, sum(gvc) * 4, dtype="f32", rcounts=gvc, root=0)
        sct = [sc[j][r] for j in range(p)]  # backward: rank r sends back what it received
        add("all_to_allv", dense_backend, sum(sct) * 4, dtype="f32", scounts=sct)
    return recs


def write_jsonl(records: List[dict], path: str) -> None:
    with open(path, "w") as fh:
        for rec in records:
            fh.write(json.dumps(rec, separators=(",", ":")) + "\n")


def load_jsonl(path: str) -> List[dict]:
    out = []
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if line:
                rec = json.loads(line)
                missing = [k for k in LOG_FIELDS if k not in rec]
                if missing:
                    raise ValueError(f"{path}: not a CommLog record (missing {missing})")
                out.append(rec)
    return out


class Replay:
    """Replays one rank's records of a trace through a Runtime. Buffers are
    created once (`prepare`), so `step()` is the timed unit; `fill(seed)`
    writes fresh inputs. Outputs stay on the object for verification."""

    def __init__(self, rt, records: List[dict], rank: int, device, backend_map: Optional[Dict] = None):
        import torch

        from .core import Buffer, DType

        self.rt, self.rank, self.torch, self.Buffer = rt, rank, torch, Buffer
        self.map = backend_map or {}
        world = rt.world_size
        by_rank: Dict[int, List[dict]] = {}
        for rec in records:
            by_rank.setdefault(int(rec["rank"]), []).append(rec)
        for v in by_rank.values():
            v.sort(key=lambda x: x["seq"])
        self.mine = by_rank[rank]
        if any(len(by_rank.get(q, [])) != len(self.mine) for q in range(world)):
            raise ValueError("trace: every rank must have the same number of records")
        self.ops = []
        for i, rec in enumerate(self.mine):
            op, dt = rec["op"], DType.from_name(rec.get("dtype", "f32"))
            td = dt.torch_dtype
            peers = [by_rank[q][i] for q in range(world)]
            if any(p_["op"] != op for p_ in peers):
                raise ValueError(f"trace: ranks disagree on op {i}")
            be = self.map.get(rec["backend"], rec["backend"])
            if op == "all_to_allv":
                sc = [int(x) for x in rec["scounts"]]
                rc = [int(peers[j]["scounts"][rank]) for j in range(world)]
                ent = {"op": op, "be": be, "sc": sc, "rc": rc,
                       "sd": _packed(sc), "rd": _packed(rc),
                       "inp": torch.empty(sum(sc), dtype=td, device=device),
                       "out": torch.empty(sum(rc), dtype=td, device=device)}
            elif op == "all_reduce":
                n = int(rec.get("count", rec["bytes"] // dt.size_bytes))
                ent = {"op": op, "be": be, "async": bool(rec.get("async")),
                       "buf": torch.empty(n, dtype=td, device=device)}
            elif op in ("all_gatherv", "gatherv"):
                rcs = [int(x) for x in rec["rcounts"]]
                root = int(rec.get("root", 0))
                ent = {"op": op, "be": be, "rc": rcs, "dp": _packed(rcs), "root": root,
                       "inp": torch.empty(rcs[rank], dtype=td, device=device),
                       "out": (torch.empty(sum(rcs), dtype=td, device=device)
                               if op == "all_gatherv" or rank == root else None)}
            else:
                raise ValueError(f"trace: op {op!r} is not replayable")
            ent["dtype"] = dt
            self.ops.append(ent)

    def fill(self, seed: int) -> None:
        g = self.torch.Generator(device=self.ops[0].get("inp", self.ops[0].get("buf")).device)
        g.manual_seed(seed * 1000 + self.rank)
        for ent in self.ops:
            t = ent.get("inp", ent.get("buf"))
            if t.is_floating_point():
                t.normal_(generator=g)
            else:
                t.random_(-1000, 1000, generator=g)

    def step(self):
        rt, B = self.rt, self.Buffer
        handles = []
        for ent in self.ops:
            op = ent["op"]
            if op == "all_to_allv":
                rt.all_to_allv(ent["be"], B(ent["out"]), B(ent["inp"]), ent["sc"], ent["rc"],
                               ent["sd"], ent["rd"])
            elif op == "all_reduce":
                h = rt.all_reduce(ent["be"], B(ent["buf"]), async_op=ent["async"])
                if ent["async"]:
                    handles.append(h)
            elif op == "all_gatherv":
                rt.all_gatherv(ent["be"], B(ent["out"]), B(ent["inp"]), ent["rc"], ent["dp"])
            else:
                rt.gatherv(ent["be"], B(ent["out"]) if ent["out"] is not None else None,
                           B(ent["inp"]), ent["root"], ent["rc"], ent["dp"])
        for h in handles:
            rt.wait(h)
        return handles


def _packed(counts):
    out, o = [], 0
    for c in counts:
        out.append(o)
        o += c
    return out

"""Loaders for the committed golden fixtures (tests/golden/, generated from
the reference by oracle/make_golden.py) and the oracle's answer for each
case. Shared by the CPU oracle tests and the GPU parity worker."""

from __future__ import annotations

import base64
import json
from pathlib import Path
from typing import List, Optional

import numpy as np

from oracle import seqref

GOLDEN = Path(__file__).resolve().parent / "golden"
NPD = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64, "u8": np.uint8}


def dec(d) -> np.ndarray:
    return np.frombuffer(base64.b64decode(d["b64"]), dtype=np.dtype(d["dtype"])).copy()


def load_selftest(p: int) -> list:
    f = GOLDEN / f"selftest_p{p}.json"
    if not f.exists():
        return []
    doc = json.loads(f.read_text())
    assert doc["world_size"] == p
    return doc["cases"]


def selftest_arrays(case: dict, field: str) -> List[np.ndarray]:
    dt = NPD[case["dtype"]]
    return [np.asarray(x, dtype=dt) for x in case[field]]


def selftest_oracle(case: dict, p: int) -> List[Optional[np.ndarray]]:
    """Oracle output per rank for one selftest-dump case (cli.py:155-343)."""
    op, dt = case["op"], NPD[case["dtype"]]
    root = case["root"]
    if op in ("scatter", "scatterv"):
        src = np.asarray(case["root_input"], dtype=dt)
        if op == "scatter":
            return seqref.scatter(src, p)
        return seqref.scatterv(src, case["scounts"], case["displs"])
    ins = selftest_arrays(case, "inputs")
    if op == "all_reduce":
        return seqref.all_reduce(ins, "sum")
    if op == "reduce":
        return seqref.reduce(ins, "sum", root)
    if op == "bcast":
        return seqref.bcast(ins, root)
    if op == "all_gather":
        return seqref.all_gather(ins)
    if op == "gather":
        return seqref.gather(ins, root)
    if op == "reduce_scatter":
        return seqref.reduce_scatter(ins, "sum")
    if op == "all_to_all_single":
        return seqref.all_to_all_single(ins)
    if op == "all_to_all":
        m = case["count"]
        blocks = [[x[j * m:(j + 1) * m] for j in range(p)] for x in ins]
        outs = seqref.all_to_all(blocks)
        return [np.concatenate(o) if o else np.zeros(0, dt) for o in outs]
    if op == "gatherv":
        return seqref.gatherv(ins, root, case["rcounts"], case["displs"])
    if op == "all_gatherv":
        return seqref.all_gatherv(ins, case["rcounts"], case["displs"])
    if op == "all_to_allv":
        sc = case["scounts"]
        return seqref.all_to_allv(ins, sc, case["sdispls"], case["rdispls"],
                                  out_counts=[sum(sc[j][r] for j in range(p)) for r in range(p)])
    raise KeyError(op)


def load_live() -> list:
    f = GOLDEN / "live_cases.json"
    return json.loads(f.read_text())["cases"] if f.exists() else []


def load_trunc16() -> dict:
    f = GOLDEN / "trunc16.json"
    return json.loads(f.read_text()) if f.exists() else {}


def trunc16_oracle(c: dict) -> list:
    """Oracle output per rank for one compressed (trunc16) record: rank r sees
    trunc16 of every other rank's data and its own data exactly."""
    p, out = c["p"], []
    for r in range(p):
        cc = dict(c)
        if c["kind"] == "all_to_all":
            cc["inputs"] = [[enc_like(seqref.trunc16(dec(b)) if q != r else dec(b)) for b in row]
                            for q, row in enumerate(c["inputs"])]
        elif c["kind"] in ("scatter", "scatterv"):  # inputs[0] holds the root's data
            x = dec(c["inputs"][0])
            cc["inputs"] = [enc_like(seqref.trunc16(x) if r != c["root"] else x)] + c["inputs"][1:]
        else:
            cc["inputs"] = [enc_like(seqref.trunc16(dec(x)) if q != r else dec(x))
                            for q, x in enumerate(c["inputs"])]
        cc["op"] = "sum"
        out.append(live_oracle(cc)[r])
    return out


def enc_like(a: np.ndarray) -> dict:
    import base64

    a = np.ascontiguousarray(a)
    return {"dtype": a.dtype.str, "b64": base64.b64encode(a.tobytes()).decode()}


def live_oracle(c: dict) -> list:
    """Oracle output per rank for one live_cases.json record."""
    kind, p, root, op = c["kind"], c["p"], c["root"], c["op"]
    if kind == "all_to_all":
        ins = [[dec(b) for b in row] for row in c["inputs"]]
        return seqref.all_to_all(ins)
    ins = [dec(x) for x in c["inputs"]]
    if kind == "all_reduce":
        return seqref.all_reduce(ins, op)
    if kind == "reduce":
        return seqref.reduce(ins, op, root)
    if kind == "reduce_scatter":
        return seqref.reduce_scatter(ins, op)
    if kind == "bcast":
        return seqref.bcast(ins, root)
    if kind == "all_gather":
        return seqref.all_gather(ins)
    if kind == "all_gatherv":
        return seqref.all_gatherv(ins, c["counts"], c["displs"])
    if kind == "gather":
        return seqref.gather(ins, root)
    if kind == "gatherv":
        return seqref.gatherv(ins, root, c["counts"], c["displs"])
    if kind == "scatter":
        return seqref.scatter(ins[0], p)
    if kind == "scatterv":
        return seqref.scatterv(ins[0], c["counts"], c["displs"])
    if kind == "all_to_all_single":
        return seqref.all_to_all_single(ins)
    if kind == "all_to_allv":
        sc = c["sc_matrix"]
        return seqref.all_to_allv(ins, sc, c["sdispls"], c["rdispls"],
                                  out_counts=[sum(sc[j][r] for j in range(p)) for r in range(p)])
    raise KeyError(kind)

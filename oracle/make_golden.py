"""Generate golden fixtures from the REFERENCE implementation (test infra).

Run here, where /root/reference exists (the GPU box never reads it):

    python oracle/make_golden.py            # writes tests/golden/*.json

Fixtures:
  selftest_p{2,4,8}.json  the reference CLI's own parity dump
                          (`mcrdl launch -n P selftest --out`, cli.py:476-491):
                          78 cases per world, all kinds, f32/i64, counts 0/1/5.
  live_cases.json         seeded cases (reference tests/cases.py make_case
                          input distributions) executed by the reference's LIVE
                          collective algorithms (run_thread_world, naive =
                          ascending-fold policy and the default policy), every
                          collective kind x p in {2,3,5,8} x {f32,i64,u8} x
                          counts {0,1,7,64}, plus f32 all_reduce sums of 1000
                          elements at p=4. Arrays are stored as base64 raw
                          little-endian bytes so floats are exact.
  cfg5_fusion.json        the reference's FusionManager (middleware.py:241-344)
                          on the cfg5 step's posting order: the
                          14 DLRM MLP gradients posted async on a fusion
                          backend FusionConfig(B = 1 MiB, T = 5 s so grouping
                          is decided by B alone), p = 2, naive policy. Records
                          every flush (seq order, member count) and the
                          posting indices that were not eligible, from the
                          reference's own CommLog.
  trunc16.json            the reference's Trunc16Codec (middleware.py:43-75):
                          decode(encode(x)) of specials + seeded normals, and
                          live COMPRESSED collectives (CompressionConfig on the
                          inproc backend) for every compressible kind at p=3.

    python oracle/make_golden.py trunc16    # only trunc16.json
    python oracle/make_golden.py cfg5       # only cfg5_fusion.json
"""

from __future__ import annotations

import base64
import importlib.util
import json
import os
import subprocess
import sys
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = ROOT / "tests" / "golden"


def enc(a) -> dict:
    a = np.ascontiguousarray(a)
    return {"dtype": a.dtype.str, "b64": base64.b64encode(a.tobytes()).decode()}


def selftest_dumps() -> None:
    env = dict(os.environ, PYTHONPATH=str(REF_SRC))
    for p in (2, 4, 8):
        out = OUT / f"selftest_p{p}.json"
        subprocess.run([sys.executable, "-m", "mcrdl", "launch", "-n", str(p), "selftest",
                        "--out", str(out)], env=env, check=True, cwd="/tmp")
        print("wrote", out)


def live_cases() -> None:
    sys.path.insert(0, str(REF_SRC))
    sys.path.insert(0, str(REF_TESTS))
    import mcrdl
    from mcrdl import AlgorithmPolicy, BackendConfig, CommOpKind, DType, run_thread_world

    spec = importlib.util.spec_from_file_location("ref_cases", REF_TESTS / "cases.py")
    cases = importlib.util.module_from_spec(spec)
    sys.modules["ref_cases"] = cases
    spec.loader.exec_module(cases)

    records = []

    def run(case, policy):
        def entry(rt, rank):
            rt.init([BackendConfig("a", transport="inproc", policy=policy)])
            req = case.build_request(rank, "a")
            rt.post(req)
            res = case.result_of(rank, req)
            rt.finalize()
            return res

        return run_thread_world(case.p, entry, timeout=60.0)

    def pack_result(kind, res):
        if res is None:
            return None
        if kind is CommOpKind.all_to_all:
            return [enc(x) for x in res]
        return enc(res)

    for kind in cases.COLLECTIVE_KINDS:
        for p in (2, 3, 5, 8):
            for dtype in (DType.f32, DType.i64, DType.u8):
                for count in (0, 1, 7, 64):
                    seed = zlib.crc32(f"{kind.value}|{p}|{dtype.name}|{count}".encode()) & 0xFFFF
                    case = cases.make_case(kind, dtype, count, p, seed=seed)
                    policy = AlgorithmPolicy.naive()
                    res = run(case, policy)
                    rec = {
                        "kind": kind.value, "p": p, "dtype": dtype.name, "count": count,
                        "root": case.root, "op": case.op.value, "policy": "naive",
                        "counts": case.counts, "displs": case.displs,
                        "sc_matrix": case.sc_matrix, "sdispls": case.sdispls,
                        "rdispls": case.rdispls,
                        "inputs": ([[enc(b) for b in row] for row in case.inputs]
                                   if kind is CommOpKind.all_to_all
                                   else [enc(x) for x in case.inputs]),
                        "outputs": [pack_result(kind, r) for r in res],
                    }
                    records.append(rec)
    # float sums with reduction-order sensitivity: naive (ascending) must be
    # bit-exact with the oracle; ring is recorded too (within tolerance only).
    for policy_name in ("naive", "ring"):
        for seed in range(4):
            case = cases.make_case(CommOpKind.all_reduce, DType.f32, 1000, 4, seed=100 + seed)
            pol = AlgorithmPolicy.naive() if policy_name == "naive" else AlgorithmPolicy(
                {CommOpKind.all_reduce: "ring"})
            res = run(case, pol)
            records.append({
                "kind": "all_reduce", "p": 4, "dtype": "f32", "count": 1000, "root": case.root,
                "op": "sum", "policy": policy_name, "counts": None, "displs": None,
                "sc_matrix": None, "sdispls": None, "rdispls": None,
                "inputs": [enc(x) for x in case.inputs],
                "outputs": [enc(r) for r in res],
            })
    out = OUT / "live_cases.json"
    out.write_text(json.dumps({"generator": "oracle/make_golden.py",
                               "reference": "mcrdl 0.1.0 (/root/reference/pkg)",
                               "cases": records}))
    print("wrote", out, len(records), "cases")


def trunc16_cases() -> None:
    sys.path.insert(0, str(REF_SRC))
    sys.path.insert(0, str(REF_TESTS))
    from mcrdl import AlgorithmPolicy, BackendConfig, CommOpKind, DType, run_thread_world
    from mcrdl.middleware import COMPRESSIBLE_KINDS, CompressionConfig, Trunc16Codec

    spec = importlib.util.spec_from_file_location("ref_cases", REF_TESTS / "cases.py")
    cases = importlib.util.module_from_spec(spec)
    sys.modules["ref_cases"] = cases
    spec.loader.exec_module(cases)

    codec = Trunc16Codec()
    special = np.array([0.0, -0.0, 1.0, -1.5, 3.14159265, np.inf, -np.inf, np.nan,
                        np.finfo(np.float32).max, np.finfo(np.float32).tiny,
                        np.float32(1.4e-45), -2.5e-42, 65504.0, 1e-3, -7.77e20], dtype=np.float32)
    rng = np.random.default_rng(7)
    x = np.concatenate([special, rng.standard_normal(1000).astype(np.float32) * 1e3])
    roundtrip = codec.decode(codec.encode(x), x.size)

    records = []
    for kind in sorted(COMPRESSIBLE_KINDS, key=lambda k: k.value):
        for count in (1, 7, 64):
            seed = zlib.crc32(f"trunc16|{kind.value}|{count}".encode()) & 0xFFFF
            case = cases.make_case(kind, DType.f32, count, 3, seed=seed)

            def entry(rt, rank, case=case):
                rt.init([BackendConfig("a", transport="inproc", policy=AlgorithmPolicy.naive(),
                                       compression=CompressionConfig())])
                req = case.build_request(rank, "a")
                rt.post(req)
                res = case.result_of(rank, req)
                rt.finalize()
                return res

            res = run_thread_world(case.p, entry, timeout=60.0)
            records.append({
                "kind": kind.value, "p": case.p, "dtype": "f32", "count": count,
                "root": case.root, "counts": case.counts, "displs": case.displs,
                "sc_matrix": case.sc_matrix, "sdispls": case.sdispls, "rdispls": case.rdispls,
                "inputs": ([[enc(b) for b in row] for row in case.inputs]
                           if kind is CommOpKind.all_to_all else [enc(v) for v in case.inputs]),
                "outputs": [None if r is None else
                            ([enc(v) for v in r] if kind is CommOpKind.all_to_all else enc(r))
                            for r in res],
            })
    out = OUT / "trunc16.json"
    out.write_text(json.dumps({"generator": "oracle/make_golden.py trunc16",
                               "reference": "mcrdl 0.1.0 Trunc16Codec + CompressionConfig",
                               "roundtrip": {"input": enc(x), "output": enc(roundtrip)},
                               "cases": records}))
    print("wrote", out, len(records), "compressed cases")


CFG5_MLP = [6656, 512, 262144, 512, 65536, 128, 490496, 1024, 1048576, 1024, 1048576, 1024,
            1024, 1]


def cfg5_fusion() -> None:
    sys.path.insert(0, str(REF_SRC))
    from mcrdl import AlgorithmPolicy, BackendConfig, Buffer, DType, run_thread_world
    from mcrdl.middleware import FusionConfig

    def entry(rt, rank):
        rt.init([BackendConfig("f", transport="inproc", policy=AlgorithmPolicy.naive(),
                               fusion=FusionConfig(max_bytes=1 << 20, max_wait=5.0))])
        bufs = [Buffer.from_values(DType.f32, np.full(n, rank + 1, dtype=np.float32))
                for n in CFG5_MLP]
        hs = [rt.all_reduce("f", b, async_op=True) for b in bufs]
        for h in hs:
            rt.wait(h)
        rt.synchronize()
        recs = sorted(rt.comm_log.records(), key=lambda r: r.seq)
        out = [{"seq": r.seq, "fused": r.fused, "members": r.members, "bytes": r.bytes}
               for r in recs if r.op == "all_reduce"]
        ok = all(np.all(b.array == 3.0) for b in bufs)
        rt.finalize()
        return out, ok

    res = run_thread_world(2, entry, timeout=60.0)
    recs, ok = res[0]
    assert ok and res[1][0] == recs, "reference ranks disagree"
    fused = [r["members"] for r in recs if r["fused"]]
    eligible = [i for i, n in enumerate(CFG5_MLP) if 4 * n <= (1 << 20)]
    doc = {"generator": "oracle/make_golden.py cfg5",
           "reference": "mcrdl 0.1.0 FusionManager (run_thread_world p=2, inproc, naive)",
           "posting_order_elems": CFG5_MLP, "dtype": "f32",
           "fusion": {"max_bytes": 1 << 20, "max_wait_s": 5.0},
           "eligible_indices": eligible,
           "flush_members": fused,
           "unfused_records": sum(1 for r in recs if not r["fused"]),
           "records": recs}
    out = OUT / "cfg5_fusion.json"
    out.write_text(json.dumps(doc, indent=1))
    print("wrote", out, "flushes", fused)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    if sys.argv[1:] == ["cfg5"]:
        cfg5_fusion()
    elif sys.argv[1:] == ["trunc16"]:
        trunc16_cases()
    else:
        selftest_dumps()
        live_cases()
        trunc16_cases()
        cfg5_fusion()

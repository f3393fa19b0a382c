"""cfg5 step trace: LogRecord-schema JSONL that the CommLog
loader and report() read unchanged, carrying what a replay needs."""

import os
from pathlib import Path

import pytest

from paper_2303_08374_b200 import trace
from paper_2303_08374_b200.middleware import LogRecord, report

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("p", [2, 4, 8])
def test_cfg5_trace_round_trip_and_schema(tmp_path, p):
    recs = trace.cfg5_trace(p)
    assert len(recs) == 18 * p
    path = tmp_path / "t.jsonl"
    trace.write_jsonl(recs, str(path))
    assert trace.load_jsonl(str(path)) == recs
    lines = path.read_text().splitlines()
    logs = [LogRecord.from_json(x) for x in lines]
    assert {x.op for x in logs} == {"all_to_allv", "all_reduce", "all_gatherv", "gatherv"}
    bd = report([str(path)])
    assert bd.rows
    for r in range(p):  # a2av counts are consistent across ranks: what r sends j receives
        mine = [x for x in recs if x["rank"] == r]
        assert mine[-1]["scounts"] == [recs[j * 18]["scounts"][r] for j in range(p)]


def test_committed_p8_trace_matches_generator():
    committed = trace.load_jsonl(str(ROOT / "profiles" / "cfg5_trace_p8.jsonl"))
    assert committed == trace.cfg5_trace(8)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not present")
def test_reference_commlog_reads_the_trace(tmp_path):
    import importlib.util
    import sys

    src = "/root/reference/pkg/src/mcrdl"
    spec = importlib.util.spec_from_file_location("mcrdl_ref_trace", f"{src}/__init__.py",
                                                  submodule_search_locations=[src])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["mcrdl_ref_trace"] = mod
    spec.loader.exec_module(mod)
    from mcrdl_ref_trace.middleware import LogRecord as RefLogRecord

    path = tmp_path / "t.jsonl"
    trace.write_jsonl(trace.cfg5_trace(4), str(path))
    recs = [RefLogRecord.from_json(x) for x in path.read_text().splitlines()]
    assert len(recs) == 72 and recs[0].op == "all_to_allv"

"""Tuning table (schema + per-size algorithm), routing and the tuner's
winner/table builder (reference dispatch.py, tuner.py semantics)."""

import json

import numpy as np
import pytest

from paper_2303_08374_b200 import Buffer, CommOpKind, CommRequest, ReduceOp, TuningTable
from paper_2303_08374_b200.dispatch import (TableEntry, bucket, load_table, message_bytes, route,
                                            save_table)
from paper_2303_08374_b200.errors import (EmptySamples, MonotonicityError, ParseError,
                                          UnroutableRequest)
from paper_2303_08374_b200.tuner import (BenchSample, SkippedCombination, build_table, parse_sizes,
                                         winner_grid)

AR, A2AV = CommOpKind.all_reduce, CommOpKind.all_to_allv


def test_table_roundtrip_with_algorithm(tmp_path):
    t = TuningTable({AR: {8: [TableEntry(262144, "nvl", "one_shot"),
                              TableEntry(1 << 30, "nvl", "two_shot")]}}, system="b200")
    p = tmp_path / "t.json"
    save_table(t, str(p))
    doc = json.loads(p.read_text())
    assert doc["tables"]["all_reduce"]["8"][0]["algorithm"] == "one_shot"
    t2 = load_table(str(p))
    assert t2.algorithm_for(AR, 8, 1000, "nvl") == "one_shot"
    assert t2.algorithm_for(AR, 8, 1 << 20, "nvl") == "two_shot"
    assert t2.algorithm_for(AR, 8, 1 << 40, "nvl") == "two_shot"  # beyond last -> last
    assert t2.algorithm_for(AR, 8, 1000, "other") is None


def test_reference_table_without_algorithm_loads():
    # PAPER.md:654-673 Table II style, reference schema (no algorithm key)
    doc = {"version": 1, "system": "thetagpu", "tables": {"all_gather": {"32": [
        {"max_bytes": 2048, "backend": "mv2"}, {"max_bytes": 8192, "backend": "nccl"},
        {"max_bytes": 32768, "backend": "sccl"}]}}}
    t = TuningTable.from_dict(doc)
    assert t.lookup(CommOpKind.all_gather, 32, 4096) == "nccl"
    assert t.lookup(CommOpKind.all_gather, 64, 100) == "mv2"  # nearest smaller world
    assert t.lookup(CommOpKind.all_gather, 16, 100) is None
    assert t.lookup_entry(CommOpKind.all_gather, 32, 1).algorithm is None


def test_table_validation_and_merge():
    with pytest.raises(MonotonicityError):
        TuningTable({AR: {2: [TableEntry(8, "a"), TableEntry(8, "b")]}})
    with pytest.raises(ParseError):
        TuningTable.from_dict({"tables": {"all_reduce": {"2": [{"backend": "a"}]}}})
    with pytest.raises(ParseError):
        TuningTable.from_dict({"tables": {"nope": {}}})
    merged = TuningTable.merge_runs([TableEntry(8, "a", "one_shot"), TableEntry(16, "a", "one_shot"),
                                     TableEntry(32, "a", "two_shot"), TableEntry(64, "a", "two_shot")])
    assert merged == [TableEntry(16, "a", "one_shot"), TableEntry(64, "a", "two_shot")]


def test_route_rules():
    t = TuningTable({AR: {2: [TableEntry(100, "x"), TableEntry(1000, "y")]}})
    assert route(t, AR, 2, 50, ["y", "x"]) == "x"
    assert route(t, AR, 2, 500, ["y", "x"]) == "y"
    assert route(None, AR, 2, 50, ["y", "x"]) == "y"
    assert route(t, A2AV, 2, 50, ["y", "x"]) == "y"  # untuned op -> first registered
    with pytest.raises(UnroutableRequest):
        route(t, AR, 2, 50, ["y"])
    with pytest.raises(UnroutableRequest):
        route(t, AR, 2, 50, [])
    assert bucket(5) == 8 and bucket(1 << 40) == 1 << 26


def test_message_bytes_canonical_sizes():
    b = Buffer(np.zeros(10, np.float32))
    assert message_bytes(CommRequest(AR, input=b, output=b, op=ReduceOp.sum), 4) == 40
    r = CommRequest(A2AV, input=Buffer(np.zeros(6, np.int64)), output=Buffer(np.zeros(6, np.int64)),
                    scounts=[1, 2, 3], rcounts=[3, 2, 1], sdispls=[0, 1, 3], rdispls=[0, 3, 5])
    assert message_bytes(r, 3) == 48
    s = CommRequest(CommOpKind.scatter, input=None, output=Buffer(np.zeros(5, np.float32)), root=0)
    assert message_bytes(s, 4) == 80


def test_message_bytes_device_counts_route_by_capacity():
    torch = pytest.importorskip("torch")
    c = torch.tensor([1, 2, 3])
    r = CommRequest(A2AV, input=Buffer(np.zeros(6, np.int64)), output=Buffer(np.zeros(6, np.int64)),
                    scounts=c, rcounts=c, sdispls=c, rdispls=c)
    assert message_bytes(r, 3) == 48


def samples_for(op, world, sizes, alpha_beta):
    out = []
    for size in sizes:
        for algo, (a, b) in alpha_beta.items():
            t = a + b * size
            out.append(BenchSample(op, "nvl", world, size, [t * 1.01, t, t * 0.99], algo))
    return out


def test_winner_grid_and_table_crossover():
    sizes = [2 ** k for k in range(3, 28)]
    # one_shot: 8 us + 1/300 GB/s ; two_shot: 20 us + 1/600 GB/s -> crossover 7.2 MB
    s = samples_for(AR, 8, sizes, {"one_shot": (8e-6, 1 / 300e9), "two_shot": (20e-6, 1 / 600e9)})
    grid = winner_grid(s)
    assert grid[(AR, 8, 8)] == ("nvl", "one_shot")
    assert grid[(AR, 8, 1 << 27)] == ("nvl", "two_shot")
    t = build_table(s)
    ents = t.tables[AR][8]
    assert [e.algorithm for e in ents] == ["one_shot", "two_shot"]
    assert ents[0].max_bytes == 1 << 22  # last size where one_shot wins
    assert t.algorithm_for(AR, 8, 5 << 20, "nvl") == "two_shot"
    assert t.algorithm_for(AR, 8, 3 << 20, "nvl") == "one_shot"


def test_winner_grid_requires_every_cell():
    s = samples_for(AR, 2, [8, 16], {"one_shot": (1e-6, 0)})
    skipped = [SkippedCombination(A2AV, "nvl", 2, n, "unsupported") for n in (8, 16)]
    grid = winner_grid(s, skipped=skipped)
    assert (A2AV, 2, 8) not in grid and (AR, 2, 16) in grid
    with pytest.raises(EmptySamples):  # a cell neither measured nor skipped
        winner_grid(s, skipped=skipped[:1])
    with pytest.raises(EmptySamples):
        winner_grid([])
    with pytest.raises(EmptySamples):
        winner_grid(s + [BenchSample(A2AV, "nvl", 2, 16, [1.0], "direct_write")])


def test_build_table_merges_worlds_into_base():
    base = build_table(samples_for(AR, 2, [8, 16], {"one_shot": (1e-6, 0)}))
    t = build_table(samples_for(AR, 8, [8, 16], {"two_shot": (1e-6, 0)}), base=base)
    assert set(t.tables[AR]) == {2, 8}


def test_parse_sizes():
    assert parse_sizes("8:64") == [8, 16, 32, 64]
    assert parse_sizes("1K,4,1M") == [4, 1024, 1 << 20]
    assert parse_sizes("8:1G")[-1] == 1 << 30


# ---------------------------------------------------- shipped algorithm table

def test_shipped_table_drives_auto_rows():
    """The measured table shipped with the package is the default source of
    AUTO (Runtime.algorithm_table -> install_tuning -> mcrdl_comm_set_tuning);
    p = 8 has no sweep yet and takes the nearest measured world's cells."""
    import json

    from paper_2303_08374_b200 import dispatch
    from paper_2303_08374_b200.core import CommOpKind

    t = dispatch.default_algorithm_table()
    assert t is not None
    rows2 = dispatch.algorithm_rows(t, CommOpKind.all_reduce, 2, "any_name")
    rows4 = dispatch.algorithm_rows(t, CommOpKind.all_reduce, 4, "any_name")
    assert [a for _, a in rows2][:1] == ["one_shot"] and rows2[-1][1] == "two_shot"
    assert [m for m, _ in rows4] == sorted(m for m, _ in rows4)
    assert dispatch.algorithm_rows(t, CommOpKind.all_reduce, 8, "x") == rows4
    doc = json.loads(dispatch.SHIPPED_TABLE.read_text())
    assert "8" in doc["untuned_worlds"]


def test_algorithm_rows_respect_backend_names():
    from paper_2303_08374_b200 import dispatch
    from paper_2303_08374_b200.core import CommOpKind

    doc = {"tables": {"all_reduce": {"2": [
        {"max_bytes": 1024, "backend": "mine", "algorithm": "one_shot"},
        {"max_bytes": 1 << 30, "backend": "mine", "algorithm": "two_shot"}]}}}
    t = dispatch.TuningTable.from_dict(doc)
    assert dispatch.algorithm_rows(t, CommOpKind.all_reduce, 2, "mine") == [
        (1024, "one_shot"), (1 << 30, "two_shot")]
    # a cell routed to another backend is not this backend's algorithm table
    assert dispatch.algorithm_rows(t, CommOpKind.all_reduce, 2, "other") == []
    assert dispatch.algorithm_rows(t, CommOpKind.all_reduce, 1, "mine") == []
    assert dispatch.algorithm_rows(None, CommOpKind.all_reduce, 2, "mine") == []


def test_runtime_algorithm_table_default_and_override(tmp_path, monkeypatch):
    from paper_2303_08374_b200 import Runtime, dispatch

    monkeypatch.delenv("MCRDL_TUNING_TABLE", raising=False)
    rt = Runtime(0, 1)
    assert rt.algorithm_table is not None and rt.tuning_table is None
    p = tmp_path / "t.json"
    p.write_text('{"tables": {"all_reduce": {"2": [{"max_bytes": 64, "backend": "nvl", '
                 '"algorithm": "two_shot"}]}}}')
    monkeypatch.setenv("MCRDL_TUNING_TABLE", str(p))
    rt = Runtime(0, 1)
    assert rt.algorithm_table is rt.tuning_table
    monkeypatch.setenv("MCRDL_ALGO_TABLE", "off")
    assert Runtime(0, 1).algorithm_table is None


def test_shipped_table_bcast_rows_end_on_chain():
    """bcast: push for small messages, then (p = 4) NVLS, then the pipelined
    chain for large ones; every shipped algorithm name is one the policy
    layer accepts for its op."""
    from paper_2303_08374_b200 import dispatch
    from paper_2303_08374_b200.collectives import ALGORITHMS
    from paper_2303_08374_b200.core import CommOpKind

    t = dispatch.default_algorithm_table()
    for w in (2, 4):
        rows = dispatch.algorithm_rows(t, CommOpKind.bcast, w, "nvl")
        assert rows[0][1] == "direct_write" and rows[-1][1] == "chain", rows
        assert all(a in ALGORITHMS[CommOpKind.bcast] for _, a in rows)
    for kind in (CommOpKind.all_reduce, CommOpKind.all_to_allv, CommOpKind.all_gatherv):
        for w in (2, 4):
            assert all(a in ALGORITHMS[kind] for _, a in dispatch.algorithm_rows(t, kind, w, "nvl"))

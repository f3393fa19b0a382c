"""Host-side API types: validation (reference core.py:421-566 semantics),
buffers, dtypes, handles, algorithm policy."""

import numpy as np
import pytest

from paper_2303_08374_b200 import (AlgorithmPolicy, Buffer, CommOpKind, CommRequest, DType,
                                   ReduceOp, Runtime, WorkHandle, element_reduce, validate)
from paper_2303_08374_b200.collectives import canonical, even_segments, bus_factor
from paper_2303_08374_b200.core import HandleState
from paper_2303_08374_b200.errors import (DuplicateBackend, UnknownTransport, UnsupportedOperation,
                                          ValidationError)


def B(n, dt=np.float32):
    return Buffer(np.zeros(n, dtype=dt))


def good_requests(p=3):
    x = B(6)
    return [
        CommRequest(CommOpKind.all_reduce, input=x, output=x, op=ReduceOp.sum),
        CommRequest(CommOpKind.reduce, input=x, output=x, op=ReduceOp.max, root=2),
        CommRequest(CommOpKind.bcast, output=x, root=0),
        CommRequest(CommOpKind.all_gather, input=B(2), output=B(2 * p)),
        CommRequest(CommOpKind.gather, input=B(2), output=None, root=1),
        CommRequest(CommOpKind.gatherv, input=B(1), output=B(4), root=0, rcounts=[1, 2, 1],
                    rdispls=[0, 1, 3]),
        CommRequest(CommOpKind.all_gatherv, input=B(1), output=B(4), rcounts=[1, 2, 1],
                    rdispls=[0, 1, 3]),
        CommRequest(CommOpKind.scatter, input=B(6), output=B(2), root=0),
        CommRequest(CommOpKind.scatterv, input=B(3), output=B(1), root=0, scounts=[1, 1, 1],
                    sdispls=[0, 1, 2]),
        CommRequest(CommOpKind.reduce_scatter, input=B(6), output=B(2), op=ReduceOp.sum),
        CommRequest(CommOpKind.all_to_all_single, input=B(6), output=B(6)),
        CommRequest(CommOpKind.all_to_all, input=[B(1)] * p, output=[B(1)] * p),
        CommRequest(CommOpKind.all_to_allv, input=B(3), output=B(3), scounts=[1, 1, 1],
                    rcounts=[1, 1, 1], sdispls=[0, 1, 2], rdispls=[2, 1, 0]),
    ]


def test_validate_accepts_well_formed_requests():
    for req in good_requests():
        validate(req, 3, 0)


@pytest.mark.parametrize("mutate", [
    lambda r: setattr(r, "op", None) if r.kind is CommOpKind.all_reduce else setattr(r, "root", 7),
    lambda r: setattr(r, "root", 5),
    lambda r: setattr(r, "scounts", [1, 1, 1]) if r.kind is not CommOpKind.all_to_allv
    and r.kind is not CommOpKind.scatterv else setattr(r, "scounts", [-1, 2, 2]),
])
def test_validate_rejects_mutations(mutate):
    rejected = 0
    for req in good_requests():
        mutate(req)
        try:
            validate(req, 3, 0)
        except ValidationError:
            rejected += 1
    assert rejected >= 10


def test_vectored_overlap_and_sum_checks():
    with pytest.raises(ValidationError, match="overlap"):
        validate(CommRequest(CommOpKind.all_gatherv, input=B(2), output=B(4), rcounts=[2, 2, 0],
                             rdispls=[0, 1, 4]), 3, 0)
    with pytest.raises(ValidationError):
        validate(CommRequest(CommOpKind.all_gatherv, input=B(2), output=B(5), rcounts=[2, 2, 0],
                             rdispls=[0, 2, 4]), 3, 0)
    with pytest.raises(ValidationError, match="rcounts\\[0\\]"):
        validate(CommRequest(CommOpKind.gatherv, input=B(3), output=B(4), root=0,
                             rcounts=[2, 2, 0], rdispls=[0, 2, 4]), 3, 0)
    # root must supply the output (core.py:513-527)
    with pytest.raises(ValidationError):
        validate(CommRequest(CommOpKind.gatherv, input=B(2), output=None, root=0,
                             rcounts=[2, 2, 0], rdispls=[0, 2, 4]), 3, 0)


def test_device_count_tensors_skip_host_sums():
    torch = pytest.importorskip("torch")
    c = torch.tensor([1, 1, 1])
    validate(CommRequest(CommOpKind.all_to_allv, input=B(3), output=B(3), scounts=c,
                         rcounts=c, sdispls=c, rdispls=c), 3, 0)
    with pytest.raises(ValidationError):
        validate(CommRequest(CommOpKind.all_to_allv, input=B(3), output=B(3), scounts=c[:2],
                             rcounts=c, sdispls=c, rdispls=c), 3, 0)


def test_buffer_wraps_numpy_and_torch_without_copy():
    torch = pytest.importorskip("torch")
    a = np.arange(4, dtype=np.int64)
    b = Buffer(a)
    assert b.array is a and b.dtype is DType.i64 and b.nbytes == 32 and not b.is_device
    t = torch.zeros(5, dtype=torch.bfloat16)
    bt = Buffer(t)
    assert bt.dtype is DType.bf16 and bt.nbytes == 10 and bt.is_tensor and not bt.is_device
    with pytest.raises(ValidationError):
        Buffer(np.zeros((2, 2), np.float32))
    with pytest.raises(ValidationError):
        Buffer(np.zeros(4, np.float32)[::2])
    with pytest.raises(ValidationError):
        Buffer(np.zeros(4, np.complex64))
    assert Buffer.zeros(DType.bf16, 3).dtype is DType.bf16


def test_buffer_checkout_guard():
    b = B(2)
    b._checkout()
    with pytest.raises(ValidationError, match="in flight"):
        b._checkout()
    b._checkin()
    b._checkout()


def test_handle_state_machine_forward_only():
    h = WorkHandle("x")
    assert h.state is HandleState.posted and not h.test()
    h.mark_in_progress()
    h.complete()
    assert h.test() and h.state is HandleState.complete
    with pytest.raises(RuntimeError):
        h._advance(HandleState.posted)
    calls = []
    h.add_done_callback(lambda hh: calls.append(hh.id))
    assert calls == [h.id]
    f = WorkHandle("x")
    f.fail(ValueError("boom"))
    with pytest.raises(ValueError):
        f.wait(0.1)
    c = WorkHandle.completed("x")
    assert c.test() and c.state is HandleState.complete
    c.wait(0.0)


def test_reduce_ops_and_element_reduce():
    assert element_reduce(np.uint8(200), np.uint8(100), ReduceOp.sum) == 44
    assert element_reduce(np.float32(1.5), np.float32(2.0), ReduceOp.max) == 2.0
    assert ReduceOp.min.identity(DType.i32) == np.iinfo(np.int32).max
    assert ReduceOp.prod.identity(DType.f64) == 1.0
    assert [op.code for op in ReduceOp] == [0, 1, 2, 3]


def test_dtype_codes_match_c_abi():
    assert [d.code for d in (DType.f32, DType.f64, DType.i32, DType.i64, DType.u8, DType.bf16)] \
        == [0, 1, 2, 3, 4, 5]
    assert DType.from_name("bf16").size_bytes == 2
    with pytest.raises(ValidationError):
        DType.from_name("f16")


def test_algorithm_policy_and_reference_aliases():
    pol = AlgorithmPolicy({CommOpKind.all_reduce: "ring", "all_to_allv": "pairwise_exchange"})
    assert pol.algorithm(CommOpKind.all_reduce) == "two_shot"
    assert pol.algorithm(CommOpKind.all_to_allv) == "direct_write"
    assert AlgorithmPolicy.naive().algorithm(CommOpKind.all_reduce) == "one_shot"
    assert canonical(CommOpKind.bcast, "binomial_tree") == "direct_write"
    with pytest.raises(ValidationError):
        AlgorithmPolicy({CommOpKind.all_to_allv: "nvls"})
    assert AlgorithmPolicy().algorithm(CommOpKind.send) == "direct"
    assert AlgorithmPolicy().algorithm(CommOpKind.recv) == "direct"
    dis = AlgorithmPolicy(disabled=[CommOpKind.bcast])
    assert not dis.supports(CommOpKind.bcast)
    with pytest.raises(UnsupportedOperation):
        dis.algorithm(CommOpKind.bcast)


def test_even_segments_and_bus_factor():
    assert even_segments(7, 3) == ([3, 2, 2], [0, 3, 5])
    assert even_segments(0, 4)[0] == [0, 0, 0, 0]
    assert bus_factor(CommOpKind.all_reduce, 8) == pytest.approx(1.75)
    assert bus_factor(CommOpKind.all_to_allv, 2) == pytest.approx(0.5)
    assert bus_factor(CommOpKind.all_reduce, 1) == 0.0


def test_runtime_rejects_host_transports_and_duplicates(monkeypatch):
    rt = Runtime(0, 1)
    with pytest.raises(UnknownTransport):
        rt.init([__import__("paper_2303_08374_b200").BackendConfig("a", transport="tcp")])
    with pytest.raises(DuplicateBackend):
        rt.init(["a", "a"])
    with pytest.raises(ValidationError):
        rt.init(["auto"])
    with pytest.raises(ValidationError):
        rt.init(["Bad"])
    with pytest.raises(UnknownTransport):
        Runtime(0, 1, fabric=object())


def test_runtime_env_defaults(monkeypatch):
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("WORLD_SIZE", "8")
    monkeypatch.setenv("LOCAL_RANK", "3")
    monkeypatch.delenv("MCRDL_RANK", raising=False)
    monkeypatch.delenv("MCRDL_WORLD_SIZE", raising=False)
    rt = Runtime()
    assert (rt.rank, rt.world_size, rt.local_device) == (3, 8, 3)
    monkeypatch.setenv("MCRDL_RANK", "1")
    monkeypatch.setenv("MCRDL_WORLD_SIZE", "2")
    rt = Runtime()
    assert (rt.rank, rt.world_size) == (1, 2)

"""FusionManager grouping semantics (reference middleware.py:241-359) on a
fake backend instance: no GPU needed, the device launch is recorded."""

import time

import numpy as np
import pytest

from paper_2303_08374_b200 import Buffer, CommOpKind, CommRequest, FusionConfig, ReduceOp
from paper_2303_08374_b200.core import WorkHandle
from paper_2303_08374_b200.errors import ValidationError
from paper_2303_08374_b200.middleware import FusionManager


class FakeInstance:
    def __init__(self, name="f"):
        self.name = name
        self.flushes = []

    def post_fused(self, members, ready, flush_request):
        self.flushes.append([m.input.count for m in members])
        h = WorkHandle(self.name, flush_request)
        h.complete()
        return h


class FakeRuntime:
    def __init__(self, inst):
        self.inst = inst

    def _instance(self, name):
        return self.inst


def req(n, dtype=np.float32, op=ReduceOp.sum, async_op=True):
    b = Buffer(np.zeros(n, dtype=dtype))
    return CommRequest(CommOpKind.all_reduce, input=b, output=b, op=op, backend="f",
                       async_op=async_op)


def make(B=64, T=10.0):
    inst = FakeInstance()
    fm = FusionManager(FakeRuntime(inst))
    return inst, fm, FusionConfig(max_bytes=B, max_wait=T)


def test_grouping_by_capacity():
    inst, fm, cfg = make(B=64)
    for n in (4, 4, 4, 4, 4):  # 16 B each: 4 members fill 64 B exactly -> flush
        fm.post(inst, cfg, req(n))
    assert inst.flushes == [[4, 4, 4, 4]]
    fm.post(inst, cfg, req(12))  # 16 + 48 = 64 -> fits, full -> flush
    assert inst.flushes[-1] == [4, 12]
    fm.post(inst, cfg, req(10))
    fm.post(inst, cfg, req(10))  # 40 + 40 > 64 -> flush first, open new
    assert inst.flushes[-1] == [10]
    assert fm.open_buffers() == 1
    fm.close()


def test_keyed_by_dtype_and_op():
    inst, fm, cfg = make(B=1024)
    fm.post(inst, cfg, req(4, np.float32))
    fm.post(inst, cfg, req(4, np.int64))
    fm.post(inst, cfg, req(4, np.float32, ReduceOp.max))
    assert fm.open_buffers() == 3
    fm.flush_backend("f")
    assert sorted(map(tuple, inst.flushes)) == [(4,), (4,), (4,)]
    fm.close()


def test_blocking_member_flushes_its_group_now():
    inst, fm, cfg = make(B=1024)
    fm.post(inst, cfg, req(4))
    fm.post(inst, cfg, req(8, async_op=False))
    assert inst.flushes == [[4, 8]]
    fm.close()


def test_timer_flushes_after_T_and_wait_hook():
    inst, fm, cfg = make(B=1 << 20, T=0.05)
    fm.post(inst, cfg, req(4))
    t0 = time.monotonic()
    while not inst.flushes and time.monotonic() - t0 < 2.0:
        time.sleep(0.01)
    assert inst.flushes == [[4]]
    # a waiter forces its group out instead of sleeping until T
    inst2, fm2, cfg2 = make(B=1 << 20, T=60.0)
    r = req(4)
    h = fm2.post(inst2, cfg2, r)
    h._flush_hook()
    assert inst2.flushes == [[4]]
    fm.close()
    fm2.close()


def test_eligibility_and_config_validation():
    inst, fm, cfg = make(B=64)
    assert fm.eligible(cfg, req(16))
    assert not fm.eligible(cfg, req(17))
    b = Buffer(np.zeros(4, np.float32))
    assert not fm.eligible(cfg, CommRequest(CommOpKind.bcast, output=b, root=0))
    with pytest.raises(ValidationError):
        FusionConfig(max_bytes=0)
    fm.close()

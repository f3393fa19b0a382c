"""GPU parity: the nvlink backend (sm_100a kernels through the C ABI, driven
by the public Runtime API) against the CPU oracle and the reference's golden
dumps, one process per GPU. Every scenario checks every rank's output:
bit-exact for movement, integer and (ascending-fold) float reductions.

World sizes run only when that many GPUs are visible (never more ranks than
GPUs: spinning kernels must not share a GPU)."""

import pytest

torch = pytest.importorskip("torch")

from gpu_launch import run_world  # noqa: E402

pytestmark = pytest.mark.gpu

SCENARIOS = ["golden", "all_reduce", "all_to_allv", "all_to_all", "gathers", "bcast_scatter",
             "reduce_family", "host_buffers", "async_fusion", "graphs", "p2p",
             "symm", "codec", "commlog",
             "order_mismatch"]


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _assert_ok(reports):
    problems = []
    for rep in reports:
        if rep["exit"] != 0 or rep["failures"]:
            problems.append(f"rank {rep['rank']} exit={rep['exit']}: "
                            + " | ".join(rep["failures"][:10]))
    assert not problems, "\n".join(problems)
    assert all(rep["checked"] > 0 for rep in reports)
    assert all((rep.get("launches") or 0) > 0 for rep in reports), "native kernels not launched"


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_parity_all_scenarios(world):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs, have {_ngpu()}")
    _assert_ok(run_world(world, SCENARIOS, timeout=900.0))


def test_smoke_entry_point():
    if _ngpu() < 1:
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.smoke()


def test_host_buffers_are_staged_through_the_device():
    """No CPU fallback: reference-style numpy Buffers on an nvlink backend are
    staged to the device and reduced by the sm_100a kernels (the partner.py
    known answers, p = 2)."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _assert_ok(run_world(2, ["host_buffers"], timeout=300.0))

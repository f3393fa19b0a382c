"""GPU parity: the nvlink backend (sm_100a kernels through the C ABI, driven
by the public Runtime API) against the CPU oracle and the reference's golden
dumps. Every scenario checks every rank's output: bit-exact for movement,
integer and (ascending-fold) float reductions.

Two layouts:
* one process per GPU (production): world sizes run when that many GPUs are
  visible;
* co-located: p thread-ranks of one process on ONE GPU (the reference's
  thread-world layout). The communicator sees the shared device,
  splits the SMs so every rank's spinning grids are resident together and has
  no NVLS; every other kernel and the whole flag protocol run as in
  production, so p = 2, 4, 8 parity runs on a single B200."""

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


@pytest.mark.parametrize("world", [2, 4, 8])
def test_parity_colocated(world):
    if _ngpu() < 1:
        pytest.skip("no GPU")
    reports = run_world(world, SCENARIOS, timeout=1500.0, colocated=True)
    _assert_ok(reports)
    assert all(rep.get("colocated") == world for rep in reports), \
        [rep.get("colocated") for rep in reports]


def test_smoke_entry_point():
    if _ngpu() < 1:
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.smoke()


def test_host_buffers_are_staged_through_the_device():
    """No CPU fallback: reference-style numpy Buffers on an nvlink backend are
    staged to the device and reduced by the sm_100a kernels (the partner.py
    known answers, p = 2)."""
    if _ngpu() < 1:
        pytest.skip("no GPU")
    _assert_ok(run_world(2, ["host_buffers"], timeout=300.0, colocated=_ngpu() < 2))

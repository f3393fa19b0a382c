"""The C-ABI library loads without a GPU and exports every entry point the
header declares; status codes map onto the reference error kinds."""

import re
from pathlib import Path

import pytest

from paper_2303_08374_b200 import errors
from paper_2303_08374_b200.nvl import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mcrdl_nvl.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(mcrdl_[a-z0-9_]+)\s*\(", text)) - {"mcrdl_allgather_fn"})


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), f"{name} not exported by {_lib.LIB_PATH.name}"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_abi_version_and_status_kinds():
    lib = _lib.load()
    assert lib.mcrdl_abi_version() == 1
    kinds = {code: lib.mcrdl_status_kind(code).decode() for code in range(11)}
    assert kinds[0] == "ok"
    for code, kind in kinds.items():
        if code == 0:
            continue
        exc = errors.from_status(code, "x")
        assert isinstance(exc, errors.CommError)
        if kind in ("validation", "order_mismatch", "timeout", "unsupported_operation",
                    "peer_disconnected", "bootstrap_timeout", "length_mismatch",
                    "not_initialized"):
            assert exc.kind == kind, (code, kind, exc.kind)


def test_status_maps_to_reference_exception_classes():
    assert isinstance(errors.from_status(2, "m"), errors.OrderMismatch)
    assert isinstance(errors.from_status(3, "m"), errors.CommTimeout)
    assert isinstance(errors.from_status(1, "m"), errors.ValidationError)


def test_comm_init_without_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import ctypes

    lib = _lib.load()
    h = ctypes.c_void_p()
    cb = ctypes.cast(None, _lib.ALLGATHER_FN)
    rc = lib.mcrdl_comm_init(ctypes.byref(h), 0, 1, 0, cb, None, 1 << 20, 1.0)
    assert rc != 0
    assert lib.mcrdl_last_error()
    assert not h.value


def test_null_communicator_is_rejected():
    lib = _lib.load()
    assert lib.mcrdl_all_reduce(None, None, None, 4, 0, 0, 0, 0, None) == 9  # not_initialized
    assert lib.mcrdl_barrier(None, 0, None) == 9
    assert lib.mcrdl_send(None, None, 0, 0, None) == 9
    assert lib.mcrdl_recv(None, None, 0, 0, None) == 9
    assert lib.mcrdl_comm_status(None) == 9


def test_launch_counter_starts_at_zero_without_gpu():
    assert _lib.launch_count() >= 0


def test_no_cpu_fallback_for_nvlink_backend():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2303_08374_b200 import Runtime
    from paper_2303_08374_b200.errors import NativeBackendMissing

    rt = Runtime(0, 1)
    with pytest.raises(NativeBackendMissing):
        rt.init(["nvl"])


def test_build_script_targets_sm100a():
    from paper_2303_08374_b200 import build

    assert "arch=compute_100a,code=sm_100a" in " ".join(build.ARCH)
    assert "-lineinfo" in build.FLAGS


def test_algorithm_codes_match_the_header():
    """collectives.ALGO_CODES (what the tuning table's algorithm names become
    in mcrdl_comm_set_tuning / the algo argument) equals mcrdl_algo_t."""
    from paper_2303_08374_b200.collectives import ALGO_CODES

    text = HEADER.read_text()
    enum = {m.group(1).lower(): int(m.group(2))
            for m in re.finditer(r"MCRDL_ALGO_([A-Z_]+)\s*=\s*(\d+)", text)}
    assert enum, "mcrdl_algo_t not found"
    for name, code in enum.items():
        assert ALGO_CODES[name] == code, name

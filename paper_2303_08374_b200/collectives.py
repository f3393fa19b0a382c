"""Algorithm registry and per-backend algorithm policy.

The reference registers host algorithms per kind (collectives.py:36-77) and
runs them over point-to-point frames (collectives.py:769-789). On B200 the
algorithms are sm_100a kernels inside one NVLink backend; this module keeps
the reference's registry/policy surface and maps it onto those kernels:

=================  ======================================================
kind               NVLink algorithms (first = default)
=================  ======================================================
all_reduce         auto, one_shot, two_shot, nvls
reduce             auto, one_shot, two_shot          (all_reduce, root keeps)
reduce_scatter     auto, two_shot                    (all_reduce + own slice)
bcast              auto, direct_write, nvls
all_gather(v)      auto, direct_write
gather(v)          auto, direct_write
scatter(v)         auto, direct_write
all_to_all*        auto, direct_write
send / recv        direct                            (per-pair mailbox ring)
=================  ======================================================

"auto" = per message size from the runtime's tuning table, else the
library's size heuristic. Reference algorithm names are accepted as aliases
so existing ``AlgorithmPolicy`` overrides keep working: ``naive`` (ascending
fold) -> one_shot, ``ring``/``recursive_doubling`` -> two_shot, the
pairwise/bruck/linear/binomial families -> direct_write.
"""

from __future__ import annotations

import math
from typing import Dict, Optional, Sequence, Tuple

from .core import CommOpKind
from .errors import UnsupportedOperation, ValidationError

_AR = ("auto", "one_shot", "two_shot", "nvls")
_MOVE = ("auto", "direct_write")

ALGORITHMS: Dict[CommOpKind, Tuple[str, ...]] = {
    CommOpKind.all_reduce: _AR,
    CommOpKind.reduce: ("auto", "one_shot", "two_shot"),
    CommOpKind.reduce_scatter: ("auto", "two_shot"),
    CommOpKind.bcast: ("auto", "direct_write", "nvls", "chain"),
    CommOpKind.all_gather: _MOVE,
    CommOpKind.all_gatherv: _MOVE,
    CommOpKind.gather: _MOVE,
    CommOpKind.gatherv: _MOVE,
    CommOpKind.scatter: _MOVE,
    CommOpKind.scatterv: _MOVE,
    CommOpKind.all_to_all_single: _MOVE,
    CommOpKind.all_to_all: _MOVE,
    CommOpKind.all_to_allv: _MOVE,
    CommOpKind.send: ("direct",),
    CommOpKind.recv: ("direct",),
}

# Every kind has a native path (send/recv: csrc/p2p.cu).
UNSUPPORTED_KINDS: frozenset = frozenset()

DEFAULT_ALGORITHMS: Dict[CommOpKind, str] = {
    k: (v[0] if v else "unsupported") for k, v in ALGORITHMS.items()
}

ALIASES: Dict[str, str] = {
    "naive": "one_shot",
    "ring": "two_shot",
    "recursive_doubling": "two_shot",
    "pairwise_exchange": "direct_write",
    "bruck": "direct_write",
    "linear": "direct_write",
    "binomial_tree": "direct_write",
}

# Native algorithm codes (include/mcrdl_nvl.h mcrdl_algo_t).
ALGO_CODES = {"auto": 0, "one_shot": 1, "two_shot": 2, "nvls": 3, "direct_write": 4, "chain": 5,
              "direct": 0}


def canonical(kind: CommOpKind, name: str) -> str:
    """Resolve an algorithm name (or reference alias) for `kind`."""
    real = ALIASES.get(name, name)
    if kind is CommOpKind.reduce_scatter and real == "one_shot":
        real = "two_shot"
    if real in ("one_shot", "two_shot") and kind not in (
            CommOpKind.all_reduce, CommOpKind.reduce, CommOpKind.reduce_scatter):
        real = "direct_write"
    if real not in ALGORITHMS[kind]:
        raise ValidationError("policy", f"{name!r} is not an algorithm for {kind.name}")
    return real


class AlgorithmPolicy:
    """Per-kind algorithm selection for one backend (collectives.py:80-114).
    Kinds may be disabled to model partial backends."""

    def __init__(self, overrides: Optional[dict] = None, *,
                 base: Optional[Dict[CommOpKind, str]] = None,
                 disabled: Sequence[CommOpKind] = ()):
        self._table = dict(base if base is not None else DEFAULT_ALGORITHMS)
        for kind, name in (overrides or {}).items():
            kind = CommOpKind(kind) if isinstance(kind, str) else kind
            self._table[kind] = canonical(kind, name)
        self._disabled = frozenset(CommOpKind(k) if isinstance(k, str) else k for k in disabled)

    @classmethod
    def naive(cls, overrides: Optional[dict] = None) -> "AlgorithmPolicy":
        """Ascending-fold policy: every reduction one-shot (bit-identical to
        the sequential oracle, as the reference's naive family is)."""
        base = dict(DEFAULT_ALGORITHMS)
        for k in (CommOpKind.all_reduce, CommOpKind.reduce):
            base[k] = "one_shot"
        return cls(overrides, base=base)

    def supports(self, kind: CommOpKind) -> bool:
        return kind not in self._disabled and kind not in UNSUPPORTED_KINDS

    def algorithm(self, kind: CommOpKind) -> str:
        if kind in self._disabled:
            raise UnsupportedOperation(f"{kind.name} disabled on this backend")
        if kind in UNSUPPORTED_KINDS:
            raise UnsupportedOperation(
                f"{kind.name} is point-to-point; the NVLink backend runs collectives only")
        return self._table[kind]


def even_segments(count: int, parts: int) -> Tuple[list, list]:
    """Ceil/floor split (collectives.py:163-171): the first count % parts
    segments get one extra element. Returns (sizes, offsets)."""
    q, r = divmod(count, parts)
    sizes = [q + (1 if i < r else 0) for i in range(parts)]
    offsets = [0]
    for s in sizes[:-1]:
        offsets.append(offsets[-1] + s)
    return sizes, offsets[:parts]


def critical_rounds(kind: CommOpKind, algorithm: str, p: int) -> int:
    """NVLink round trips on the critical path of each algorithm (the
    reference counts payload message rounds, collectives.py:792-829). Every
    NVSwitch algorithm here is single-hop, so this is 1 or 2."""
    if p == 1:
        return 0
    algorithm = ALIASES.get(algorithm, algorithm)
    if algorithm == "two_shot":
        return 2
    if algorithm == "auto":
        return 1 if kind is not CommOpKind.reduce_scatter else 2
    return 1


def bus_factor(kind: CommOpKind, p: int) -> float:
    """nccl-tests bus-bandwidth factor: busbw = algbw * factor."""
    if p <= 1:
        return 0.0
    if kind in (CommOpKind.all_reduce,):
        return 2.0 * (p - 1) / p
    if kind in (CommOpKind.bcast, CommOpKind.reduce):
        return 1.0
    if kind in (CommOpKind.send, CommOpKind.recv):
        return 2.0  # timed as the tuner's 0<->1 ping-pong: S each way per sample
    return (p - 1) / p


def log2ceil(p: int) -> int:
    return 0 if p <= 1 else math.ceil(math.log2(p))

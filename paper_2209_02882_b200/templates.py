"""Template families: which of the four Sgap corners covers a point, and the
divisibility gates that decide whether it is templated under a KernelConfig.

Mirrors ``spmmlab.templates`` (``/root/reference/pkg/src/spmmlab/templates.py``):
``template_family`` (82-99), the per-family builders' gates and split factors
(114-202) and ``algorithm_template`` (220-235).  The reference builds a CIN
schedule from these factors; on the B200 path the factors feed the device
kernels directly, so a template here is just the resolved factors.  The same
gates are implemented in C (``sgap_build_kernel``) for non-Python callers;
both are pinned by ``tests/golden/space.json``.
"""

from __future__ import annotations

from dataclasses import dataclass

from .lowering import KernelConfig
from .space import AmountKind, DataKind, SchedulePoint, legality_rule

__all__ = [
    "FAMILIES", "FAMILY_NNZ_MULTIPLE", "FAMILY_NNZ_ONE", "FAMILY_ROW_MULTIPLE",
    "FAMILY_ROW_RECIPROCAL", "AlgorithmTemplate", "IllegalPointError", "algorithm_template",
    "kernel_name", "template_family",
]

FAMILY_NNZ_MULTIPLE = "nnz-multiple"
FAMILY_ROW_MULTIPLE = "row-multiple"
FAMILY_ROW_RECIPROCAL = "row-reciprocal"
FAMILY_NNZ_ONE = "nnz-one"
FAMILIES = (FAMILY_NNZ_MULTIPLE, FAMILY_ROW_MULTIPLE, FAMILY_ROW_RECIPROCAL, FAMILY_NNZ_ONE)

# the paper's names for the corners
STRATEGY = {
    FAMILY_NNZ_MULTIPLE: "EB+SR",
    FAMILY_ROW_MULTIPLE: "RB+SR",
    FAMILY_ROW_RECIPROCAL: "RB+PR",
    FAMILY_NNZ_ONE: "EB+PR",
}


class IllegalPointError(ValueError):
    """Point rejected by legality rule ``rule``."""

    def __init__(self, rule: int):
        super().__init__(f"illegal point (rule {rule})")
        self.rule = rule


@dataclass(frozen=True)
class AlgorithmTemplate:
    """A templated point: family plus resolved split factors.

    ``chunk`` is the unit count of one logical block -- nonzero positions
    (nnz families), rows (row-multiple) or fused (i, k) cells
    (row-reciprocal); ``block_size`` is the reference's thread-block size.
    """

    family: str
    point: SchedulePoint
    config: KernelConfig
    g: int
    c: int
    r: int
    chunk: int
    block_size: int


def kernel_name(family: str) -> str:
    return "spmm_" + family.replace("-", "_")


def template_family(point: SchedulePoint) -> str | None:
    """The corner covering a legal point, or None; illegal points raise."""
    rule = legality_rule(point)
    if rule is not None:
        raise IllegalPointError(rule)
    if point.col_amount.kind is AmountKind.RECIPROCAL:
        return None
    kind, r = point.data_amount.kind, point.r
    if point.data_kind is DataKind.NNZ:
        if kind is AmountKind.ONE:
            return FAMILY_NNZ_ONE
        return FAMILY_NNZ_MULTIPLE if (kind is AmountKind.MULTIPLE and r == 1) else None
    if kind is AmountKind.RECIPROCAL:
        return FAMILY_ROW_RECIPROCAL if r == point.data_amount.param else None
    return FAMILY_ROW_MULTIPLE if r == 1 else None


def _factors(family: str, g: int, c: int, r: int, n: int, p: int):
    """(chunk, block_size) or None when a divisibility gate fails."""
    if n % c:
        return None
    if family == FAMILY_NNZ_ONE:
        if (p * c) % n:
            return None
        npb = p * c // n  # one position per thread, n/c column tiles per block
        if r > 1 and (32 % r or npb % r or r > npb):
            return None
        return npb, p
    if family == FAMILY_NNZ_MULTIPLE:
        if (p * c) % n or (p * g * c) % n:
            return None
        chunk = p * g * c // n
        threads = (p * c // n) * c  # chunk/g walkers x c column lanes
        if threads % 32:
            return None
        return chunk, threads
    if family == FAMILY_ROW_MULTIPLE:
        if (p * g * c) % n or (p * c) % n:
            return None
        return p * g * c // n, p
    if family == FAMILY_ROW_RECIPROCAL:
        if (c * p) % g or p % g or 32 % g:
            return None
        return c * p // g, p
    raise ValueError(family)


def algorithm_template(point: SchedulePoint, config: KernelConfig) -> AlgorithmTemplate | None:
    """Resolve a legal point under ``config``; None when no corner covers it
    or its factors do not divide out; IllegalPointError for illegal points."""
    family = template_family(point)
    if family is None:
        return None
    g, c = point.data_amount.factor, point.col_amount.factor
    got = _factors(family, g, c, point.r, config.n, config.p)
    if got is None:
        return None
    chunk, block = got
    return AlgorithmTemplate(family, point, config, g, c, point.r, chunk, block)

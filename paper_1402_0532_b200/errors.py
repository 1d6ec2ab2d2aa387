"""Exception classes and operation counting, mirroring operator.py:39-109.

Counting is the reference's only metric: one complex ⊙ costs 4 sign, 8 abs and
6 add operations (operator.py:86-90).  The GPU kernels never count per element;
the host fills counters analytically (ndft N², nfft N(log2N+1), lag n per row),
exactly the numbers the reference accumulates.
"""

from __future__ import annotations

from dataclasses import dataclass


class DomainError(ValueError):
    """An operand is NaN or infinite."""


class ContractError(ValueError):
    """A call violates an interface precondition (shape, size, range)."""


@dataclass(frozen=True)
class OpCountReport:
    """Immutable snapshot of accumulated operation counts."""

    sign_ops: int = 0
    abs_ops: int = 0
    add_ops: int = 0
    complex_mf_ops: int = 0
    complex_mul_ops: int = 0

    def __add__(self, other: "OpCountReport") -> "OpCountReport":
        return OpCountReport(
            self.sign_ops + other.sign_ops,
            self.abs_ops + other.abs_ops,
            self.add_ops + other.add_ops,
            self.complex_mf_ops + other.complex_mf_ops,
            self.complex_mul_ops + other.complex_mul_ops,
        )


@dataclass
class OpCounter:
    """Mutable accumulator; single owner, merged by summation (operator.py:67-109)."""

    sign_ops: int = 0
    abs_ops: int = 0
    add_ops: int = 0
    complex_mf_ops: int = 0
    complex_mul_ops: int = 0

    def count_real(self, n: int = 1) -> None:
        self.sign_ops += n
        self.abs_ops += 2 * n
        self.add_ops += n

    def count_complex(self, n: int = 1) -> None:
        self.sign_ops += 4 * n
        self.abs_ops += 8 * n
        self.add_ops += 6 * n
        self.complex_mf_ops += n

    def count_complex_mul(self, n: int = 1) -> None:
        self.complex_mul_ops += n

    def merge(self, other) -> None:
        self.sign_ops += other.sign_ops
        self.abs_ops += other.abs_ops
        self.add_ops += other.add_ops
        self.complex_mf_ops += other.complex_mf_ops
        self.complex_mul_ops += other.complex_mul_ops

    def report(self) -> OpCountReport:
        return OpCountReport(self.sign_ops, self.abs_ops, self.add_ops,
                             self.complex_mf_ops, self.complex_mul_ops)

"""Error classes of the hot path.

The names and the hierarchy are those of the reference taxonomy
(pkg/src/flashfps/errors.py:8-73) so that code catching the reference's
exceptions keeps working unchanged; all of them are raised by host-side
validation before any device work is queued.  KernelError is new: the
reference has no device code, and this package never degrades to a CPU path.
"""

__all__ = [
    "FlashFpsError", "EmptyCloud", "NonFiniteCoordinate", "BudgetOutOfRange",
    "SeedOutOfRange", "PruneLeavesNothing", "SeedNotInCandidates",
    "BudgetsNotMonotone", "BudgetExceedsCloud", "PrefixTooLong",
    "UnsupportedFormat", "KernelError",
]


class FlashFpsError(Exception):
    """Root of every error the package raises."""


class EmptyCloud(FlashFpsError):
    """Zero points were supplied."""


class NonFiniteCoordinate(FlashFpsError):
    """NaN/Inf coordinate; ``index`` is the first offending point."""

    def __init__(self, index: int, message: str | None = None):
        self.index = int(index)
        if message is None:
            message = f"non-finite coordinate at point index {self.index}"
        super().__init__(message)


class BudgetOutOfRange(FlashFpsError):
    """A sample budget outside [1, N]."""


class SeedOutOfRange(FlashFpsError):
    """A seed index outside [0, N)."""


class PruneLeavesNothing(FlashFpsError):
    """Candidate pruning admitted no point (cannot happen for 0 <= p < 1)."""


class SeedNotInCandidates(FlashFpsError):
    """The seed lies beyond the candidate prefix kept by pruning."""


class BudgetsNotMonotone(FlashFpsError):
    """Layer budgets increase somewhere (or none were given)."""


class BudgetExceedsCloud(FlashFpsError):
    """The first layer asks for more points than the cloud has."""


class PrefixTooLong(FlashFpsError):
    """A reused prefix longer than the cached layer (or empty)."""


class UnsupportedFormat(FlashFpsError):
    """A serialized FPSC cache blob failed validation."""


class KernelError(FlashFpsError):
    """The CUDA library is missing or a device call failed."""

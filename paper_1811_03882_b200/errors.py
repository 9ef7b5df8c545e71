"""Exception hierarchy of the offload tuner.

Mirrors the reference's error classes one for one (reference
`pkg/src/acctuner/errors.py:6-48`) so callers that branch on exception type,
and the CLI's exit-code table, behave identically.  Two classes are new and
belong to the B200 execution path: `DeviceError` (a CUDA call or the native
library failed -- infrastructure trouble, never converted into a penalty,
the same contract as `SpawnError`) and `ParityError` (a GPU result disagreed
with the checker it was compared against).
"""

from __future__ import annotations


class AutotunerError(Exception):
    """Root of every error this package raises."""


class ParseError(AutotunerError):
    """Source text outside the C subset; carries the offending position."""

    def __init__(self, message: str, line: int, col: int, path: str = "<source>"):
        self.message = message
        self.line = line
        self.col = col
        self.path = path
        super().__init__(f"{path}:{line}:{col}: {message}")


class ProfileError(AutotunerError):
    """The loop-count profile is unreadable, malformed or incomplete."""


class ModelError(AutotunerError):
    """Evaluator configuration (cost model, gpu config) is unusable."""


class InvalidGenome(AutotunerError):
    """A genome string is malformed or selects nested loops."""


class EmptyGenome(AutotunerError):
    """The program has no offloadable loop, so the gene length is zero."""


class PlanMismatch(AutotunerError):
    """A transfer plan names a loop the program does not have."""


class SpawnError(AutotunerError):
    """An evaluator subprocess could not be started."""


class ExternalOracleError(AutotunerError):
    """The external compile-probe command could not be started."""


class DomainError(AutotunerError):
    """A fitness was requested for a non-positive measured time."""


class DeviceError(ModelError):
    """The CUDA runtime or the sm_100a kernel library reported a failure.

    Subclasses ModelError so the CLI maps it to the evaluator-failure exit
    code (14), exactly like the reference maps a broken evaluator.
    """


class ParityError(AutotunerError):
    """A device result differs from the checker beyond the stated tolerance."""

"""Exception hierarchy for the mesh-intersection backend.

Mirrors the reference package's hierarchy (``maniconn/errors.py:4-53``) so a
caller that catches ``ManiconnError`` / ``ConfigError`` / ``NumericsError`` /
``FileFormatError`` keeps working when it switches to ``backend="cuda"``.  The
CLI exit-code mapping of the reference spec (2 config, 3 numerics,
4 I/O) is carried as ``exit_code``.

Two classes are new and specific to the device path:

* ``BackendError`` — the CUDA library is missing, or a CUDA call failed.
  says "device/backend failure surfaces as a task error with the layer-pair
  id"; the id is carried in ``task``.
* ``CapacityError`` — internal: the device hit buffer overflowed.  The host
  grows the buffer and reruns, so users only see it if the rerun also fails.
"""
from __future__ import annotations


class ManiconnError(Exception):
    """Base class for all package-specific errors (errors.py:4)."""

    exit_code = 1


class ConfigError(ManiconnError):
    """Bad or missing configuration / arguments (errors.py:8; exit code 2)."""

    exit_code = 2


class NumericsError(ManiconnError):
    """Numerical failure in a stage (errors.py:12; exit code 3)."""

    exit_code = 3


class SingularSystemError(NumericsError):
    """A linear system was too ill-conditioned to solve reliably (errors.py:32)."""

    def __init__(self, message, condition=None):
        super().__init__(message)
        self.condition = condition


class FileFormatError(ManiconnError):
    """Malformed binary or text artifact file (errors.py:52; exit code 4)."""

    exit_code = 4


class BackendError(ManiconnError):
    """The CUDA backend failed (library missing, CUDA error).

    ``task`` is the layer-pair id ``(n1, sign1, n2, sign2)`` when known
    (SPEC.md:473), ``status`` the C-ABI status code.
    """

    exit_code = 3

    def __init__(self, message, task=None, status=None):
        if task is not None:
            message = f"layer pair {task}: {message}"
        super().__init__(message)
        self.task = task
        self.status = status


class CapacityError(BackendError):
    """Device hit buffer too small; ``required`` is the exact hit count."""

    def __init__(self, message, required=0, task=None):
        super().__init__(message, task=task, status=1)
        self.required = required

"""Exception hierarchy for the mesh-intersection backend.

When the reference package is importable (``maniconn``, e.g. a maintainer plugging
this backend into it), its own classes are used: ``ConfigError``
here IS ``maniconn.errors.ConfigError`` (likewise ``ManiconnError``,
``NumericsError``, ``SingularSystemError``, ``FileFormatError``;
``maniconn/errors.py:4-53``), so a reference caller's ``except ManiconnError`` /
``except ConfigError`` catches this backend's errors unchanged.  Without it,
stand-ins with the same names, bases and constructor arguments are defined.

Two classes are new and specific to the device path, both ``ManiconnError``s:

* ``BackendError`` — the CUDA library is missing, or a CUDA call failed.
  says "device/backend failure surfaces as a task error with the layer-pair id";
  the id is carried in ``task``.
* ``CapacityError`` — internal: a device output buffer overflowed.  The host grows
  the buffer and reruns, so users only see it if the rerun also fails.

CLI exit codes (2 config, 3 numerics, 4 I/O) come from ``exit_code``,
by class, so the reference's classes need no extra attributes.
"""
from __future__ import annotations

try:  # the reference's own hierarchy, when the reference package is installed
    from maniconn import errors as _reference
except ImportError:  # pragma: no cover - depends on the environment
    _reference = None

if _reference is not None:
    ManiconnError = _reference.ManiconnError
    ConfigError = _reference.ConfigError
    NumericsError = _reference.NumericsError
    SingularSystemError = _reference.SingularSystemError
    FileFormatError = _reference.FileFormatError
else:
    class ManiconnError(Exception):
        """Base class for all package-specific errors (maniconn/errors.py:4)."""

    class ConfigError(ManiconnError):
        """Bad or missing configuration / arguments (maniconn/errors.py:8; exit code 2)."""

    class NumericsError(ManiconnError):
        """Numerical failure in a stage (maniconn/errors.py:12; exit code 3)."""

    class SingularSystemError(NumericsError):
        """Ill-conditioned linear system (maniconn/errors.py:32)."""

        def __init__(self, message, condition=None):
            super().__init__(message)
            self.condition = condition

    class FileFormatError(ManiconnError):
        """Malformed binary or text artifact (maniconn/errors.py:52; exit code 4)."""

REFERENCE_CLASSES = _reference is not None


class BackendError(ManiconnError):
    """The CUDA backend failed (library missing, CUDA error).

    ``task`` is the layer-pair id ``(n1, sign1, n2, sign2)`` when known
    (SPEC.md:473), ``status`` the C-ABI status code.
    """

    def __init__(self, message, task=None, status=None):
        if task is not None:
            message = f"layer pair {task}: {message}"
        super().__init__(message)
        self.task = task
        self.status = status


class CapacityError(BackendError):
    """Device output buffer too small; ``required`` is the exact count."""

    def __init__(self, message, required=0, task=None):
        super().__init__(message, task=task, status=1)
        self.required = required


def exit_code(exc: BaseException) -> int:
    """CLI exit code of an error: 2 config, 3 numerics / backend, 4 I/O."""
    if isinstance(exc, ConfigError):
        return 2
    if isinstance(exc, (NumericsError, BackendError)):
        return 3
    if isinstance(exc, (FileFormatError, OSError)):
        return 4
    return 1

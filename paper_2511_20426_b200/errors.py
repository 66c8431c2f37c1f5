"""Error taxonomy of the B200 build.

Mirrors the reference's exception classes (``errors.py:4-35`` of the
``blockcascade`` package) so that callers catching them keep working, and adds
the mapping from the C-ABI status codes (``include/bcb200.h``) onto them:

    BC_OK = 0, BC_ERR_CONTRACT = 1, BC_ERR_NUMERIC = 2, BC_ERR_CUDA = 3
"""

from __future__ import annotations


class CascadeError(Exception):
    """Root of every error this package raises."""


class InvalidInputError(CascadeError, ValueError):
    """A user-supplied value (config field, schedule, prompt, flag) is bad.

    ``fields`` lists the offending config keys when they are known.
    """

    def __init__(self, message, fields=None):
        super().__init__(message)
        self.fields = list(fields) if fields else []


class ContractViolation(CascadeError):
    """A documented precondition between two internal layers was broken."""


class NumericError(CascadeError):
    """Non-finite values reached a numeric kernel (device flag or host check)."""


class IterationError(CascadeError):
    """One batch entry of an iteration failed; carries its block/pass."""

    def __init__(self, message, block_index=None, pass_index=None):
        super().__init__(message)
        self.block_index = block_index
        self.pass_index = pass_index


class DeviceError(CascadeError, RuntimeError):
    """CUDA / NCCL failure reported by the native library (status 3), or the
    native library is missing on a machine that needs it."""


_STATUS = {1: ContractViolation, 2: NumericError, 3: DeviceError}


def raise_for_status(code: int, what: str, detail: str = "") -> None:
    """Translate a C-ABI status code into the matching exception."""
    if code == 0:
        return
    cls = _STATUS.get(code, DeviceError)
    msg = f"{what} failed with status {code}"
    if detail:
        msg += f": {detail}"
    raise cls(msg)

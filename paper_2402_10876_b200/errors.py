"""Error taxonomy of the TW/TEW path.

Mirrors ``tilesparse.errors`` (reference pkg/src/tilesparse/errors.py:4-17) so
callers can catch the same classes.  The C-ABI library reports failures as
integer status codes; :func:`raise_for_status` maps them back:

==========  =========================  ======================================
status      exception                  reference meaning (cli.py exit code)
==========  =========================  ======================================
0           --                         success (EXIT_OK)
2           InvalidInputError          bad shapes / params (EXIT_INVALID_INPUT)
4           CorruptEncodingError       malformed CTO offsets (also exit 2)
3           ContractViolationError     overlay overlaps payload (EXIT 3)
5           DeviceError                CUDA launch / driver failure (new)
==========  =========================  ======================================
"""

from __future__ import annotations


class TileSparseError(Exception):
    """Root of every error raised by this package."""


class InvalidInputError(TileSparseError, ValueError):
    """Caller data breaks a documented precondition."""


class ContractViolationError(TileSparseError, RuntimeError):
    """Composed structures break an API contract (e.g. overlay overlaps tiles)."""


class CorruptEncodingError(TileSparseError, ValueError):
    """A CTO encoding (in memory or on disk) fails validation."""


class DeviceError(TileSparseError, RuntimeError):
    """The CUDA extension is missing, or a launch / driver call failed."""


STATUS_OK = 0
STATUS_INVALID_INPUT = 2
STATUS_CONTRACT = 3
STATUS_CORRUPT = 4
STATUS_CUDA = 5

_STATUS_TO_EXC = {
    STATUS_INVALID_INPUT: InvalidInputError,
    STATUS_CONTRACT: ContractViolationError,
    STATUS_CORRUPT: CorruptEncodingError,
    STATUS_CUDA: DeviceError,
}


def raise_for_status(status: int, message: str) -> None:
    """Raise the exception class that corresponds to a C-ABI status code."""
    if status == STATUS_OK:
        return
    exc = _STATUS_TO_EXC.get(int(status), DeviceError)
    raise exc(message or f"native call failed with status {status}")

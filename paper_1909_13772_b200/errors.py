"""Exception hierarchy of the drop-in API.

Same names and meaning as the reference (pkg/src/blocksim/errors.py:12-49) so
callers' `except ValidationError` keeps working after switching backends.
"""


class BlocksimError(Exception):
    """Base class for all package errors."""


class ValidationError(BlocksimError):
    """Bad configuration, bad arguments, unsupported case (errors.py:12)."""


class TopologyError(BlocksimError):
    """Illegal block forest layout for the sweep (errors.py:36)."""


class NumericsError(BlocksimError):
    """Non-positive density / divergence (errors.py:44)."""


class SyncError(BlocksimError):
    """Distributed body state is inconsistent (errors.py:40)."""


class TypeTagError(BlocksimError):
    """A debug type tag or wire dtype code did not match (errors.py:20)."""


class BufferUnderflowError(BlocksimError):
    """Read past the end of a receive buffer (errors.py:24)."""


class BackendError(BlocksimError):
    """The CUDA kernel library is missing or a launch failed.  There is no
    CPU fallback: every compute call goes through the sm_100a library."""


class UnrecoverableError(BlocksimError):
    """A checkpoint cannot restore the lost state (errors.py:48)."""

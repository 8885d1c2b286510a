"""Exception hierarchy of the reference (errors.hpp:10-81), raised from C-ABI status codes."""
from __future__ import annotations


class Error(RuntimeError):
    """errors.hpp:10 — base class of all library errors."""


class DimensionError(Error):
    """errors.hpp:19 — operand shapes do not conform."""


class IndexError(Error):  # noqa: A001  (the reference's name)
    """errors.hpp:25 — block or node index outside the partition."""


class NumericalError(Error):
    """errors.hpp:31 — non-finite values; carries the last good iteration."""

    def __init__(self, what: str, last_good_iteration: int = 0):
        super().__init__(what)
        self._last_good = int(last_good_iteration)

    def last_good_iteration(self) -> int:
        return self._last_good


class SingularityError(Error):
    """errors.hpp:48 — factorization breakdown."""


class PartitionError(Error):
    """errors.hpp:54 — invalid or non-divisible partition."""


class ParameterError(Error):
    """errors.hpp:60 — invalid scalar parameter."""


class FormatError(Error):
    """errors.hpp:64 — malformed file contents; carries the byte offset of the defect."""

    def __init__(self, what: str, byte_offset: int = 0):
        super().__init__(what)
        self._offset = int(byte_offset)

    def byte_offset(self) -> int:
        return self._offset


class IoError(Error):
    """errors.hpp:75 — underlying I/O failure (open/read/write)."""


class MetricsError(Error):
    """errors.hpp:78 — recovery metrics undefined."""


class DeviceError(Error):
    """CUDA / driver failure (no reference counterpart; ADMM_E_CUDA)."""


class StateError(Error):
    """API misuse (ADMM_E_STATE)."""


class NcclError(Error):
    """NCCL failure inside a multi-GPU plan (ADMM_E_NCCL; no reference counterpart)."""


class ObserverStop(Error):
    """ADMM_E_OBSERVER: the observer callback stopped the solve (the mirror re-raises the
    observer's own exception instead)."""


STATUS = {1: DimensionError, 2: IndexError, 3: NumericalError, 4: SingularityError,
          5: PartitionError, 6: ParameterError, 7: DeviceError, 8: StateError, 9: FormatError,
          10: IoError, 11: NcclError, 12: ObserverStop}


def check(status: int) -> None:
    """Map an admm_status to the reference exception class (no-op for ADMM_OK)."""
    if status == 0:
        return
    from . import _lib
    msg = _lib.lib.admm_last_error().decode(errors="replace")
    cls = STATUS.get(status, Error)
    if cls is NumericalError:
        raise NumericalError(msg, _lib.lib.admm_last_good_iteration())
    if cls is FormatError:
        raise FormatError(msg, _lib.lib.admm_cmat_error_offset())
    raise cls(msg)

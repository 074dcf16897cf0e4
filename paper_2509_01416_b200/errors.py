"""Exception hierarchy mirroring the reference's proj/core/include/snop/errors.hpp:8-41; C-ABI
status codes (include/snop_cuda.h snop_status) map 1:1 onto these classes."""


class Error(RuntimeError):
    """snop::Error"""


class InvalidArgument(Error):
    """snop::InvalidArgument — bad call arguments or malformed inputs (CLI exit 1)."""


class NumericalError(Error):
    """snop::NumericalError — non-finite values, division guards (CLI exit 3)."""


class DegenerateProblem(NumericalError):
    """snop::DegenerateProblem — eigenproblem without a usable fission source."""


class IoError(Error):
    """snop::IoError"""


class ConfigError(Error):
    """snop::ConfigError"""


class CudaError(Error):
    """Device/runtime failure (no reference analogue)."""


_BY_STATUS = {1: InvalidArgument, 2: NumericalError, 3: DegenerateProblem, 4: IoError, 5: ConfigError, 6: CudaError}


def raise_for_status(status: int, message: str) -> None:
    raise _BY_STATUS.get(status, Error)(message or f"snop status {status}")

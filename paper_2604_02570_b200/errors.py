"""Exception hierarchy mirroring the reference's include/wsvd/errors.hpp:9-31
(and its CLI exit codes, tools/wsvd_main.cpp:632-653)."""


class WsvdError(RuntimeError):
    """Base class for all library errors (wsvd::Error)."""
    exit_code = 1


class ShapeError(WsvdError, ValueError):
    """Dimension or state precondition violated (wsvd::ShapeError)."""
    exit_code = 2


class ConfigError(WsvdError, ValueError):
    """Invalid configuration supplied by the caller (wsvd::ConfigError)."""
    exit_code = 2


class NumericError(WsvdError, ArithmeticError):
    """Non-finite values, counter mismatch (wsvd::NumericError)."""
    exit_code = 3


class IoError(WsvdError, OSError):
    """Filesystem / serialization problems (wsvd::IoError)."""
    exit_code = 4


class CudaError(WsvdError):
    """CUDA / NCCL failure, or no sm_100 device: there is no CPU fallback."""
    exit_code = 1

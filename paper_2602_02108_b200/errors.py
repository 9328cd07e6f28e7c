"""Error taxonomy of the reference (common.hpp:15-29), mapped from oomb_status."""


class OombError(RuntimeError):
    code = 9


class ConfigError(OombError):
    code = 1


class ShapeError(OombError):
    code = 2


class StateError(OombError):
    code = 3


class ResidencyError(OombError):
    code = 4


class IoError(OombError):
    code = 5


class CudaError(OombError):
    code = 6


_BY_CODE = {c.code: c for c in (ConfigError, ShapeError, StateError, ResidencyError, IoError, CudaError)}


def raise_for_status(code: int, msg: str) -> None:
    raise _BY_CODE.get(code, OombError)(msg)

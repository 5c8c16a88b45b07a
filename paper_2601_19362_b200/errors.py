"""Python mirror of the reference error taxonomy (inc/types.hpp:14-48).

Each class corresponds to one odc_status code of include/odc/odc.h, so code
that catches the reference's exception kinds behaves the same here.
"""


class OdcError(RuntimeError):
    code = -1


class ParamError(OdcError, ValueError):  # ODC_ERR_PARAM (ParamError / FormatError)
    code = 2


class InfeasibleError(OdcError):  # ODC_ERR_INFEASIBLE
    code = 3


class InvariantError(OdcError, AssertionError):  # ODC_ERR_INVARIANT
    code = 4


class ProtocolError(OdcError):  # ODC_ERR_PROTOCOL
    code = 5


class StateError(OdcError):  # ODC_ERR_STATE
    code = 6


class ModeError(OdcError):  # ODC_ERR_MODE
    code = 7


class DeviceError(OdcError):  # ODC_ERR_CUDA (no reference counterpart)
    code = 8


class BarrierTimeout(DeviceError):  # ODC_ERR_TIMEOUT (no reference counterpart)
    code = 9


class RangeError(DeviceError):  # ODC_ERR_RANGE: FIXED push saturation / non-finite (no reference counterpart)
    code = 10


_BY_CODE = {c.code: c for c in (ParamError, InfeasibleError, InvariantError, ProtocolError, StateError, ModeError,
                                DeviceError, BarrierTimeout, RangeError)}


def from_status(code: int, msg: str) -> OdcError:
    return _BY_CODE.get(code, DeviceError)(msg)

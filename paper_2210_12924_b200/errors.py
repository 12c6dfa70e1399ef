"""Exception hierarchy mirroring memplan's (proj/include/memplan/errors.hpp:24-76).

Messages are prefixed with the class name exactly as MEMPLAN_DEFINE_ERROR does
(errors.hpp:39-44), so ``str(InvalidOrder("x")) == "InvalidOrder: x"``.
"""


class Error(RuntimeError):
    """memplan::Error (errors.hpp:24-28)."""

    def __init__(self, what: str = ""):
        name = type(self).__name__
        msg = what if type(self) is Error or what.startswith(name + ": ") else f"{name}: {what}"
        super().__init__(msg)


class ParseError(Error):
    pass


class CycleDetected(Error):
    pass


class DanglingEndpoint(Error):
    pass


class DuplicateId(Error):
    pass


class ControlEdgeWithSize(Error):
    pass


class InvalidStructure(Error):
    pass


class InvalidSpec(Error):
    pass


class InvalidOrder(Error):
    pass


class NonTopological(Error):
    pass


class Capacity(Error):
    """Caller buffer too small (MP_E_CAPACITY); no reference analogue."""


class DeviceError(Error):
    """CUDA failure or no sm_100 device (MP_E_CUDA / MP_E_OOM / MP_E_NO_DEVICE).

    There is no CPU fallback: every compute call raises this without a B200.
    """

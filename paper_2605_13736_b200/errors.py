"""Exceptions raised by the binding, named as in SPEC.md."""


class MDSError(RuntimeError):
    code = None


class DimensionError(MDSError):
    code = -1


class MalformedMatrixError(MDSError):
    code = -2


class CompressionError(MDSError):
    code = -3


class NumericError(MDSError):
    code = -4


class SingularError(MDSError):
    code = -5


class NotInteriorError(MDSError):
    code = -6


class CudaError(MDSError):
    code = -7


class WorkspaceError(MDSError):
    code = -8


_BY_CODE = {c.code: c for c in (DimensionError, MalformedMatrixError, CompressionError, NumericError, SingularError,
                                NotInteriorError, CudaError, WorkspaceError)}


def raise_for(code, what=""):
    cls = _BY_CODE.get(int(code), MDSError)
    raise cls(f"{what}: mds status {code}")

"""Exception classes mirroring the reference (triangulation.py:18-27,
order.py:19-20) and the mapping from C ABI status codes."""
from __future__ import annotations


class MeshError(ValueError):
    """Invalid or unsupported mesh input (reference triangulation.py:18)."""


class NonTriangleFace(MeshError):
    """A face with other than three vertices (reference triangulation.py:22)."""


class NonManifoldEdge(MeshError):
    """An edge shared by more than two triangles (reference triangulation.py:26)."""


class FieldError(ValueError):
    """Invalid scalar-field input (reference order.py:19)."""


class ConstraintNotExtremum(ValueError):
    """A preserve-set vertex is not an extremum of the input order."""


class LocalizeError(RuntimeError):
    """A region has no admissible boundary minimum (_kernels.py:479-480, status 1)."""


class NoSaddleError(ValueError):
    """Every extremum of one kind was discarded, so no region has a saddle."""


class VerifyError(RuntimeError):
    """verify_constraints still fails after maxIterations outer iterations."""


class LTSNativeError(RuntimeError):
    """CUDA / workspace / argument failure inside liblts_sm100.so."""


def error_for_code(rc: int, msg: str) -> Exception:
    from . import _native as N
    cls = {
        N.E_FIELD_NONFINITE: FieldError,
        N.E_BAD_DIMS: MeshError,
        N.E_CONSTRAINT_NOT_EXTREMUM: ConstraintNotExtremum,
        N.E_LOCALIZE_NO_MIN: LocalizeError,
        N.E_VERIFY_FAILED_AT_CAP: VerifyError,
        N.E_NO_SADDLE: NoSaddleError,
    }.get(rc, LTSNativeError)
    return cls(f"[lts rc={rc}] {msg}")

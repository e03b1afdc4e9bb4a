"""Exception types of the solve path, mirroring pkg/src/rbffd/errors.py.

When the reference package ``rbffd`` is importable the classes here also
derive from the reference's own classes, so callers written against the
reference (``except rbffd.errors.InstabilityError``) keep working when they
switch to this package.
"""

from __future__ import annotations

try:  # optional: only to let reference-side `except` clauses catch ours
    from rbffd import errors as _ref  # type: ignore
except Exception:  # pragma: no cover - the GPU box has no reference
    _ref = None


def _bases(name: str, default: type) -> tuple:
    ref_cls = getattr(_ref, name, None) if _ref is not None else None
    return (ref_cls,) if ref_cls is not None else (default,)


class ParameterError(*_bases("ParameterError", ValueError)):
    """A caller-supplied parameter is out of its documented range (errors.py:4)."""


class InstabilityError(*_bases("InstabilityError", RuntimeError)):
    """The explicit iteration produced a non-finite field (errors.py:21-27)."""

    def __init__(self, message, step=None, max_abs=None):
        RuntimeError.__init__(self, message)
        self.step = step
        self.max_abs = max_abs


class SteadyStateTimeout(*_bases("SteadyStateTimeout", RuntimeError)):
    """Run-to-steady mode hit its step cap before reaching tolerance (errors.py:30-36)."""

    def __init__(self, message, steps=None, residual=None):
        RuntimeError.__init__(self, message)
        self.steps = steps
        self.residual = residual


class DegenerateStencilError(*_bases("DegenerateStencilError", RuntimeError)):
    """A local weight system is singular or numerically rank-deficient
    (errors.py:8-18): carries the offending node index and its coordinates."""

    def __init__(self, message, node_index=None, position=None):
        RuntimeError.__init__(self, message)
        self.node_index = node_index
        self.position = position


class DeviceError(RuntimeError):
    """A CUDA error reported by the C ABI (status RBF_ERR_CUDA)."""

"""Exception classes with the reference's names, bases and messages.

pkg/src/hull3d/oracle.py:23-25 (DegenerateInputError), merge.py:29-39
(MergeOverflowError, BridgeWalkError), store.py:24-30 (ChainError, LogError).
Device status codes (include/hull3d_b200.h) map onto them exactly as the
reference's ``_check`` helpers map its kernel codes (merge.py:59-72,
store.py:33-43).
"""

from __future__ import annotations

NIL = -1
E_OVERFLOW = -1
E_BRIDGE = -2
E_CHAIN = -3
E_COUNT = -4
E_UNTERMINATED = -5
E_TIES = -6
E_COINCIDENT = -7
E_COLLINEAR = -8
E_COPLANAR = -9
E_NOFACETS = -10
E_CAPACITY = -11
E_NONFINITE = -12
E_ARG = -100
E_CUDA = -101


class DegenerateInputError(ValueError):
    """Input violates the general-position contract in a way that makes
    facet decisions ambiguous."""


class MergeOverflowError(RuntimeError):
    """Merged log would exceed its 2*(R-L) slice: degenerate input or bug."""


class BridgeWalkError(RuntimeError):
    """Initial bridge walk overran the group size: chains were not valid
    convex chains (degenerate input or bug)."""


class ChainError(RuntimeError):
    """act() reached a sentinel neighbor: the caller broke a chain
    precondition (or fed the engine degenerate input)."""


class LogError(RuntimeError):
    """A log slice was unterminated or a replay count overran it."""


class DeviceError(RuntimeError):
    """CUDA runtime failure inside the B200 library."""


def check_merge(code: int) -> int:
    """merge.py:59-72 mapping (merge jobs, level runs, carries)."""
    if code >= 0:
        return code
    if code == E_OVERFLOW:
        raise MergeOverflowError(
            "merged event log overflow: input violates the general-position "
            "contract (or upstream state is corrupt)"
        )
    if code == E_BRIDGE:
        raise BridgeWalkError("bridge walk exceeded the group size")
    if code == E_CHAIN:
        raise BridgeWalkError("chain state corrupt: act() hit a sentinel neighbor")
    return _common(code, f"merge failed with kernel error code {code}")


def check_store(code: int) -> int:
    """store.py:33-43 mapping (act, replay, extract, log length)."""
    if code >= 0:
        return code
    if code == E_CHAIN:
        raise ChainError("act() on a point with a sentinel neighbor")
    if code == E_COUNT:
        raise LogError("replay count exceeds the event log length")
    if code == E_UNTERMINATED:
        raise LogError("event log has no terminator inside its slice")
    return _common(code, f"kernel error code {code}")


def check_api(code: int) -> int:
    """api.py:186-256 input errors raised by the device presort/epilogue."""
    if code >= 0:
        return code
    if code == E_NONFINITE:
        raise ValueError("coordinates must be finite")
    if code == E_TIES:
        raise DegenerateInputError("duplicate x coordinates survived perturbation")
    if code == E_COINCIDENT:
        raise DegenerateInputError("all points coincide")
    if code == E_COLLINEAR:
        raise DegenerateInputError("all points are collinear")
    if code == E_COPLANAR:
        raise DegenerateInputError("all points are coplanar")
    if code == E_NOFACETS:
        raise DegenerateInputError("no facets produced; input is degenerate")
    return check_merge(code)


def _common(code: int, default: str) -> int:
    if code == E_CUDA:
        from ._lib import last_error

        raise DeviceError(f"CUDA error in the B200 hull library: {last_error()}")
    if code == E_CAPACITY:
        raise MergeOverflowError("fixed-capacity device buffer exceeded")
    if code == E_ARG:
        raise ValueError("invalid argument to the B200 hull library")
    raise RuntimeError(default)

"""Typed errors mirroring ``bertopt::Error`` (proj/core/include/bertopt/errors.hpp:24-48).

Status codes come from ``bo_status`` in include/bertopt_b200.h.
"""
from __future__ import annotations


class BertoptError(RuntimeError):
    status = -1


class ShapeMismatch(BertoptError):
    status = 1


class NonFiniteGradient(BertoptError):
    status = 2


class OverflowDetected(BertoptError):
    status = 3


class LengthMismatch(BertoptError):
    status = 4


class InvalidConfig(BertoptError):
    status = 5


class BucketLayoutMismatch(BertoptError):
    status = 6


class PeerDisconnected(BertoptError):
    status = 7


class WatchdogTimeout(BertoptError):
    status = 8


class ProtocolError(BertoptError):
    status = 9


class IoFailure(BertoptError):
    status = 10


class CudaError(BertoptError):
    status = 20


class NcclError(BertoptError):
    status = 21


class NoDevice(BertoptError):
    status = 22


_BY_STATUS = {c.status: c for c in (ShapeMismatch, NonFiniteGradient, OverflowDetected,
                                     LengthMismatch, InvalidConfig, BucketLayoutMismatch,
                                     PeerDisconnected, WatchdogTimeout, ProtocolError, IoFailure,
                                     CudaError, NcclError, NoDevice)}


def from_status(status: int, msg: str) -> BertoptError:
    cls = _BY_STATUS.get(status, BertoptError)
    return cls(f"{cls.__name__}: {msg}")

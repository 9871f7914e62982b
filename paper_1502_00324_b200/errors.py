"""Exception types, named as in the reference, and the status mapping of the C ABI."""

from __future__ import annotations


class PoolConfigError(Exception):
    """Pool parameters cannot produce a non-empty pool for this image (pool.py:28)."""


class EmptyPoolError(Exception):
    """The domain pool has no entries at the requested level (matcher.py:34)."""


def raise_for_status(rc: int, msg: str):
    from . import _native as N

    if rc == N.FC_ERR_POOL_CONFIG:
        raise PoolConfigError(msg)
    if rc == N.FC_ERR_EMPTY_POOL:
        raise EmptyPoolError(msg)
    if rc in (N.FC_ERR_ARG, N.FC_ERR_TILE_SIZE, N.FC_ERR_DIMS):
        raise ValueError(msg)
    if rc == N.FC_ERR_NO_DEVICE:
        raise N.DeviceUnavailableError(msg)
    raise N.DeviceError(f"status {rc}: {msg}")

"""Device plumbing: PyTorch supplies device allocations and the CUDA stream;
everything that computes lives in libdyngpu.so.

A global "device epoch" counts device-side mutations of persistent state
(backward accumulating into gradients, trainer updates).  Host mirrors of
parameters remember the epoch they were synced at and download lazily; host
writes mark a mirror dirty and it is uploaded before the next device use
(SURVEY 8(b) "host-visible storage coherence").
"""

from __future__ import annotations

import threading

from . import errors

_torch = None
_state = threading.local()
EPOCH = [0]
DIRTY: set = set()  # objects with a pending host->device upload (have ._upload())


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise errors.ConfigError(
            "the B200 backend needs a CUDA device (no CPU fallback); graph construction works "
            "without one, execution does not"
        )
    return t


def device():
    t = require_cuda()
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    t = require_cuda()
    return int(t.cuda.current_stream().cuda_stream)


def empty_bytes(nbytes: int):
    t = require_cuda()
    return t.empty(max(int(nbytes), 256), dtype=t.uint8, device=device())


def zeros_f32(n: int):
    t = require_cuda()
    return t.zeros(max(int(n), 1), dtype=t.float32, device=device())


def bump_epoch() -> None:
    EPOCH[0] += 1


def flush_dirty() -> None:
    """Upload every host-dirtied mirror before a device operation."""
    if DIRTY:
        for obj in list(DIRTY):
            obj._upload()
        DIRTY.clear()

"""ctypes binding of the C-ABI executor library (include/dyngpu.h).

The library is built in-tree (`make` / `__graft_entry__.build()`) as
paper_1701_03980_b200/libdyngpu.so.  There is no CPU fallback: if the library
or a CUDA device is missing, every execution entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import errors

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdyngpu.so")

# op codes (dyngpu.h dg_op) keyed by the reference registry names (ops.py:98-527)
OP_CODES = {
    "input": 0,
    "parameter": 1,
    "lookup": 2,
    "lookup_batch": 3,
    "add": 4,
    "cmult": 5,
    "scalar_mul": 6,
    "tanh": 7,
    "logistic": 8,
    "matmul": 9,
    "affine": 10,
    "concatenate": 11,
    "pick_range": 12,
    "softmax": 13,
    "pickneglogsoftmax": 14,
    "pickneglogsoftmax_batch": 15,
    "sum_batches": 16,
}

# dg_node, 13 x int32 (dyngpu.h)
NODE_DTYPE = np.dtype(
    [
        ("kind", np.int32),
        ("n_in", np.int32),
        ("in_off", np.int32),
        ("rank", np.int32),
        ("dims", np.int32, (4,)),
        ("batch", np.int32),
        ("aux_i_off", np.int32),
        ("aux_i_len", np.int32),
        ("aux_f_off", np.int32),
        ("aux_f_len", np.int32),
    ]
)

EXPORTS = (
    "dg_last_error", "dg_abi_version",
    "dg_param_register", "dg_param_rebind", "dg_param_release",
    "dg_touched_count", "dg_touched_get", "dg_touched_add", "dg_touched_clear",
    "dg_graph_create", "dg_graph_destroy", "dg_graph_set_stream", "dg_graph_renew", "dg_graph_append",
    "dg_forward", "dg_backward", "dg_value", "dg_gradient", "dg_value_ptr",
    "dg_graph_counters", "dg_graph_plan_stats", "dg_profile_enable", "dg_profile_read", "dg_profile_reset",
    "dg_trainer_create", "dg_trainer_destroy", "dg_trainer_set", "dg_trainer_attach", "dg_trainer_update",
    "dg_trainer_step_count", "dg_trainer_set_step",
    "dg_lookup_pack", "dg_lookup_merge", "dg_scale",
)

_lock = threading.Lock()
_lib = None

c_i32, c_i64, c_f32, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
c_size = ctypes.c_size_t


def _declare(lib):
    sig = {
        "dg_last_error": (ctypes.c_char_p, []),
        "dg_abi_version": (ctypes.c_int, []),
        "dg_param_register": (ctypes.c_int, [ctypes.c_int, c_i64, c_i64, c_vp, c_vp, ctypes.POINTER(c_i64)]),
        "dg_param_rebind": (ctypes.c_int, [c_i64, c_vp, c_vp]),
        "dg_param_release": (ctypes.c_int, [c_i64]),
        "dg_touched_count": (ctypes.c_int, [c_i64, ctypes.POINTER(c_i64)]),
        "dg_touched_get": (ctypes.c_int, [c_i64, c_vp, c_i64]),
        "dg_touched_add": (ctypes.c_int, [c_i64, c_vp, c_i64]),
        "dg_touched_clear": (ctypes.c_int, [c_i64]),
        "dg_graph_create": (ctypes.c_int, [ctypes.c_int, c_vp, c_size, c_vp, c_size, c_vp, c_size, ctypes.POINTER(c_vp)]),
        "dg_graph_destroy": (ctypes.c_int, [c_vp]),
        "dg_graph_set_stream": (ctypes.c_int, [c_vp, c_vp]),
        "dg_graph_renew": (ctypes.c_int, [c_vp]),
        "dg_graph_append": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_i32, c_vp, c_i64, c_vp, c_i64]),
        "dg_forward": (ctypes.c_int, [c_vp, c_i32]),
        "dg_backward": (ctypes.c_int, [c_vp, c_i32]),
        "dg_value": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i64]),
        "dg_gradient": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i64]),
        "dg_value_ptr": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(c_vp)]),
        "dg_graph_counters": (ctypes.c_int, [c_vp, c_vp]),
        "dg_graph_plan_stats": (ctypes.c_int, [c_vp, c_vp]),
        "dg_profile_enable": (ctypes.c_int, [c_vp, ctypes.c_uint32]),
        "dg_profile_read": (ctypes.c_int, [c_vp, c_i32, c_vp]),
        "dg_profile_reset": (ctypes.c_int, [c_vp]),
        "dg_schedule_stats": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp]),
        "dg_schedule_rnn_stats": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp]),
        "dg_rnn_trace": (ctypes.c_int, [c_vp, c_i64]),
        "dg_trainer_create": (ctypes.c_int, [ctypes.c_int, c_f32, c_f32, c_f32, c_f32, c_f32, c_f32, ctypes.c_int,
                                              ctypes.POINTER(c_vp)]),
        "dg_trainer_destroy": (ctypes.c_int, [c_vp]),
        "dg_trainer_set": (ctypes.c_int, [c_vp, c_f32, ctypes.c_int]),
        "dg_trainer_attach": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
        "dg_trainer_update": (ctypes.c_int, [c_vp, c_vp]),
        "dg_trainer_step_count": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i64)]),
        "dg_trainer_set_step": (ctypes.c_int, [c_vp, c_i64]),
        "dg_lookup_pack": (ctypes.c_int, [c_i64, c_vp, c_vp, c_i64, ctypes.POINTER(c_i64), c_vp]),
        "dg_lookup_merge": (ctypes.c_int, [c_i64, ctypes.c_int32, c_vp, c_vp, c_vp, c_f32, c_vp]),
        "dg_scale": (ctypes.c_int, [c_vp, c_i64, c_f32, c_vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


PROFILE_CLASSES = ("gemm_fwd", "gemm_dx", "gemm_dw", "pnls_fwd", "pnls_bwd", "elementwise", "gather",
                   "scatter_add", "bias_colsum", "other", "rnn_fwd", "rnn_bwd")


def lib():
    """Load libdyngpu.so (once).  Raises if it is missing: no CPU fallback."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise errors.ConfigError(
                        f"native executor {LIB_PATH} is not built; run `make` or __graft_entry__.build()"
                    )
                handle = ctypes.CDLL(LIB_PATH)
                _declare(handle)
                _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a dg_status onto the reference exception taxonomy (errors.py)."""
    if rc == 0:
        return
    msg = (lib().dg_last_error() or b"").decode("utf-8", "replace")
    if rc == 1:
        pool, req, rem = msg.split("|")
        raise errors.PoolExhausted(pool, int(req), int(rem))
    cls = {
        2: errors.NonScalarLoss,
        3: errors.StaleExpression,
        4: errors.ShapeError,
        5: errors.IndexOutOfBounds,
        6: errors.BadShape,
        7: errors.DeviceError,
        8: errors.ConfigError,
    }.get(rc, errors.DyncoreError)
    raise cls(msg)


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (interop only)."""
    return int(t.data_ptr())

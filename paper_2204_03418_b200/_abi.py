"""ctypes declarations of the C ABI in include/co.h (argument marshalling only).

The shared library ``libco_b200.so`` is built in-tree by ``build.py``.  There
is no fallback: if the library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libco_b200.so")
if os.environ.get("CO_LIB_VARIANT"):            # experiment builds only (build.py --variant)
    LIB_PATH = os.path.join(_HERE, f"libco_b200_{os.environ['CO_LIB_VARIANT']}.so")

CO_OK, CO_ERR_ARG, CO_ERR_SHAPE, CO_ERR_LENGTH, CO_ERR_UNSUPPORTED, CO_ERR_CUDA, CO_ERR_OOM = 0, -1, -2, -3, -4, -5, -6
CO_F32, CO_BF16 = 0, 1
CO_ACT_NONE, CO_ACT_RELU = 0, 1
CO_STATE_PSUM, CO_STATE_RAW, CO_STATE_AUTO = 0, 1, 2
STATE_LAYOUTS = {"psum": CO_STATE_PSUM, "raw": CO_STATE_RAW, "auto": CO_STATE_AUTO}
CO_KERNEL_AUTO, CO_KERNEL_DIRECT, CO_KERNEL_DENSE_TC, CO_KERNEL_DEPTHWISE, CO_KERNEL_POOL, CO_KERNEL_COPY = range(6)
KERNELS = {"auto": CO_KERNEL_AUTO, "direct": CO_KERNEL_DIRECT, "dense_tc": CO_KERNEL_DENSE_TC,
           "depthwise": CO_KERNEL_DEPTHWISE, "pool": CO_KERNEL_POOL, "copy": CO_KERNEL_COPY}
CO_OP_CONV, CO_OP_MAX_POOL, CO_OP_AVG_POOL, CO_OP_DELAY = 0, 1, 2, 3
OPS = {"conv": CO_OP_CONV, "max": CO_OP_MAX_POOL, "avg": CO_OP_AVG_POOL, "delay": CO_OP_DELAY}
KERNEL_NAMES = {v: k for k, v in KERNELS.items()}
# defaults of the documented options (include/co.h co_set_option)
OPTION_DEFAULTS = {"tc_mode": 0, "khalo": 1, "pair": 0, "kpair": 0, "eg": 0, "mc": 1, "pdl": 1, "chunk": 1,
                   "chunk_flat": 0, "chunk_st": 0, "chunk_t": 0, "pool_band": 1, "pool_vh": -1, "pool_g": 0, "log": 0,
                   "stem": 1, "dw_seg": 1, "mha_ring": 1, "pool_seg": 1}

# every entry point include/co.h declares (checked by tests/test_abi_load.py)
EXPORTS = ["co_conv_create", "co_conv_destroy", "co_conv_info", "co_delay", "co_kernel_name",
           "co_forward_step", "co_forward_step_host", "co_forward_steps_host", "co_forward_steps", "co_steps_ready_count",
           "co_forward", "co_forward_out_len", "co_state_bytes", "co_state_get", "co_state_set",
           "co_state_clean", "co_stack_create", "co_stack_destroy", "co_stack_step", "co_stack_step_host", "co_stack_steps_host", "co_stack_delay",
           "co_stack_clean", "co_state_clean_streams", "co_stream_ready", "co_stack_clean_streams",
           "co_stack_stream_ready", "co_parallel_create", "co_parallel_destroy", "co_parallel_step",
           "co_parallel_forward", "co_parallel_clean", "co_parallel_delay", "co_parallel_out_channels", "co_mha_create", "co_mha_destroy", "co_mha_step", "co_mha_forward", "co_mha_clean",
           "co_mha_delay", "co_mha_state_bytes", "co_mha_state_get", "co_mha_state_set", "co_residual_create", "co_residual_destroy", "co_residual_step", "co_residual_forward",
           "co_residual_clean", "co_residual_delay", "co_stack_graph_create", "co_stack_graph_period", "co_graph_upload", "co_graph_launch",
           "co_graph_info", "co_graph_destroy", "co_set_option", "co_get_option", "co_option_name",
           "co_last_error", "co_abi_version"]


class CoMhaDesc(C.Structure):
    _fields_ = [("embed_dim", C.c_int32), ("num_heads", C.c_int32), ("window", C.c_int32),
                ("n_streams", C.c_int64), ("out_dtype", C.c_int32)]


class CoConvDesc(C.Structure):
    _fields_ = [("spatial_rank", C.c_int32), ("in_channels", C.c_int32), ("out_channels", C.c_int32),
                ("groups", C.c_int32), ("kernel", C.c_int32 * 3), ("stride", C.c_int32 * 3),
                ("padding", C.c_int32 * 3), ("dilation", C.c_int32 * 3), ("in_spatial", C.c_int32 * 2),
                ("n_streams", C.c_int64), ("in_dtype", C.c_int32), ("w_dtype", C.c_int32),
                ("out_dtype", C.c_int32), ("activation", C.c_int32), ("kernel_choice", C.c_int32),
                ("state_layout", C.c_int32), ("op", C.c_int32)]


class CoInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("head", C.c_int32), ("ring_slots", C.c_int32), ("delay", C.c_int32),
                ("receptive_field", C.c_int32), ("stride_t", C.c_int32), ("padding_t", C.c_int32),
                ("out_spatial", C.c_int32 * 2), ("kernel_used", C.c_int32), ("state_layout", C.c_int32)]


class CoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"co error {code}: {msg}")
        self.code = code


_lock = threading.Lock()
_lib = None


def lib():
    """Load libco_b200.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2204_03418_b200.build`")
            L = C.CDLL(LIB_PATH)
            vp, i64p = C.c_void_p, C.POINTER(C.c_int64)
            L.co_conv_create.argtypes = [C.POINTER(CoConvDesc), vp, vp, C.c_int, C.POINTER(vp)]
            L.co_conv_destroy.argtypes = [vp]
            L.co_conv_info.argtypes = [vp, C.POINTER(CoInfo)]
            L.co_delay.argtypes = [vp, i64p]
            L.co_kernel_name.argtypes = [vp]
            L.co_kernel_name.restype = C.c_char_p
            L.co_forward_step.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_int), vp]
            L.co_forward_step_host.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_int), vp]
            L.co_forward_steps_host.argtypes = [vp, vp, C.c_int64, vp, C.POINTER(C.c_uint8), i64p, vp]
            L.co_stack_steps_host.argtypes = [vp, vp, C.c_int64, vp, C.POINTER(C.c_uint8), i64p, vp]
            L.co_forward_steps.argtypes = [vp, vp, C.c_int64, vp, C.POINTER(C.c_uint8), i64p, C.c_int, C.c_int, vp]
            L.co_steps_ready_count.argtypes = [vp, C.c_int64, C.c_int, i64p]
            L.co_forward.argtypes = [vp, vp, C.c_int64, vp, i64p, vp]
            L.co_forward_out_len.argtypes = [vp, C.c_int64, i64p]
            L.co_state_bytes.argtypes = [vp, C.POINTER(C.c_size_t)]
            L.co_state_get.argtypes = [vp, vp, C.c_size_t, C.POINTER(CoInfo), vp]
            L.co_state_set.argtypes = [vp, vp, C.c_size_t, C.POINTER(CoInfo), vp]
            L.co_state_clean.argtypes = [vp, vp]
            L.co_stack_create.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(vp)]
            L.co_stack_destroy.argtypes = [vp]
            L.co_stack_step.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_int), vp]
            L.co_stack_step_host.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_int), vp]
            L.co_stack_delay.argtypes = [vp, i64p]
            L.co_stack_clean.argtypes = [vp, vp]
            L.co_state_clean_streams.argtypes = [vp, C.POINTER(C.c_uint8), vp]
            L.co_stream_ready.argtypes = [vp, C.POINTER(C.c_uint8)]
            L.co_stack_clean_streams.argtypes = [vp, C.POINTER(C.c_uint8), vp]
            L.co_stack_stream_ready.argtypes = [vp, C.POINTER(C.c_uint8)]
            L.co_parallel_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.POINTER(vp)]
            L.co_parallel_destroy.argtypes = [vp]
            L.co_parallel_step.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_int), vp]
            L.co_parallel_forward.argtypes = [vp, vp, C.c_int64, vp, i64p, vp]
            L.co_parallel_clean.argtypes = [vp, vp]
            L.co_parallel_delay.argtypes = [vp, i64p]
            L.co_parallel_out_channels.argtypes = [vp, C.POINTER(C.c_int32)]
            L.co_mha_create.argtypes = [C.POINTER(CoMhaDesc), vp, vp, vp, vp, C.c_int, C.POINTER(vp)]
            L.co_mha_destroy.argtypes = [vp]
            L.co_mha_step.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_int), vp]
            L.co_mha_forward.argtypes = [vp, vp, C.c_int64, vp, vp]
            L.co_mha_clean.argtypes = [vp, vp]
            L.co_mha_delay.argtypes = [vp, i64p]
            L.co_mha_state_bytes.argtypes = [vp, C.POINTER(C.c_size_t)]
            L.co_mha_state_get.argtypes = [vp, vp, C.c_size_t, i64p, vp]
            L.co_mha_state_set.argtypes = [vp, vp, C.c_size_t, C.c_int64, vp]
            L.co_residual_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
            L.co_residual_destroy.argtypes = [vp]
            L.co_residual_step.argtypes = [vp, vp, vp, C.c_int, C.POINTER(C.c_int), vp]
            L.co_residual_forward.argtypes = [vp, vp, C.c_int64, vp, i64p, vp]
            L.co_residual_clean.argtypes = [vp, vp]
            L.co_residual_delay.argtypes = [vp, i64p, i64p]
            L.co_stack_graph_create.argtypes = [vp, C.c_int64, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]
            L.co_graph_upload.argtypes = [vp, vp]
            L.co_stack_graph_period.argtypes = [vp, i64p]
            L.co_graph_launch.argtypes = [vp, i64p, vp]
            L.co_graph_info.argtypes = [vp, i64p, C.POINTER(C.c_int)]
            L.co_graph_destroy.argtypes = [vp]
            L.co_set_option.argtypes = [C.c_char_p, C.c_int64]
            L.co_get_option.argtypes = [C.c_char_p, i64p]
            L.co_option_name.argtypes = [C.c_int]
            L.co_option_name.restype = C.c_char_p
            L.co_last_error.restype = C.c_char_p
            L.co_abi_version.restype = C.c_int
            _lib = L
    return _lib


def check(rc: int):
    if rc != CO_OK:
        raise CoError(rc, lib().co_last_error().decode())

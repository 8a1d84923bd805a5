"""ctypes binding of the sm_100a C-ABI library (include/ppll.h).

The library is built in-tree (``paper_2411_12780_b200/lib/libppll_b200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_2411_12780_b200/csrc``.  There
is no fallback: if the library is missing, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PPLL_LIB") or os.path.join(_HERE, "lib", "libppll_b200.so")

PPLL_OK, PPLL_ERR_ARG, PPLL_ERR_CUDA, PPLL_ERR_UNSUPPORTED, PPLL_ERR_CLOSED = 0, 1, 2, 3, 4
F32, BF16 = 0, 1
ERRBIT_LABEL, ERRBIT_LOSS, ERRBIT_PARAM, ERRBIT_STEP, ERRBIT_GRAD = 1, 2, 4, 8, 16
ERRBIT_SYNC = 32
GEMM_AUTO, GEMM_SIMT, GEMM_TCGEN05 = 0, 1, 2

_vp, _i, _i64, _f, _d, _u64 = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double, C.c_uint64

# name -> (restype, argtypes); every symbol include/ppll.h declares
SIGNATURES = {
    "ppll_abi_version": (_i, []),
    "ppll_last_error": (C.c_char_p, []),
    "ppll_launch_count": (_u64, []),
    "ppll_set_gemm_engine": (None, [_i]),
    "ppll_set_attn_engine": (None, [_i]),
    "ppll_gemm_timeline": (_vp, []),
    "ppll_linear_fwd": (_i, [_i, _i, _i, _vp, _i, _vp, _vp, _vp, _i, _vp, _i, _i, _i, _vp]),
    "ppll_linear_fwd_ex": (_i, [_i, _i, _i, _vp, _i, _vp, _vp, _vp, _i, _i, _vp, _i, _vp, _i,
                                _vp, _i, _i, _vp]),
    "ppll_linear_dgrad_ex": (_i, [_i, _i, _i, _vp, _i, _vp, _vp, _i, _i, _vp, _i, _i, _vp]),
    "ppll_linear_dgrad": (_i, [_i, _i, _i, _vp, _i, _vp, _vp, _i, _vp, _i, _i, _vp]),
    "ppll_linear_wgrad": (_i, [_i, _i, _i, _vp, _i, _vp, _i, _vp, _vp, _i, _vp]),
    "ppll_softmax_xent": (_i, [_i, _i, _vp, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp]),
    "ppll_nesterov_step": (_i, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _i, _f, _f, _f, _vp, _vp]),
    "ppll_cosine_lr": (_d, [_i, _d, _d, _i]),
    "ppll_set_local_optimizer": (_i, [_vp, _i, _vp, _f, _f, _f]),
    "ppll_cast": (_i, [_i64, _vp, _i, _vp, _i, _vp]),
    "ppll_ew": (_i, [_i, _i64, _i64, _vp, _vp, _f, _vp, _i, _vp, _vp]),
    "ppll_colsum": (_i, [_i, _i, _vp, _vp, _i, _vp]),
    "ppll_sum_all": (_i, [_i64, _vp, _vp, _i, _vp, _vp]),
    "ppll_conv3x3_bf16": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp]),
    "ppll_conv3x3_bf16_ex": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp]),
    "ppll_conv3x3_wgrad_ws_floats": (C.c_long, [_i, _i, _i, _i, _i]),
    "ppll_conv3x3_wgrad_bf16": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, C.c_long, _vp]),
    "ppll_gather_rows": (_i, [_i, _i64, _vp, _vp, _vp, _i, _vp, _vp, _vp]),
    "ppll_gather_rows_u8": (_i, [_i, _i64, _vp, _vp, _vp, _i, _vp, _vp, _vp]),
    "ppll_events_elapsed": (_i, [_i, _vp, C.c_uint64, _vp]),
    "ppll_set_pdl": (_i, [_i]),
    "ppll_set_gpu_exclusive": (_i, [_i]),
    "ppll_count_correct": (_i, [_i, _i, _vp, _i, _i, _vp, _vp, _vp]),
    "ppll_stage_create": (_vp, [_i, _i, _vp, _vp, _vp, _vp, _i64, _i, _i, _vp, _vp, _vp, _vp,
                                _vp, _vp, _i, _vp, _vp, _f, _f]),
    "ppll_stage_destroy": (None, [_vp]),
    "ppll_stage_step": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ppll_stage_block_forward": (_i, [_vp, _i, _vp, _vp, _vp]),
    "ppll_stage_block_backward": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp]),
    "ppll_stage_forward": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ppll_vit_stage_create": (_vp, [_vp, _vp, _i64, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _f, _f]),
    "ppll_vit_stage_destroy": (None, [_vp]),
    "ppll_vit_stage_step": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ppll_vit_stage_forward": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ppll_layernorm_bwd_ws_floats": (C.c_long, [_i, _i]),
    "ppll_layernorm_fwd": (_i, [_i, _i, _vp, C.c_long, _vp, _vp, _vp, C.c_long, _vp, _vp, _i, _vp]),
    "ppll_layernorm_bwd": (_i, [_i, _i, _vp, C.c_long, _vp, C.c_long, _vp, _vp, _vp, _vp, C.c_long,
                                _vp, C.c_long, _vp, _vp, _vp, _vp, C.c_long, _i, _vp]),
    "ppll_batchnorm_ws_floats": (C.c_long, [_i, _i]),
    "ppll_batchnorm_fwd": (_i, [_i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, C.c_long, _i,
                                _vp]),
    "ppll_batchnorm_bwd": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_long, _i,
                                _vp]),
    "ppll_set_ring_timeout_ms": (None, [C.c_longlong]),
    "ppll_ring_stall": (_i, [_vp, _i]),
    "ppll_attn_fwd_bf16": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp]),
    "ppll_attn_bwd_bf16": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ppll_vit_stage_block_forward": (_i, [_vp, _i, _vp, _vp, _vp]),
    "ppll_vit_stage_block_backward": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp]),
    "ppll_resnet_stage_create": (_vp, [_vp, _vp, _vp, _vp, _i64, _i, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _i, _vp, _vp, _f, _f]),
    "ppll_resnet_stage_destroy": (None, [_vp]),
    "ppll_resnet_stage_step": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ppll_resnet_stage_forward": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ppll_resnet_stage_block_forward": (_i, [_vp, _i, _vp, _vp, _vp]),
    "ppll_resnet_stage_block_backward": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp]),
    "ppll_ring_publish": (_i, [_vp, _i, _vp]),
    "ppll_ring_wait": (_i, [_vp, _i, _vp]),
    "ppll_ring_release": (_i, [_vp, _vp]),
    "ppll_ring_wait_credit": (_i, [_vp, _i, _vp]),
    "ppll_ipc_get_handle": (_i, [_vp, _vp]),
    "ppll_ipc_open_handle": (_i, [_vp, _vp]),
    "ppll_ipc_close_handle": (_i, [_vp]),
    "ppll_enable_peer": (_i, [_i]),
    "ppll_copy_async": (_i, [_vp, _vp, C.c_size_t, _vp]),
    "ppll_dev_alloc": (_vp, [C.c_size_t]),
    "ppll_dev_free": (_i, [_vp]),
    "ppll_stream_sync": (_i, [_vp]),
}

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A C-ABI call failed (CUDA error or invalid argument)."""


def load():
    """Load the library (idempotent).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"PPLL CUDA library not built ({LIB_PATH} missing); run "
                    "`python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != PPLL_OK:
        msg = load().ppll_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (rc={rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream) -> int:
    return stream.cuda_stream if stream is not None else 0


def launch_count() -> int:
    return int(load().ppll_launch_count())

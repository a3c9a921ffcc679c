"""ctypes binding of libattnpred.so (include/attnpred.h).

This is the only way the package reaches compute: there is no CPU fallback.
If the in-tree library is missing, importing the compute modules raises
:class:`NativeLibraryMissing` (build it with ``python -c "import
__graft_entry__ as g; g.build()"``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors as E

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libattnpred.so"

AP_OK, AP_EPARAM, AP_ECONFIG, AP_ESTATE, AP_ENUMERIC, AP_ECUDA, AP_EFORMAT, AP_ECORRUPT, AP_EVALID, AP_EIO = range(10)
AP_F32, AP_F64, AP_BF16 = 0, 1, 2
PREC = {"fp32": 0, "fp16x3": 1, "fp16": 2}

_ERR = {
    AP_EPARAM: E.ParameterError,
    AP_ECONFIG: E.ConfigError,
    AP_ESTATE: E.StateError,
    AP_ENUMERIC: E.NumericError,
    AP_ECUDA: E.DeviceError,
    AP_EFORMAT: E.FormatError,
    AP_ECORRUPT: E.CorruptionError,
    AP_EVALID: E.ValidationError,
    AP_EIO: OSError,
}


class NativeLibraryMissing(ImportError):
    pass


class MapState(ctypes.Structure):
    _fields_ = [
        ("n_pushed", ctypes.c_int64), ("r_pushed", ctypes.c_int64), ("row_len", ctypes.c_int64),
        ("counter", ctypes.c_int64), ("mid_clip", ctypes.c_int64), ("width", ctypes.c_int32),
        ("r_width", ctypes.c_int32), ("n_mid", ctypes.c_int32), ("r_wgen", ctypes.c_int32),
        ("tie_n", ctypes.c_int32), ("prev_kth", ctypes.c_uint32),
    ]


class Selector(ctypes.Structure):
    _fields_ = [
        ("n_maps", ctypes.c_int32), ("history", ctypes.c_int32), ("block", ctypes.c_int32),
        ("w_max", ctypes.c_int32), ("k_mid", ctypes.c_int32), ("sink", ctypes.c_int32),
        ("local", ctypes.c_int32), ("calib_period", ctypes.c_int32), ("update_interval", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("ring", ctypes.c_void_p), ("rmap", ctypes.c_void_p), ("rsum", ctypes.c_void_p),
        ("slot_width", ctypes.c_void_p), ("slot_xmax", ctypes.c_void_p),
        ("state", ctypes.c_void_p), ("scores", ctypes.c_void_p), ("mid_blocks", ctypes.c_void_p),
        ("mid_mask", ctypes.c_void_p), ("status", ctypes.c_void_p), ("tie_ws", ctypes.c_void_p),
        ("k_map", ctypes.c_void_p), ("fused_done", ctypes.c_void_p),
    ]


class AttnLayerDesc(ctypes.Structure):
    """ap_attn_layer (include/attnpred.h)."""

    _fields_ = [
        ("n_seq", ctypes.c_int32), ("n_q_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("t_max", ctypes.c_int32), ("n_splits", ctypes.c_int32),
        ("block", ctypes.c_int32), ("w_max", ctypes.c_int32),
        ("q", ctypes.c_void_p), ("k_cache", ctypes.c_void_p), ("v_cache", ctypes.c_void_p),
        ("seq_len", ctypes.c_void_p), ("out", ctypes.c_void_p), ("lse", ctypes.c_void_p),
        ("partial", ctypes.c_void_p), ("bmax", ctypes.c_void_p), ("counters", ctypes.c_void_p),
    ]


class VPages(ctypes.Structure):
    """ap_vpages (include/attnpred.h)."""

    _fields_ = [
        ("k_cap", ctypes.c_int32), ("sink_pages", ctypes.c_int32), ("recent_pages", ctypes.c_int32),
        ("pad_", ctypes.c_int32), ("host_t_max", ctypes.c_int64),
        ("pages", ctypes.c_void_p), ("host_v", ctypes.c_void_p), ("mid_page", ctypes.c_void_p),
        ("old_blocks", ctypes.c_void_p), ("old_pages", ctypes.c_void_p), ("old_n", ctypes.c_void_p),
        ("bytes_copied", ctypes.c_void_p),
    ]


MAP_STATE_BYTES = ctypes.sizeof(MapState)  # 64


class TraceHeaderC(ctypes.Structure):
    """ap_trace_header (include/attnpred.h)."""

    _fields_ = [(n, ctypes.c_int32) for n in ("num_layers", "num_heads", "prefill_len", "num_decode_steps",
                                               "has_qk", "head_dim", "first_step_offset", "pad_")]

_P = ctypes.c_void_p
_I32, _I64 = ctypes.c_int32, ctypes.c_int64

# symbol -> (restype, argtypes); the table is also what tests check the .so exports
SIGNATURES = {
    "ap_version": (ctypes.c_int, []),
    "ap_last_error": (ctypes.c_char_p, []),
    "ap_device_sm_count": (ctypes.c_int, []),
    "ap_set_weights": (ctypes.c_int, [_P, _P]),
    "ap_max_pool": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _I64, _I32, _P, ctypes.c_int, _I64, _P]),
    "ap_expand_indices": (ctypes.c_int, [_P, _I32, _I32, _I64, _P, _P, _P, _P]),
    "ap_topk": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _I32, _I32, _P, _I64, _P, _P, _P]),
    "ap_predict_forward": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _I64, _P, _I64, _P, ctypes.c_int, _P, _P]),
    "ap_sel_reset": (ctypes.c_int, [ctypes.POINTER(Selector), _P]),
    "ap_sel_push_rows": (ctypes.c_int, [ctypes.POINTER(Selector), _P, ctypes.c_int, _I64, _I64, ctypes.c_int, _P]),
    "ap_sel_push_compressed": (ctypes.c_int, [ctypes.POINTER(Selector), _P, _I64, _I64, ctypes.c_int, _P]),
    "ap_sel_step": (ctypes.c_int, [ctypes.POINTER(Selector), ctypes.c_int, _P]),
    "ap_sel_step_grid": (ctypes.c_int, [ctypes.POINTER(Selector), ctypes.c_int, ctypes.c_int, _P]),
    "ap_set_sm_reserve": (ctypes.c_int, [ctypes.c_int]),
    "ap_sm_budget": (ctypes.c_int, []),
    "ap_sel_grid_ctas": (ctypes.c_int, [ctypes.c_int]),
    "ap_sel_tie_ws_bytes": (ctypes.c_int64, [_I32]),
    "ap_sel_tie_stats": (ctypes.c_int, [_P, _P]),
    "ap_sel_set_tie_guard": (ctypes.c_int, [ctypes.c_int, ctypes.c_float, ctypes.c_float]),
    "ap_sel_set_tie_guard_f16": (ctypes.c_int, [ctypes.c_float, ctypes.c_float]),
    "ap_attn_dense": (ctypes.c_int, [ctypes.POINTER(AttnLayerDesc), ctypes.c_int, ctypes.POINTER(Selector),
                                     _I32, _I32, _I32, ctypes.c_int, _P]),
    "ap_attn_set_calib_kernel": (ctypes.c_int, [ctypes.c_int]),
    "ap_attn_sparse": (ctypes.c_int, [ctypes.POINTER(AttnLayerDesc), ctypes.POINTER(Selector), _I32, _I32, _I32,
                                      ctypes.c_int, _P]),
    "ap_attn_sparse_prefetch": (ctypes.c_int, [ctypes.POINTER(AttnLayerDesc), ctypes.POINTER(Selector), _I32, _I32,
                                               _I32, _P]),
    "ap_prefetch": (ctypes.c_int, [ctypes.POINTER(Selector), ctypes.POINTER(VPages), _I32, _I32, _I32, _I32, _P]),
    "ap_v_append": (ctypes.c_int, [_P, _I32, _I32, _P, ctypes.POINTER(VPages), _I32, _I32, _P]),
    "ap_v_pages_init": (ctypes.c_int, [ctypes.POINTER(VPages), _I64, _I64, _P]),
    "ap_attn_sparse_paged": (ctypes.c_int, [ctypes.POINTER(AttnLayerDesc), ctypes.POINTER(Selector), _I32, _I32,
                                            _I32, ctypes.c_int, ctypes.POINTER(VPages), _I32, _P]),
    "ap_rmsnorm": (ctypes.c_int, [_P, _P, _P, _P, _I32, _I32, ctypes.c_float, _P]),
    "ap_rope_append": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, _P, _P, _I32, ctypes.c_float, _P]),
    "ap_silu_mul": (ctypes.c_int, [_P, _P, _I32, _I32, _P]),
    "ap_advance": (ctypes.c_int, [_P, _I32, _I32, _P]),
    "ap_advance_embed": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _P, _I32, _P]),
    "ap_gemv": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, ctypes.c_float, _P, _P, _P]),
    "ap_gemm_tc_workspace_bytes": (ctypes.c_int64, [_I32, _I32, _I32]),
    "ap_gemm_tc": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _P, ctypes.c_int64, _P]),
    "ap_argmax_workspace_bytes": (ctypes.c_int64, [_I32]),
    "ap_argmax_rows": (ctypes.c_int, [_P, _I32, _I64, _P, _I64, _P, _P]),
    "ap_gemv_qkv_rope": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, ctypes.c_float, _P, _P,
                                        _P, _P, _I32, ctypes.c_float, _P]),
    # .att1 trace container (host code)
    "ap_trace_check_header": (ctypes.c_int, [ctypes.POINTER(TraceHeaderC)]),
    "ap_trace_check_row": (ctypes.c_int, [_P, _I64, _I32, _I32, _I32]),
    "ap_trace_nbytes": (_I64, [ctypes.POINTER(TraceHeaderC)]),
    "ap_trace_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_P)]),
    "ap_trace_open_memory": (ctypes.c_int, [_P, _I64, ctypes.POINTER(_P)]),
    "ap_trace_close": (None, [_P]),
    "ap_trace_get_header": (ctypes.c_int, [_P, ctypes.POINTER(TraceHeaderC)]),
    "ap_trace_validate": (ctypes.c_int, [_P]),
    "ap_trace_read_rows": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I64, _I64]),
    "ap_trace_gather_step": (ctypes.c_int, [_P, _I32, _P, _I64, _I64]),
    "ap_trace_read_qk": (ctypes.c_int, [_P, _I32, _I32, _P, _P]),
    "ap_trace_writer_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(TraceHeaderC), ctypes.POINTER(_P)]),
    "ap_trace_writer_append_row": (ctypes.c_int, [_P, _P, _I64]),
    "ap_trace_writer_append_qk": (ctypes.c_int, [_P, _P, _P]),
    "ap_trace_writer_finish": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
    "ap_trace_writer_bytes": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    "ap_trace_writer_free": (None, [_P]),
    # forecaster training (predictor.backward / train)
    "ap_train_workspace_bytes": (ctypes.c_int64, [_I32, _I32, _I32]),
    "ap_train_backward": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _P, _P, _P, _P, ctypes.c_int64, _P]),
    "ap_adam_step": (ctypes.c_int, [_P, _P, _P, _P, _I32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, _I64, _P]),
    "ap_forward_f64_workspace_bytes": (ctypes.c_int64, [_I32, _I32, _I32]),
    "ap_predict_forward_f64": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, _I64, _P, ctypes.c_int64, _P]),
}

_lib = None


def load():
    """Load (once) and return the native library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("ATTNPRED_LIB", LIB_PATH))
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path} not found: the CUDA path is the only implementation; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # optional symbols are checked by callers / tests
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def fn(name: str):
    lib = load()
    f = getattr(lib, name, None)
    if f is None:
        raise NativeLibraryMissing(f"{LIB_PATH.name} does not export {name}")
    if name in SIGNATURES:
        f.restype, f.argtypes = SIGNATURES[name]
    return f


def check(rc: int, what: str = "") -> None:
    """Map a synchronous AP_E* status to the reference exception classes."""
    if rc == AP_OK:
        return
    msg = load().ap_last_error()
    text = msg.decode() if msg else what
    raise _ERR.get(rc, E.DeviceError)(text or f"{what} failed with status {rc}")


def raise_device_status(code: int, what: str) -> None:
    """Map a device status word (set by kernels) to an exception."""
    if code == 0:
        return
    msgs = {
        AP_ENUMERIC: f"{what}: non-finite values encountered",
        AP_EPARAM: f"{what}: index out of range",
    }
    raise _ERR.get(code, E.DeviceError)(msgs.get(code, f"{what}: device status {code}"))


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)

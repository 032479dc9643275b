"""ctypes loader for libamun.so (the C-ABI in include/amun.h).

No fallback: if the library is missing or fails to load, importing the
binding raises. Build it with `python -c "import __graft_entry__ as g; g.build()"`.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# AMUN_LIB may point at an alternative build of the same ABI (experiments).
LIB_PATH = os.environ.get("AMUN_LIB", os.path.join(_HERE, "libamun.so"))

AMUN_OK, AMUN_EINVAL, AMUN_EUNSUPPORTED, AMUN_ECUDA = 0, 1, 2, 3
AMUN_F32, AMUN_BF16, AMUN_E4M3, AMUN_TF32X3, AMUN_MXFP4 = 0, 1, 2, 3, 4
AMUN_MAX_K = 16
AMUN_MAX_COLUMNS = 16

EXPORTS = [
    "amun_abi_version", "amun_last_error", "amun_status_string", "amun_ol_create",
    "amun_ol_destroy", "amun_ol_workspace_bytes", "amun_ol_partial_stride",
    "amun_output_layer", "amun_output_layer_dev", "amun_ol_scores", "amun_ol_select", "amun_output_layer_partial",
    "amun_merge_partials", "amun_argmax", "amun_debug_logits", "amun_bench_variant", "amun_compact",
    "amun_beam_advance_workspace_bytes", "amun_beam_advance", "amun_output_layer_e4m3",
    "amun_ol_scores_e4m3", "amun_quantize_e4m3", "amun_output_layer_partial_e4m3",
    "amun_argmax_e4m3", "amun_split_tf32x3", "amun_oneshot_buffer_bytes", "amun_oneshot_alloc",
    "amun_oneshot_free", "amun_oneshot_open", "amun_oneshot_close", "amun_output_layer_oneshot",
    "amun_output_layer_oneshot_emulated", "amun_sentence_alive", "amun_ol_workspace_init",
    "amun_debug_timeline", "amun_ol_launches_per_call", "amun_oneshot_error",
    "amun_mxfp4_sf_bytes", "amun_quantize_mxfp4", "amun_output_layer_mxfp4", "amun_ol_scores_mxfp4",
    "amun_argmax_mxfp4", "amun_debug_logits_mxfp4",
]
AMUN_ONESHOT_MAX_G = 8


class amun_column(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("row_bytes", ctypes.c_int64)]


class AmunError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "AMUN_OK", 1: "AMUN_EINVAL", 2: "AMUN_EUNSUPPORTED", 3: "AMUN_ECUDA"}

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    st = ctypes.c_int
    sig = {
        "amun_abi_version": (i32, []),
        "amun_last_error": (ctypes.c_char_p, []),
        "amun_status_string": (ctypes.c_char_p, [st]),
        "amun_ol_create": (st, [ctypes.POINTER(vp), i32, i32, i32, i32, i32, i32, i32, i32, i32]),
        "amun_ol_destroy": (st, [vp]),
        "amun_ol_workspace_bytes": (sz, [vp]),
        "amun_ol_partial_stride": (i32, [vp]),
        "amun_ol_workspace_init": (st, [vp, vp, vp]),
        "amun_debug_timeline": (st, [vp, vp]),
        "amun_ol_launches_per_call": (i32, [vp, i32]),
        "amun_oneshot_error": (st, [vp, vp]),
        "amun_output_layer": (st, [vp, vp, vp, vp, vp, vp, i32, i32, vp, i32, vp, vp, vp, vp]),
        "amun_output_layer_dev": (st, [vp, vp, vp, vp, vp, vp, vp, i32, vp, i32, vp, vp, vp, vp]),
        "amun_ol_scores": (st, [vp, vp, vp, vp, i32, vp, vp]),
        "amun_ol_select": (st, [vp, vp, vp, vp, i32, i32, vp, i32, vp, vp, vp]),
        "amun_output_layer_partial": (st, [vp, vp, vp, vp, i32, vp, vp, vp]),
        "amun_merge_partials": (st, [vp, vp, i32, vp, vp, i32, i32, vp, i32, vp, vp, vp]),
        "amun_argmax": (st, [vp, vp, vp, vp, i32, vp, vp, vp, vp]),
        "amun_debug_logits": (st, [vp, vp, vp, vp, i32, vp, vp, vp]),
        "amun_bench_variant": (st, [vp, vp, vp, vp, i32, i32, vp, vp]),
        "amun_compact": (st, [ctypes.POINTER(amun_column), i32, vp, i32, vp, i32, vp, vp, vp, vp, vp]),
        "amun_beam_advance_workspace_bytes": (sz, [i32, i32]),
        "amun_output_layer_e4m3": (st, [vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, i32, vp, vp,
                                        vp, vp]),
        "amun_ol_scores_e4m3": (st, [vp, vp, vp, vp, vp, vp, i32, i32, vp, vp]),
        "amun_quantize_e4m3": (st, [vp, i32, i32, i32, vp, vp, vp]),
        "amun_output_layer_partial_e4m3": (st, [vp, vp, vp, vp, vp, vp, i32, vp, vp, vp]),
        "amun_argmax_e4m3": (st, [vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp]),
        "amun_split_tf32x3": (st, [vp, i32, i32, i32, vp, vp]),
        "amun_mxfp4_sf_bytes": (sz, [i32, i32]),
        "amun_quantize_mxfp4": (st, [vp, i32, i32, i32, vp, vp, vp]),
        "amun_output_layer_mxfp4": (st, [vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp, i32, vp, vp,
                                         vp, vp]),
        "amun_ol_scores_mxfp4": (st, [vp, vp, vp, vp, vp, vp, i32, i32, vp, vp]),
        "amun_argmax_mxfp4": (st, [vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp]),
        "amun_debug_logits_mxfp4": (st, [vp, vp, vp, vp, vp, vp, i32, vp, vp, vp]),
        "amun_oneshot_buffer_bytes": (sz, [vp, i32]),
        "amun_sentence_alive": (st, [vp, i32, vp, vp, vp]),
        "amun_oneshot_alloc": (st, [vp, i32, ctypes.POINTER(vp), vp]),
        "amun_oneshot_free": (st, [vp]),
        "amun_oneshot_open": (st, [vp, i32, ctypes.POINTER(vp)]),
        "amun_oneshot_close": (st, [vp]),
        "amun_output_layer_oneshot": (st, [vp, vp, vp, vp, vp, vp, i32, i32, vp, i32,
                                           ctypes.POINTER(vp), i32, i32, vp, vp, vp, vp]),
        "amun_output_layer_oneshot_emulated": (st, [ctypes.POINTER(vp), i32, vp, ctypes.POINTER(vp),
                                                    ctypes.POINTER(vp), vp, vp, i32, i32, vp, i32,
                                                    ctypes.POINTER(vp), ctypes.POINTER(vp),
                                                    ctypes.POINTER(vp), ctypes.POINTER(vp), vp]),
        "amun_beam_advance": (st, [vp, vp, i32, i32, ctypes.c_int64, i32, i32,
                                   ctypes.POINTER(amun_column), i32, vp, vp, vp, vp, vp, vp, vp,
                                   vp]),
    }
    alt = "AMUN_LIB" in os.environ   # an older build (A/B experiments) may lack newer calls
    for name, (res, args) in sig.items():
        if alt and not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != AMUN_OK:
        msg = load().amun_last_error().decode(errors="replace")
        raise AmunError(status, msg)

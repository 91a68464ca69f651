"""ctypes binding of libstpc_b200.so (include/stpc_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every entry point raises ``NativeUnavailable`` instead of
computing anything on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CodecError

LIB_PATH = os.environ.get(
    "STPC_B200_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstpc_b200.so"))

STPC_NSTAT = 9
(STAT_REJECTED, STAT_DROPPED, STAT_KEPT, STAT_VALID, STAT_TEMPORAL, STAT_FALLBACK,
 STAT_RESIDUAL, STAT_ESCAPES, STAT_EPS_BAND) = range(STPC_NSTAT)
(BUF_BEST, BUF_CLS, BUF_RUN_S, BUF_RUN_LEN, BUF_RUN_ABC, BUF_N_RUNS, BUF_REF_OK, BUF_REF_C,
 BUF_PAYLOAD, BUF_VBITS) = range(10)

# every symbol include/stpc_b200.h declares
EXPORTS = [
    "stpc_encoder_create", "stpc_encoder_destroy", "stpc_encode_device", "stpc_encode_host", "stpc_encoder_wait",
    "stpc_encode_host_gather", "stpc_result_host_blobs",
    "stpc_result_groups", "stpc_result_blobs", "stpc_result_device_blobs",
    "stpc_result_copy_blobs", "stpc_result_frame_stats", "stpc_result_payload_lengths",
    "stpc_encoder_buffer", "stpc_project", "stpc_malloc", "stpc_free", "stpc_memcpy_d2h",
    "stpc_memcpy_h2d", "stpc_host_scatter", "stpc_device_count", "stpc_last_error", "stpc_version",
    "stpc_encoder_profile", "stpc_encoder_stage_ms", "stpc_stage_name", "stpc_launch_count",
    "stpc_decoder_create", "stpc_decoder_destroy", "stpc_decoder_load", "stpc_decoder_load_gather",
    "stpc_decoder_heads", "stpc_decode_transforms",
    "stpc_decoder_frames", "stpc_decoder_total_points", "stpc_decoder_points",
    "stpc_decoder_device_points", "stpc_entropy_encode",
]

# stpc_decoder_* status kinds
DEC_TRUNCATED, DEC_MALFORMED, DEC_CHECKSUM, DEC_VERSION = 1, 2, 3, 4


class NativeUnavailable(CodecError):
    """libstpc_b200 is not built or no CUDA device is present (no CPU fallback)."""


class StpcDecodeGeom(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int32) for name in ("w", "h", "tile_w", "tile_h", "n_frames", "k_index")] + [
        ("range_quant", ctypes.c_double), ("r_max", ctypes.c_double)]


class StpcConfig(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("tile_w", ctypes.c_int32),
        ("tile_h", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("h", ctypes.c_int32),
        ("n_frames", ctypes.c_int32),
        ("k_index", ctypes.c_int32),
        ("points_f64", ctypes.c_int32),
        ("tau", ctypes.c_double),
        ("theta_r", ctypes.c_double),
        ("phi_r", ctypes.c_double),
        ("phi_offset", ctypes.c_double),
        ("range_quant", ctypes.c_double),
        ("r_max", ctypes.c_double),
        ("cond_limit", ctypes.c_double),
    ]


_lock = threading.Lock()
_lib = None


def load(require_device: bool = False):
    """Load (never build) the in-tree library and declare its signatures."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} missing; build it with `python -m paper_2008_06972_b200.build`"
                )
            L = ctypes.CDLL(LIB_PATH)
            P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
            sig = {
                "stpc_encoder_create": ([ctypes.POINTER(StpcConfig), P, P, P, P, ctypes.POINTER(P)], ctypes.c_int),
                "stpc_encoder_destroy": ([P], None),
                "stpc_encode_device": ([P, I32, P, P, P, P], ctypes.c_int),
                "stpc_encode_host": ([P, I32, P, P, P, P, I64, P], ctypes.c_int),
                "stpc_result_groups": ([P], I32),
                "stpc_result_blobs": ([P, P, P], ctypes.c_int),
                "stpc_result_device_blobs": ([P], P),
                "stpc_result_copy_blobs": ([P, P, I64, P], ctypes.c_int),
                "stpc_result_frame_stats": ([P, P], ctypes.c_int),
                "stpc_result_payload_lengths": ([P, P], ctypes.c_int),
                "stpc_encoder_buffer": ([P, I32, ctypes.POINTER(P), ctypes.POINTER(I64)], ctypes.c_int),
                "stpc_project": ([P, I32, P, I32, P, I32, I32, D, D, D, P, P, P, P], ctypes.c_int),
                "stpc_malloc": ([ctypes.POINTER(P), I64], ctypes.c_int),
                "stpc_free": ([P], ctypes.c_int),
                "stpc_memcpy_d2h": ([P, P, I64], ctypes.c_int),
                "stpc_memcpy_h2d": ([P, P, I64], ctypes.c_int),
                "stpc_host_scatter": ([P, P, P, P, I32], ctypes.c_int),
                "stpc_device_count": ([], ctypes.c_int),
                "stpc_last_error": ([], ctypes.c_char_p),
                "stpc_version": ([], ctypes.c_char_p),
                "stpc_encoder_profile": ([P, I32], ctypes.c_int),
                "stpc_encoder_stage_ms": ([P, P, I32], I32),
                "stpc_stage_name": ([I32], ctypes.c_char_p),
                "stpc_launch_count": ([], ctypes.c_uint64),
                "stpc_encoder_wait": ([P, P], ctypes.c_int),
                "stpc_encode_host_gather": ([P, I32, P, P, P, P], ctypes.c_int),
                "stpc_result_host_blobs": ([P], P),
                "stpc_decoder_create": ([ctypes.POINTER(P)], ctypes.c_int),
                "stpc_decoder_destroy": ([P], None),
                "stpc_decoder_load": ([P, P, I32, P, I32, P, P], ctypes.c_int),
                "stpc_decoder_load_gather": ([P, P, P, I32, P, P], ctypes.c_int),
                "stpc_decoder_heads": ([P, I32, P, P, P], ctypes.c_int),
                "stpc_decode_transforms": ([P, I64, P, I32, I32, I32, D, P, P, P], ctypes.c_int),
                "stpc_decoder_frames": ([P, ctypes.POINTER(StpcDecodeGeom), P, I32, P, P, P, P, P, P, P, P, P],
                                        ctypes.c_int),
                "stpc_decoder_total_points": ([P], I64),
                "stpc_decoder_points": ([P, P, I32, I64, P], ctypes.c_int),
                "stpc_decoder_device_points": ([P], P),
                "stpc_entropy_encode": ([P, P, I32, P, I64, P], ctypes.c_int),
            }
            for name, (args, res) in sig.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
    if require_device and _lib.stpc_device_count() < 1:
        raise NativeUnavailable("no CUDA device visible to libstpc_b200 (no CPU fallback)")
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.stpc_last_error().decode(errors="replace") if _lib is not None else "?"
        raise CodecError(f"libstpc_b200 error {rc}: {msg}")

"""ctypes binding of the vitdec_b200 C-ABI (include/vitdec_b200.h).

The shared library is built in-tree (``make -C paper_2011_09337_b200`` or
``__graft_entry__.build()``). There is no fallback: if the library is missing
every entry point raises, and without a CUDA device the decode calls fail
with ``VD_ECUDA``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

# VITDEC_LIB selects another build of the same library (kernel tuning A/B runs).
LIB_PATH = Path(os.environ.get("VITDEC_LIB") or Path(__file__).resolve().with_name("libvitdec_b200.so"))

VD_OK, VD_EINVAL, VD_ECUDA, VD_EUNSUPPORTED, VD_ENOMEM = 0, 1, 2, 3, 4


class VdFrameCfg(C.Structure):
    """struct vd_frame_cfg (reference decoder.hpp:20-31 FrameConfig)."""

    _fields_ = [
        ("f", C.c_int32),
        ("v1", C.c_int32),
        ("v2", C.c_int32),
        ("f0", C.c_int32),
        ("start", C.c_int32),
        ("reserved", C.c_int32),
        ("seed", C.c_uint64),
    ]


class VdStats(C.Structure):
    """struct vd_stats (reference decoder.hpp:33-37 DecodeStats)."""

    _fields_ = [("frames", C.c_int64), ("stages", C.c_int64), ("tracebacks", C.c_int64)]


class VdPuncture(C.Structure):
    """struct vd_puncture (reference codec.hpp:13-33 PuncturePattern)."""

    _fields_ = [("b", C.c_int32), ("period", C.c_int32), ("mask", C.c_void_p)]


class VdExec(C.Structure):
    _fields_ = [("num_devices", C.c_int32), ("devices", C.POINTER(C.c_int32)), ("chunk_stages", C.c_int64)]


P = C.c_void_p
I32, I64, U64, DBL = C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); the complete set of symbols include/vitdec_b200.h declares.
SIGNATURES = {
    "vd_code_create": (I32, [I32, I32, P, C.POINTER(P)]),
    "vd_code_destroy": (None, [P]),
    "vd_code_k": (I32, [P]),
    "vd_code_b": (I32, [P]),
    "vd_code_tables": (I32, [P, P, P, P, P, P]),
    "vd_code_fast_path": (I32, [P]),
    "vd_code_jit_check": (I32, [P]),
    "vd_frame_cfg_validate": (I32, [C.POINTER(VdFrameCfg), I32]),
    "vd_frame_stats": (I32, [C.POINTER(VdFrameCfg), I64, C.POINTER(VdStats)]),
    "vd_partition_frames": (I32, [C.POINTER(VdFrameCfg), I64, I32, P]),
    "vd_decode_i8_device": (I32, [P, C.POINTER(VdFrameCfg), I64, P, I64, I64, I64, P, I64, P, I32, P]),
    "vd_decode_f64_device": (I32, [P, C.POINTER(VdFrameCfg), I64, P, I64, I64, I64, P, I64, P, I32, P]),
    "vd_frame_window": (I32, [C.POINTER(VdFrameCfg), I64, I64, I64, C.POINTER(I64), C.POINTER(I64)]),
    "vd_decode_batch_i8_device": (I32, [P, C.POINTER(VdFrameCfg), I32, P, P, P, C.POINTER(VdStats), I32, P]),
    "vd_decode_batch_f64_device": (I32, [P, C.POINTER(VdFrameCfg), I32, P, P, P, C.POINTER(VdStats), I32, P]),
    "vd_decode_batch_i8": (I32, [P, C.POINTER(VdFrameCfg), I32, P, P, P, C.POINTER(VdStats), C.POINTER(VdExec)]),
    "vd_decode_i8": (I32, [P, C.POINTER(VdFrameCfg), P, I64, P, C.POINTER(VdStats), C.POINTER(VdExec)]),
    "vd_decode_f64": (I32, [P, C.POINTER(VdFrameCfg), P, I64, P, C.POINTER(VdStats), C.POINTER(VdExec)]),
    "vd_serial_decode_f64": (I32, [P, P, I64, P, C.POINTER(VdStats), I32]),
    "vd_synth_llr_i8_device": (I32, [P, I64, DBL, DBL, U64, P, P, I32, P]),
    "vd_synth_llr_i8_range_device": (I32, [P, I64, I64, DBL, DBL, U64, P, P, I32, P]),
    "vd_kernel_launches": (U64, []),
    "vd_count_bit_errors_device": (I32, [P, P, I64, P, I32, P]),
    "vd_puncture_validate": (I32, [C.POINTER(VdPuncture)]),
    "vd_depuncture_stages": (I32, [C.POINTER(VdPuncture), I64, C.POINTER(I64)]),
    "vd_depuncture_i8_device": (I32, [C.POINTER(VdPuncture), P, I64, P, I32, P]),
    "vd_depuncture_f64": (I32, [C.POINTER(VdPuncture), P, I64, P]),
    "vd_decode_punctured_i8": (I32, [P, C.POINTER(VdFrameCfg), C.POINTER(VdPuncture), P, I64, P, C.POINTER(VdStats),
                                     C.POINTER(VdExec)]),
    "vd_decode_punctured_i8_device": (I32, [P, C.POINTER(VdFrameCfg), C.POINTER(VdPuncture), P, I64, P, P,
                                            C.POINTER(VdStats), I32, P]),
    "vd_decode_i4": (I32, [P, C.POINTER(VdFrameCfg), P, I64, P, C.POINTER(VdStats), C.POINTER(VdExec)]),
    "vd_unpack_i4_device": (I32, [P, I64, P, I32, P]),
    "vd_last_error": (C.c_char_p, []),
    "vd_version": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libvitdec_b200.so (once). Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `make -C paper_2011_09337_b200` "
                    "(or __graft_entry__.build()); there is no CPU fallback"
                )
            h = C.CDLL(os.fspath(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


class VitdecError(RuntimeError):
    """A non-VD_EINVAL failure of the C-ABI (CUDA error, unsupported, OOM)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def check(status: int) -> None:
    """Map vd_status to Python: VD_EINVAL -> ValueError (the reference's
    std::invalid_argument, same message), anything else -> VitdecError."""
    if status == VD_OK:
        return
    msg = lib().vd_last_error().decode()
    if status == VD_EINVAL:
        raise ValueError(msg)
    raise VitdecError(status, msg)

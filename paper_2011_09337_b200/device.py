"""Device-resident entry points (HBM in, HBM out) for benchmarks and tests.

These pass raw device pointers and a CUDA stream handle straight to the
C-ABI; torch tensors are used only as device allocations / streams
(plumbing). The decode itself is ``vd_decode_i8_device`` (the hot path).
"""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib
from .api import FrameConfig, Trellis


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(stream) -> int:
    if stream is None:
        return 0
    return int(getattr(stream, "cuda_stream", stream))


def decode_i8_device(trellis: Trellis, cfg: FrameConfig, n: int, llr, llr_stage0: int, frame_begin: int,
                     frame_end: int, out, out_stage0: int, sigma=None, device: int = -1, stream=None) -> None:
    """vd_decode_i8_device on torch CUDA tensors (llr: int8, out: int32/uint32
    words, sigma: optional int64 [frames, S])."""
    c = cfg.to_c()
    check(lib().vd_decode_i8_device(trellis.handle, C.byref(c), int(n), _ptr(llr), int(llr_stage0),
                                    int(frame_begin), int(frame_end), _ptr(out), int(out_stage0), _ptr(sigma),
                                    int(device), _stream(stream)))


def decode_f64_device(trellis: Trellis, cfg: FrameConfig, n: int, llr, llr_stage0: int, frame_begin: int,
                      frame_end: int, out, out_stage0: int, sigma=None, device: int = -1, stream=None) -> None:
    c = cfg.to_c()
    check(lib().vd_decode_f64_device(trellis.handle, C.byref(c), int(n), _ptr(llr), int(llr_stage0),
                                     int(frame_begin), int(frame_end), _ptr(out), int(out_stage0), _ptr(sigma),
                                     int(device), _stream(stream)))


def decode_batch_i8_device(trellis: Trellis, cfg: FrameConfig, block_stages, llr, out, device: int = -1,
                           stream=None):
    """vd_decode_batch_i8_device: independent blocks (host list of stage
    counts) concatenated in the int8 device tensor ``llr``; packed bits of
    every block, back to back, into ``out``. Returns the summed stats."""
    import numpy as np

    from ._lib import VdStats

    lens = np.ascontiguousarray(np.asarray(block_stages, np.int64))
    c = cfg.to_c()
    st = VdStats()
    check(lib().vd_decode_batch_i8_device(trellis.handle, C.byref(c), int(lens.size), lens.ctypes.data, _ptr(llr),
                                          _ptr(out), C.byref(st), int(device), _stream(stream)))
    return st


def synth_llr_i8(trellis: Trellis, n: int, sigma: float, scale: float, seed: int, llr, bits=None, device: int = -1,
                 stream=None) -> None:
    """Fill an int8 device tensor with n stages of synthetic AWGN LLRs."""
    check(lib().vd_synth_llr_i8_device(trellis.handle, int(n), float(sigma), float(scale),
                                       int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(llr), _ptr(bits), int(device),
                                       _stream(stream)))


def synth_llr_i8_range(trellis: Trellis, t_begin: int, n: int, sigma: float, scale: float, seed: int, llr,
                       bits=None, device: int = -1, stream=None) -> None:
    """Stages [t_begin, t_begin + n) of the synth_llr_i8 stream (a shard's window)."""
    check(lib().vd_synth_llr_i8_range_device(trellis.handle, int(t_begin), int(n), float(sigma), float(scale),
                                             int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(llr), _ptr(bits), int(device),
                                             _stream(stream)))


def count_bit_errors(a, b, n_bits: int, count, device: int = -1, stream=None) -> None:
    check(lib().vd_count_bit_errors_device(_ptr(a), _ptr(b), int(n_bits), _ptr(count), int(device),
                                           _stream(stream)))


def depuncture_i8_device(pattern, punctured, n_punctured: int, llr, device: int = -1, stream=None) -> None:
    """vd_depuncture_i8_device: punctured int8 device tensor -> stage-major
    int8 block (0 at punctured positions) in ``llr`` (4-byte aligned)."""
    pc = pattern.to_c()
    check(lib().vd_depuncture_i8_device(C.byref(pc), _ptr(punctured), int(n_punctured), _ptr(llr), int(device),
                                        _stream(stream)))


def decode_punctured_i8_device(trellis: Trellis, cfg: FrameConfig, pattern, punctured, n_punctured: int, scratch,
                               out, device: int = -1, stream=None) -> None:
    """vd_decode_punctured_i8_device: device depuncture into ``scratch`` then
    the framed decode of every frame into ``out``."""
    c = cfg.to_c()
    pc = pattern.to_c()
    check(lib().vd_decode_punctured_i8_device(trellis.handle, C.byref(c), C.byref(pc), _ptr(punctured),
                                              int(n_punctured), _ptr(scratch), _ptr(out), None, int(device),
                                              _stream(stream)))

"""B200-native framed soft-decision Viterbi decoder (arXiv 2011.09337 hot path).

The decode path is hand-written sm_100a CUDA behind a C-ABI
(include/vitdec_b200.h, libvitdec_b200.so). This package is the Python
mirror of the reference C++ API (``vitdec::``) over that C-ABI; see
DESIGN.md and INTEGRATION.md.
"""
from ._lib import LIB_PATH, VitdecError, lib
from .api import (
    CodeSpec,
    DecodeOutput,
    DecodeStats,
    FrameConfig,
    PuncturePattern,
    TracebackStart,
    Trellis,
    build_trellis,
    depuncture_stages,
    frame_stats,
    frame_window,
    framed_decode,
    framed_decode_batch,
    framed_decode_punctured,
    framed_decode_stream,
    framed_decode_stream_i4,
    pack_bits,
    pack_i4,
    partition_frames,
    serial_decode,
    unpack_bits,
    unpack_i4,
)

__all__ = [
    "LIB_PATH",
    "VitdecError",
    "lib",
    "CodeSpec",
    "DecodeOutput",
    "DecodeStats",
    "FrameConfig",
    "PuncturePattern",
    "TracebackStart",
    "Trellis",
    "build_trellis",
    "depuncture_stages",
    "frame_stats",
    "frame_window",
    "framed_decode",
    "framed_decode_batch",
    "framed_decode_punctured",
    "framed_decode_stream",
    "framed_decode_stream_i4",
    "pack_bits",
    "pack_i4",
    "partition_frames",
    "serial_decode",
    "unpack_bits",
    "unpack_i4",
]

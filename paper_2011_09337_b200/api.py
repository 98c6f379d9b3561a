"""Python mirror of the reference vitdec decoder API over the C-ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(reference proj/include/vitdec/trellis.hpp, decoder.hpp): ``CodeSpec``,
``build_trellis``, ``FrameConfig`` (with ``validate``), ``framed_decode``,
``serial_decode``, ``DecodeOutput``/``DecodeStats``. ``std::invalid_argument``
becomes ``ValueError`` with the same message. All decoding runs on the GPU
through libvitdec_b200.so; there is no Python/CPU decode path.

LLR blocks follow the reference ``LlrBlock`` convention: a B x N array
(rows = code outputs, columns = stages). A C-contiguous (N, B) array or a
flat stage-major stream is accepted by the ``*_stream`` helpers.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import VD_EUNSUPPORTED, VdPuncture, VdExec, VdFrameCfg, VdStats, VitdecError, check, lib

__all__ = [
    "CodeSpec",
    "Trellis",
    "build_trellis",
    "TracebackStart",
    "FrameConfig",
    "DecodeStats",
    "DecodeOutput",
    "framed_decode",
    "serial_decode",
    "framed_decode_stream",
    "frame_stats",
    "partition_frames",
    "frame_window",
    "unpack_bits",
    "pack_bits",
]


@dataclass
class CodeSpec:
    """reference trellis.hpp:14-25."""

    k: int = 0
    b: int = 0
    polys: list = field(default_factory=list)

    @staticmethod
    def from_octal(k: int, octal_csv: str) -> "CodeSpec":
        polys = []
        for tok in octal_csv.split(","):
            if not tok:
                continue
            try:
                polys.append(int(tok, 8))
            except ValueError:
                raise ValueError("bad octal polynomial: " + tok) from None
        return CodeSpec(k, len(polys), polys)

    def num_states(self) -> int:
        return 1 << (self.k - 1)

    def base_rate(self) -> float:
        return 1.0 / self.b

    def polys_octal(self) -> str:
        return ",".join(format(p, "o") for p in self.polys)


class Trellis:
    """reference trellis.hpp:30-76, backed by a C-ABI ``vd_code``."""

    def __init__(self, spec: CodeSpec):
        if spec.k >= 2 and spec.b >= 2 and len(spec.polys) != spec.b:
            raise ValueError("polynomial count must equal B")
        self.spec = spec
        polys = (C.c_uint32 * max(spec.b, 1))(*([int(p) for p in spec.polys] + [0] * max(0, spec.b - len(spec.polys))))
        h = C.c_void_p()
        check(lib().vd_code_create(spec.k, spec.b, C.cast(polys, C.c_void_p), C.byref(h)))
        self._h = h
        s = 1 << (spec.k - 1)
        self._next = np.zeros(2 * s, np.uint32)
        self._out = np.zeros(2 * s, np.uint32)
        self._pred = np.zeros(2 * s, np.uint32)
        self._in_out = np.zeros(2 * s, np.uint32)
        cp = C.c_int32()
        check(
            lib().vd_code_tables(
                h, self._next.ctypes.data, self._out.ctypes.data, self._pred.ctypes.data, self._in_out.ctypes.data,
                C.addressof(cp),
            )
        )
        self._cp = bool(cp.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().vd_code_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def num_states(self) -> int:
        return 1 << (self.spec.k - 1)

    def constraint_length(self) -> int:
        return self.spec.k

    def outputs_per_bit(self) -> int:
        return self.spec.b

    def next_state(self, state: int, inp: int) -> int:
        return int(self._next[state * 2 + inp])

    def branch_output(self, state: int, inp: int) -> int:
        return int(self._out[state * 2 + inp])

    def predecessors(self, state: int):
        return int(self._pred[state * 2]), int(self._pred[state * 2 + 1])

    def incoming_output(self, state: int, which: int) -> int:
        return int(self._in_out[state * 2 + which])

    def branch_input(self, state: int) -> int:
        return state >> (self.spec.k - 2)

    def complement_paired(self) -> bool:
        return self._cp

    def incoming_output_data(self) -> np.ndarray:
        return self._in_out

    def fast_path(self) -> bool:
        """Whether the register-resident kernel (vd_fast.cu) serves this code."""
        return bool(lib().vd_code_fast_path(self._h))


def build_trellis(spec: CodeSpec) -> Trellis:
    return Trellis(spec)


class TracebackStart(enum.IntEnum):
    kStoredMax = 0
    kRandom = 1


@dataclass
class FrameConfig:
    """reference decoder.hpp:20-31."""

    f: int = 0
    v1: int = 0
    v2: int = 0
    f0: int = 0
    start: TracebackStart = TracebackStart.kStoredMax
    seed: int = 0

    def to_c(self) -> VdFrameCfg:
        # the C-ABI fields are int32: refuse values ctypes would silently truncate
        for name in ("f", "v1", "v2", "f0"):
            v = int(getattr(self, name))
            if not -(1 << 31) <= v < (1 << 31):
                raise ValueError(f"FrameConfig.{name} = {v} does not fit the decoder's int32 field")
        return VdFrameCfg(int(self.f), int(self.v1), int(self.v2), int(self.f0), int(self.start), 0,
                          int(self.seed) & 0xFFFFFFFFFFFFFFFF)

    def validate(self, pattern_period: int = 1) -> None:
        c = self.to_c()
        check(lib().vd_frame_cfg_validate(C.byref(c), pattern_period))


@dataclass
class DecodeStats:
    frames: int = 0
    stages: int = 0
    tracebacks: int = 0


@dataclass
class DecodeOutput:
    bits: np.ndarray
    stats: DecodeStats


def unpack_bits(packed: np.ndarray, n: int) -> np.ndarray:
    """LSB-first packed uint32 words -> n uint8 bits."""
    by = np.ascontiguousarray(packed, dtype=np.uint32).view(np.uint8)
    return np.unpackbits(by, bitorder="little")[:n].copy()


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """uint8 0/1 bits -> LSB-first packed uint32 words."""
    bits = np.asarray(bits, dtype=np.uint8)
    n = bits.size
    pad = (-n) % 32
    by = np.packbits(np.concatenate([bits, np.zeros(pad, np.uint8)]), bitorder="little")
    return by.view(np.uint32).copy()


def _stats(s: VdStats) -> DecodeStats:
    return DecodeStats(int(s.frames), int(s.stages), int(s.tracebacks))


def _exec(gpus: int, chunk_stages: int = 0, devices=None) -> VdExec:
    """vd_exec: `devices` (a list of device indices, repeats allowed) shards the
    frames over those devices; else gpus > 0 -> devices 0 .. gpus-1, 0 -> the
    current device."""
    if devices:
        arr = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        ex = VdExec(len(devices), C.cast(arr, C.POINTER(C.c_int32)), int(chunk_stages))
        ex._keep = arr  # the array must outlive the call
        return ex
    return VdExec(int(gpus) if gpus and gpus > 0 else 0, None, int(chunk_stages))


def _check_block(llr: np.ndarray, trellis: Trellis) -> None:
    # reference decoder.cpp:92-97
    if llr.ndim != 2 or llr.shape[1] < 1:
        raise ValueError("empty llr block")
    if llr.shape[0] != trellis.outputs_per_bit():
        raise ValueError("llr row count must equal B")


def framed_decode_stream(llr_stream: np.ndarray, n: int, trellis: Trellis, cfg: FrameConfig, gpus: int = 0,
                         chunk_stages: int = 0, devices=None):
    """Native entry: stage-major stream (int8 or float64, n*B values) ->
    (packed uint32 bits, DecodeStats), through vd_decode_i8 / vd_decode_f64."""
    arr = np.ascontiguousarray(llr_stream)
    if arr.size != n * trellis.outputs_per_bit():
        raise ValueError("stream length is not n * B")
    out = np.zeros((n + 31) // 32, np.uint32)
    st = VdStats()
    c = cfg.to_c()
    ex = _exec(gpus, chunk_stages, devices)
    if arr.dtype == np.int8:
        check(lib().vd_decode_i8(trellis.handle, C.byref(c), arr.ctypes.data, n, out.ctypes.data, C.byref(st),
                                 C.byref(ex)))
    elif arr.dtype == np.float64:
        check(lib().vd_decode_f64(trellis.handle, C.byref(c), arr.ctypes.data, n, out.ctypes.data, C.byref(st),
                                  C.byref(ex)))
    else:
        raise TypeError("llr stream must be int8 or float64")
    return out, _stats(st)


def _as_stream(llr: np.ndarray) -> np.ndarray:
    """B x N block -> stage-major stream; integer-valued blocks in
    [-127, 127] become int8 (decoded exactly by the fixed-point kernels)."""
    stream = np.ascontiguousarray(np.asarray(llr).T)
    if stream.dtype == np.int8:
        return stream.reshape(-1)
    d = stream.astype(np.float64, copy=False).reshape(-1)
    if np.all(np.abs(d) <= 127.0) and np.all(np.rint(d) == d):
        return d.astype(np.int8)
    return d


def framed_decode(llr: np.ndarray, trellis: Trellis, cfg: FrameConfig, workers: int = 1,
                  gpus: int = 0) -> DecodeOutput:
    """reference decoder.hpp:74-79. ``llr`` is B x N (LlrBlock layout)."""
    llr = np.asarray(llr)
    _check_block(llr, trellis)
    cfg.validate()
    n = llr.shape[1]
    packed, st = framed_decode_stream(_as_stream(llr), n, trellis, cfg, gpus=gpus)
    return DecodeOutput(unpack_bits(packed, n), st)


def framed_decode_batch(blocks, trellis: Trellis, cfg: FrameConfig, gpu: int = -1) -> list:
    """Independent framed decodes of several int8 blocks in one device pass
    (vd_decode_batch_i8): ``blocks`` is a list of stage-major int8 streams
    (n_j * B values each) or of B x n_j LlrBlocks. Equivalent to calling
    framed_decode on every block (reference run_ber_sweep, berlab.cpp:63-88).
    Returns [(bits uint8[n_j], DecodeStats)] with per-block stats."""
    b = trellis.outputs_per_bit()
    streams = []
    for blk in blocks:
        a = np.asarray(blk)
        if a.ndim == 2:
            _check_block(a, trellis)
            a = _as_stream(a)
        if a.dtype != np.int8:
            raise TypeError("batched decode takes int8 LLR blocks")
        if a.size == 0 or a.size % b:
            raise ValueError("empty llr block" if a.size == 0 else "stream length is not n * B")
        streams.append(np.ascontiguousarray(a).reshape(-1))
    if not streams:
        raise ValueError("batch needs at least one block")
    cfg.validate()
    lens = np.array([s.size // b for s in streams], np.int64)
    cat = np.concatenate(streams)
    total = int(lens.sum())
    out = np.zeros((total + 31) // 32, np.uint32)
    st = VdStats()
    c = cfg.to_c()
    dev = C.c_int32(int(gpu))
    ex = VdExec(1, C.pointer(dev), 0) if gpu >= 0 else VdExec(0, None, 0)
    check(lib().vd_decode_batch_i8(trellis.handle, C.byref(c), len(streams), lens.ctypes.data, cat.ctypes.data,
                                   out.ctypes.data, C.byref(st), C.byref(ex)))
    bits = unpack_bits(out, total)
    res, off = [], 0
    for n in lens:
        res.append((bits[off:off + n], frame_stats(cfg, int(n))))
        off += int(n)
    return res


def serial_decode(llr: np.ndarray, trellis: Trellis) -> DecodeOutput:
    """reference decoder.cpp:101-129 (one frame, no overlap, on the GPU)."""
    llr = np.asarray(llr)
    _check_block(llr, trellis)
    n = llr.shape[1]
    stream = _as_stream(llr)
    if stream.dtype == np.int8:
        if n > 0x7FFFFFFF:  # one frame of n stages: f is an int32 (vd_serial_decode_f64's limit too)
            raise VitdecError(VD_EUNSUPPORTED, "serial decode limited to 2^31-1 stages")
        packed, st = framed_decode_stream(stream, n, trellis, FrameConfig(f=n), chunk_stages=n)
    else:
        packed = np.zeros((n + 31) // 32, np.uint32)
        s = VdStats()
        check(lib().vd_serial_decode_f64(trellis.handle, stream.ctypes.data, n, packed.ctypes.data, C.byref(s), -1))
        st = _stats(s)
    return DecodeOutput(unpack_bits(packed, n), st)


def frame_stats(cfg: FrameConfig, n: int) -> DecodeStats:
    c = cfg.to_c()
    s = VdStats()
    check(lib().vd_frame_stats(C.byref(c), n, C.byref(s)))
    return _stats(s)


def partition_frames(cfg: FrameConfig, n: int, parts: int) -> list:
    c = cfg.to_c()
    first = np.zeros(parts + 1, np.int64)
    check(lib().vd_partition_frames(C.byref(c), n, parts, first.ctypes.data))
    return [int(x) for x in first]


def frame_window(cfg: FrameConfig, n: int, frame_begin: int, frame_end: int):
    c = cfg.to_c()
    b, e = C.c_int64(), C.c_int64()
    check(lib().vd_frame_window(C.byref(c), n, frame_begin, frame_end, C.byref(b), C.byref(e)))
    return int(b.value), int(e.value)


# ---- puncturing (reference codec.hpp:13-33, decoder.hpp:69-72) -------------------


class PuncturePattern:
    """reference codec.hpp:13-33: B rows x ``period`` columns, column-major
    ``mask[col * b + row]`` (1 keeps the coded bit)."""

    def __init__(self, b: int, period: int, mask, name: str = ""):
        self.b = int(b)
        self.period = int(period)
        self.mask = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8).reshape(-1))
        self.name = name

    @staticmethod
    def parse(rows: str) -> "PuncturePattern":
        """reference codec.cpp:25-58: rows separated by ';', e.g. "110;101"."""
        lines = rows.split(";")
        b, period = len(lines), len(lines[0])
        mask = np.zeros(b * period, np.uint8)
        for r, line in enumerate(lines):
            if len(line) != period:
                raise ValueError("puncture mask rows differ in length")
            for c, ch in enumerate(line):
                if ch not in "01":
                    raise ValueError("puncture mask must be 0/1")
                mask[c * b + r] = ch == "1"
        p = PuncturePattern(b, period, mask, rows)
        p.validate()
        return p

    @staticmethod
    def named(name: str) -> "PuncturePattern":
        """reference codec.cpp:60-74: "r12", "r23", "r34" or an explicit mask."""
        table = {"r12": "1;1", "r23": "11;10", "r34": "110;101"}
        p = PuncturePattern.parse(table.get(name, name))
        p.name = name
        return p

    def at(self, row: int, col: int) -> int:
        return int(self.mask[col * self.b + row])

    def kept_per_period(self) -> int:
        return int(self.mask.sum())

    def rate(self) -> float:
        return self.period / self.kept_per_period()

    def is_identity(self) -> bool:
        return self.kept_per_period() == self.b * self.period

    def to_c(self) -> VdPuncture:
        return VdPuncture(self.b, self.period, self.mask.ctypes.data)

    def validate(self) -> None:
        """reference codec.cpp:12-23 (VD_EINVAL -> ValueError, same message)."""
        c = self.to_c()
        check(lib().vd_puncture_validate(C.byref(c)))


def depuncture_stages(n_punctured: int, pattern: PuncturePattern) -> int:
    """Stages a punctured stream covers (reference decoder.cpp:141-152 rules)."""
    c = pattern.to_c()
    n = C.c_int64()
    check(lib().vd_depuncture_stages(C.byref(c), int(n_punctured), C.byref(n)))
    return int(n.value)


def framed_decode_punctured(punctured: np.ndarray, pattern: PuncturePattern, trellis: Trellis, cfg: FrameConfig,
                            gpus: int = 0, chunk_stages: int = 0):
    """framed_decode(depuncture(stream, pattern), trellis, cfg) (reference
    berlab.cpp:79-84, vitdec_cli.cpp:172-176) on an int8 punctured stream:
    only the punctured bytes go over PCIe, depuncture runs on the device
    (vd_decode_punctured_i8). Returns (packed uint32 bits, n_stages, DecodeStats)."""
    arr = np.ascontiguousarray(punctured)
    if arr.dtype != np.int8:
        raise TypeError("punctured stream must be int8")
    arr = arr.reshape(-1)
    n = depuncture_stages(arr.size, pattern)
    out = np.zeros(max((n + 31) // 32, 1), np.uint32)
    st = VdStats()
    c = cfg.to_c()
    pc = pattern.to_c()
    ex = _exec(gpus, chunk_stages)
    check(lib().vd_decode_punctured_i8(trellis.handle, C.byref(c), C.byref(pc), arr.ctypes.data, arr.size,
                                       out.ctypes.data, C.byref(st), C.byref(ex)))
    return out, n, _stats(st)


# ---- 4-bit LLR wire format -----------------------------------


def pack_i4(llr: np.ndarray) -> np.ndarray:
    """int8 LLRs in [-8, 7] (stage-major) -> 4-bit wire format: element i in
    nibble i, low nibble first (include/vitdec_b200.h)."""
    a = np.ascontiguousarray(llr, dtype=np.int8).reshape(-1)
    if a.size and (a.min() < -8 or a.max() > 7):
        raise ValueError("4-bit LLRs must lie in [-8, 7]")
    nib = (a.astype(np.int16) & 0xF).astype(np.uint8)
    if nib.size % 2:
        nib = np.concatenate([nib, np.zeros(1, np.uint8)])
    return (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8)


def unpack_i4(packed: np.ndarray, count: int) -> np.ndarray:
    """Inverse of pack_i4 (host reference for the device unpack)."""
    p = np.ascontiguousarray(packed, dtype=np.uint8)
    nib = np.empty(p.size * 2, np.uint8)
    nib[0::2] = p & 0xF
    nib[1::2] = p >> 4
    v = nib[:count].astype(np.int8)
    return np.where(v >= 8, v - 16, v).astype(np.int8)


def framed_decode_stream_i4(llr4: np.ndarray, n: int, trellis: Trellis, cfg: FrameConfig, gpus: int = 0,
                            chunk_stages: int = 0):
    """framed_decode on a 4-bit wire-format stream (vd_decode_i4) -> (packed bits, DecodeStats)."""
    arr = np.ascontiguousarray(llr4, dtype=np.uint8).reshape(-1)
    if arr.size * 2 < n * trellis.outputs_per_bit():
        raise ValueError("4-bit stream shorter than n * B values")
    out = np.zeros((n + 31) // 32, np.uint32)
    st = VdStats()
    c = cfg.to_c()
    ex = _exec(gpus, chunk_stages)
    check(lib().vd_decode_i4(trellis.handle, C.byref(c), arr.ctypes.data, n, out.ctypes.data, C.byref(st),
                             C.byref(ex)))
    return out, _stats(st)

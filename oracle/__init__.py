"""CPU ORACLE — test infrastructure only (the checker, never the product).

ctypes wrappers over
  * ``oracle/liboracle.so``  — the plain-C restatement of the reference
    decode path (oracle/vd_oracle.c), built by ``make -C oracle``; travels to
    the GPU box as a prebuilt file;
  * ``oracle/_ref/libvitdec_ref.so`` — the REFERENCE's own sources compiled
    in place (``make -C oracle ref``; only where /root/reference exists).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package. Parity is pinned by tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libvitdec_ref.so"

P, I32, I64, U64, DBL = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double

_DECODE_ARGS = [I32, I32, P, P, I64, I32, I32, I32, I32, I32, U64]


class _Lib:
    def __init__(self, path: Path, prefix: str, sigs: dict):
        self.path = path
        self.h = C.CDLL(os.fspath(path))
        self.prefix = prefix
        for name, (res, args) in sigs.items():
            fn = getattr(self.h, prefix + name)
            fn.restype = res
            fn.argtypes = args

    def fn(self, name):
        return getattr(self.h, self.prefix + name)

    def check(self, st: int):
        if st != 0:
            msg = self.fn("last_error")().decode()
            raise ValueError(msg) if st == 1 else RuntimeError(msg)


_ORACLE_SIGS = {
    "last_error": (C.c_char_p, []),
    "mix_seed": (U64, [U64, U64]),
    "sigma_from_ebn0": (DBL, [DBL, DBL]),
    "trellis": (I32, [I32, I32, P, P, P, P, P, P]),
    "framed_decode_f64": (I32, _DECODE_ARGS + [P, P, P]),
    "framed_decode_i8": (I32, _DECODE_ARGS + [P, P, P]),
    "framed_decode_range_i8": (I32, _DECODE_ARGS + [I64, I64, P]),
    "serial_decode_f64": (I32, [I32, I32, P, P, I64, P, P]),
    "random_bits": (None, [I64, U64, P]),
    "encode": (I32, [I32, I32, P, P, I64, P]),
    "awgn_bpsk": (None, [P, I64, DBL, U64, P]),
    "gen_bench_block": (I32, [I32, I32, P, I64, DBL, U64, P, P]),
    "gen_sweep_block": (I32, [I32, I32, P, I64, DBL, U64, P, P]),
    "quantize_i8": (None, [P, I64, DBL, P]),
    "puncture_i8": (I32, [I32, I32, P, P, I64, P, P]),
    "depuncture_i8": (I32, [I32, I32, P, P, I64, P, I64, P]),
}

_REF_SIGS = {
    "last_error": (C.c_char_p, []),
    "mix_seed": (U64, [U64, U64]),
    "sigma_from_ebn0": (DBL, [DBL, DBL]),
    "trellis": (I32, [I32, I32, P, P, P, P, P, P]),
    "framed_decode_f64": (I32, _DECODE_ARGS + [I32, P, P]),
    "framed_decode_i8": (I32, _DECODE_ARGS + [I32, P, P]),
    "serial_decode_f64": (I32, [I32, I32, P, P, I64, P, P]),
    "gen_bench_block": (I32, [I32, I32, P, I64, DBL, U64, P, P]),
    "gen_sweep_block": (I32, [I32, I32, P, I64, DBL, U64, P, P]),
    "ber_sweep": (I32, [I32, I32, P, C.c_char_p, I32, I32, I32, I32, I32, U64, I32, P, I32, I64, I64, U64, I32,
                        P, P]),
    "depuncture": (I32, [C.c_char_p, P, I64, P, I64, P]),
}

_oracle = None
_ref = None


def oracle() -> _Lib:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle` (or __graft_entry__.build())")
        _oracle = _Lib(ORACLE_SO, "vdo_", _ORACLE_SIGS)
    return _oracle


def reference():
    """The reference library compiled from /root/reference, or None."""
    global _ref
    if _ref is None and REF_SO.exists():
        _ref = _Lib(REF_SO, "vdref_", _REF_SIGS)
    return _ref


def _polys(polys):
    arr = (C.c_uint32 * len(polys))(*[int(p) for p in polys])
    return arr


class Backend:
    """Uniform interface over the oracle restatement or the reference."""

    def __init__(self, lib: _Lib, is_ref: bool):
        self.lib = lib
        self.is_ref = is_ref

    def mix_seed(self, seed: int, salt: int) -> int:
        return int(self.lib.fn("mix_seed")(seed & (2**64 - 1), salt & (2**64 - 1)))

    def sigma_from_ebn0(self, ebn0: float, rate: float) -> float:
        return float(self.lib.fn("sigma_from_ebn0")(ebn0, rate))

    def trellis(self, k, b, polys):
        s = 1 << (k - 1)
        t = [np.zeros(2 * s, np.uint32) for _ in range(4)]
        cp = C.c_int32()
        self.lib.check(self.lib.fn("trellis")(k, b, _polys(polys), *[x.ctypes.data for x in t], C.addressof(cp)))
        return (*t, bool(cp.value))

    def framed_decode(self, k, b, polys, llr, n, f, v1=0, v2=0, f0=0, start=0, seed=0, workers=1, want_sigma=False):
        """llr: stage-major stream (int8 or float64) of n*b values -> (bits, stats, sigma|None)."""
        llr = np.ascontiguousarray(llr)
        bits = np.zeros(n, np.uint8)
        stats = np.zeros(3, np.int64)
        kind = "i8" if llr.dtype == np.int8 else "f64"
        if kind == "f64":
            llr = llr.astype(np.float64, copy=False)
        args = [k, b, _polys(polys), llr.ctypes.data, n, f, v1, v2, f0, start, seed & (2**64 - 1)]
        sigma = None
        if self.is_ref:
            self.lib.check(self.lib.fn("framed_decode_" + kind)(*args, workers, bits.ctypes.data, stats.ctypes.data))
        else:
            nf = (n + f - 1) // f
            sig_ptr = None
            if want_sigma:
                sigma = np.zeros((nf, 1 << (k - 1)), np.float64)
                sig_ptr = sigma.ctypes.data
            self.lib.check(self.lib.fn("framed_decode_" + kind)(*args, bits.ctypes.data, stats.ctypes.data, sig_ptr))
        return bits, tuple(int(x) for x in stats), sigma

    def serial_decode(self, k, b, polys, llr, n):
        llr = np.ascontiguousarray(llr, dtype=np.float64)
        bits = np.zeros(n, np.uint8)
        if self.is_ref:
            stats = np.zeros(3, np.int64)
            self.lib.check(self.lib.fn("serial_decode_f64")(k, b, _polys(polys), llr.ctypes.data, n,
                                                            bits.ctypes.data, stats.ctypes.data))
        else:
            self.lib.check(self.lib.fn("serial_decode_f64")(k, b, _polys(polys), llr.ctypes.data, n,
                                                            bits.ctypes.data, None))
        return bits

    def gen_bench_block(self, k, b, polys, n, ebn0, seed):
        rx = np.zeros(n * b, np.float64)
        sent = np.zeros(n, np.uint8)
        self.lib.check(self.lib.fn("gen_bench_block")(k, b, _polys(polys), n, ebn0, seed, rx.ctypes.data,
                                                      sent.ctypes.data))
        return rx, sent

    def gen_sweep_block(self, k, b, polys, n, sigma, block_seed):
        rx = np.zeros(n * b, np.float64)
        sent = np.zeros(n, np.uint8)
        self.lib.check(self.lib.fn("gen_sweep_block")(k, b, _polys(polys), n, sigma, block_seed & (2**64 - 1),
                                                      rx.ctypes.data, sent.ctypes.data))
        return rx, sent


def port() -> Backend:
    return Backend(oracle(), False)


def ref_backend():
    r = reference()
    return None if r is None else Backend(r, True)


def quantize(y: np.ndarray, scale: float = 32.0) -> np.ndarray:
    """q = clamp(nearbyint(scale*y), -127, 127) via the C oracle (exact libm semantics)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    q = np.zeros(y.size, np.int8)
    oracle().fn("quantize_i8")(y.ctypes.data, y.size, scale, q.ctypes.data)
    return q


def framed_decode_range_i8(k, b, polys, llr, n, f, v1, v2, f0, start, seed, frame_begin, frame_end):
    """Oracle decode of frames [frame_begin, frame_end) only (shard parity)."""
    llr = np.ascontiguousarray(llr, dtype=np.int8)
    bits = np.zeros(n, np.uint8)
    o = oracle()
    o.check(o.fn("framed_decode_range_i8")(k, b, _polys(polys), llr.ctypes.data, n, f, v1, v2, f0, start,
                                           seed & (2**64 - 1), frame_begin, frame_end, bits.ctypes.data))
    return bits


def _mask_arr(mask_rows):
    """Rows as strings ("110;101", reference PuncturePattern::parse) -> (b, period, column-major u8 mask)."""
    rows = mask_rows.split(";")
    b, period = len(rows), len(rows[0])
    m = np.zeros(b * period, np.uint8)
    for r, line in enumerate(rows):
        for c, ch in enumerate(line):
            m[c * b + r] = ch == "1"
    return b, period, m


def puncture_i8(mask_rows: str, llr: np.ndarray, n_stages: int) -> np.ndarray:
    """Oracle puncture (reference codec.cpp:88-103) of an int8 stage-major stream."""
    b, period, m = _mask_arr(mask_rows)
    llr = np.ascontiguousarray(llr, dtype=np.int8)
    out = np.zeros(max(llr.size, 1), np.int8)
    n_out = C.c_int64()
    o = oracle()
    o.check(o.fn("puncture_i8")(b, period, m.ctypes.data, llr.ctypes.data, n_stages, out.ctypes.data,
                                C.addressof(n_out)))
    return out[: n_out.value].copy()


def depuncture_i8(mask_rows: str, punctured: np.ndarray):
    """Oracle depuncture (reference decoder.cpp:131-163) -> (stage-major int8 block, n_stages)."""
    b, period, m = _mask_arr(mask_rows)
    punctured = np.ascontiguousarray(punctured, dtype=np.int8)
    o = oracle()
    stages = C.c_int64()
    o.check(o.fn("depuncture_i8")(b, period, m.ctypes.data, punctured.ctypes.data, punctured.size, None, 0,
                                  C.addressof(stages)))
    out = np.zeros(max(stages.value * b, 1), np.int8)
    o.check(o.fn("depuncture_i8")(b, period, m.ctypes.data, punctured.ctypes.data, punctured.size, out.ctypes.data,
                                  out.size, C.addressof(stages)))
    return out[: stages.value * b].copy(), stages.value

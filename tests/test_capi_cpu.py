"""CPU-side checks of the C-ABI library (no GPU compute).

* libvitdec_b200.so loads and exports every symbol include/vitdec_b200.h
  declares;
* host logic behind the boundary: trellis tables, validation messages
  (identical to the reference's std::invalid_argument texts), DecodeStats,
  frame windows and the multi-GPU frame partition;
* the decode entry points refuse to run without a CUDA device (no CPU
  fallback).
"""
import re

import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd
from paper_2011_09337_b200._lib import SIGNATURES, VitdecError, lib

ROOT = __import__("pathlib").Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "vitdec_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(vd_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    declared = header_symbols()
    assert declared, "no declarations parsed"
    assert declared == set(SIGNATURES), declared ^ set(SIGNATURES)
    h = lib()
    for name in declared:
        assert hasattr(h, name), name
    assert b"sm_100a" in h.vd_version()


@pytest.mark.parametrize("k,polys", [(3, "7,5"), (7, "171,133"), (7, "133,171,165"), (9, "561,753"), (2, "3,1"),
                                     (3, "3,5"), (6, "53,75,47,71"), (12, "4335,5723")])
def test_trellis_tables_match_oracle(k, polys):
    spec = vd.CodeSpec.from_octal(k, polys)
    t = vd.build_trellis(spec)
    nxt, out, pred, io, cp = oracle.port().trellis(k, spec.b, spec.polys)
    assert np.array_equal(t._next, nxt) and np.array_equal(t._out, out)
    assert np.array_equal(t._pred, pred) and np.array_equal(t.incoming_output_data(), io)
    assert t.complement_paired() == cp
    assert t.num_states() == 1 << (k - 1)
    assert spec.polys_octal() == polys


@pytest.mark.parametrize("spec,msg", [
    (vd.CodeSpec(1, 2, [1, 1]), "constraint length must be >= 2"),
    (vd.CodeSpec(3, 1, [5]), "need at least 2 outputs per bit"),
    (vd.CodeSpec(3, 2, [7, 0]), "zero generator polynomial"),
    (vd.CodeSpec(3, 2, [7, 0x10]), "generator polynomial wider than K bits"),
    (vd.CodeSpec(3, 2, [7]), "polynomial count must equal B"),
    (vd.CodeSpec(17, 2, [1, 1]), "constraint length too large"),
])
def test_trellis_validation_messages(spec, msg):
    # reference test_trellis.cpp:46-52 / trellis.cpp:38-53
    with pytest.raises(ValueError, match=msg):
        vd.build_trellis(spec)


def test_from_octal_rejects_bad_digits():
    with pytest.raises(ValueError, match="bad octal polynomial"):
        vd.CodeSpec.from_octal(7, "171,189")


def test_frame_config_validation():
    # reference test_decoder.cpp:207-215
    cfg = vd.FrameConfig(f=32, v1=8, v2=8, f0=40)
    with pytest.raises(ValueError, match=r"f0 must be in \[0, f\]"):
        cfg.validate()
    cfg.f0 = 16
    cfg.validate()
    with pytest.raises(ValueError, match="multiples of the puncture period"):
        cfg.validate(3)
    cfg.validate(2)
    with pytest.raises(ValueError, match="frame size f must be >= 1"):
        vd.FrameConfig(f=0).validate()
    with pytest.raises(ValueError, match="overlaps must be >= 0"):
        vd.FrameConfig(f=4, v1=-1).validate()


def test_stats_kat_and_random_against_oracle():
    # reference test_decoder.cpp:289-295
    s = vd.frame_stats(vd.FrameConfig(f=32, v1=8, v2=8, f0=16), 100)
    assert (s.frames, s.tracebacks) == (4, 7)
    rng = np.random.default_rng(5)
    port = oracle.port()
    for _ in range(60):
        n = int(rng.integers(1, 3000))
        f = int(rng.integers(1, 400))
        cfg = vd.FrameConfig(f, int(rng.integers(0, 300)), int(rng.integers(0, 300)), int(rng.integers(0, f + 1)))
        _, st, _ = port.framed_decode(7, 2, [0o171, 0o133], np.zeros(2 * n), n, cfg.f, cfg.v1, cfg.v2, cfg.f0)
        got = vd.frame_stats(cfg, n)
        assert (got.frames, got.stages, got.tracebacks) == st


def test_partition_and_windows():
    rng = np.random.default_rng(6)
    for _ in range(100):
        n = int(rng.integers(1, 100000))
        f = int(rng.integers(1, 600))
        cfg = vd.FrameConfig(f, int(rng.integers(0, 64)), int(rng.integers(0, 64)))
        nf = -(-n // f)
        for parts in (1, 2, 3, 8):
            first = vd.partition_frames(cfg, n, parts)
            assert first[0] == 0 and first[-1] == nf and all(a <= b for a, b in zip(first, first[1:]))
            for a in first[1:-1]:
                if 0 < a < nf:
                    assert (a * f) % 32 == 0  # output shards start on a packed word
            for a, b in zip(first, first[1:]):
                if a < b:
                    lo, hi = vd.frame_window(cfg, n, a, b)
                    assert lo == max(a * f - cfg.v1, 0) and hi == min(min(b * f, n) + cfg.v2, n)


def test_decode_requires_a_gpu():
    """No CUDA device here: the decode path must fail loudly, not fall back."""
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    t = vd.build_trellis(vd.CodeSpec.from_octal(7, "171,133"))
    with pytest.raises(VitdecError, match="no CUDA device"):
        vd.framed_decode(np.ones((2, 64), np.int8), t, vd.FrameConfig(f=32, v1=4, v2=4))


def test_block_checks():
    t = vd.build_trellis(vd.CodeSpec.from_octal(7, "171,133"))
    with pytest.raises(ValueError, match="empty llr block"):
        vd.framed_decode(np.zeros((2, 0)), t, vd.FrameConfig(f=4))
    with pytest.raises(ValueError, match="llr row count must equal B"):
        vd.framed_decode(np.zeros((3, 5)), t, vd.FrameConfig(f=4))

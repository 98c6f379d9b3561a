"""Large constraint lengths, K = 13 .. 16 (the reference accepts K <= 16,
trellis.cpp:44): the CTA-per-frame path (vd_bigk.cu) against fixtures the
reference itself produced (tests/golden/make_golden_bigk.py) and against the
C oracle, bit-exact: decoded bits, DecodeStats and final path metrics.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def bigk():
    meta = json.loads((GOLD / "bigk_vectors.json").read_text())
    return meta, dict(np.load(GOLD / "bigk_vectors.npz"))


def _unpack(a, n):
    return np.unpackbits(np.asarray(a, np.uint8), bitorder="little")[:n]


def test_oracle_matches_reference_fixtures(bigk):
    """CPU: the C oracle reproduces the reference's K = 13..16 decodes."""
    meta, arr = bigk
    port = oracle.port()
    for c in meta["cases"]:
        cfg = c["cfg"]
        bits, st, _ = port.framed_decode(c["k"], c["b"], c["polys"], arr[c["name"] + "_llr"], c["n"], cfg["f"],
                                         cfg["v1"], cfg["v2"], cfg["f0"], cfg["start"], cfg["seed"])
        assert np.array_equal(bits, _unpack(arr[c["name"] + "_bits"], c["n"])), c["name"]
        assert list(st) == c["stats"], c["name"]


@pytest.mark.gpu
def test_gpu_matches_reference_fixtures(bigk):
    meta, arr = bigk
    for c in meta["cases"]:
        t = vd.build_trellis(vd.CodeSpec(c["k"], c["b"], c["polys"]))
        cfg = c["cfg"]
        fc = vd.FrameConfig(cfg["f"], cfg["v1"], cfg["v2"], cfg["f0"], vd.TracebackStart(cfg["start"]), cfg["seed"])
        packed, st = vd.framed_decode_stream(arr[c["name"] + "_llr"], c["n"], t, fc)
        assert np.array_equal(vd.unpack_bits(packed, c["n"]), _unpack(arr[c["name"] + "_bits"], c["n"])), c["name"]
        assert [st.frames, st.stages, st.tracebacks] == c["stats"], c["name"]


@pytest.mark.gpu
@pytest.mark.parametrize("code", [(13, 2, [0o15627, 0o12345]), (16, 3, [0o123457, 0o164355, 0o177777])],
                         ids=["K13B2", "K16B3"])
def test_gpu_vs_oracle_bits_and_metrics(code):
    """Random configs (serial / parallel traceback / random start / f >= N),
    int8 and real-valued LLRs; final path metrics of every frame == oracle."""
    import torch

    from paper_2011_09337_b200.device import decode_f64_device, decode_i8_device

    k, b, polys = code
    port = oracle.port()
    t = vd.build_trellis(vd.CodeSpec(k, b, polys))
    rng = np.random.default_rng(k)
    for n, cfg in ((700, vd.FrameConfig(256, 20, 20)), (600, vd.FrameConfig(150, 25, 40, 30)),
                   (500, vd.FrameConfig(128, 10, 30, 32, vd.TracebackStart.kRandom, 5)),
                   (300, vd.FrameConfig(400, 0, 0))):
        for real in (False, True):
            y = np.repeat(rng.choice([-1.0, 1.0], n), b) + rng.standard_normal(n * b)
            llr = y * 3.0 if real else np.clip(np.rint(y * 32), -127, 127).astype(np.int8)
            exp, st, sig = port.framed_decode(k, b, polys, llr, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start),
                                              cfg.seed, want_sigma=True)
            nf = -(-n // cfg.f)
            dl = torch.from_numpy(np.ascontiguousarray(llr)).cuda()
            out = torch.zeros((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
            sigma = torch.zeros((nf, 1 << (k - 1)), dtype=torch.float64 if real else torch.int64, device="cuda")
            (decode_f64_device if real else decode_i8_device)(t, cfg, n, dl, 0, 0, nf, out, 0, sigma)
            torch.cuda.synchronize()
            got = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
            assert np.array_equal(got, exp), (code, cfg, real)
            assert np.array_equal(sigma.cpu().numpy().astype(np.float64), sig), (code, cfg, real)

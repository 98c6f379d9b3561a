"""4-bit LLR wire format: pack/unpack host round trip (CPU);
device unpack and the streaming decode vd_decode_i4 bit-identical to the int8
path on the same values and to the oracle (GPU), including chunk starts on odd
nibbles (B = 3) and multi-chunk streaming."""
import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd


def test_pack_unpack_round_trip():
    rng = np.random.default_rng(5)
    for n in (0, 1, 2, 3, 17, 4096, 100_001):
        a = rng.integers(-8, 8, n).astype(np.int8)
        p = vd.pack_i4(a)
        assert p.size == (n + 1) // 2
        assert np.array_equal(vd.unpack_i4(p, n), a)
    with pytest.raises(ValueError):
        vd.pack_i4(np.array([9], np.int8))


@pytest.mark.gpu
def test_device_unpack_matches_host():
    import torch

    rng = np.random.default_rng(6)
    for n in (1, 7, 8, 9, 1000, 1 << 20, (1 << 20) + 5):
        a = rng.integers(-8, 8, n).astype(np.int8)
        p = torch.from_numpy(vd.pack_i4(a)).cuda()
        out = torch.full((n + 16,), 99, dtype=torch.int8, device="cuda")
        vd.api.check(vd.lib().vd_unpack_i4_device(p.data_ptr(), n, out.data_ptr(), -1, None))
        got = out.cpu().numpy()
        assert np.array_equal(got[:n], a), n
        assert (got[n:] == 99).all()


@pytest.mark.gpu
@pytest.mark.parametrize("code", [(7, 2, [0o171, 0o133]), (7, 3, [0o133, 0o171, 0o165]), (3, 2, [7, 5])],
                         ids=lambda c: f"K{c[0]}B{c[1]}")
def test_i4_stream_decode_matches_int8_and_oracle(code):
    k, b, polys = code
    t = vd.build_trellis(vd.CodeSpec(k, b, polys))
    port = oracle.port()
    rng = np.random.default_rng(7 + k + b)
    for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32), vd.FrameConfig(100, 14, 30)):
        n = int(rng.integers(50_000, 90_000))
        rx, _ = port.gen_bench_block(k, b, polys, n, 3.0, n)
        q = np.clip(np.rint(rx * 4.0), -7, 7).astype(np.int8)  # a 4-bit quantiser
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0)
        p4 = vd.pack_i4(q)
        for chunk in (0, 3333):  # 3333-stage chunks: B = 3 chunk windows start on odd nibbles
            packed, stats = vd.framed_decode_stream_i4(p4, n, t, cfg, chunk_stages=chunk)
            got = vd.unpack_bits(packed, n)
            assert np.array_equal(got, exp), (code, cfg, chunk)
            assert (stats.frames, stats.stages, stats.tracebacks) == st
        p8, _ = vd.framed_decode_stream(q, n, t, cfg)
        assert np.array_equal(p8, packed)

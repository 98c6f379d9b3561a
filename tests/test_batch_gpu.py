"""GPU parity of the batched multi-block decode.

Reference behaviour: run_ber_sweep decodes every block of a BER point with its
own framed_decode call (berlab.cpp:63-88), so each block has its own frame
grid clipped at both of its ends and its random-start salt counts frames from
the block start (decoder.cpp:224). vd_decode_batch_* must equal exactly that:
per-block oracle decodes, bit for bit, for any mix of block lengths.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd

pytestmark = pytest.mark.gpu

K7 = (7, 2, [0o171, 0o133])


@pytest.fixture(scope="module")
def port():
    return oracle.port()


def trellis(k, b, polys):
    return vd.build_trellis(vd.CodeSpec(k, b, list(polys)))


CFGS = [vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32),
        vd.FrameConfig(128, 20, 40, 32, vd.TracebackStart.kRandom, 11), vd.FrameConfig(64, 64, 0, 1),
        vd.FrameConfig(100, 14, 30, 30)]


@pytest.mark.parametrize("code", [K7, (7, 3, [0o133, 0o171, 0o165]), (9, 2, [0o561, 0o753]), (3, 2, [7, 5])],
                         ids=lambda c: f"K{c[0]}B{c[1]}")
def test_batch_equals_per_block_decodes(code, port):
    k, b, polys = code
    t = trellis(k, b, polys)
    rng = np.random.default_rng(4242 + k * 3 + b)
    for ci, cfg in enumerate(CFGS):
        # ragged mix: single stages, non-multiples of 4 (misaligned block
        # starts -> those blocks' frames all take the generic kernel), and
        # long blocks with many interior frames
        lens = [1, 2, 3, 31, 33, 257, 1000, 4099, 65536, 20000, 777, 12345][: 6 + ci * 2]
        rng.shuffle(lens)
        blocks, exp = [], []
        for j, n in enumerate(lens):
            rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(0, 4)), 1000 * ci + j)
            q = oracle.quantize(rx, [32.0, 4.0][j % 2])
            blocks.append(q)
            exp.append(port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start),
                                          cfg.seed))
        got = vd.framed_decode_batch(blocks, t, cfg)
        for j, ((bits, st), (eb, est, _)) in enumerate(zip(got, exp)):
            bad = np.flatnonzero(bits != eb)
            assert bad.size == 0, (code, cfg, lens[j], bad[:10])
            assert (st.frames, st.stages, st.tracebacks) == est


def test_batch_ber_point_int8(port):
    """One BER point the way the reference harness builds it (16 blocks of
    65536 bits, block seeds mix_seed(seed, p*0x100000 + blk)), quantised to
    int8: the batched decode's error count equals the per-block oracle's."""
    t = trellis(*K7)
    sigma = port.sigma_from_ebn0(2.0, 0.5)
    blocks, sent_all, exp_err = [], [], 0
    cfg = vd.FrameConfig(256, 20, 20)
    for blk in range(16):
        rx, sent = port.gen_sweep_block(*K7, 65536, sigma, port.mix_seed(7, blk))
        q = oracle.quantize(rx, 32.0)
        blocks.append(q)
        sent_all.append(sent)
        eb, _, _ = port.framed_decode(*K7, q, 65536, cfg.f, cfg.v1, cfg.v2)
        exp_err += int(np.count_nonzero(eb != sent))
    got = vd.framed_decode_batch(blocks, t, cfg)
    err = sum(int(np.count_nonzero(bits != s)) for (bits, _), s in zip(got, sent_all))
    assert err == exp_err
    assert err > 0


def test_batch_device_fp64(port):
    """vd_decode_batch_f64_device on real-valued LLRs (FP64 kernel): identical
    to per-block reference-order double decodes."""
    import torch

    t = trellis(*K7)
    cfg = vd.FrameConfig(64, 16, 24, 16)
    lens = [500, 1, 1234, 64, 3000]
    streams, exp = [], []
    for j, n in enumerate(lens):
        rx, _ = port.gen_bench_block(*K7, n, 1.5, 50 + j)
        streams.append(rx)
        exp.append(port.framed_decode(*K7, rx, n, cfg.f, cfg.v1, cfg.v2, cfg.f0)[0])
    cat = torch.from_numpy(np.concatenate(streams)).cuda()
    total = sum(lens)
    out = torch.zeros((total + 31) // 32, dtype=torch.int32, device="cuda")
    arr = np.array(lens, np.int64)
    c = cfg.to_c()
    st = vd._lib.VdStats()
    vd._lib.check(vd.lib().vd_decode_batch_f64_device(t.handle, C.byref(c), len(lens), arr.ctypes.data,
                                                      cat.data_ptr(), out.data_ptr(), C.byref(st), -1, 0))
    torch.cuda.synchronize()
    bits = vd.unpack_bits(out.cpu().numpy().view(np.uint32), total)
    off = 0
    for n, e in zip(lens, exp):
        assert np.array_equal(bits[off:off + n], e), n
        off += n
    assert st.frames == sum(-(-n // cfg.f) for n in lens)


def test_batch_errors():
    t = trellis(*K7)
    with pytest.raises(ValueError, match="empty llr block"):
        vd.framed_decode_batch([np.zeros(10, np.int8), np.zeros(0, np.int8)], t, vd.FrameConfig(4))
    with pytest.raises(ValueError, match="at least one block"):
        vd.framed_decode_batch([], t, vd.FrameConfig(4))


@pytest.mark.parametrize("code", [K7, (7, 3, [0o133, 0o171, 0o165]), (9, 2, [0o561, 0o753])],
                         ids=lambda c: f"K{c[0]}B{c[1]}")
def test_batch_head_and_tail_classes(code, port):
    """Many blocks (the BER-sweep shape) so the fast kernel takes the block
    heads (zero-padded head copies) and the clipped-v2 tails (one launch per
    distinct v2'); block lengths chosen to give several tail classes."""
    k, b, polys = code
    t = trellis(k, b, polys)
    rng = np.random.default_rng(77 + k + b)
    for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(128, 24, 40), vd.FrameConfig(256, 20, 20, 0,
                                                                                          vd.TracebackStart.kRandom, 3),
                vd.FrameConfig(160, 20, 48, 32)):
        lens = [int(x) for x in rng.choice([8192, 8192 + 4, 8192 + 12, 8192 + 36, 4096 + 8, 6000], size=300)]
        blocks, exp = [], []
        for j, n in enumerate(lens):
            rx, _ = port.gen_bench_block(k, b, polys, n, 2.5, 50_000 + j)
            q = oracle.quantize(rx, 32.0)
            blocks.append(q)
        got = vd.framed_decode_batch(blocks, t, cfg)
        for j, n in enumerate(lens[:120]):  # oracle on a subset of blocks (time)
            eb, est, _ = port.framed_decode(k, b, polys, blocks[j], n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start),
                                            cfg.seed)
            bits, st = got[j]
            bad = np.flatnonzero(bits != eb)
            assert bad.size == 0, (code, cfg, n, bad[:10])
            assert (st.frames, st.stages, st.tracebacks) == est

"""GPU parity: the sm_100a decode path vs the reference (golden vectors) and
vs the CPU oracle, bit-exact, through the C-ABI.

Bar: identical decoded bits and DecodeStats for the same
int8 LLRs and frame configuration; identical final path metrics (integer
metrics, renormalisation offset re-added); real-valued LLRs via the FP64
kernel identical too. Full-size runs use size-independent properties
(sampled-window parity, noiseless round trips, chunk/shard invariance).
"""
import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd
from conftest import unpack

pytestmark = pytest.mark.gpu

K7 = (7, 2, [0o171, 0o133])


def trellis(k, b, polys):
    return vd.build_trellis(vd.CodeSpec(k, b, list(polys)))


def block(stream, b):
    """Stage-major stream -> B x N block (reference LlrBlock layout)."""
    return np.asarray(stream).reshape(-1, b).T


@pytest.fixture(scope="module")
def port():
    return oracle.port()


def test_golden_framed_cases(golden):
    meta, arr = golden
    for c in meta["cases"]:
        t = trellis(c["k"], c["b"], c["polys"])
        cfg = vd.FrameConfig(**{k: v for k, v in c["cfg"].items() if k != "start"},
                             start=vd.TracebackStart(c["cfg"]["start"]))
        out = vd.framed_decode(block(arr[c["name"] + "_llr"], c["b"]), t, cfg)
        assert np.array_equal(out.bits, unpack(arr[c["name"] + "_bits"], c["n"])), c["name"]
        assert [out.stats.frames, out.stats.stages, out.stats.tracebacks] == c["stats"], c["name"]


def test_golden_serial_cases(golden):
    meta, arr = golden
    for c in meta["serial"]:
        t = trellis(c["k"], c["b"], c["polys"])
        out = vd.serial_decode(block(arr[c["name"] + "_llr"], c["b"]), t)
        assert np.array_equal(out.bits, unpack(arr[c["name"] + "_bits"], c["n"])), c["name"]
        assert (out.stats.frames, out.stats.stages, out.stats.tracebacks) == (1, c["n"], 1)


CODES = [(2, 2, [3, 1]), (3, 2, [7, 5]), (3, 2, [3, 5]), (3, 2, [6, 5]), (4, 3, [0o13, 0o15, 0o17]),
         (5, 2, [0o23, 0o35]), (6, 4, [0o53, 0o75, 0o47, 0o71]), (7, 2, [0o171, 0o133]),
         (7, 3, [0o133, 0o171, 0o165]), (8, 2, [0o247, 0o371]), (9, 2, [0o561, 0o753]),
         (9, 3, [0o557, 0o663, 0o711]), (10, 2, [0o1167, 0o1545])]


@pytest.mark.parametrize("code", CODES, ids=lambda c: f"K{c[0]}B{c[1]}")
def test_random_configs_vs_oracle(code, port):
    k, b, polys = code
    t = trellis(k, b, polys)
    rng = np.random.default_rng(1000 + k * 10 + b)
    for it in range(10):
        n = int(rng.integers(1, 5000))
        f = int(rng.integers(1, 400))
        cfg = vd.FrameConfig(f, int(rng.integers(0, 80)), int(rng.integers(0, 80)), int(rng.integers(0, f + 1)),
                             vd.TracebackStart(int(rng.integers(0, 2))), int(rng.integers(0, 2**63)))
        scale = [32.0, 4.0, 1.0][it % 3]
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(-1, 4)), int(rng.integers(0, 2**32)))
        llr = oracle.quantize(rx, scale) if it < 7 else rx
        exp, st, _ = port.framed_decode(k, b, polys, llr, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        out = vd.framed_decode(block(llr, b), t, cfg)
        assert np.array_equal(out.bits, exp), (k, b, n, cfg, scale)
        assert (out.stats.frames, out.stats.stages, out.stats.tracebacks) == st


def test_headline_config_c1(port):
    """Config 1: K=7 r1/2, 1M info bits at 3 dB, int8 scale 32 — both frame
    configurations of the minimum slice."""
    n = 1_000_000
    rx, sent = port.gen_bench_block(*K7, n, 3.0, 1)
    q = oracle.quantize(rx, 32.0)
    t = trellis(*K7)
    for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32)):
        exp, st, _ = port.framed_decode(*K7, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0)
        packed, stats = vd.framed_decode_stream(q, n, t, cfg)
        assert np.array_equal(vd.unpack_bits(packed, n), exp)
        assert (stats.frames, stats.stages, stats.tracebacks) == st
        assert np.count_nonzero(exp != sent) < n * 1e-3  # sane BER at 3 dB


def test_path_metric_parity(port):
    """Final per-frame path metrics of the int8 kernel == oracle's doubles."""
    import torch

    for k, b, polys in [K7, (9, 2, [0o561, 0o753]), (7, 3, [0o133, 0o171, 0o165]), (3, 2, [7, 5])]:
        n = 6000
        rx, _ = port.gen_bench_block(k, b, polys, n, 2.0, 17)
        q = oracle.quantize(rx, 32.0)
        for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(100, 13, 45, 32), vd.FrameConfig(n, 0, 0)):
            _, _, sig = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, want_sigma=True)
            nf = -(-n // cfg.f)
            t = trellis(k, b, polys)
            llr = torch.from_numpy(q).cuda()
            out = torch.zeros((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
            sigma = torch.zeros((nf, 1 << (k - 1)), dtype=torch.int64, device="cuda")
            from paper_2011_09337_b200.device import decode_i8_device

            decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0, sigma)
            torch.cuda.synchronize()
            assert np.array_equal(sigma.cpu().numpy().astype(np.float64), sig), (k, cfg)


def test_fp64_path_is_bit_exact_on_real_llrs(port):
    rng = np.random.default_rng(7)
    for k, b, polys in [K7, (9, 2, [0o561, 0o753]), (4, 3, [0o13, 0o15, 0o17])]:
        n = 3000
        llr = rng.standard_normal(n * b) * 1.7
        for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(128, 20, 40, 32, vd.TracebackStart.kRandom, 9)):
            exp, st, _ = port.framed_decode(k, b, polys, llr, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start),
                                            cfg.seed)
            out = vd.framed_decode(block(llr, b), trellis(k, b, polys), cfg)
            assert np.array_equal(out.bits, exp)
        assert np.array_equal(vd.serial_decode(block(llr, b), trellis(k, b, polys)).bits,
                              port.serial_decode(k, b, polys, llr, n))


def test_chunking_and_shard_invariance(port):
    """Output is identical for any streaming chunk size and for frame-range
    shards decoded separately (the multi-GPU decomposition, on one device)."""
    import torch

    from paper_2011_09337_b200.device import decode_i8_device

    n = 200_003
    rx, _ = port.gen_bench_block(*K7, n, 2.5, 99)
    q = oracle.quantize(rx)
    t = trellis(*K7)
    for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(100, 30, 45, 25, vd.TracebackStart.kRandom, 4)):
        exp, _, _ = port.framed_decode(*K7, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        for chunk in (0, 4096, 50_000):
            packed, _ = vd.framed_decode_stream(q, n, t, cfg, chunk_stages=chunk)
            assert np.array_equal(vd.unpack_bits(packed, n), exp), chunk
        for parts in (2, 3, 8):
            first = vd.partition_frames(cfg, n, parts)
            merged = np.zeros((n + 31) // 32, np.uint32)
            for a, bnd in zip(first, first[1:]):
                if a == bnd:
                    continue
                lo, hi = vd.frame_window(cfg, n, a, bnd)
                llr = torch.from_numpy(q[lo * 2:hi * 2].copy()).cuda()  # only this shard's halo window
                out0 = (a * cfg.f) // 32 * 32
                words = (min(bnd * cfg.f, n) - out0 + 31) // 32
                out = torch.zeros(words, dtype=torch.int32, device="cuda")
                decode_i8_device(t, cfg, n, llr, lo, a, bnd, out, out0)
                torch.cuda.synchronize()
                merged[out0 // 32:out0 // 32 + words] |= out.cpu().numpy().view(np.uint32)
            assert np.array_equal(vd.unpack_bits(merged, n), exp), parts


def test_large_stream_sampled_windows(port):
    """2^25-stage synthetic stream decoded on device; frames in sampled
    windows must equal an oracle decode of just that window re-based to the
    frame grid."""
    import torch

    from paper_2011_09337_b200.device import decode_i8_device, synth_llr_i8

    n = 1 << 25
    t = trellis(*K7)
    cfg = vd.FrameConfig(256, 20, 20)
    llr = torch.empty(n * 2, dtype=torch.int8, device="cuda")
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    synth_llr_i8(t, n, 0.7071, 32.0, 123, llr, bits)
    nf = n // cfg.f
    out = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)
    host_llr = llr.cpu().numpy()
    rng = np.random.default_rng(3)
    for m0 in [0, nf - 8, *rng.integers(1, nf - 8, 6).tolist()]:
        m1 = m0 + 8
        origin = max(m0 - 1, 0) * cfg.f  # ceil(v1/f) = 1 frame of lead-in
        end = min(m1 * cfg.f + cfg.v2, n)
        sub = host_llr[origin * 2:end * 2]
        exp, _, _ = port.framed_decode(*K7, sub, end - origin, cfg.f, cfg.v1, cfg.v2)
        lo, hi = m0 * cfg.f - origin, m1 * cfg.f - origin
        assert np.array_equal(vd.unpack_bits(got, n)[origin + lo:origin + hi], exp[lo:hi]), m0
    # decoded vs sent: sane BER at 3 dB
    errs = np.unpackbits((got ^ bits.cpu().numpy().view(np.uint32)).view(np.uint8)).sum()
    assert errs < n * 1e-3


def test_ber_sweep_counts_match_reference(golden, port):
    """Config 2 parity: the reference run_ber_sweep recipe (berlab.cpp:42-99)
    with the GPU decoding each 65536-bit block reproduces the reference's own
    error counts exactly (unquantised doubles -> FP64 kernel)."""
    meta, _ = golden
    for sw in meta["ber_sweeps"]:
        t = trellis(*K7)
        for p, ebn0 in enumerate(sw["ebn0"]):
            sigma = port.sigma_from_ebn0(ebn0, 0.5)
            errors = 0
            nblk = -(-sw["bits_per_point"] // sw["block_bits"])
            for blk in range(nblk):
                n = min(sw["block_bits"], sw["bits_per_point"] - blk * sw["block_bits"])
                rx, sent = port.gen_sweep_block(*K7, n, sigma, port.mix_seed(sw["seed"], p * 0x100000 + blk))
                if sw["frame"] is None:
                    bits = vd.serial_decode(block(rx, 2), t).bits
                else:
                    f, v1, v2, f0, start, seed = sw["frame"]
                    bits = vd.framed_decode(block(rx, 2), t,
                                            vd.FrameConfig(f, v1, v2, f0, vd.TracebackStart(start), seed)).bits
                errors += int(np.count_nonzero(bits != sent))
            assert errors == sw["errors"][p], (sw["frame"], ebn0)


def test_error_behaviour_on_gpu():
    t = trellis(*K7)
    with pytest.raises(ValueError, match="empty llr block"):
        vd.framed_decode(np.zeros((2, 0)), t, vd.FrameConfig(f=4))
    with pytest.raises(ValueError, match="frame size f must be >= 1"):
        vd.framed_decode(np.zeros((2, 10)), t, vd.FrameConfig(f=0))
    with pytest.raises(ValueError, match="llr row count must equal B"):
        vd.serial_decode(np.zeros((3, 10)), t)


FAST_CODES = [(7, 2, [0o171, 0o133]), (7, 2, [0o133, 0o171]), (9, 2, [0o561, 0o753]), (9, 2, [0o753, 0o561]),
              (5, 2, [0o23, 0o35]), (6, 2, [0o53, 0o75]), (8, 2, [0o247, 0o371]),
              (7, 3, [0o133, 0o171, 0o165]), (9, 3, [0o557, 0o663, 0o711])]


@pytest.mark.parametrize("code", FAST_CODES, ids=lambda c: f"K{c[0]}B{c[1]}_{c[2][0]:o}")
def test_fast_path_vs_oracle(code, port):
    """The register-resident kernel (interior frames) + generic kernel (edge
    frames) against the oracle over many frame configurations."""
    k, b, polys = code
    t = trellis(k, b, polys)
    assert t.fast_path(), "fast path should serve this code"
    rng = np.random.default_rng(2000 + k)
    cfgs = [vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32), vd.FrameConfig(64, 16, 24, 16),
            vd.FrameConfig(128, 20, 40, 32, vd.TracebackStart.kRandom, 5), vd.FrameConfig(100, 14, 30, 30),
            vd.FrameConfig(512, 42, 42), vd.FrameConfig(32, 0, 35), vd.FrameConfig(64, 64, 0, 1)]
    for i, cfg in enumerate(cfgs):
        n = int(rng.integers(60_000, 120_000))
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(0, 4)), 77 + i)
        q = oracle.quantize(rx, [32.0, 4.0][i % 2])
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        packed, stats = vd.framed_decode_stream(q, n, t, cfg)
        got = vd.unpack_bits(packed, n)
        bad = np.flatnonzero(got != exp)
        assert bad.size == 0, (k, cfg, n, bad[:10], bad.size)
        assert (stats.frames, stats.stages, stats.tracebacks) == st


def test_fast_path_metrics(port):
    import torch

    from paper_2011_09337_b200.device import decode_i8_device

    for k, b, polys in [K7, (9, 2, [0o561, 0o753]), (7, 3, [0o133, 0o171, 0o165])]:
        n = 50_000
        rx, _ = port.gen_bench_block(k, b, polys, n, 2.0, 3)
        q = oracle.quantize(rx, 32.0)
        t = trellis(k, b, polys)
        for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 46, 32)):
            _, _, sig = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, want_sigma=True)
            nf = -(-n // cfg.f)
            llr = torch.from_numpy(q).cuda()
            out = torch.zeros((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
            sigma = torch.zeros((nf, 1 << (k - 1)), dtype=torch.int64, device="cuda")
            decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0, sigma)
            torch.cuda.synchronize()
            got = sigma.cpu().numpy().astype(np.float64)
            bad = np.flatnonzero(np.any(got != sig, axis=1))
            assert bad.size == 0, (k, cfg, bad[:5])


@pytest.mark.parametrize("code", [(7, 2, [0o171, 0o133]), (7, 3, [0o133, 0o171, 0o165]), (9, 2, [0o561, 0o753])],
                         ids=lambda c: f"K{c[0]}B{c[1]}")
def test_fast_path_full_int8_range(code, port):
    """Every int8 value, -128 included (outside the quantiser's range but legal
    input): the fast kernel's offset-binary negation must stay exact."""
    k, b, polys = code
    t = trellis(k, b, polys)
    rng = np.random.default_rng(99 + k + b)
    n = 40_000
    q = rng.integers(-128, 128, n * b).astype(np.int8)
    q[rng.random(n * b) < 0.2] = -128
    for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 44, 32)):
        exp, _, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        packed, _ = vd.framed_decode_stream(q, n, t, cfg)
        got = vd.unpack_bits(packed, n)
        assert np.array_equal(got, exp), (code, cfg, np.flatnonzero(got != exp)[:10])


@pytest.mark.parametrize("rows", [0, 37])
@pytest.mark.parametrize("code", [K7, (7, 3, [0o133, 0o171, 0o165]), (9, 2, [0o561, 0o753]), (5, 2, [0o23, 0o35])],
                         ids=lambda c: f"K{c[0]}B{c[1]}" if isinstance(c, tuple) else str(c))
def test_global_spill_tier(code, rows, port, monkeypatch):
    """Survivor rows spilled to global scratch (the long-frame tier): the test
    hook VITDEC_SPILL_ROWS caps the shared-memory rows so every config below
    keeps stages [t_gl, L) in global memory; bit-exact vs the oracle."""
    monkeypatch.setenv("VITDEC_SPILL_ROWS", str(rows))
    k, b, polys = code
    t = trellis(k, b, polys)
    rng = np.random.default_rng(500 + k + rows)
    cfgs = [vd.FrameConfig(256, 20, 20), vd.FrameConfig(1024, 42, 42), vd.FrameConfig(320, 20, 45, 32),
            vd.FrameConfig(500, 26, 51), vd.FrameConfig(384, 20, 40, 64, vd.TracebackStart.kRandom, 9)]
    for i, cfg in enumerate(cfgs):
        n = int(rng.integers(80_000, 140_000))
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(1, 4)), 900 + i)
        q = oracle.quantize(rx, 32.0)
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        packed, stats = vd.framed_decode_stream(q, n, t, cfg)
        got = vd.unpack_bits(packed, n)
        bad = np.flatnonzero(got != exp)
        assert bad.size == 0, (k, rows, cfg, n, bad[:10], bad.size)
        assert (stats.frames, stats.stages, stats.tracebacks) == st


def test_long_frames_full_size_sampled_windows(port):
    """f = 1024 at 2^25 stages (a full-GPU launch: the natural spill layout,
    12 warps per SM with TMEM + smem + global rows): sampled frame windows
    re-decoded by the oracle are bit-identical; BER sane."""
    import torch

    from paper_2011_09337_b200.device import count_bit_errors, decode_i8_device, synth_llr_i8

    t = trellis(*K7)
    n = 1 << 25
    for cfg in (vd.FrameConfig(1024, 42, 42), vd.FrameConfig(512, 20, 63)):
        f, v1, v2 = cfg.f, cfg.v1, cfg.v2
        llr = torch.empty(n * 2, dtype=torch.int8, device="cuda")
        bits = torch.empty(n // 32, dtype=torch.int32, device="cuda")
        out = torch.empty(n // 32 + 1, dtype=torch.int32, device="cuda")
        synth_llr_i8(t, n, 0.7, 32.0, 4321, llr, bits)
        decode_i8_device(t, cfg, n, llr, 0, 0, -(-n // f), out, 0)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        count_bit_errors(out, bits, n, cnt)
        torch.cuda.synchronize()
        assert int(cnt.item()) < n * 2e-3
        got_all = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
        q = llr.cpu().numpy()
        rng = np.random.default_rng(f)
        nf = n // f
        for m0 in list(rng.integers(1, nf - 8, 6)) + [0, nf - 4]:
            m1 = min(m0 + 4, nf)
            g0 = max(m0 - (-(-v1 // f)), 0)  # window origin on the frame grid
            lo, hi = g0 * f, min(m1 * f + v2, n)
            exp, _, _ = port.framed_decode(*K7, q[lo * 2:hi * 2], hi - lo, f, v1, v2)
            a, b2 = (m0 - g0) * f, (m1 - g0) * f
            assert np.array_equal(got_all[m0 * f:m1 * f], exp[a:b2]), (cfg, m0)


@pytest.mark.parametrize("code", [K7, (7, 3, [0o133, 0o171, 0o165]), (3, 2, [7, 5]), (5, 2, [0o23, 0o35]),
                                  (6, 2, [0o53, 0o75]), (4, 3, [0o13, 0o15, 0o17])],
                         ids=lambda c: f"K{c[0]}B{c[1]}")
def test_serial_decode_segment_parallel(code, port):
    """Long single frames (serial_decode, f >= N) take the exact segment-
    parallel decoder (max-plus transfer matrices per segment, sequential
    boundary combine, per-segment re-run + traceback): bit-identical to the
    oracle, including tie-heavy inputs (scale 1 -> LLRs in {-1, 0, 1})."""
    k, b, polys = code
    t = trellis(k, b, polys)
    rng = np.random.default_rng(31 + k * b)
    for n, scale in ((8192, 32.0), (8193, 4.0), (65543, 1.0), (300_001, 32.0)):
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(0, 3)), n + k)
        q = oracle.quantize(rx, scale)
        exp = port.serial_decode(k, b, polys, q.astype(np.float64), n)
        out = vd.serial_decode(block(q, b), t)
        bad = np.flatnonzero(out.bits != exp)
        assert bad.size == 0, (code, n, scale, bad[:10], bad.size)
        assert (out.stats.frames, out.stats.stages, out.stats.tracebacks) == (1, n, 1)
    # one long frame with overlaps inside a longer stream (f >= n - ... : single frame, clipped window)
    n = 50_000
    rx, _ = port.gen_bench_block(k, b, polys, n, 2.0, 99)
    q = oracle.quantize(rx, 32.0)
    cfg = vd.FrameConfig(60_000, 0, 0)
    exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2)
    packed, stats = vd.framed_decode_stream(q, n, t, cfg)
    assert np.array_equal(vd.unpack_bits(packed, n), exp)


def test_concurrent_host_calls_pageable_and_pinned(port):
    """The reference's BER sweep calls framed_decode from several host threads
    at once (berlab.cpp:63-88): concurrent vd_decode_i8 calls (per-thread
    streams and pinned staging of pageable buffers) all equal the oracle."""
    import threading

    import torch

    t = trellis(*K7)
    cfg = vd.FrameConfig(256, 20, 20)
    jobs = []
    for i in range(6):
        n = 150_000 + 4099 * i
        rx, _ = port.gen_bench_block(*K7, n, 2.0, 700 + i)
        q = oracle.quantize(rx, 32.0)
        if i % 2:
            q = torch.from_numpy(q).pin_memory().numpy()  # pinned input for half the jobs
        exp, _, _ = port.framed_decode(*K7, q, n, 256, 20, 20)
        jobs.append((q, n, exp))
    results = [None] * len(jobs)

    def run(i):
        q, n, _ = jobs[i]
        for _ in range(3):
            packed, _ = vd.framed_decode_stream(q, n, t, cfg, chunk_stages=1 << 15)
            results[i] = vd.unpack_bits(packed, n)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for (q, n, exp), got in zip(jobs, results):
        assert np.array_equal(got, exp)


@pytest.mark.parametrize("polys", [[0o171, 0o133], [0o133, 0o171]])
def test_small_launch_kernel_vs_oracle(polys, port, monkeypatch):
    """Small launches (fewer 16-frame warps than schedulers) run the
    8-states-per-lane kernel (csrc/vd_small_dev.cuh); bit-exact vs the oracle
    and vs the 16-states-per-lane kernel (VITDEC_SMALL=0) over frame
    configurations incl. subframe / random-start tracebacks, v1 not a multiple
    of the 3-stage blocks, padded head frames and generic tail frames."""
    k, b = 7, 2
    t = trellis(k, b, polys)
    rng = np.random.default_rng(4242 + polys[0])
    cfgs = [vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32), vd.FrameConfig(64, 16, 24, 16),
            vd.FrameConfig(128, 20, 40, 32, vd.TracebackStart.kRandom, 5), vd.FrameConfig(100, 14, 30, 30),
            vd.FrameConfig(512, 42, 42), vd.FrameConfig(32, 0, 35), vd.FrameConfig(96, 7, 11, 0)]
    for i, cfg in enumerate(cfgs):
        n = int(rng.integers(50_000, 400_000))
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(0, 4)), 300 + i)
        q = oracle.quantize(rx, [32.0, 4.0][i % 2])
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        for small in ("1", "0"):
            monkeypatch.setenv("VITDEC_SMALL", small)
            packed, stats = vd.framed_decode_stream(q, n, t, cfg)
            got = vd.unpack_bits(packed, n)
            bad = np.flatnonzero(got != exp)
            assert bad.size == 0, (small, cfg, n, bad[:10], bad.size)
            assert (stats.frames, stats.stages, stats.tracebacks) == st


@pytest.mark.parametrize("inputs", ["noise", "saturated", "minus3dB_scale1", "3dB"])
def test_small_launch_extreme_inputs_vs_oracle(inputs, port, monkeypatch):
    """The small kernel (lagged renormalisation: metrics must stay inside
    int16 over 12 stages of growth) on pure-noise, saturated (+-127 only) and
    -3 dB tie-heavy (scale 1) LLRs as well as 3 dB ones, over frame
    geometries with whole-word output (so the output is not pre-zeroed);
    bit-exact vs the oracle through the host and the device calls."""
    import torch

    from paper_2011_09337_b200.device import decode_i8_device

    k, b, polys = K7
    t = trellis(k, b, polys)
    rng = np.random.default_rng({"noise": 1, "saturated": 4, "minus3dB_scale1": 2, "3dB": 3}[inputs])
    cfgs = [(256, 20, 20), (128, 0, 0), (512, 42, 42), (160, 5, 9), (256, 3, 63), (416, 30, 2)]
    for i, (f, v1, v2) in enumerate(cfgs):
        n = 32 * int(rng.integers(2_000, 20_000))
        if inputs == "noise":
            q = rng.integers(-127, 128, size=b * n, dtype=np.int8)
        elif inputs == "saturated":
            q = (rng.integers(0, 2, size=b * n, dtype=np.int8) * 2 - 1) * np.int8(127)
        else:
            rx, _ = port.gen_bench_block(k, b, polys, n, -3.0 if inputs != "3dB" else 3.0, 700 + i)
            q = oracle.quantize(rx, 1.0 if inputs != "3dB" else 32.0)
        q = q.astype(np.int8)
        exp, st, _ = port.framed_decode(k, b, polys, q, n, f, v1, v2, 0)
        cfg = vd.FrameConfig(f, v1, v2)
        monkeypatch.setenv("VITDEC_SMALL", "1")
        packed, stats = vd.framed_decode_stream(q, n, t, cfg)
        got = vd.unpack_bits(packed, n)
        assert np.array_equal(got, exp), (inputs, n, cfg, np.flatnonzero(got != exp)[:8])
        assert (stats.frames, stats.stages, stats.tracebacks) == st
        out = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        decode_i8_device(t, cfg, n, torch.from_numpy(q).cuda(), 0, 0, -(-n // f), out, 0)
        torch.cuda.synchronize()
        got2 = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
        assert np.array_equal(got2, exp), (inputs, n, cfg, "device", np.flatnonzero(got2 != exp)[:8])


@pytest.mark.parametrize("cfg", [(256, 20, 20, 0), (320, 20, 45, 32), (256, 20, 20, 0, 7)],
                         ids=["f256", "f320f0_32", "n_unaligned"])
def test_small_launch_whole_words_over_stale_output(cfg, port):
    """Small launches with 32-aligned frame / subframe boundaries write every
    output word whole and skip the output zeroing: an output buffer full of
    stale ones must come back exactly equal to the oracle's bits (an unaligned
    stream end keeps the zeroing)."""
    import torch

    from paper_2011_09337_b200.device import decode_i8_device

    f, v1, v2, f0 = cfg[:4]
    n = 3200 * 32 + (cfg[4] if len(cfg) > 4 else 0)
    k, b, polys = K7
    rx, _ = port.gen_bench_block(k, b, polys, n, 2.5, 99 + f)
    q = oracle.quantize(rx, 32.0)
    exp, _, _ = port.framed_decode(k, b, polys, q, n, f, v1, v2, f0)
    t = trellis(k, b, polys)
    fc = vd.FrameConfig(f, v1, v2, f0)
    nf = -(-n // f)
    llr = torch.from_numpy(q).cuda()
    out = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")
    decode_i8_device(t, fc, n, llr, 0, 0, nf, out, 0)
    torch.cuda.synchronize()
    got = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
    assert np.array_equal(got, exp), np.flatnonzero(got != exp)[:10]


@pytest.mark.parametrize("code", [K7, (7, 2, [0o133, 0o171]), (7, 3, [0o133, 0o171, 0o165]),
                                  (9, 2, [0o561, 0o753]), (6, 2, [0o53, 0o75])],
                         ids=["K7a", "K7b", "K7c", "K9a", "K6a"])
def test_random_geometry_mid_sizes_vs_oracle(code, port):
    """Random frame geometries (f, v1, v2, f0, traceback start) at sizes where
    the fast kernels take the launch (small-launch kernel with its clipped tail
    segments and whole-word output, or the 16-states-per-lane kernel with head
    padding and generic edge frames), through the host streaming call and the
    device call into a stale output buffer; bit-exact vs the oracle."""
    import torch

    from paper_2011_09337_b200.device import decode_i8_device

    k, b, polys = code
    t = trellis(k, b, polys)
    rng = np.random.default_rng(9000 + k * 10 + b + polys[0])
    for it in range(16):
        n = int(rng.integers(20_000, 300_000))
        f = int(rng.choice([32, 64, 96, 128, 200, 256, 320, 480, 512]))
        f0 = int(rng.choice([0, 0, 32, f // 2 if f >= 64 else 0, int(rng.integers(1, f + 1))]))
        cfg = vd.FrameConfig(f, int(rng.integers(0, 60)), int(rng.integers(0, 80)), f0,
                             vd.TracebackStart(int(rng.integers(0, 2))), int(rng.integers(0, 2**63)))
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(0, 4)), int(rng.integers(0, 2**32)))
        q = oracle.quantize(rx, [32.0, 4.0][it % 2])
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        packed, stats = vd.framed_decode_stream(q, n, t, cfg)
        got = vd.unpack_bits(packed, n)
        assert np.array_equal(got, exp), (code, n, cfg, np.flatnonzero(got != exp)[:8])
        assert (stats.frames, stats.stages, stats.tracebacks) == st
        out = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        decode_i8_device(t, cfg, n, torch.from_numpy(q).cuda(), 0, 0, -(-n // f), out, 0)
        torch.cuda.synchronize()
        got2 = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
        assert np.array_equal(got2, exp), (code, n, cfg, "device", np.flatnonzero(got2 != exp)[:8])


@pytest.mark.parametrize("code", [K7, (7, 2, [0o165, 0o117])], ids=["K7a", "K7jit"])
def test_round_split_sizes_vs_oracle(code, port):
    """Mid-size launches where the 16-states-per-lane kernel runs one round
    of 4- / 8-warp CTAs with its edge frames on the small-launch kernel beside
    it, and multi-round launches whose partial last round (a few frame groups)
    goes to the small kernel after it together with the tail edge frames
    (csrc/vd_fast.cuh launch_variant): bit-exact vs the oracle, decoded into a
    stale output buffer, over the sizes around those splits."""
    import torch

    from paper_2011_09337_b200.device import decode_i8_device

    k, b, polys = code
    t = trellis(k, b, polys)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    slots = 12 * sms  # 16-frame groups per round of 12-warp CTAs
    rng = np.random.default_rng(777 + polys[0])
    cases = []
    for f, v1, v2, f0 in ((256, 20, 20, 0), (320, 20, 45, 32)):
        for groups in (2 * sms + 5, 7 * sms, slots + 1, slots + 250):  # one round (4 / 8 warps); round + remainder
            cases.append((vd.FrameConfig(f, v1, v2, f0), groups * 16 * f - int(rng.integers(1, f))))
    for i, (cfg, n) in enumerate(cases):
        rx, _ = port.gen_bench_block(k, b, polys, n, 2.5, 4000 + i)
        q = oracle.quantize(rx, 32.0)
        exp, _, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0)
        out = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        decode_i8_device(t, cfg, n, torch.from_numpy(q).cuda(), 0, 0, -(-n // cfg.f), out, 0)
        torch.cuda.synchronize()
        got = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
        bad = np.flatnonzero(got != exp)
        assert bad.size == 0, (code, cfg, n, bad[:8], bad.size)
        if i % 4 == 3:
            # host streaming in chunks whose decodes split the same way (each
            # chunk's window starts inside the stream: llr_stage0 > 0)
            chunk = (slots + 100) * 16 * cfg.f
            packed, _ = vd.framed_decode_stream(q, n, t, cfg, chunk_stages=chunk)
            got = vd.unpack_bits(packed, n)
            assert np.array_equal(got, exp), (code, cfg, n, "chunked", np.flatnonzero(got != exp)[:8])

"""Run-time (NVRTC) instantiations of the fast kernel for codes outside the
precompiled list (csrc/vd_jit.cu).

The reference's ACS is code-generic through the trellis tables
(proj/src/decoder.cpp:53-76, trellis.cpp:57-100); the fast kernel bakes the
polynomials into compile-time table selections, so every code with
5 <= K <= 10 and B in {2, 3, 4} (complement-paired or not) gets its own
instantiation compiled on first use. CPU tests: the envelope and the NVRTC compile of the embedded
sources (no GPU needed). GPU tests: bit-exact parity with the oracle and
identical results with the JIT disabled (generic kernel).
"""
import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd

# codes that are NOT among the precompiled instantiations: complement-paired
# ones, and ones whose polynomials miss the newest or the oldest tap (their
# butterfly edges are not complement pairs: four distinct edge labels)
JIT_CODES = [
    (7, 2, [0o165, 0o117]),
    (7, 3, [0o171, 0o133, 0o145]),
    (5, 3, [0o25, 0o33, 0o37]),
    (6, 2, [0o65, 0o57]),
    (8, 3, [0o225, 0o331, 0o367]),
    (9, 2, [0o657, 0o435]),
    (7, 2, [0o170, 0o133]),         # not paired: 0170 misses the oldest tap
    (5, 2, [0o22, 0o35]),           # not paired
    (8, 2, [0o247, 0o170]),         # not paired: neither edge bit is common
    (10, 2, [0o1157, 0o1753]),      # K = 10: 32 lanes per frame pair, 2 frames per warp
    (10, 3, [0o1157, 0o1753, 0o1331]),
    (9, 4, [0o765, 0o671, 0o513, 0o473]),   # rate 1/4, K = 9 (cdma2000 r1/4)
    (7, 4, [0o117, 0o127, 0o155, 0o171]),
]


def trellis(spec):
    k, b, polys = spec
    return vd.build_trellis(vd.CodeSpec(k, b, list(polys)))


def test_jit_envelope(monkeypatch):
    lib = vd.lib()
    for spec in JIT_CODES:
        assert trellis(spec).fast_path(), spec
    # K outside 5..9 -> generic kernel
    t = trellis((4, 2, [0o17, 0o13]))
    assert lib.vd_code_jit_check(t.handle) == vd.api.VD_EUNSUPPORTED
    assert not trellis((4, 2, [0o17, 0o13])).fast_path()
    assert not trellis((11, 2, [0o2335, 0o3277])).fast_path()
    monkeypatch.setenv("VITDEC_JIT", "0")
    assert not trellis(JIT_CODES[0]).fast_path()
    assert trellis((7, 2, [0o171, 0o133])).fast_path()  # precompiled: unaffected


def test_jit_compiles_embedded_sources():
    """NVRTC compiles the sources embedded in the library for sm_100a (what a
    GPU box does on first use of a new code)."""
    t = trellis(JIT_CODES[0])
    st = vd.lib().vd_code_jit_check(t.handle)
    assert st == 0, vd.lib().vd_last_error()


@pytest.mark.gpu
@pytest.mark.parametrize("spec", JIT_CODES, ids=lambda s: f"K{s[0]}B{s[1]}")
def test_jit_fast_path_vs_oracle(spec, monkeypatch, tmp_path):
    monkeypatch.setenv("VITDEC_JIT_CACHE", str(tmp_path))  # compile in this test, not from a cache
    k, b, polys = spec
    port = oracle.port()
    t = trellis(spec)
    assert t.fast_path()
    rng = np.random.default_rng(7000 + k * 10 + b)
    # TMEM + smem survivor store; subframe tracebacks; long frames (global spill tier)
    cfgs = [vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32), vd.FrameConfig(1024, 42, 42)]
    for i, cfg in enumerate(cfgs):
        n = int(rng.integers(150_000, 220_000))
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(1, 4)), 11 + i)
        q = oracle.quantize(rx, [32.0, 4.0][i % 2])
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0)
        packed, stats = vd.framed_decode_stream(q, n, t, cfg)
        got = vd.unpack_bits(packed, n)
        bad = np.flatnonzero(got != exp)
        assert bad.size == 0, (spec, cfg, n, bad[:10], bad.size)
        assert (stats.frames, stats.stages, stats.tracebacks) == st
        if i == 0:
            monkeypatch.setenv("VITDEC_JIT", "0")  # generic kernel: same bits
            packed0, _ = vd.framed_decode_stream(q, n, t, cfg)
            assert np.array_equal(vd.unpack_bits(packed0, n), exp)
            monkeypatch.delenv("VITDEC_JIT")


@pytest.mark.gpu
def test_jit_concurrent_first_use(monkeypatch, tmp_path):
    """Several host threads decoding codes that need a run-time instantiation
    at the same moment (first use of each, one shared per-process cache):
    every thread gets its code's kernel and the oracle's bits."""
    import threading

    monkeypatch.setenv("VITDEC_JIT_CACHE", str(tmp_path))
    port = oracle.port()
    specs = [(7, 2, [0o117, 0o165]), (6, 2, [0o57, 0o65]), (7, 2, [0o117, 0o165]), (9, 2, [0o435, 0o657])]
    cfg = vd.FrameConfig(256, 20, 20)
    jobs, res = [], [None] * len(specs)
    for i, (k, b, polys) in enumerate(specs):
        n = 80_000 + 999 * i
        rx, _ = port.gen_bench_block(k, b, polys, n, 2.5, 500 + i)
        q = oracle.quantize(rx)
        exp, _, _ = port.framed_decode(k, b, polys, q, n, 256, 20, 20)
        jobs.append((trellis((k, b, polys)), q, n, exp))

    def run(i):
        t, q, n, _ = jobs[i]
        packed, _ = vd.framed_decode_stream(q, n, t, cfg)
        res[i] = vd.unpack_bits(packed, n)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for (_, _, _, exp), got in zip(jobs, res):
        assert got is not None and np.array_equal(got, exp)


@pytest.mark.gpu
@pytest.mark.parametrize("spec", [(10, 3, [0o1157, 0o1753, 0o1331]), (10, 2, [0o1157, 0o1753]),
                                  (9, 3, [0o557, 0o663, 0o711]), (10, 4, [0o1157, 0o1753, 0o1331, 0o1475])],
                         ids=["K10B3", "K10B2", "K9B3", "K10B4"])
def test_metric_range_at_saturated_llrs(spec, monkeypatch, tmp_path):
    """The int16 metric range at its extreme: every LLR +-127 (random signs and
    a long all-+127 run), K = 9 / 10 with B = 3 / 4 (the largest spreads the
    fast kernel admits), bit-exact vs the oracle."""
    monkeypatch.setenv("VITDEC_JIT_CACHE", str(tmp_path))
    k, b, polys = spec
    rng = np.random.default_rng(k * 100 + b)
    n = 120_000
    q = rng.choice(np.array([-127, 127], np.int8), size=n * b)
    q[: 3000 * b] = 127
    port = oracle.port()
    t = trellis(spec)
    assert t.fast_path()
    for cfg in (vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32)):
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0)
        packed, stats = vd.framed_decode_stream(q, n, t, cfg)
        got = vd.unpack_bits(packed, n)
        assert np.array_equal(got, exp), (spec, cfg, np.flatnonzero(got != exp)[:10])


SMALL_JIT_CODES = [
    (9, 2, [0o561, 0o753]),         # K = 8 / 9: the 16-states-per-lane kernel either way
    (8, 2, [0o247, 0o170]),         # not paired
    (6, 2, [0o65, 0o57]),
    (5, 2, [0o22, 0o35]),           # not paired
    (7, 2, [0o165, 0o117]),
]


@pytest.mark.gpu
@pytest.mark.parametrize("spec", SMALL_JIT_CODES, ids=lambda s: f"K{s[0]}_{s[2][0]:o}")
def test_jit_small_launch_vs_oracle(spec, monkeypatch, tmp_path):
    """Small launches of rate-1/2 codes with K <= 7 other than the two
    precompiled K = 7 ones run a run-time instantiation of the 8-states-per-lane kernel
    (csrc/vd_small_dev.cuh): bit-exact vs the oracle and vs the
    16-states-per-lane kernel (VITDEC_SMALL=0), over subframe, random-start,
    head-padded and clipped-tail geometries."""
    monkeypatch.setenv("VITDEC_JIT_CACHE", str(tmp_path))
    k, b, polys = spec
    port = oracle.port()
    t = trellis(spec)
    rng = np.random.default_rng(9100 + k * 10 + polys[0])
    cfgs = [vd.FrameConfig(256, 20, 20), vd.FrameConfig(320, 20, 45, 32),
            vd.FrameConfig(128, 20, 40, 32, vd.TracebackStart.kRandom, 5), vd.FrameConfig(100, 14, 30, 30),
            vd.FrameConfig(96, 7, 11, 0)]
    for i, cfg in enumerate(cfgs):
        n = int(rng.integers(40_000, 200_000))
        rx, _ = port.gen_bench_block(k, b, polys, n, float(rng.uniform(0, 4)), 700 + i)
        q = oracle.quantize(rx, [32.0, 4.0][i % 2])
        exp, st, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        for small in ("1", "0"):
            monkeypatch.setenv("VITDEC_SMALL", small)
            packed, stats = vd.framed_decode_stream(q, n, t, cfg)
            got = vd.unpack_bits(packed, n)
            bad = np.flatnonzero(got != exp)
            assert bad.size == 0, (spec, small, cfg, n, bad[:10], bad.size)
            assert (stats.frames, stats.stages, stats.tracebacks) == st

"""Puncturing: oracle restatement pinned to the reference, C-ABI validation
(CPU), and the device depuncture + punctured framed decode (GPU).

Reference anchors: PuncturePattern (codec.hpp:13-33, codec.cpp:12-74),
puncture (codec.cpp:88-103), depuncture (decoder.cpp:131-163) and its unit
test (test_decoder.cpp:160-204); the punctured chain run by run_ber_sweep
(berlab.cpp:74-84) and the CLI (vitdec_cli.cpp:172-176).
Bar: bit-exact (depunctured bytes, decoded bits, DecodeStats).
"""
import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd

K7 = (7, 2, [0o171, 0o133])
PATTERNS = ["r12", "r23", "r34", "1101;1011", "110;011;101", "10;01;11"]


def _b(pattern):
    return len(pattern.split(";")) if ";" in pattern else 2


def _rows(name):
    return {"r12": "1;1", "r23": "11;10", "r34": "110;101"}.get(name, name)


# ---------------------------------------------------------------- CPU ------


def test_oracle_depuncture_kats():
    # test_decoder.cpp:161-177: identity and rate-2/3 reinsertion
    blk, n = oracle.depuncture_i8("1;1", np.array([1, 2, 3, 4], np.int8))
    assert n == 2 and blk[1 * 2 + 1] == 4
    blk, n = oracle.depuncture_i8("11;10", np.array([10, 20, 30], np.int8))
    assert n == 2 and list(blk) == [10, 20, 30, 0]
    # test_decoder.cpp:198-203: inconsistent length
    with pytest.raises(ValueError, match="punctured length inconsistent with pattern"):
        oracle.depuncture_i8("11;10", np.array([1, 2, 3, 4], np.int8))


@pytest.mark.parametrize("name", ["r23", "r34"])
def test_oracle_depuncture_matches_reference(name):
    ref = oracle.reference()
    if ref is None:
        pytest.skip("reference library not built (oracle/_ref)")
    import ctypes as C

    rng = np.random.default_rng(7)
    for n_stages in (1, 2, 3, 7, 60, 601):
        full = rng.integers(-127, 128, n_stages * 2).astype(np.int8)
        punct = oracle.puncture_i8(_rows(name), full, n_stages)
        ours, n = oracle.depuncture_i8(_rows(name), punct)
        d = punct.astype(np.float64)
        out = np.zeros(n_stages * 2 + 8, np.float64)
        st = C.c_int64()
        ref.check(ref.fn("depuncture")(name.encode(), d.ctypes.data, d.size, out.ctypes.data, out.size,
                                       C.addressof(st)))
        assert st.value == n == n_stages
        assert np.array_equal(out[: n * 2], ours.astype(np.float64))


@pytest.mark.parametrize("pattern", PATTERNS)
def test_oracle_puncture_depuncture_round_trip(pattern):
    rows = _rows(pattern)
    b, period, mask = oracle._mask_arr(rows)
    rng = np.random.default_rng(3)
    for n_stages in (1, period, 5 * period + 1, 1000):
        full = rng.integers(-127, 128, n_stages * b).astype(np.int8)
        blk, n = oracle.depuncture_i8(rows, oracle.puncture_i8(rows, full, n_stages))
        assert n == n_stages
        keep = np.array([mask[(t % period) * b + r] for t in range(n_stages) for r in range(b)], bool)
        assert np.array_equal(blk[keep], full[keep]) and not blk[~keep].any()


def test_capi_puncture_validation_messages():
    with pytest.raises(ValueError, match="puncture mask drops an entire stage"):
        vd.PuncturePattern(2, 2, [1, 1, 0, 0]).validate()
    with pytest.raises(ValueError, match="puncture mask shape mismatch"):
        vd.PuncturePattern(0, 2, [1]).validate()
    with pytest.raises(ValueError, match="puncture mask rows differ in length"):
        vd.PuncturePattern.parse("11;1")
    with pytest.raises(ValueError, match="puncture mask must be 0/1"):
        vd.PuncturePattern.parse("12;11")
    with pytest.raises(vd.VitdecError):
        vd.PuncturePattern(2, 600, np.ones(1200)).validate()  # GPU envelope: period * B <= 1024
    p = vd.PuncturePattern.named("r34")
    assert (p.b, p.period, p.kept_per_period(), p.rate()) == (2, 3, 4, 0.75)


@pytest.mark.parametrize("pattern", PATTERNS)
def test_capi_depuncture_stage_count_matches_oracle(pattern):
    rows = _rows(pattern)
    p = vd.PuncturePattern.parse(rows)
    for length in range(0, 40):
        try:
            _, want = oracle.depuncture_i8(rows, np.zeros(length, np.int8))
        except ValueError as e:
            with pytest.raises(ValueError, match=str(e)):
                vd.depuncture_stages(length, p)
            continue
        assert vd.depuncture_stages(length, p) == want


# ---------------------------------------------------------------- GPU ------


def _punctured_case(k, b, polys, rows, n_stages, seed, ebn0=3.0):
    port = oracle.port()
    rx, sent = port.gen_bench_block(k, b, polys, n_stages, ebn0, seed)
    full = oracle.quantize(rx, 32.0)
    return oracle.puncture_i8(rows, full, n_stages), sent


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", PATTERNS)
def test_device_depuncture_bit_exact(pattern):
    import torch

    rows = _rows(pattern)
    b = len(rows.split(";"))
    p = vd.PuncturePattern.parse(rows)
    rng = np.random.default_rng(11)
    for n_stages in (1, 2, 5, 4097, 100_003):
        full = rng.integers(-127, 128, n_stages * b).astype(np.int8)
        punct = oracle.puncture_i8(rows, full, n_stages)
        want, n = oracle.depuncture_i8(rows, punct)
        dev_in = torch.from_numpy(punct.copy()).cuda()
        dev_out = torch.full((n * b + 4,), 77, dtype=torch.int8, device="cuda")
        pc = p.to_c()
        import ctypes as C

        vd.api.check(vd.lib().vd_depuncture_i8_device(C.byref(pc), dev_in.data_ptr(), punct.size,
                                                      dev_out.data_ptr(), -1, None))
        got = dev_out.cpu().numpy()
        assert np.array_equal(got[: n * b], want), (pattern, n_stages)
        assert (got[n * b:] == 77).all()  # nothing written past the block


CFGS = [vd.FrameConfig(256, 20, 20), vd.FrameConfig(60, 12, 24), vd.FrameConfig(240, 24, 48, 48),
        vd.FrameConfig(96, 0, 36, 32, vd.TracebackStart.kRandom, seed=5)]


@pytest.mark.gpu
@pytest.mark.parametrize("pattern", ["r23", "r34", "1101;1011"])
def test_punctured_framed_decode_matches_oracle(pattern):
    rows = _rows(pattern)
    k, b, polys = K7
    t = vd.build_trellis(vd.CodeSpec(k, b, polys))
    port = oracle.port()
    p = vd.PuncturePattern.parse(rows)
    for n_stages in (12, 997, 60_000):
        punct, sent = _punctured_case(k, b, polys, rows, n_stages, seed=n_stages)
        full, n = oracle.depuncture_i8(rows, punct)
        for cfg in CFGS:
            exp, st, _ = port.framed_decode(k, b, polys, full, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start),
                                            cfg.seed)
            for chunk in (0, 4096):
                packed, n2, stats = vd.framed_decode_punctured(punct, p, t, cfg, chunk_stages=chunk)
                assert n2 == n
                got = vd.unpack_bits(packed, n)
                assert np.array_equal(got, exp), (pattern, n_stages, cfg, chunk)
                assert (stats.frames, stats.stages, stats.tracebacks) == st


@pytest.mark.gpu
def test_punctured_r13_code_and_device_entry():
    import ctypes as C

    import torch

    k, b, polys = 7, 3, [0o133, 0o171, 0o165]
    rows = "110;011;101"
    t = vd.build_trellis(vd.CodeSpec(k, b, polys))
    p = vd.PuncturePattern.parse(rows)
    punct, sent = _punctured_case(k, b, polys, rows, 50_000, seed=9)
    full, n = oracle.depuncture_i8(rows, punct)
    cfg = vd.FrameConfig(256, 20, 20)
    exp, st, _ = oracle.port().framed_decode(k, b, polys, full, n, 256, 20, 20)
    dev_in = torch.from_numpy(punct.copy()).cuda()
    scratch = torch.empty(n * b, dtype=torch.int8, device="cuda")
    out = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    s = vd.api.VdStats()
    c, pc = cfg.to_c(), p.to_c()
    vd.api.check(vd.lib().vd_decode_punctured_i8_device(t.handle, C.byref(c), C.byref(pc), dev_in.data_ptr(),
                                                        punct.size, scratch.data_ptr(), out.data_ptr(), C.byref(s),
                                                        -1, None))
    torch.cuda.synchronize()
    got = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
    assert np.array_equal(got, exp)
    assert (s.frames, s.stages, s.tracebacks) == st
    # B mismatch between the pattern and the code -> check_block's message
    with pytest.raises(ValueError, match="llr row count must equal B"):
        vd.framed_decode_punctured(punct[: punct.size // 3 * 3], vd.PuncturePattern.named("r23"), t, cfg)


@pytest.mark.gpu
def test_punctured_noiseless_round_trip_large():
    """Size-independent property at 4 Mi stages: noiseless r3/4 decode is exact."""
    import torch

    k, b, polys = K7
    t = vd.build_trellis(vd.CodeSpec(k, b, polys))
    n = 1 << 22
    rows = "110;101"
    code = vd.lib()
    llr = torch.empty(n * b, dtype=torch.int8, device="cuda")
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    vd.api.check(code.vd_synth_llr_i8_device(t.handle, n, 0.0, 32.0, 1234, llr.data_ptr(), bits.data_ptr(), -1,
                                             None))
    torch.cuda.synchronize()
    punct = oracle.puncture_i8(rows, llr.cpu().numpy(), n)
    packed, n2, _ = vd.framed_decode_punctured(punct, vd.PuncturePattern.parse(rows), t, vd.FrameConfig(256, 24, 48))
    assert n2 == n
    assert np.array_equal(packed, bits.cpu().numpy().view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["r23", "r34"])
def test_drop_in_depuncture_f64_matches_reference(name):
    """vd_depuncture_f64 (the device gather behind the drop-in
    vitdec::depuncture) on real-valued streams == the reference's depuncture."""
    ref = oracle.reference()
    if ref is None:
        pytest.skip("reference library not built (oracle/_ref)")
    import ctypes as C

    from paper_2011_09337_b200._lib import VdPuncture, check, lib

    rows = _rows(name)
    b, period, mask = oracle._mask_arr(rows)
    m = np.ascontiguousarray(mask, np.uint8)
    pc = VdPuncture(b, period, m.ctypes.data)
    rng = np.random.default_rng(11)
    kept = int(m.sum())
    for n_p in (1, kept, kept * 5 + 2, 100_003 // kept * kept):
        d = rng.normal(size=n_p)
        st = C.c_int64()
        out = np.zeros(2 * n_p + 8, np.float64)
        status = ref.fn("depuncture")(name.encode(), d.ctypes.data, d.size, out.ctypes.data, out.size, C.addressof(st))
        n_stages = C.c_int64()
        ours_status = lib().vd_depuncture_stages(C.byref(pc), n_p, C.byref(n_stages))
        if status != 0:
            assert ours_status != 0
            continue
        check(ours_status)
        assert n_stages.value == st.value
        got = np.zeros(n_stages.value * b, np.float64)
        check(lib().vd_depuncture_f64(C.byref(pc), d.ctypes.data, n_p, got.ctypes.data))
        assert np.array_equal(got, out[:n_stages.value * b]), (name, n_p)


FUSED_CASES = [(K7, "r23", (256, 20, 20)), (K7, "r23", (128, 16, 42)), (K7, "r34", (255, 21, 21)),
               (K7, "r34", (240, 24, 48)),
               # other rate-1/2 codes: run-time instantiations of the fused kernel
               ((7, 2, [0o133, 0o171]), "r23", (256, 20, 20)), ((9, 2, [0o561, 0o753]), "r34", (240, 45, 45)),
               ((5, 2, [0o23, 0o35]), "r23", (128, 16, 24)),  # K != 7: the separate pass
               ((8, 2, [0o247, 0o170]), "r34", (252, 30, 30))]


@pytest.mark.gpu
@pytest.mark.parametrize("code,pattern,cfg", FUSED_CASES,
                         ids=[f"K{c[0]}_{c[2][0]:o}_{p}_{g[0]}" for c, p, g in FUSED_CASES])
def test_fused_depuncture_device_decode(code, pattern, cfg, monkeypatch, tmp_path):
    """Depuncture fused into the fast kernel's LLR staging (vd_fast_dev.cuh
    Punct: the kernel gathers the punctured stream into its shared-memory LLR
    ring, re-inserting the zeros; the default) == the oracle's framed_decode
    of the depunctured block, and == the separate-pass path
    (VITDEC_PUNCT_FUSED=0); edge frames come from dense copies of their
    windows. The fused kernel is checked to be the one that ran."""
    import ctypes as C

    import torch
    from torch.profiler import ProfilerActivity, profile

    monkeypatch.setenv("VITDEC_JIT_CACHE", str(tmp_path))
    k, b, polys = code
    rows = _rows(pattern)
    t = vd.build_trellis(vd.CodeSpec(k, b, polys))
    p = vd.PuncturePattern.parse(rows)
    fc = vd.FrameConfig(*cfg)
    for n_stages in (cfg[0] * 40 + 7, 200_001, 1 << 20):
        punct, sent = _punctured_case(k, b, polys, rows, n_stages, seed=n_stages + cfg[0])
        full, n = oracle.depuncture_i8(rows, punct)
        exp, st, _ = oracle.port().framed_decode(k, b, polys, full, n, fc.f, fc.v1, fc.v2)
        dev_in = torch.from_numpy(punct.copy()).cuda()
        res = {}
        for fused in ("1", "0"):
            monkeypatch.setenv("VITDEC_PUNCT_FUSED", fused)
            scratch = torch.empty(n * b, dtype=torch.int8, device="cuda")
            out = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")  # stale bits must be cleared
            s = vd.api.VdStats()
            c, pc = fc.to_c(), p.to_c()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                vd.api.check(vd.lib().vd_decode_punctured_i8_device(t.handle, C.byref(c), C.byref(pc),
                                                                    dev_in.data_ptr(), punct.size, scratch.data_ptr(),
                                                                    out.data_ptr(), C.byref(s), -1, None))
                torch.cuda.synchronize()
            if n_stages == 1 << 20:
                ran = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
                # (odd f or v1: the fast kernel needs 4-byte aligned frame windows, plan())
                takes_fused = fused == "1" and cfg[0] % 2 == 0 and cfg[1] % 2 == 0 and k == 7
                assert any("Punct<" in x for x in ran) == takes_fused, (fused, ran)
            res[fused] = vd.unpack_bits(out.cpu().numpy().view(np.uint32), n)
            assert (s.frames, s.stages, s.tracebacks) == st
        bad = np.flatnonzero(res["1"] != exp)
        assert bad.size == 0, (pattern, cfg, n_stages, bad[:10], bad.size)
        assert np.array_equal(res["0"], exp)

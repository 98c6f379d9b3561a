"""Pin the CPU oracle (oracle/vd_oracle.c) before trusting it.

1. The reference's own known-answer tests for the decode path, restated
   (reference proj/tests/test_decoder.cpp, test_trellis.cpp, test_codec.cpp).
2. Golden vectors produced by running the reference itself
   (tests/golden/make_golden.py over oracle/_ref/libvitdec_ref.so).
3. When the reference library is present (build container), random
   cross-checks of oracle vs reference.
"""
import itertools

import numpy as np
import pytest

import oracle
from conftest import unpack

K7 = (7, 2, [0o171, 0o133])


@pytest.fixture(scope="module")
def port():
    return oracle.port()


def ml_decode(llr_stream, n, k, b, polys):
    """Brute force over all 2^n messages x 2^(K-1) start states
    (reference tests/oracle.hpp:50-67)."""
    best, best_m = None, None
    llr = np.asarray(llr_stream).reshape(n, b)
    for start in range(1 << (k - 1)):
        for msg in range(1 << n):
            reg = start << 1
            m = 0.0
            bits = []
            for t in range(n):
                u = (msg >> t) & 1
                bits.append(u)
                reg = (reg >> 1) | (u << (k - 1))
                for i in range(b):
                    c = bin(polys[i] & reg).count("1") & 1
                    m += -llr[t, i] if c else llr[t, i]
            if best is None or m > best_m:
                best, best_m = bits, m
    return np.array(best, np.uint8)


# ---- reference KATs --------------------------------------------------------

def test_trellis_75_all_branches(port):
    # test_trellis.cpp:30-44
    nxt, out, pred, io, cp = port.trellis(3, 2, [7, 5])
    table = [(0, 0, 0, 0b00), (0, 1, 2, 0b11), (1, 0, 0, 0b11), (1, 1, 2, 0b00),
             (2, 0, 1, 0b10), (2, 1, 3, 0b01), (3, 0, 1, 0b01), (3, 1, 3, 0b10)]
    for s, u, n, bo in table:
        assert nxt[s * 2 + u] == n and out[s * 2 + u] == bo


def test_trellis_standard_and_k2(port):
    # test_trellis.cpp:11-28
    *_, cp = port.trellis(*K7)
    assert cp
    nxt, out, *_ = port.trellis(2, 2, [0b11, 0b01])
    assert nxt[0] == 0 and out[0] == 0


@pytest.mark.parametrize("k,b,polys,msg", [
    (1, 2, [1, 1], "constraint length must be >= 2"),
    (3, 1, [5], "need at least 2 outputs per bit"),
    (3, 2, [7, 0], "zero generator polynomial"),
    (3, 2, [7, 0x10], "generator polynomial wider than K bits"),
    (17, 2, [1, 1], "constraint length too large"),
])
def test_trellis_validation(port, k, b, polys, msg):
    # test_trellis.cpp:46-52, trellis.cpp:38-53
    with pytest.raises(ValueError, match=msg):
        port.trellis(k, b, polys)


def test_encoder_impulse(port):
    # test_codec.cpp:17-20: (7,5) impulse {1,0,0} -> 1,1,1,0,1,1
    bits = np.array([1, 0, 0], np.uint8)
    coded = np.zeros(6, np.uint8)
    o = oracle.oracle()
    o.check(o.fn("encode")(3, 2, oracle._polys([7, 5]), bits.ctypes.data, 3, coded.ctypes.data))
    assert coded.tolist() == [1, 1, 1, 0, 1, 1]


def test_stats_kat(port):
    # test_decoder.cpp:289-295
    llr = np.zeros(200, np.float64)
    _, stats, _ = port.framed_decode(*K7, llr, 100, 32, 8, 8, 16)
    assert stats[0] == 4 and stats[2] == 7


def test_exact_ties_take_second_predecessor(port):
    # test_decoder.cpp:81-89: all-zero metrics -> every ACS is a tie -> i2;
    # traceback from state 0 (lowest index on ties) walks 0,1,3,...,63,63,...
    n = 40
    bits = port.serial_decode(*K7, np.zeros(2 * n), n)
    expect = np.ones(n, np.uint8)
    expect[-6:] = 0
    assert np.array_equal(bits, expect)


def test_serial_matches_ml_oracle(port):
    # test_decoder.cpp:134-143
    rng = np.random.default_rng(37)
    for _ in range(12):
        n = int(rng.integers(4, 9))
        llr = rng.uniform(-2, 2, size=2 * n)
        assert np.array_equal(port.serial_decode(3, 2, [7, 5], llr, n), ml_decode(llr, n, 3, 2, [7, 5]))


def test_noiseless_roundtrip_and_single_flip(port):
    # test_decoder.cpp:122-132, 145-152
    for k, polys in [(3, [7, 5]), (5, [0o23, 0o35]), (7, [0o171, 0o133])]:
        rx, sent = port.gen_bench_block(k, 2, polys, 200, 300.0, 31)  # effectively noiseless
        assert np.array_equal(port.serial_decode(k, 2, polys, np.sign(rx), 200), sent)
    rx, sent = port.gen_bench_block(*K7, 64, 300.0, 41)
    llr = np.sign(rx)
    llr[30 * 2 + 1] *= -1
    assert np.array_equal(port.serial_decode(*K7, llr, 64), sent)


def test_framed_properties(port):
    rng = np.random.default_rng(53)
    # single frame == serial (test_decoder.cpp:222-232)
    for _ in range(5):
        n = int(rng.integers(50, 250))
        llr = rng.standard_normal(2 * n)
        a, _, _ = port.framed_decode(*K7, llr, n, n + 10)
        assert np.array_equal(a, port.serial_decode(*K7, llr, n))
    llr = rng.standard_normal(2000) * 1.5
    # f0 == f matches f0 == 0 (test_decoder.cpp:244-252)
    a, _, _ = port.framed_decode(*K7, llr, 1000, 128, 20, 40, 0)
    b, _, _ = port.framed_decode(*K7, llr, 1000, 128, 20, 40, 128)
    assert np.array_equal(a, b)
    # random start: seed-deterministic and seed-sensitive (test_decoder.cpp:263-273)
    a, _, _ = port.framed_decode(*K7, llr, 1000, 128, 20, 40, 32, 1, 5)
    b, _, _ = port.framed_decode(*K7, llr, 1000, 128, 20, 40, 32, 1, 5)
    c, _, _ = port.framed_decode(*K7, llr, 1000, 128, 20, 40, 32, 1, 6)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    # scaling invariance (test_decoder.cpp:275-287)
    base, _, _ = port.framed_decode(*K7, llr, 1000, 64, 16, 24, 16)
    for s in (0.1, 3.0, 1000.0):
        assert np.array_equal(port.framed_decode(*K7, llr * s, 1000, 64, 16, 24, 16)[0], base)


# ---- golden vectors from the reference --------------------------------------

def test_golden_framed_cases(port, golden):
    meta, arr = golden
    for c in meta["cases"]:
        cfg = c["cfg"]
        bits, stats, _ = port.framed_decode(c["k"], c["b"], c["polys"], arr[c["name"] + "_llr"], c["n"], cfg["f"],
                                            cfg["v1"], cfg["v2"], cfg["f0"], cfg["start"], cfg["seed"])
        assert np.array_equal(bits, unpack(arr[c["name"] + "_bits"], c["n"])), c["name"]
        assert list(stats) == c["stats"], c["name"]


def test_golden_serial_cases(port, golden):
    meta, arr = golden
    for c in meta["serial"]:
        bits = port.serial_decode(c["k"], c["b"], c["polys"], arr[c["name"] + "_llr"], c["n"])
        assert np.array_equal(bits, unpack(arr[c["name"] + "_bits"], c["n"])), c["name"]


def test_golden_data_chain(port, golden):
    _, arr = golden
    rx, sent = port.gen_bench_block(*K7, 2000, 3.0, 1)
    assert np.array_equal(rx, arr["chain_bench_rx"]) and np.array_equal(sent, arr["chain_bench_sent"])
    rx, sent = port.gen_sweep_block(7, 3, [0o133, 0o171, 0o165], 1500, 0.8, port.mix_seed(7, 0x100000 + 3))
    assert np.array_equal(rx, arr["chain_sweep_rx"]) and np.array_equal(sent, arr["chain_sweep_sent"])


def test_golden_trellis(port, golden):
    meta, arr = golden
    for code, (k, b, polys) in meta["codes"].items():
        nxt, out, pred, io, cp = port.trellis(k, b, polys)
        assert np.array_equal(np.stack([nxt, out, pred, io]), arr[f"trellis_{code}"])
        assert int(cp) == int(arr[f"trellis_{code}_cp"][0])


def test_golden_ber_sweep_counts(port, golden):
    """The oracle reproduces the reference run_ber_sweep error counts
    (berlab.cpp:42-99) through the same per-block recipe."""
    meta, _ = golden
    sw = meta["ber_sweeps"][0]
    f, v1, v2, f0, start, seed = sw["frame"]
    for p, ebn0 in enumerate(sw["ebn0"][1:], start=1):
        sigma = port.sigma_from_ebn0(ebn0, 0.5)
        errors = 0
        nblk = -(-sw["bits_per_point"] // sw["block_bits"])
        for blk in range(nblk):
            n = min(sw["block_bits"], sw["bits_per_point"] - blk * sw["block_bits"])
            rx, sent = port.gen_sweep_block(*K7, n, sigma, port.mix_seed(sw["seed"], p * 0x100000 + blk))
            bits, _, _ = port.framed_decode(*K7, rx, n, f, v1, v2, f0, start, seed)
            errors += int(np.count_nonzero(bits != sent))
        assert errors == sw["errors"][p]


# ---- cross-check against the reference library (build container only) --------

@pytest.mark.skipif(oracle.ref_backend() is None, reason="reference library not built here")
def test_random_cross_check_vs_reference(port):
    ref = oracle.ref_backend()
    rng = np.random.default_rng(99)
    codes = [(3, 2, [7, 5]), (7, 2, [0o171, 0o133]), (7, 3, [0o133, 0o171, 0o165]), (9, 2, [0o561, 0o753]),
             (3, 2, [3, 5]), (2, 2, [3, 1])]
    for (k, b, polys), it in itertools.product(codes, range(6)):
        n = int(rng.integers(1, 600))
        f = int(rng.integers(1, 200))
        cfg = (f, int(rng.integers(0, 50)), int(rng.integers(0, 50)), int(rng.integers(0, f + 1)),
               int(rng.integers(0, 2)), int(rng.integers(0, 2**62)))
        llr = rng.integers(-127, 128, n * b).astype(np.int8) if it % 2 else rng.standard_normal(n * b)
        a = port.framed_decode(k, b, polys, llr, n, *cfg)
        r = ref.framed_decode(k, b, polys, llr, n, *cfg, workers=2)
        assert np.array_equal(a[0], r[0]) and a[1] == r[1]

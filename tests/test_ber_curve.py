"""BASELINE config C2: K=7 r1/2 BER-vs-Eb/N0 curves (0-6 dB) over a sweep of
frame length f and convergence depth v2 (traceback depth 5K..10K), GPU vs the
CPU oracle.

* Exact: every BER point is built the way reference run_ber_sweep builds it
  (berlab.cpp:42-99: per-block seeds mix_seed(seed, p * 0x100000 + blk),
  random_bits -> encode -> BPSK -> AWGN, one framed_decode per block), the
  soft values quantised to int8 (scale 32); the GPU batched decode must make
  exactly the oracle's bit errors, point by point.
* Monte-Carlo: an independent large-sample GPU curve (device-side synthetic
  AWGN, 2^24 bits per point) must agree with the oracle's curve (reference
  data chain, 2^20 bits per point) within binomial tolerance.
"""
import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd

pytestmark = pytest.mark.gpu

K7 = (7, 2, [0o171, 0o133])
EBN0 = [0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0]
GRID = [(32, 35), (128, 49), (256, 42), (1024, 70)]  # (f, v2); v1 = 20
BLOCK_BITS, BLOCKS = 8192, 6
SEED = 2024


def _point_blocks(port, ebn0, p):
    sigma = port.sigma_from_ebn0(ebn0, 0.5)
    blocks, sents = [], []
    for blk in range(BLOCKS):
        rx, sent = port.gen_sweep_block(*K7, BLOCK_BITS, sigma, port.mix_seed(SEED, p * 0x100000 + blk))
        blocks.append(oracle.quantize(rx, 32.0))
        sents.append(sent)
    return blocks, sents


@pytest.mark.parametrize("f,v2", GRID)
def test_ber_curve_error_counts_match_oracle(f, v2):
    port = oracle.port()
    t = vd.build_trellis(vd.CodeSpec(*K7))
    cfg = vd.FrameConfig(f, 20, v2)
    prev = None
    for p, ebn0 in enumerate(EBN0):
        blocks, sents = _point_blocks(port, ebn0, p)
        got = vd.framed_decode_batch(blocks, t, cfg)
        e_gpu = sum(int(np.count_nonzero(b != s)) for (b, _), s in zip(got, sents))
        e_ora = 0
        for q, s in zip(blocks, sents):
            bits, _, _ = port.framed_decode(*K7, q, BLOCK_BITS, f, 20, v2)
            e_ora += int(np.count_nonzero(bits != s))
        assert e_gpu == e_ora, (f, v2, ebn0)
        if prev is not None and prev > 50:
            assert e_gpu <= prev, (f, v2, ebn0)  # BER falls with Eb/N0
        prev = e_gpu


MC_BLOCKS = 128  # oracle side: 128 x 8192 = 2^20 bits per point


def test_large_sample_curve_within_monte_carlo_tolerance():
    """GPU curve at 2^24 bits/point (device AWGN) vs the oracle's curve at
    2^20 bits/point (reference data chain, run_ber_sweep block recipe): |p1 -
    p2| within 4 sigma of the pooled binomial estimate (+ 3 % relative for
    the generators' differing float / double noise samples; both sides use
    the same int8 quantiser). Points where the oracle sees < 20 errors get a
    one-sided bound instead."""
    from concurrent.futures import ThreadPoolExecutor
    import os

    import torch

    port = oracle.port()
    t = vd.build_trellis(vd.CodeSpec(*K7))
    cfg = vd.FrameConfig(256, 20, 42)
    n = 1 << 24
    from paper_2011_09337_b200.device import count_bit_errors, decode_i8_device, synth_llr_i8

    llr = torch.empty(n * 2, dtype=torch.int8, device="cuda")
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    out = torch.empty((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for p, ebn0 in enumerate(EBN0[:5]):
        sigma = port.sigma_from_ebn0(ebn0, 0.5)
        synth_llr_i8(t, n, sigma, 32.0, 77 + p, llr, bits)
        decode_i8_device(t, cfg, n, llr, 0, 0, (n + 255) // 256, out, 0)
        cnt.zero_()
        count_bit_errors(out, bits, n, cnt)
        torch.cuda.synchronize()
        p_gpu = int(cnt.item()) / n
        sigma_p = port.sigma_from_ebn0(ebn0, 0.5)

        def one(blk):
            rx, sent = port.gen_sweep_block(*K7, BLOCK_BITS, sigma_p, port.mix_seed(SEED + 1, p * 0x100000 + blk))
            b, _, _ = port.framed_decode(*K7, oracle.quantize(rx, 32.0), BLOCK_BITS, 256, 20, 42)
            return int(np.count_nonzero(b != sent))

        with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
            e = sum(ex.map(one, range(MC_BLOCKS)))
        m = MC_BLOCKS * BLOCK_BITS
        p_ora = e / m
        if e < 20:  # too few oracle errors for a two-sample check: one-sided bound
            assert p_gpu < 30.0 / m, (ebn0, p_gpu, p_ora)
            continue
        pooled = (p_gpu * n + e) / (n + m)
        tol = 4.0 * np.sqrt(pooled * (1 - pooled) * (1.0 / n + 1.0 / m)) + 0.03 * pooled
        assert abs(p_gpu - p_ora) <= tol, (ebn0, p_gpu, p_ora, tol)

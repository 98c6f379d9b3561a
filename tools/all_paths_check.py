"""Small decodes through every kernel family, each checked bit-exactly
against the C oracle (one process, a few seconds; compute-sanitizer is not
available on the GPU pool, so this is the quick all-paths check):

    python tools/all_paths_check.py

Paths: fast kernel (K=7 / K=9 / B=3, TMEM + smem survivors, subframe
traceback), small-launch kernel (interior, head and clipped tail frames),
run-time (NVRTC) fast and small instantiations, fused depuncture, generic
warp-per-frame kernel (int8 and FP64 metrics), K=13 CTA-per-frame kernel,
exact segment-parallel serial decode, batched blocks.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402  (checker only)
import paper_2011_09337_b200 as vd  # noqa: E402


def main():
    port = oracle.port()
    fails = []

    def check(name, got, exp):
        ok = np.array_equal(got, exp)
        print(f"{name:48s} {'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            fails.append(name)

    def stream(k, b, polys, n, cfg, small, name, ebn0=2.5, scale=32.0, seed=1):
        os.environ["VITDEC_SMALL"] = small
        rx, _ = port.gen_bench_block(k, b, polys, n, ebn0, seed)
        q = oracle.quantize(rx, scale)
        exp, _, _ = port.framed_decode(k, b, polys, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        t = vd.build_trellis(vd.CodeSpec(k, b, polys))
        packed, _ = vd.framed_decode_stream(q, n, t, cfg)
        check(name, vd.unpack_bits(packed, n), exp)
        return q

    K7 = (7, 2, [0o171, 0o133])
    stream(*K7, 40_000, vd.FrameConfig(256, 20, 20), "0", "fast K=7 f=256/20/20")
    stream(*K7, 40_000, vd.FrameConfig(320, 20, 45, 32), "0", "fast K=7 subframes f0=32")
    stream(*K7, 40_000, vd.FrameConfig(1024, 42, 42), "0", "fast K=7 f=1024 (global spill tier)")
    stream(9, 2, [0o561, 0o753], 30_000, vd.FrameConfig(256, 20, 20), "0", "fast K=9")
    stream(7, 3, [0o133, 0o171, 0o165], 30_000, vd.FrameConfig(256, 20, 20), "0", "fast K=7 B=3")
    stream(*K7, 40_000 + 17, vd.FrameConfig(256, 20, 20), "1", "small K=7 (head + tail frames)")
    stream(*K7, 40_000, vd.FrameConfig(320, 20, 45, 32), "1", "small K=7 subframes")
    stream(7, 2, [0o165, 0o117], 30_000, vd.FrameConfig(256, 20, 20), "1", "small, run-time instantiation")
    stream(7, 2, [0o165, 0o117], 30_000, vd.FrameConfig(256, 20, 20), "0", "fast, run-time instantiation")
    stream(3, 2, [7, 5], 20_000, vd.FrameConfig(100, 13, 45, 32), "1", "generic K=3 int8")
    stream(13, 2, [0o16561, 0o11643], 3_000, vd.FrameConfig(256, 20, 20), "1", "K=13 CTA-per-frame")

    # FP64 metrics (real-valued LLRs)
    n = 8_000
    rx, _ = port.gen_bench_block(*K7, n, 2.0, 5)
    t = vd.build_trellis(vd.CodeSpec(*K7))
    exp, _, _ = port.framed_decode(*K7, rx, n, 256, 20, 20)
    got = vd.framed_decode(rx.reshape(n, 2).T.copy(), t, vd.FrameConfig(256, 20, 20))
    check("generic FP64 metrics", np.asarray(got.bits), exp)

    # serial decode (one frame over the block, segment-parallel)
    q = oracle.quantize(rx, 32.0)
    exp = port.serial_decode(*K7, q, n)
    got = vd.serial_decode(q.reshape(n, 2).T.copy().astype(np.float64), t)
    check("serial decode (segment-parallel)", np.asarray(got.bits), exp)

    # fused depuncture (r2/3 on K=7) vs oracle depuncture + decode
    n = 30_000
    rx, _ = port.gen_bench_block(*K7, n, 3.0, 9)
    q = oracle.quantize(rx, 32.0)
    pat = vd.PuncturePattern.named("r23")
    pq = oracle.puncture_i8("11;10", q, n)
    dq, nd = oracle.depuncture_i8("11;10", pq)
    exp, _, _ = port.framed_decode(*K7, dq, nd, 240, 24, 24)
    packed, nn, _ = vd.framed_decode_punctured(pq, pat, t, vd.FrameConfig(240, 24, 24))
    check("fused depuncture r2/3", vd.unpack_bits(packed, nn), exp)

    # batched blocks
    blocks, exps = [], []
    for i in range(3):
        m = 5_000 + 333 * i
        rx, _ = port.gen_bench_block(*K7, m, 2.0, 20 + i)
        qb = oracle.quantize(rx, 32.0)
        exps.append(port.framed_decode(*K7, qb, m, 256, 20, 20)[0])
        blocks.append(qb)
    outs = vd.framed_decode_batch(blocks, t, vd.FrameConfig(256, 20, 20))
    for i, ((bits, _), e) in enumerate(zip(outs, exps)):
        check(f"batched block {i}", np.asarray(bits), e)

    print("FAILED: " + ", ".join(fails) if fails else "all paths bit-exact")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

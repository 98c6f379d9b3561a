"""End-to-end host-buffer decode from PAGEABLE vs pinned numpy buffers
(framed_decode_stream -> vd_decode_i8; K=7 r1/2 f=256/20/20), wall-clock
Gbps per call, printed as one JSON line.

    python tools/bench_pageable.py [--stages 2^28] [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=0, help="chunk_stages (0: library default 2^24)")
    a = ap.parse_args()

    import numpy as np
    import torch

    import paper_2011_09337_b200 as vd

    t = vd.build_trellis(vd.CodeSpec(7, 2, [0o171, 0o133]))
    cfg = vd.FrameConfig(256, 20, 20)
    n = a.stages
    rng = np.random.default_rng(1)
    pageable = rng.integers(-127, 128, size=2 * n, dtype=np.int8)
    pinned_t = torch.empty(2 * n, dtype=torch.int8, pin_memory=True)
    pinned = pinned_t.numpy()
    pinned[:] = pageable
    res = {}
    ref = None
    for name, arr in (("pageable", pageable), ("pinned_in", pinned)):
        vd.framed_decode_stream(arr, n, t, cfg, chunk_stages=a.chunk)  # warm-up (staging buffers, pool)
        best = 0.0
        for _ in range(a.reps):
            t0 = time.perf_counter()
            out, _ = vd.framed_decode_stream(arr, n, t, cfg, chunk_stages=a.chunk)
            best = max(best, n / (time.perf_counter() - t0) / 1e9)
        if ref is None:
            ref = out
        assert np.array_equal(out, ref)
        res[name] = round(best, 2)
    print(json.dumps({"workload": f"K=7 r1/2 f=256/20/20, {n} stages, framed_decode_stream (vd_decode_i8)",
                      "chunk_stages": a.chunk or (1 << 24), "gbps_wall": res, "note": "output buffer is a pageable numpy array in both rows"}))


if __name__ == "__main__":
    main()

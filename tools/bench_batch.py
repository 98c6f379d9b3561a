"""Batched multi-block decode throughput on one B200 (the BER-sweep shape:
reference run_ber_sweep decodes blocks of block_bits independently,
berlab.cpp:63-88) vs the same stages as one stream.

    python tools/bench_batch.py [--block-bits 65536] [--blocks 16384] [--frame 256,20,20]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block-bits", type=int, default=65536)
    ap.add_argument("--blocks", type=int, default=16384)
    ap.add_argument("--frame", default="256,20,20")
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()

    import torch

    import paper_2011_09337_b200 as vd
    from paper_2011_09337_b200.device import decode_batch_i8_device, decode_i8_device, synth_llr_i8

    t = vd.build_trellis(vd.CodeSpec(7, 2, [0o171, 0o133]))
    f, v1, v2 = [int(x) for x in a.frame.split(",")]
    cfg = vd.FrameConfig(f, v1, v2)
    n = a.block_bits * a.blocks
    s = torch.cuda.Stream()
    llr = torch.empty(n * 2, dtype=torch.int8, device="cuda")
    synth_llr_i8(t, n, 0.7, 32.0, 5, llr, None, -1, s)
    out = torch.empty((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
    import numpy as np
    lens = np.full(a.blocks, a.block_bits, np.int64)

    def timed(fn):
        for _ in range(2):
            fn()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.steps):
            fn()
        e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1) / a.steps * 1e-3

    tb = timed(lambda: decode_batch_i8_device(t, cfg, lens, llr, out, -1, s))
    ts = timed(lambda: decode_i8_device(t, cfg, n, llr, 0, 0, (n + f - 1) // f, out, 0, None, -1, s))
    print(json.dumps({"block_bits": a.block_bits, "blocks": a.blocks, "frame": a.frame,
                      "batched_gbps": n / tb / 1e9, "one_stream_gbps": n / ts / 1e9,
                      "batched_ms": tb * 1e3, "one_stream_ms": ts * 1e3}))


if __name__ == "__main__":
    main()

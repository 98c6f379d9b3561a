"""serial_decode (one frame over the whole block, reference decoder.cpp:101-129)
on one B200: the exact segment-parallel int8 path vs the FP64 warp-per-frame
kernel, host buffers in and out (the drop-in call), K=7 r1/2.

    python tools/bench_serial.py
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np

    import paper_2011_09337_b200 as vd

    t = vd.build_trellis(vd.CodeSpec(7, 2, [0o171, 0o133]))
    for n in (65536, 1 << 20, 1 << 24):
        q = np.random.default_rng(1).integers(-60, 60, (2, n)).astype(np.int8)
        for _ in range(2):
            vd.serial_decode(q, t)
        t0 = time.perf_counter()
        vd.serial_decode(q, t)
        dt = time.perf_counter() - t0
        line = {"n": n, "int8_segment_parallel_mbps": n / dt / 1e6}
        if n <= 1 << 20:
            d = q.astype(np.float64) * 0.37
            vd.serial_decode(d, t)
            t0 = time.perf_counter()
            vd.serial_decode(d, t)
            line["f64_warp_per_frame_mbps"] = n / (time.perf_counter() - t0) / 1e6
        print(json.dumps(line))


if __name__ == "__main__":
    main()

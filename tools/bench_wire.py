"""End-to-end (pinned host buffers -> GPU -> packed bits on the host) decode
throughput with the int8 input (vd_decode_i8, 2 B per r1/2 stage over PCIe)
vs the 4-bit wire format (vd_decode_i4, 1 B per stage), K=7 r1/2 f=256/20/20.

    python tools/bench_wire.py [--stages N] [--reps R]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=1 << 30)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2011_09337_b200 as vd

    n = a.stages
    t = vd.build_trellis(vd.CodeSpec(7, 2, [0o171, 0o133]))
    cfg = vd.FrameConfig(256, 20, 20)
    rng = np.random.default_rng(1)
    q = rng.integers(-7, 8, n * 2, dtype=np.int8)
    h8 = torch.from_numpy(q).pin_memory()
    h4 = torch.from_numpy(vd.pack_i4(q)).pin_memory()
    o8 = torch.empty((n + 31) // 32, dtype=torch.int32).pin_memory()
    o4 = torch.empty((n + 31) // 32, dtype=torch.int32).pin_memory()
    lib = vd.lib()
    c = cfg.to_c()
    st = vd._lib.VdStats()

    def run(fn):
        fn()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            fn()
        return (time.perf_counter() - t0) / a.reps

    s8 = run(lambda: vd._lib.check(lib.vd_decode_i8(t.handle, C.byref(c), h8.data_ptr(), n, o8.data_ptr(),
                                                    C.byref(st), None)))
    s4 = run(lambda: vd._lib.check(lib.vd_decode_i4(t.handle, C.byref(c), h4.data_ptr(), n, o4.data_ptr(),
                                                    C.byref(st), None)))
    print(json.dumps({"stages": n, "e2e_gbps_int8": n / s8 / 1e9, "e2e_gbps_i4": n / s4 / 1e9,
                      "h2d_bytes_int8": 2 * n, "h2d_bytes_i4": n, "identical": bool(torch.equal(o8, o4))}))


if __name__ == "__main__":
    main()

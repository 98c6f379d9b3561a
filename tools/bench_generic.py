"""Throughput of the generic kernel paths on one B200 (device-resident):
FP64 metrics on real-valued LLRs (bit-exact to the reference on any input)
and int8 codes outside the fast kernel's compile-time list.

    python tools/bench_generic.py [--stages N]
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
    ap.add_argument("--stages", type=int, default=1 << 24)
    a = ap.parse_args()
    import torch

    import paper_2011_09337_b200 as vd
    from paper_2011_09337_b200.device import decode_f64_device, decode_i8_device

    n = a.stages
    cfg = vd.FrameConfig(256, 20, 20)
    out = torch.empty((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    for (k, b, polys), kind in [((7, 2, [0o171, 0o133]), "f64"), ((3, 2, [7, 5]), "i8"), ((5, 2, [0o27, 0o31]), "i8"),
                                ((7, 2, [0o171, 0o133]), "i8")]:
        t = vd.build_trellis(vd.CodeSpec(k, b, polys))
        nf = (n + 255) // 256
        if kind == "f64":
            llr = torch.randn(n * b, dtype=torch.float64, device="cuda")
            s = timed(lambda: decode_f64_device(t, cfg, n, llr, 0, 0, nf, out, 0))
        else:
            llr = torch.randint(-60, 60, (n * b,), dtype=torch.int8, device="cuda")
            s = timed(lambda: decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0))
        print(json.dumps({"code": f"K={k} B={b} {[oct(p) for p in polys]}", "llr": kind,
                          "kernel": "fast" if (kind == "i8" and t.fast_path()) else "generic",
                          "gbps": n / s / 1e9}))


if __name__ == "__main__":
    main()

"""Latency of the generic (warp-per-frame) kernel on ONE frame: device time of
vd_decode_i8_device over a single frame of a code the fast kernel does not
take, for several window lengths -> cycles per stage (the latency that edge
frames put on the critical path of small launches such as C1).

    python tools/probe_generic_latency.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2011_09337_b200 as vd  # noqa: E402
from paper_2011_09337_b200.device import decode_i8_device  # noqa: E402


def main():
    codes = {"K7 (170,133) generic": (7, 2, [0o170, 0o133]), "K5 (23,35) generic-only code": (5, 2, [0o22, 0o35])}
    mhz = 1965.0
    for name, (k, b, polys) in codes.items():
        t = vd.build_trellis(vd.CodeSpec(k, b, polys))
        for f, v1, v2, f0 in ((64, 20, 0, 0), (256, 20, 20, 0), (320, 20, 45, 32), (1024, 42, 42, 0)):
            cfg = vd.FrameConfig(f, v1, v2, f0)
            n = 4 * (f + v1 + v2)
            llr = torch.randint(-60, 60, (n * b,), dtype=torch.int8, device="cuda")
            out = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
            m = 1  # an interior frame: window f + v1 + v2
            for _ in range(3):
                decode_i8_device(t, cfg, n, llr, 0, m, m + 1, out, 0)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            reps = 20
            ev[0].record()
            for _ in range(reps):
                decode_i8_device(t, cfg, n, llr, 0, m, m + 1, out, 0)
            ev[1].record()
            torch.cuda.synchronize()
            us = ev[0].elapsed_time(ev[1]) / reps * 1e3
            L = f + v1 + v2
            print(json.dumps({"code": name, "cfg": [f, v1, v2, f0], "window": L, "us": round(us, 2),
                              "cycles_per_stage": round(us * mhz / L, 1), "fast_path": t.fast_path()}))


if __name__ == "__main__":
    main()

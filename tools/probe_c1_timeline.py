"""Device timeline of one small decode (C1: 1 M bits, K=7 r1/2) under the
torch profiler (CUPTI): every kernel / memset of the step with its start
offset and duration, to see what besides the decode kernel is on the critical
path of a latency-bound launch.

    python tools/probe_c1_timeline.py [--frame f,v1,v2[,f0]] [--stages N]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2011_09337_b200 as vd  # noqa: E402
from paper_2011_09337_b200.device import decode_i8_device, synth_llr_i8  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frame", default="256,20,20")
    ap.add_argument("--stages", type=int, default=1_000_000)
    a = ap.parse_args()
    vals = [int(x) for x in a.frame.split(",")]
    cfg = vd.FrameConfig(*vals)
    n = a.stages
    t = vd.build_trellis(vd.CodeSpec(7, 2, [0o171, 0o133]))
    llr = torch.empty(n * 2, dtype=torch.int8, device="cuda")
    synth_llr_i8(t, n, 0.7071, 32.0, 1, llr, None)
    nf = -(-n // cfg.f)
    out = torch.zeros(n // 32 + 2, dtype=torch.int32, device="cuda")
    for _ in range(5):
        decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0)
        torch.cuda.synchronize()
    import time

    reps = 200
    torch.cuda.synchronize()
    t_a = time.perf_counter()
    for _ in range(reps):
        decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0)
    t_b = time.perf_counter()
    torch.cuda.synchronize()
    t_c = time.perf_counter()
    print(f"host enqueue {1e6 * (t_b - t_a) / reps:.1f} us/call, wall {1e6 * (t_c - t_a) / reps:.1f} us/call")
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start if evs else 0
    for e in evs:
        print(f"{e.time_range.start - t0:9.1f} us  {e.time_range.elapsed_us():8.1f} us  {e.name[:90]}")


if __name__ == "__main__":
    main()

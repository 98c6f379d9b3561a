"""Host<->device copy ceiling on the bench box: pinned H2D / D2H bandwidth of
one large copy and of 64 MiB chunks on two streams (the e2e path's bound).

    python tools/pcie_probe.py   -> one JSON line (GB/s)
"""
from __future__ import annotations

import json

import torch


def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


def main():
    n = 2 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    chunk = 64 << 20
    s = [torch.cuda.Stream(), torch.cuda.Stream()]

    def chunked_h2d():
        for i, o in enumerate(range(0, n, chunk)):
            with torch.cuda.stream(s[i % 2]):
                d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
        for x in s:
            torch.cuda.current_stream().wait_stream(x)

    out = {
        "h2d_one_copy_GBps": bw(lambda: d.copy_(h, non_blocking=True), n),
        "d2h_one_copy_GBps": bw(lambda: h.copy_(d, non_blocking=True), n),
        "h2d_64MiB_chunks_2_streams_GBps": bw(chunked_h2d, n),
        "bytes": n,
    }
    print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in out.items()}))


if __name__ == "__main__":
    main()

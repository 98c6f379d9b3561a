"""Per-piece latency of one framed decode launch (GPU): head edge frames,
tail edge frames, interior (fast kernel) frames and the whole range, each
timed alone with CUDA events on the launching stream. Used to find where
small-stream latency goes; prints one line per piece.

    python -m paper_2011_09337_b200.microbench.latency_probe [--stages N]
"""
import argparse
import json

import torch

import paper_2011_09337_b200 as vd
from paper_2011_09337_b200 import device as dev


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=1 << 20)
    ap.add_argument("--k", type=int, default=7)
    ap.add_argument("--polys", default="171,133")
    ap.add_argument("--f", type=int, default=256)
    ap.add_argument("--v", type=int, default=20)
    a = ap.parse_args()
    n = a.stages
    tr = vd.build_trellis(vd.CodeSpec.from_octal(a.k, a.polys))
    cfg = vd.FrameConfig(a.f, a.v, a.v, 0, vd.TracebackStart.kStoredMax, 0)
    b = tr.outputs_per_bit()
    llr = torch.empty(n * b, dtype=torch.int8, device="cuda")
    dev.synth_llr_i8(tr, n, 0.7, 32.0, 5, llr, stream=torch.cuda.current_stream())
    out = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    nf = (n + a.f - 1) // a.f
    st = torch.cuda.current_stream()
    pieces = {
        "all": (0, nf),
        "head1": (0, 1),
        "tail1": (nf - 1, nf),
        "interior": (1, nf - 1),
        "one_interior": (nf // 2, nf // 2 + 1),
        "64_interior": (nf // 2, nf // 2 + 64),
    }
    res = {}
    # effective SM clock of a 1-CTA launch: torch.cuda._sleep spins N cycles
    res["sleep_1M_cycles"] = timed(lambda: torch.cuda._sleep(1_000_000))
    for name, (fb, fe) in pieces.items():
        res[name] = timed(lambda: dev.decode_i8_device(tr, cfg, n, llr, 0, fb, fe, out, 0, stream=st))
    llrd = llr.to(torch.float64)
    res["f64_one_interior"] = timed(lambda: dev.decode_f64_device(tr, cfg, n, llrd, 0, nf // 2, nf // 2 + 1, out, 0,
                                                                 stream=st))
    res["f64_all"] = timed(lambda: dev.decode_f64_device(tr, cfg, n, llrd, 0, 0, nf, out, 0, stream=st), reps=3)
    print(json.dumps({"stages": n, "k": a.k, "us": {k: round(v, 1) for k, v in res.items()}}))


if __name__ == "__main__":
    main()

"""Punctured decode on one B200: device depuncture kernel (HBM roofline),
depuncture + framed decode from HBM, and the host-buffer e2e call
(vd_decode_punctured_i8: only punctured bytes cross PCIe) vs the
unpunctured e2e call.

    python tools/bench_puncture.py [--stages N] [--patterns r23,r34] [--steps K]

Prints one JSON line per pattern. Inputs: device-synthesised int8 LLRs
(K=7 171/133, 3 dB, scale 32), punctured on the host by the oracle's
restatement of reference puncture (codec.cpp:88-103) — data setup only.
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
    ap.add_argument("--patterns", default="r23,r34")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e-stages", type=int, default=1 << 28)
    ap.add_argument("--k", type=int, default=7)
    ap.add_argument("--polys", default="171,133", help="octal generators of the rate-1/2 mother code")
    ap.add_argument("--frame", default="240,24,24", help="f,v1,v2 (multiples of the periods 2 and 3)")
    a = ap.parse_args()

    import numpy as np
    import torch

    import oracle
    import paper_2011_09337_b200 as vd
    from paper_2011_09337_b200.device import (decode_i8_device, decode_punctured_i8_device, depuncture_i8_device,
                                              synth_llr_i8)

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {
        "hbm_gbs": 6650.0}
    t = vd.build_trellis(vd.CodeSpec(a.k, 2, [int(x, 8) for x in a.polys.split(",")]))
    cfg = vd.FrameConfig(*[int(x) for x in a.frame.split(",")])  # multiples of the periods 2 and 3 (decoder.cpp:14-19)
    n = a.stages
    s = torch.cuda.Stream()
    full = torch.empty(n * 2, dtype=torch.int8, device="cuda")
    synth_llr_i8(t, n, (1.0 / (2 * 0.5 * 10 ** 0.3)) ** 0.5, 32.0, 99, full, None, -1, s)
    s.synchronize()
    full_h = full.cpu().numpy()
    out = torch.empty((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
    nf = (n + cfg.f - 1) // cfg.f

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.steps):
            fn()
        e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1) / a.steps * 1e-3

    base_s = timed(lambda: decode_i8_device(t, cfg, n, full, 0, 0, nf, out, 0, None, -1, s))
    ref_out = out.clone()
    # unpunctured e2e (pinned host buffers)
    ne = min(a.e2e_stages, n)
    lib = vd.lib()
    c = cfg.to_c()
    host_full = torch.from_numpy(full_h[: ne * 2]).pin_memory()
    host_out = torch.empty((ne + 31) // 32, dtype=torch.int32).pin_memory()
    st = vd._lib.VdStats()

    def e2e(fn, reps=3):
        fn()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return (time.perf_counter() - t0) / reps

    e2e_full = e2e(lambda: vd._lib.check(lib.vd_decode_i8(t.handle, C.byref(c), host_full.data_ptr(), ne,
                                                          host_out.data_ptr(), C.byref(st), None)))
    for name in a.patterns.split(","):
        p = vd.PuncturePattern.named(name)
        rows = {"r23": "11;10", "r34": "110;101"}.get(name, name)
        punct_h = oracle.puncture_i8(rows, full_h, n)
        punct = torch.from_numpy(punct_h).cuda()
        scratch = torch.empty(n * 2, dtype=torch.int8, device="cuda")
        dep_s = timed(lambda: depuncture_i8_device(p, punct, punct_h.size, scratch, -1, s))
        # correctness: the depunctured block (the separate pass's output, read
        # before the fused run rewrites the scratch with its edge windows) equals
        # the oracle's on a sampled prefix
        want, _ = oracle.depuncture_i8(rows, punct_h[: min(punct_h.size, 1 << 24) // p.kept_per_period()
                                                     * p.kept_per_period()])
        ok_dep = bool(np.array_equal(scratch[: want.size].cpu().numpy(), want))
        import os

        os.environ["VITDEC_PUNCT_FUSED"] = "0"  # A/B: separate depuncture pass + decode
        dec_s = timed(lambda: decode_punctured_i8_device(t, cfg, p, punct, punct_h.size, scratch, out, -1, s))
        sep_out = out.clone()
        os.environ["VITDEC_PUNCT_FUSED"] = "1"  # depuncture fused into the fast kernel's LLR staging (default)
        fused_s = timed(lambda: decode_punctured_i8_device(t, cfg, p, punct, punct_h.size, scratch, out, -1, s))
        fused_same = bool(torch.equal(out[: n // 32], sep_out[: n // 32]))
        os.environ.pop("VITDEC_PUNCT_FUSED")
        # e2e host-buffer punctured call on the first ne stages
        pe = oracle.puncture_i8(rows, full_h[: ne * 2], ne)
        host_p = torch.from_numpy(pe).pin_memory()
        pc = p.to_c()
        e2e_p = e2e(lambda: vd._lib.check(lib.vd_decode_punctured_i8(t.handle, C.byref(c), C.byref(pc),
                                                                     host_p.data_ptr(), pe.size,
                                                                     host_out.data_ptr(), C.byref(st), None)))
        dep_bytes = punct_h.size + n * 2
        print(json.dumps({
            "pattern": name, "stages": n, "code": f"K={a.k} ({a.polys})", "cfg": f"f,v1,v2={a.frame} (period-aligned)",
            "depuncture": {"ms": dep_s * 1e3, "GBps": dep_bytes / dep_s / 1e9, "hbm_peak": peaks["hbm_gbs"],
                           "frac": dep_bytes / dep_s / 1e9 / peaks["hbm_gbs"], "bytes": dep_bytes,
                           "matches_oracle": ok_dep},
            "device_gbps": {"unpunctured_decode": n / base_s / 1e9, "depuncture_plus_decode": n / dec_s / 1e9,
                            "depuncture_share": dep_s / dec_s, "fused_depuncture_decode": n / fused_s / 1e9,
                            "fused_vs_separate": dec_s / fused_s, "fused_matches_separate": fused_same},
            "e2e_gbps": {"unpunctured": ne / e2e_full / 1e9, "punctured": ne / e2e_p / 1e9,
                         "h2d_bytes_punctured": int(pe.size), "h2d_bytes_unpunctured": ne * 2},
        }))
        del punct, scratch


if __name__ == "__main__":
    main()

"""BER-vs-Eb/N0 curves on one B200 (BASELINE config C2: K=7 r1/2, f / v2
sweep, 0-6 dB), printed as JSON lines.

    python tools/ber_curve.py [--bits 2^24] [--oracle-bits 98304]

Per (f, v2) and Eb/N0: GPU BER on --bits device-synthesised int8 LLRs
(scale 32) and, for reference, the CPU oracle's BER (the reference's data
chain and decoder restatement) on --oracle-bits bits built by the
run_ber_sweep recipe (berlab.cpp:42-99).
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
    ap.add_argument("--bits", type=int, default=1 << 24)
    ap.add_argument("--oracle-bits", type=int, default=6 * 8192)
    a = ap.parse_args()

    import numpy as np
    import torch

    import oracle
    import paper_2011_09337_b200 as vd
    from paper_2011_09337_b200.device import count_bit_errors, decode_i8_device, synth_llr_i8

    k7 = (7, 2, [0o171, 0o133])
    port = oracle.port()
    t = vd.build_trellis(vd.CodeSpec(*k7))
    n = a.bits
    llr = torch.empty(n * 2, dtype=torch.int8, device="cuda")
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    out = torch.empty((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for f, v2 in [(32, 35), (64, 42), (128, 49), (256, 42), (512, 63), (1024, 70)]:
        cfg = vd.FrameConfig(f, 20, v2)
        curve = []
        for p, ebn0 in enumerate([0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0]):
            sigma = port.sigma_from_ebn0(ebn0, 0.5)
            synth_llr_i8(t, n, sigma, 32.0, 1000 + p, llr, bits)
            decode_i8_device(t, cfg, n, llr, 0, 0, (n + f - 1) // f, out, 0)
            cnt.zero_()
            count_bit_errors(out, bits, n, cnt)
            torch.cuda.synchronize()
            e_gpu = int(cnt.item())
            e_ora, m = 0, 0
            blk = 8192
            for b in range(a.oracle_bits // blk):
                rx, sent = port.gen_sweep_block(*k7, blk, sigma, port.mix_seed(7, p * 0x100000 + b))
                dec, _, _ = port.framed_decode(*k7, oracle.quantize(rx, 32.0), blk, f, 20, v2)
                e_ora += int(np.count_nonzero(dec != sent))
                m += blk
            curve.append({"ebn0_db": ebn0, "gpu_bits": n, "gpu_errors": e_gpu, "gpu_ber": e_gpu / n,
                          "oracle_bits": m, "oracle_errors": e_ora, "oracle_ber": e_ora / max(m, 1)})
        print(json.dumps({"code": "K=7 (171,133) r1/2", "f": f, "v1": 20, "v2": v2, "int8_scale": 32,
                          "curve": curve}))


if __name__ == "__main__":
    main()

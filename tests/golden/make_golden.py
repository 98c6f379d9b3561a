"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Requires oracle/_ref/libvitdec_ref.so, i.e. the reference's own sources
(/root/reference/proj/src/*.cpp) compiled in place by ``make -C oracle ref``
— only possible in the build container. The fixtures are committed so the
GPU box (which has no /root/reference) can check the CUDA path and the C
oracle against the reference's outputs.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent

CODES = {
    "k3_75": (3, 2, [0o7, 0o5]),
    "k5_2335": (5, 2, [0o23, 0o35]),
    "k7_171133": (7, 2, [0o171, 0o133]),
    "k7_r13": (7, 3, [0o133, 0o171, 0o165]),
    "k9_561753": (9, 2, [0o561, 0o753]),
    "k2_31": (2, 2, [0o3, 0o1]),
    "k3_65_lsbfree": (3, 2, [0o6, 0o5]),   # not LSB-complement: generic 4-metric ACS
    "k3_35_msbfree": (3, 2, [0o3, 0o5]),   # complement_paired() == false
    "k4_r13": (4, 3, [0o13, 0o15, 0o17]),
    "k6_r14": (6, 4, [0o53, 0o75, 0o47, 0o71]),
}

# (name, code, n, cfg(f, v1, v2, f0, start, seed), input kind, ebn0/scale)
CASES = [
    ("c1_serialtb", "k7_171133", 4096, (256, 20, 20, 0, 0, 0), "q32", 3.0),
    ("c1_paralleltb", "k7_171133", 4096, (320, 20, 45, 32, 0, 0), "q32", 3.0),
    ("c1_random", "k7_171133", 3000, (128, 20, 40, 32, 1, 5), "q32", 2.0),
    ("c1_random_seed6", "k7_171133", 3000, (128, 20, 40, 32, 1, 6), "q32", 2.0),
    ("ties_q4", "k7_171133", 2048, (64, 20, 24, 16, 0, 0), "q4", 1.0),
    ("f_ge_n", "k7_171133", 700, (1000, 0, 0, 0, 0, 0), "q32", 2.5),
    ("v1_gt_f", "k7_171133", 1500, (16, 40, 30, 0, 0, 0), "q32", 2.5),
    ("f0_not_div_f", "k7_171133", 1777, (100, 13, 27, 30, 0, 0), "q32", 2.5),
    ("f0_eq_f", "k7_171133", 1000, (128, 20, 40, 128, 0, 0), "q32", 1.5),
    ("f1", "k7_171133", 300, (1, 3, 5, 0, 0, 0), "q32", 2.0),
    ("f0_1", "k7_171133", 500, (20, 5, 7, 1, 0, 0), "q32", 2.0),
    ("no_overlap", "k7_171133", 999, (37, 0, 0, 0, 0, 0), "q32", 3.0),
    ("n1", "k7_171133", 1, (256, 20, 20, 0, 0, 0), "q32", 3.0),
    ("n2", "k5_2335", 2, (1, 1, 1, 1, 0, 0), "q32", 3.0),
    ("n3_random", "k5_2335", 3, (2, 1, 1, 1, 1, 9), "q32", 3.0),
    ("r13", "k7_r13", 3000, (256, 20, 20, 0, 0, 0), "q32", 2.0),
    ("r13_ptb", "k7_r13", 3000, (128, 16, 42, 32, 0, 0), "q32", 1.5),
    ("k9", "k9_561753", 3000, (256, 20, 20, 0, 0, 0), "q32", 2.5),
    ("k9_ptb", "k9_561753", 3000, (320, 20, 45, 32, 0, 0), "q32", 2.0),
    ("k9_random", "k9_561753", 2000, (128, 10, 50, 40, 1, 77), "q32", 1.5),
    ("k3", "k3_75", 2000, (64, 8, 16, 0, 0, 0), "q32", 2.0),
    ("k2", "k2_31", 1000, (32, 4, 8, 8, 0, 0), "q32", 2.0),
    ("k3_lsbfree", "k3_65_lsbfree", 1500, (64, 8, 16, 16, 0, 0), "q32", 2.0),
    ("k3_msbfree", "k3_35_msbfree", 1500, (64, 8, 16, 0, 0, 0), "q32", 2.0),
    ("k4_r13", "k4_r13", 1200, (50, 10, 10, 25, 0, 0), "q32", 2.0),
    ("k6_r14", "k6_r14", 1200, (64, 12, 12, 0, 0, 0), "q32", 1.0),
    ("k5", "k5_2335", 2500, (100, 15, 25, 20, 1, 3), "q32", 2.0),
    # real-valued LLRs: the FP64-metric kernel must match bit for bit
    ("f64_c1", "k7_171133", 3000, (256, 20, 20, 0, 0, 0), "f64", 2.0),
    ("f64_ptb", "k7_171133", 3000, (320, 20, 45, 32, 0, 0), "f64", 1.5),
    ("f64_random", "k7_171133", 2000, (128, 20, 40, 32, 1, 11), "f64", 1.0),
    ("f64_k9", "k9_561753", 1500, (128, 20, 30, 0, 0, 0), "f64", 1.5),
    ("f64_r13", "k7_r13", 1500, (128, 20, 30, 64, 0, 0), "f64", 1.0),
    ("f64_k3", "k3_75", 1000, (1000, 0, 0, 0, 0, 0), "f64", 0.5),
]


def main() -> None:
    ref = oracle.ref_backend()
    if ref is None:
        raise SystemExit("oracle/_ref/libvitdec_ref.so not built (make -C oracle ref)")
    arrays = {}
    meta = []
    for i, (name, code, n, cfg, kind, param) in enumerate(CASES):
        k, b, polys = CODES[code]
        rx, sent = ref.gen_bench_block(k, b, polys, n, param if kind != "q4" else param, 1000 + i)
        if kind == "q32":
            llr = oracle.quantize(rx, 32.0)
        elif kind == "q4":
            llr = oracle.quantize(rx, 4.0)
        else:
            llr = rx
        f, v1, v2, f0, start, seed = cfg
        bits, stats, _ = ref.framed_decode(k, b, polys, llr, n, f, v1, v2, f0, start, seed, workers=2)
        arrays[f"{name}_llr"] = llr
        arrays[f"{name}_bits"] = np.packbits(bits, bitorder="little")
        arrays[f"{name}_sent"] = np.packbits(sent, bitorder="little")
        meta.append({"name": name, "code": code, "k": k, "b": b, "polys": polys, "n": n,
                     "cfg": {"f": f, "v1": v1, "v2": v2, "f0": f0, "start": start, "seed": seed},
                     "kind": kind, "stats": list(stats)})
    # serial_decode cases (reference decoder.cpp:101-129)
    serial = []
    for j, (code, n) in enumerate([("k7_171133", 2000), ("k3_75", 300), ("k9_561753", 800), ("k7_r13", 600)]):
        k, b, polys = CODES[code]
        rx, _ = ref.gen_bench_block(k, b, polys, n, 1.0, 5000 + j)
        name = f"serial_{code}"
        arrays[f"{name}_llr"] = rx
        arrays[f"{name}_bits"] = np.packbits(ref.serial_decode(k, b, polys, rx, n), bitorder="little")
        serial.append({"name": name, "code": code, "k": k, "b": b, "polys": polys, "n": n})
    # the data chain itself (pins the oracle's mt19937_64 + polar restatement)
    rx, sent = ref.gen_bench_block(7, 2, [0o171, 0o133], 2000, 3.0, 1)
    arrays["chain_bench_rx"] = rx
    arrays["chain_bench_sent"] = sent
    rx, sent = ref.gen_sweep_block(7, 3, [0o133, 0o171, 0o165], 1500, 0.8, ref.mix_seed(7, 0x100000 + 3))
    arrays["chain_sweep_rx"] = rx
    arrays["chain_sweep_sent"] = sent
    # trellis tables
    for code, (k, b, polys) in CODES.items():
        nxt, out, pred, io, cp = ref.trellis(k, b, polys)
        arrays[f"trellis_{code}"] = np.stack([nxt, out, pred, io])
        arrays[f"trellis_{code}_cp"] = np.array([int(cp)])
    np.savez_compressed(OUT / "reference_vectors.npz", **arrays)

    # BER sweep counts of the reference harness itself (run_ber_sweep,
    # berlab.cpp:42-99): the GPU sweep must reproduce these error counts.
    sweeps = []
    for frame in [(256, 20, 20, 0, 0, 0), (320, 20, 45, 32, 0, 0), None]:
        ebn0 = [1.0, 2.0, 3.0]
        e = np.zeros(3, np.int64)
        bcount = np.zeros(3, np.int64)
        r = oracle.reference()
        fr = frame or (0, 0, 0, 0, 0, 0)
        eb = (oracle.C.c_double * 3)(*ebn0)
        polys = (oracle.C.c_uint32 * 2)(0o171, 0o133)
        r.check(r.fn("ber_sweep")(7, 2, polys, b"r12", fr[0], fr[1], fr[2], fr[3], fr[4], fr[5], 0, eb, 3,
                                  200000, 65536, 7, 4, e.ctypes.data, bcount.ctypes.data))
        sweeps.append({"frame": frame, "ebn0": ebn0, "bits_per_point": 200000, "block_bits": 65536, "seed": 7,
                       "errors": e.tolist(), "bits": bcount.tolist()})
    (OUT / "reference_vectors.json").write_text(json.dumps({"cases": meta, "serial": serial, "codes": CODES,
                                                            "ber_sweeps": sweeps}, indent=1))
    print(f"wrote {len(meta)} framed cases, {len(serial)} serial cases, {len(sweeps)} BER sweeps")


if __name__ == "__main__":
    main()

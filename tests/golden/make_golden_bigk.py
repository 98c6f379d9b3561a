"""Golden fixtures for large constraint lengths (K = 13 .. 16), produced by
the REFERENCE (oracle/_ref/libvitdec_ref.so, the reference's own sources
compiled in place; reference trellis.cpp:44 accepts K <= 16).

    python tests/golden/make_golden_bigk.py   ->  tests/golden/bigk_vectors.{json,npz}

Cases cover int8-valued and real-valued LLRs, serial traceback, stored-max
parallel traceback, random start and f >= N, at sizes the reference decodes
in seconds (its ACS costs ~9 ns per state-stage).
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
    "k13": (13, 2, [0o15627, 0o12345]),
    "k14_r13": (14, 3, [0o23457, 0o31651, 0o27133]),
    "k15": (15, 2, [0o46513, 0o63251]),
    "k16": (16, 2, [0o123457, 0o164355]),
}
# (name, code, n, cfg(f, v1, v2, f0, start, seed), kind)
CASES = [
    ("k13_serialtb", "k13", 1500, (256, 20, 40, 0, 0, 0), "q32"),
    ("k13_ptb_real", "k13", 900, (200, 30, 60, 50, 0, 0), "real"),
    ("k14_r13", "k14_r13", 800, (256, 24, 48, 0, 0, 0), "q32"),
    ("k14_random", "k14_r13", 700, (160, 20, 40, 40, 1, 11), "q32"),
    ("k15_fgen", "k15", 400, (1000, 0, 0, 0, 0, 0), "q4"),
    ("k16_framed", "k16", 600, (256, 20, 60, 0, 0, 0), "q32"),
    ("k16_ptb", "k16", 500, (200, 16, 48, 40, 0, 0), "real"),
]


def main():
    ref = oracle.ref_backend()
    if ref is None:
        raise SystemExit("reference library not built: make -C oracle ref")
    rng = np.random.default_rng(2026)
    meta = {"codes": {k: [v[0], v[1], v[2]] for k, v in CODES.items()}, "cases": []}
    arrays = {}
    for name, code, n, cfg, kind in CASES:
        k, b, polys = CODES[code]
        if kind == "real":
            llr = rng.standard_normal(n * b) * 2.0 + np.repeat(rng.choice([-1.0, 1.0], n), b)
        else:
            scale = 32.0 if kind == "q32" else 4.0
            y = np.repeat(rng.choice([-1.0, 1.0], n), b) + rng.standard_normal(n * b) * 0.8
            llr = np.clip(np.rint(y * scale), -127, 127).astype(np.int8)
        bits, stats, _ = ref.framed_decode(k, b, polys, llr, n, *cfg, workers=4)
        arrays[name + "_llr"] = llr
        arrays[name + "_bits"] = np.packbits(bits, bitorder="little")
        meta["cases"].append({"name": name, "k": k, "b": b, "polys": polys, "n": n,
                              "cfg": dict(zip(["f", "v1", "v2", "f0", "start", "seed"], cfg)),
                              "kind": kind, "stats": list(stats)})
        print(name, stats)
    (OUT / "bigk_vectors.json").write_text(json.dumps(meta, indent=1))
    np.savez_compressed(OUT / "bigk_vectors.npz", **arrays)


if __name__ == "__main__":
    main()

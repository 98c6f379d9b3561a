"""Run the integer-pipe microbenchmarks (alu_peak.cu) on the current GPU.

Writes profiles/alu_peak.json: per-op warp-instructions per SM clock, the SM
clock seen by the kernels, and the packed-ACS lane-op peak used as the ALU
roofline denominator by bench.py:

    tops = (lane-ops per SM clock of the VIADD.16x2 + VIADDMNMX mix) x SMs x clock

Usage: python paper_2011_09337_b200/microbench/run_alu_peak.py
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
NAMES = ["VIADD.16x2", "VIMNMX.S16x2", "VIADD.16x2+VIADDMNMX (ACS mix)", "IADD3", "IMAD", "PRMT", "LOP3",
         "VIADD.16x2+IMAD", "VIMNMX+IMAD", "SHFL.BFLY(+IADD)", "VIMNMX(pred)+SEL",
         "ACS pair VIADD.16x2+VIADDMNMX (1:1, the fast kernel's)"]
ACS = NAMES[11]


def main(out=ROOT / "profiles" / "alu_peak.json"):
    lib = C.CDLL(str(ROOT / "paper_2011_09337_b200" / "libvd_microbench.so"))
    lib.vdmb_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_double)]
    lib.vdmb_instr_per_iter.argtypes = [C.c_int]
    sms = lib.vdmb_sm_count()
    blocks, threads, iters = sms * 8, 256, 40000
    res = {}
    for op, name in enumerate(NAMES):
        ms, cyc = C.c_float(), C.c_double()
        st = lib.vdmb_run(op, blocks, threads, iters, C.byref(ms), C.byref(cyc))
        if st != 0:
            raise SystemExit(f"op {op} failed: {st}")
        warps = blocks * threads // 32
        instr = warps * iters * lib.vdmb_instr_per_iter(op)  # warp-instructions of the measured kind
        per_sm_clk = instr / (sms * cyc.value)
        mhz = cyc.value / (ms.value * 1e3)
        res[name] = {"warp_instr_per_sm_clk": per_sm_clk, "ms": ms.value, "sm_mhz_seen": mhz}
        print(f"{name:34s} {per_sm_clk:6.3f} warp-instr/SM/clk   ({ms.value:.2f} ms, {mhz:.0f} MHz)")
    acs = res[ACS]
    # the packed ACS pair makes one new register (2 frames x 1 state, 2 adds +
    # 1 compare-select each = 6 lane-ops) per 2 instructions: 3 lane-ops per
    # warp-lane instruction
    lane_ops_per_clk = acs["warp_instr_per_sm_clk"] * 32 * 3
    tops_seen = lane_ops_per_clk * sms * acs["sm_mhz_seen"] * 1e6 / 1e12
    dual = 4 * 32 * 3  # 1 warp-instr / clk / SMSP with the fmaheavy and alu pipes each at 0.5
    summary = {
        "source": "microbenchmark paper_2011_09337_b200/microbench/alu_peak.cu op 11 (the fast kernel's "
                  "VIADD.16x2 -> VIADDMNMX.S16x2 ACS pair), run by run_alu_peak.py on the bench box",
        "acs_warp_instr_per_sm_clk": acs["warp_instr_per_sm_clk"],
        "lane_ops_per_sm_clk": lane_ops_per_clk,
        "dual_issue_lane_ops_per_sm_clk": dual,
        "sms": sms,
        "sm_mhz_seen": acs["sm_mhz_seen"],
        "tops": tops_seen,
        "tops_at_1965mhz": lane_ops_per_clk * sms * 1965e6 / 1e12,
        "dual_issue_tops_at_1965mhz": dual * sms * 1965e6 / 1e12,
        "ops": res,
    }
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: v for k, v in summary.items() if k != "ops"}))


if __name__ == "__main__":
    main(Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "alu_peak.json")

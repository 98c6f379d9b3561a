"""Measure the decode kernel's DRAM traffic per decoded bit with ncu and write
profiles/decode_traffic.json (read by bench.py for roofline.traffic).

Run on the GPU box (one GPU; ncu replays the kernel):
    python tools/ncu_traffic.py [C5 C3 C4 ...]

For each workload: one bench.py process at 2^30 stages (C1: its own size)
under ncu, the first decode-kernel launch (fast_kernel; C1: small_kernel) after the warm-up captured with
dram__bytes_read.sum + dram__bytes_write.sum; bytes_per_bit = (read + write)
/ stages. The per-bit figure is size-independent (the kernel streams the
LLRs once): the algorithmic figure is B + 1/8 bytes per bit.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SIZES = {"C5": 1 << 30, "C1": 1_000_000, "C3": 1 << 26, "C4": 1 << 28, "U3": 1 << 28}


def measure(workload: str) -> dict:
    stages = SIZES[workload]
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "-k", "regex:(fast|small)_kernel", "--launch-skip", "1", "-c", "1", "--csv", "--clock-control", "none",
           sys.executable, str(ROOT / "bench.py"), "--workload", workload, "--stages", str(stages), "--steps", "1",
           "--warmup", "1", "--no-cpu", "--e2e-steps", "1", "--e2e-stages", "1048576"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    vals = {}
    kernel = None
    for row in csv.DictReader(io.StringIO("\n".join(rows))):
        kernel = row["Kernel Name"]
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
                 "ms": 1e-3, "s": 1.0}.get(unit, 1.0)
        vals[row["Metric Name"]] = v * scale
    if "dram__bytes_read.sum" not in vals:
        raise SystemExit(f"{workload}: ncu produced no metrics:\n{r.stdout[-2000:]}\n{r.stderr[-2000:]}")
    total = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    return {"stages": stages, "kernel": kernel, "dram_read_bytes": vals["dram__bytes_read.sum"],
            "dram_write_bytes": vals["dram__bytes_write.sum"], "launch_s": vals.get("gpu__time_duration.sum"),
            "bytes_per_bit": total / stages}


def main(workloads):
    import os

    out = Path(os.environ.get("VITDEC_TRAFFIC_OUT", ROOT / "profiles" / "decode_traffic.json"))
    head = os.environ.get("VITDEC_TREE") or subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True,
                                                           text=True, cwd=ROOT).stdout
    d = json.loads(out.read_text()) if out.exists() else {}
    d.setdefault("workloads", {})
    d.pop("bytes_per_bit", None)  # round-1 single-figure format
    for w in workloads:
        d["workloads"][w] = measure(w)
        print(w, json.dumps(d["workloads"][w]))
        out.write_text(json.dumps(d, indent=1))  # (each workload as it is measured)
    d["source"] = (f"tools/ncu_traffic.py (ncu dram__bytes_read.sum + dram__bytes_write.sum of one decode kernel "
                   f"launch: fast_kernel, C1 small_kernel), tree {head.strip() or '?'} (+ working changes), {time.strftime('%Y-%m-%d')}")
    out.write_text(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or ["C5"])

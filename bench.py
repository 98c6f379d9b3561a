"""Benchmark: decoded info Gbps, K=7 r1/2 soft-decision framed Viterbi on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (driver, N > 1)

Workload (BASELINE.json configs[4], "C5"): K=7 (171,133) rate 1/2, int8 LLRs
(scale 32, Eb/N0 3 dB, synthetic, generated in HBM), frames f=256, v1=v2=20,
serial traceback. A step decodes the rank's whole resident stream of
--stages stages (default 2^32 = 4 Gi info bits per GPU; weak scaling: each
rank owns its own stream, frames are independent, no collective on the data
path). Inputs (8 GiB) exceed L2, so no flush is needed between steps.

value: device-timed (CUDA events on the decode stream, max over ranks)
       whole-job info bits / s.
e2e:   the same metric through the reference-facing host call
       (vd_decode_i8: pinned host LLRs -> H2D -> kernel -> D2H packed bits,
       streamed in chunks), timed per step around the call.
roofline: the decode kernel against its binding roof (integer ALU; the HBM
       roof is reported alongside), see DESIGN.md §4.
cpu_baseline: the reference's own framed_decode (oracle/_ref, compiled from
       the reference sources) with all host threads, on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

K7 = (7, 2, [0o171, 0o133])
F, V1, V2 = 256, 20, 20
F0 = 0
SCALE = 32.0
EBN0 = 3.0

# BASELINE.json configs that fit one GPU. C5 (the default) is the headline;
# the others are measured with --workload for DESIGN.md (same metric).
WORKLOADS = {
    "C5": ((7, 2, [0o171, 0o133]), 1 << 32, "C5: K=7 r1/2 (171,133) framed decode, f=256 v1=20 v2=20 serial traceback"),
    "C1": ((7, 2, [0o171, 0o133]), 1_000_000, "C1: K=7 r1/2 (171,133), 1M info bits, f=256 v1=20 v2=20"),
    "C3": ((7, 3, [0o133, 0o171, 0o165]), 1 << 26, "C3: K=7 r1/3 (133,171,165), 64 Mi info bits, f=256 v1=20 v2=20"),
    "C4": ((9, 2, [0o561, 0o753]), 1 << 28, "C4: K=9 r1/2 (561,753), 256 Mi info bits, f=256 v1=20 v2=20"),
    "U3": ((9, 3, [0o557, 0o663, 0o711]), 1 << 28, "UMTS K=9 r1/3 (557,663,711), 256 Mi info bits, f=256 v1=20 v2=20"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="C5")
    ap.add_argument("--stages", type=int, default=0, help="info bits per rank per step (0: the workload's)")
    ap.add_argument("--e2e-stages", type=int, default=1 << 30, help="info bits per e2e step (host buffers)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=8.0, help="target wall time of the CPU baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--frame", default="", help="f,v1,v2[,f0] frame configuration override (default 256,20,20)")
    a = ap.parse_args()
    if a.frame:
        global F, V1, V2, F0
        vals = [int(x) for x in a.frame.split(",")]
        F, V1, V2 = vals[:3]
        F0 = vals[3] if len(vals) > 3 else 0
    a.code, default_n, a.workload_desc = WORKLOADS[a.workload]
    if a.stages <= 0:
        a.stages = default_n
    return a


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------- clocks ----

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU arms -----

def cpu_reference_rate(target_s: float, threads: int | None = None, code=K7):
    """The reference framed_decode (oracle/_ref, all host threads) or, if the
    reference library is absent, the single-threaded C oracle port. Returns
    (Gbps, cores, kind, sample description)."""
    import numpy as np

    import oracle

    port = oracle.port()
    ref = oracle.ref_backend()
    cores = threads or os.cpu_count() or 1
    kind = "reference" if ref is not None else "port"
    if ref is None:
        cores = 1
    backend = ref if ref is not None else port
    # probe on a small block, then size the sample for ~target_s of wall time
    n = 1 << 16
    rx, _ = port.gen_bench_block(*code, n, EBN0, 1)
    q = oracle.quantize(rx, SCALE)
    t0 = time.perf_counter()
    backend.framed_decode(*code, q, n, F, V1, V2, F0, workers=cores)
    rate = n / max(time.perf_counter() - t0, 1e-6)
    n = int(min(max(rate * target_s, 1 << 16), 1 << 26))
    rx, _ = port.gen_bench_block(*code, n, EBN0, 2)
    q = oracle.quantize(rx, SCALE)
    t0 = time.perf_counter()
    backend.framed_decode(*code, q, n, F, V1, V2, F0, workers=cores)
    dt = time.perf_counter() - t0
    sample = (f"{n} info bits (K={code[0]} B={code[1]}, int8 q=rint(32y) at {EBN0} dB, f={F}/v1={V1}/v2={V2}/f0={F0}), "
              f"{'reference framed_decode, workers=' + str(cores) if ref else 'C oracle port, 1 thread'}")
    return n / dt / 1e9, cores, kind, sample, dt


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per_step = []
    info = None
    for i in range(args.warmup + args.steps):
        info = cpu_reference_rate(min(args.cpu_seconds, 20.0) / 4)
        if i >= args.warmup:
            per_step.append(info)
    gbps = sorted(x[0] for x in per_step)[len(per_step) // 2]
    _, cores, kind, sample, dt = per_step[-1]
    line = {
        "metric": "decoded info Gbps (K=7 r1/2 soft)", "value": gbps, "unit": "Gbps", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference random_bits/encode/BPSK/AWGN chain, int8-quantised)",
        "config": {"workload": "K=7 r1/2 (171,133) framed f=256 v1=20 v2=20, CPU sample per step",
                   "sample": sample},
        "cpu_baseline": {"value": gbps, "unit": "Gbps", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": gbps, "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------ GPU arm ------

def alu_ops_per_bit(stats_stages: int, n: int, s: int = 64) -> float:
    """Algorithmic integer ops per decoded bit: 2 adds + 1 compare-select per
    state per processed stage."""
    return 3.0 * s * stats_stages / n


def run_ours(args):
    import numpy as np
    import torch

    import paper_2011_09337_b200 as vd
    from paper_2011_09337_b200.device import decode_i8_device, synth_llr_i8

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Plumbing test hook: VITDEC_BENCH_ONE_DEVICE=1 puts every rank on cuda:0
    # with the gloo backend (NCCL refuses two ranks on one GPU), so the N > 1
    # path (barriers, max-over-ranks timing, rank-0 reporting) can be exercised
    # on a one-GPU box. Numbers from such a run are not scaling measurements.
    one_dev = os.environ.get("VITDEC_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    red_dev = torch.device("cpu") if one_dev else dev  # gloo reduces CPU tensors

    t = vd.build_trellis(vd.CodeSpec(*args.code))
    B = args.code[1]
    cfg = vd.FrameConfig(F, V1, V2, F0)
    n = args.stages
    nf = (n + F - 1) // F
    stats = vd.frame_stats(cfg, n)
    stream = torch.cuda.Stream(device=dev)
    llr = torch.empty(n * B, dtype=torch.int8, device=dev)
    bits = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
    out = torch.empty((n + 31) // 32 + 1, dtype=torch.int32, device=dev)
    with torch.cuda.stream(stream):
        synth_llr_i8(t, n, (1.0 / (2 * (1.0 / B) * 10 ** (EBN0 / 10))) ** 0.5, SCALE, 1234 + rank, llr, bits, local, stream)
    stream.synchronize()

    def step():
        decode_i8_device(t, cfg, n, llr, 0, 0, nf, out, 0, None, local, stream)

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    # correctness guard on the timed data: decoded vs sent BER must be sane
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    vd.device.count_bit_errors(out, bits, n, cnt, local, stream)
    stream.synchronize()
    ber = int(cnt.item()) / n

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if dist:
        tt = torch.tensor([ms], device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    ms_step = ms / args.steps
    total_bits = n * world
    gbps = total_bits / (ms_step * 1e-3) / 1e9

    # ---- e2e through the host-buffer C-ABI call (pinned memory) -----------
    ne = min(args.e2e_stages, n)
    host_llr = torch.empty(ne * B, dtype=torch.int8, pin_memory=True)
    host_llr.copy_(llr[: ne * B])
    host_out = torch.empty((ne + 31) // 32, dtype=torch.int32, pin_memory=True)
    lib = vd.lib()
    c = cfg.to_c()
    dev_idx = C.c_int32(local)
    ex = vd._lib.VdExec(1, C.pointer(dev_idx), 0)
    st = vd._lib.VdStats()

    def e2e_step():
        vd._lib.check(lib.vd_decode_i8(t.handle, C.byref(c), host_llr.data_ptr(), ne, host_out.data_ptr(),
                                       C.byref(st), C.byref(ex)))

    e2e_step()
    if dist:
        dist.barrier()
    e2e_reps = max(args.e2e_steps, 1)
    t0 = time.perf_counter()
    for _ in range(e2e_reps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / e2e_reps
    if dist:
        tt = torch.tensor([e2e_s], device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_gbps = ne * world / e2e_s / 1e9
    # e2e result must equal the device-resident decode of the same prefix
    words = ne // 32
    same = bool(torch.equal(host_out[:words], out[:words].cpu()))

    # ---- roofline ----------------------------------------------------------
    # Binding roof: integer ALU. The packed ACS (VIADD.16x2 on the fmaheavy
    # pipe + VIADDMNMX.S16x2 on the alu pipe, each 0.5 warp-instr/clk/SMSP as
    # measured with ncu in profiles/r01_pipe_probe_ncu.csv) retires 2 states x
    # 3 ops per instruction pair: 4 SMSP x 32 lanes x 0.5 x 6 = 384 lane-ops
    # per SM clock. HBM roof reported alongside.
    peaks, peak_src = measured_peaks()
    clocks = clk.summary()
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = sms * 384 * sm_mhz * 1e6 / 1e12
    alu_src = (f"{sms} SM x 384 packed-ACS lane-ops/clk (ncu-measured pipe rates, profiles/r01_pipe_probe_ncu.csv) "
               f"x {sm_mhz:.0f} MHz (median SM clock during the timed region)")
    ops_bit = alu_ops_per_bit(stats.stages, n, 1 << (args.code[0] - 1))
    bits_per_s_kernel = n / (ms_step * 1e-3)
    alu_achieved = ops_bit * bits_per_s_kernel / 1e12
    hbm_bytes = n * B + n / 8  # int8 LLR read once + packed output
    hbm_achieved = hbm_bytes / (ms_step * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "decode_traffic.json"
    if tp.exists() and args.workload == "C5":
        traffic = json.loads(tp.read_text()).get("bytes_per_bit", 0) * n

    result = None
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            g, cores, kind, sample, _ = cpu_reference_rate(args.cpu_seconds, code=args.code)
            cpu = {"value": g, "unit": "Gbps", "cores": cores, "kind": kind, "sample": sample}
        result = {
            "metric": "decoded info Gbps (K=7 r1/2 soft)" if args.workload in ("C5", "C1") else
                      f"decoded info Gbps (K={args.code[0]} B={args.code[1]} soft)",
            "value": gbps,
            "unit": "Gbps",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "int8 LLR / int32 path metrics" if not t.fast_path() else "int8 LLR / int16x2 path metrics",
            "data": "synthetic: random message, K=7 encoder, BPSK+AWGN at 3 dB, int8 q=rint(32y), generated in HBM",
            "config": {
                "workload": args.workload_desc if not args.frame else
                            f"{args.workload_desc.split(',')[0]}, frame override f={F} v1={V1} v2={V2} f0={F0}",
                "info_bits_per_gpu_per_step": n,
                "frames_per_gpu": nf,
                "parallelism": f"frame shards x{world} (no collective)",
                "l2": (f"inputs ({B} B/bit x {n} bits = {n * B / 2**30:.2f} GiB) exceed L2; no flush needed"
                       if n * B > 256 << 20 else
                       f"inputs ({n * B / 2**20:.1f} MiB) fit in L2: steps re-read them warm (latency-bound size)"),
                "kernel": "fast (register-resident)" if t.fast_path() else "generic (warp per frame)",
                "ber_check": ber,
            },
            "roofline": {
                "bound": "alu",
                "achieved": alu_achieved,
                "peak": alu_peak,
                "unit": "Tops",
                "frac": alu_achieved / alu_peak,
                "traffic": traffic,
                "ops_per_bit": ops_bit,
                "peak_source": alu_src,
                "hbm": {"achieved": hbm_achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm_achieved / peaks["hbm_gbs"], "bytes_per_bit": hbm_bytes / n,
                        "peak_source": peak_src},
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_gbps, "unit": "Gbps", "h2d_bytes_per_step": ne * B,
                    "d2h_bytes_per_step": ((ne + 31) // 32) * 4, "info_bits_per_step": ne,
                    "matches_device_decode": same},
            "gpu_launches": 3 * args.steps,  # per step: head/tail edge frames (generic) + fast kernel
            "clocks": clocks,
        }
        print(json.dumps(result))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return result


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

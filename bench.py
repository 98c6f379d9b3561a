"""Benchmark: decoded info Gbps, K=7 r1/2 soft-decision framed Viterbi on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (driver, N > 1)

Workload (BASELINE.json configs[4], "C5"): K=7 (171,133) rate 1/2, int8 LLRs
(scale 32, Eb/N0 3 dB, synthetic, generated in HBM), frames f=256, v1=v2=20,
serial traceback. A step decodes ONE stream of --stages stages (default
2^32 = 4 Gi info bits) sharded over the N ranks (strong scaling, BASELINE C5
"4G info bits sharded across 1/2/4/8"): rank r owns a contiguous, output-word
aligned frame range (vd_partition_frames) and holds only its LLR window (the
frames' stages plus the v1 / v2 halo, synthesised on its own device: every
value is a pure function of (seed, stage)); no collective on the data path.
After timing, rank 0 gathers the packed slices and checks them against its
own 1-GPU decode of the whole stream (identity_vs_1gpu_decode). A secondary
weak-scaling line (every rank its own whole stream) is added for N > 1.
Inputs (8 GiB at N = 1) exceed L2, so no flush is needed between steps.

value: device-timed (CUDA events on the decode stream, max over ranks)
       whole-stream info bits / s.
e2e:   the same metric through the reference-facing host call
       (vd_decode_i8: pinned host LLRs -> H2D -> kernel -> D2H packed bits,
       streamed in chunks; each rank its 1/N share), timed around the call.
e2e_reference_api (N = 1, C5): the reference's own C++ signature,
       vitdec::framed_decode(LlrBlock of doubles) -> bytes, 2^26 bits
       (tools/bench_dropin.cpp): conversion, staging and unpack included.
roofline: the decode kernel against its binding roof (integer ALU: the
       measured ACS-pair rate of profiles/alu_peak.json, and the dual-issue
       bound; the HBM roof alongside), see DESIGN.md §4. traffic: DRAM bytes
       of this round's ncu capture (profiles/decode_traffic.json).
gpu_launches: kernels this library launched inside the timed region
       (vd_kernel_launches() counter around it).
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
    ap.add_argument("--no-weak", action="store_true", help="skip the secondary weak-scaling line (N > 1)")
    ap.add_argument("--frame", default="", help="f,v1,v2[,f0] frame configuration override (default 256,20,20)")
    ap.add_argument("--polys", default="", help="octal generator polynomials overriding the workload's code "
                    "(B = their count; e.g. 165,117: a code served by a run-time kernel instantiation)")
    ap.add_argument("--k", type=int, default=0, help="constraint length for --polys (0: the workload's)")
    a = ap.parse_args()
    if a.frame:
        global F, V1, V2, F0
        vals = [int(x) for x in a.frame.split(",")]
        F, V1, V2 = vals[:3]
        F0 = vals[3] if len(vals) > 3 else 0
    a.code, default_n, a.workload_desc = WORKLOADS[a.workload]
    if a.polys:
        k = a.k or a.code[0]
        polys = [int(x, 8) for x in a.polys.split(",")]
        b = len(polys)  # rate 1/B from the polynomial count
        if any(p >> k for p in polys):
            raise SystemExit(f"--polys: polynomials of at most K={k} bits")
        a.code = (k, b, polys)
        a.workload_desc += f", code overridden: ({','.join(oct(p)[2:] for p in polys)})"

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

class CpuArm:
    """The reference's own framed_decode (oracle/_ref, compiled from the
    reference sources, all host threads) or, if that library is absent, the
    single-threaded C oracle port, on a bounded sample of the workload: a
    contiguous stream of `n` info bits from the reference's data chain
    (random_bits -> encode -> BPSK -> AWGN, berlab.cpp:138-142), int8-quantised
    (q = rint(32 y)) and handed to framed_decode as doubles."""

    def __init__(self, code, n=None, target_s=8.0, threads=None):
        import oracle

        self.code = code
        self.port = oracle.port()
        ref = oracle.ref_backend()
        self.kind = "reference" if ref is not None else "port"
        self.backend = ref if ref is not None else self.port
        self.cores = (threads or os.cpu_count() or 1) if ref is not None else 1
        if n is None:
            # probe the rate, then size the sample for ~target_s (>= 2^26 bits
            # when that fits in 4 x target_s: ">= 64 Mi-bit prefix")
            m = 1 << 16
            q = self._gen(m, 1)
            t0 = time.perf_counter()
            self._decode(q, m)
            rate = m / max(time.perf_counter() - t0, 1e-6)
            n = int(min(max(rate * target_s, 1 << 16), 1 << 28))
            if n < (1 << 26) and rate * 4 * target_s >= (1 << 26):
                n = 1 << 26
        self.n = n
        self.q = self._gen(n, 2)

    def _gen(self, n, seed):
        import oracle

        rx, _ = self.port.gen_bench_block(*self.code, n, EBN0, seed)
        return oracle.quantize(rx, SCALE)

    def _decode(self, q, n):
        self.backend.framed_decode(*self.code, q, n, F, V1, V2, F0, workers=self.cores)

    def time_once(self):
        t0 = time.perf_counter()
        self._decode(self.q, self.n)
        return time.perf_counter() - t0

    def sample(self):
        k, b = self.code[0], self.code[1]
        who = f"reference framed_decode, workers={self.cores}" if self.kind == "reference" else "C oracle port, 1 thread"
        return (f"{self.n} info bits (K={k} B={b}, int8 q=rint(32y) at {EBN0} dB, f={F}/v1={V1}/v2={V2}/f0={F0}), "
                f"{who}")


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    arm = CpuArm(args.code, target_s=min(args.cpu_seconds, 20.0) / 4)
    for _ in range(args.warmup):
        arm.time_once()
    dts = sorted(arm.time_once() for _ in range(args.steps))
    dt = dts[len(dts) // 2]  # median step
    gbps = arm.n / dt / 1e9
    line = {
        "metric": "decoded info Gbps (K=7 r1/2 soft)", "value": gbps, "unit": "Gbps", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference random_bits/encode/BPSK/AWGN chain, int8-quantised)",
        "config": {"workload": "K=7 r1/2 (171,133) framed f=256 v1=20 v2=20, CPU sample per step (median step)",
                   "sample": arm.sample()},
        "cpu_baseline": {"value": gbps, "unit": "Gbps", "cores": arm.cores, "kind": arm.kind, "sample": arm.sample()},
        "e2e": {"value": gbps, "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------ GPU arm ------

def alu_ops_per_bit(stats_stages: int, n: int, s: int = 64) -> float:
    """Algorithmic integer ops per decoded bit: 2 adds + 1 compare-select per
    state per processed stage."""
    return 3.0 * s * stats_stages / n


def alu_peaks(sms: int, sm_mhz: float):
    """(measured ACS-pair Tops, its source, dual-issue bound Tops). The
    measured rate is profiles/alu_peak.json (microbench/run_alu_peak.py on a
    B200: the fast kernel's VIADD.16x2 -> VIADDMNMX.S16x2 pair); the dual-issue
    bound is 1 warp-instruction / clk / SMSP with the fmaheavy and alu pipes
    each at 0.5 (profiles/r01_pipe_probe_ncu.csv) x 3 lane-ops per packed
    instruction = 384 lane-ops / clk / SM."""
    dual = sms * 384 * sm_mhz * 1e6 / 1e12
    p = ROOT / "profiles" / "alu_peak.json"
    if p.exists():
        d = json.loads(p.read_text())
        if "acs_warp_instr_per_sm_clk" in d:
            tops = d["lane_ops_per_sm_clk"] * sms * sm_mhz * 1e6 / 1e12
            src = (f"profiles/alu_peak.json: ACS pair measured at {d['acs_warp_instr_per_sm_clk']:.3f} warp-instr/SM/clk "
                   f"({d['lane_ops_per_sm_clk']:.0f} lane-ops/clk/SM) x {sms} SM x {sm_mhz:.0f} MHz")
            return tops, src, dual
    return dual, "dual-issue bound (profiles/alu_peak.json absent)", dual


def kernel_traffic(workload: str):
    """DRAM bytes per decoded bit of the decode kernel from this round's ncu
    capture (tools/ncu_traffic.py -> profiles/decode_traffic.json), or None."""
    tp = ROOT / "profiles" / "decode_traffic.json"
    if not tp.exists():
        return None, None
    d = json.loads(tp.read_text())
    w = d.get("workloads", {}).get(workload)
    if not w:
        return None, None
    return w["bytes_per_bit"], d.get("source")


def dropin_e2e(args):
    """End to end through the reference-facing C++ call itself,
    vitdec::framed_decode(LlrBlock of doubles) -> std::vector<uint8_t> bits
    (paper_2011_09337_b200/bench_dropin, tools/bench_dropin.cpp): includes the
    integer check / double -> int8 conversion, pageable staging and the byte
    unpack that the native int8 call of `e2e` skips. Secondary to `e2e`."""
    exe = ROOT / "paper_2011_09337_b200" / "bench_dropin"
    if not exe.exists():
        return None
    n = 1 << 26
    try:
        r = subprocess.run([str(exe), str(n), "3"], capture_output=True, text=True, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 - report, do not fail the headline line
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    d["path"] = ("vitdec::framed_decode(const LlrBlock&, ...) C++ drop-in: B x N doubles in, bytes out, "
                 "host conversion + pageable staging + H2D + decode + D2H + unpack timed per call (median)")
    return d


def run_ours(args):
    import numpy as np
    import torch

    import paper_2011_09337_b200 as vd
    from paper_2011_09337_b200.device import count_bit_errors, decode_i8_device, synth_llr_i8_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Plumbing test hook: VITDEC_BENCH_ONE_DEVICE=1 puts every rank on cuda:0
    # with the gloo backend (NCCL refuses two ranks on one GPU), so the N > 1
    # path (shards, barriers, max-over-ranks timing, identity gather, rank-0
    # reporting) can be exercised on a one-GPU box. Not a scaling measurement.
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

    def max_over_ranks(x):
        if not dist:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    t = vd.build_trellis(vd.CodeSpec(*args.code))
    B = args.code[1]
    S = 1 << (args.code[0] - 1)
    cfg = vd.FrameConfig(F, V1, V2, F0)
    n = args.stages  # the WHOLE stream (strong scaling: shared by the ranks)
    nf = (n + F - 1) // F
    sigma = (1.0 / (2 * (1.0 / B) * 10 ** (EBN0 / 10))) ** 0.5
    seed = 1234
    stream = torch.cuda.Stream(device=dev)

    # ---- this rank's shard: contiguous word-aligned frames + v1/v2 halo -----
    first = vd.partition_frames(cfg, n, world)
    fb, fe = first[rank], first[rank + 1]
    wb, we = vd.frame_window(cfg, n, fb, fe) if fe > fb else (0, 0)
    out0, out1 = fb * F, min(fe * F, n)
    llr = torch.empty(max(we - wb, 1) * B, dtype=torch.int8, device=dev)
    words = (out1 - out0 + 31) // 32
    out = torch.empty(words + 1, dtype=torch.int32, device=dev)
    bits = torch.empty(words + 1, dtype=torch.int32, device=dev)
    with torch.cuda.stream(stream):
        if fe > fb:
            synth_llr_i8_range(t, wb, we - wb, sigma, SCALE, seed, llr, None, local, stream)
            synth_llr_i8_range(t, out0, out1 - out0, sigma, SCALE, seed, None, bits, local, stream)
    stream.synchronize()

    def step():
        if fe > fb:
            decode_i8_device(t, cfg, n, llr, wb, fb, fe, out, out0, None, local, stream)

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    if fe > fb:
        count_bit_errors(out, bits, out1 - out0, cnt, local, stream)
    stream.synchronize()
    errs = int(cnt.item())

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    lib = vd.lib()
    l0 = lib.vd_kernel_launches()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    launches = (lib.vd_kernel_launches() - l0) / args.steps  # this rank's kernels per step
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    if dist:
        dist.barrier()
    ms_step = ms / args.steps
    gbps = n / (ms_step * 1e-3) / 1e9  # whole stream / slowest rank

    # ---- 1-GPU identity (N > 1): rank 0 decodes the whole stream alone ----
    identity = None
    if dist:
        tot = torch.tensor([errs], dtype=torch.int64, device=red_dev)
        dist.all_reduce(tot)
        errs = int(tot.item())
        maxw = (max(min(first[r + 1] * F, n) - first[r] * F for r in range(world)) + 31) // 32
        mine = torch.zeros(maxw, dtype=torch.int32, device=red_dev)
        mine[:words] = out[:words].to(red_dev)
        gathered = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
        if one_dev:
            dist.gather(mine, gathered, dst=0)
        else:
            allg = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(allg, mine)
            gathered = allg if rank == 0 else None
        if rank == 0:
            del llr
            torch.cuda.empty_cache()
            full_llr = torch.empty(n * B, dtype=torch.int8, device=dev)
            full_out = torch.empty((n + 31) // 32 + 1, dtype=torch.int32, device=dev)
            synth_llr_i8_range(t, 0, n, sigma, SCALE, seed, full_llr, None, local, stream)
            decode_i8_device(t, cfg, n, full_llr, 0, 0, nf, full_out, 0, None, local, stream)
            stream.synchronize()
            ok = True
            for r in range(world):
                a0, a1 = first[r] * F, min(first[r + 1] * F, n)
                w = (a1 - a0 + 31) // 32
                if w == 0:
                    continue
                ref = full_out[a0 // 32:a0 // 32 + w].cpu()
                ok &= bool(torch.equal(gathered[r][:w].cpu(), ref))
            identity = ok
            del full_llr, full_out
            torch.cuda.empty_cache()
        dist.barrier()

    # ---- weak scaling (secondary, N > 1): every rank its own whole stream ---
    weak = None
    if dist and not args.no_weak:
        nw = n
        del out, bits
        if rank != 0:
            del llr
        torch.cuda.empty_cache()
        wl = torch.empty(nw * B, dtype=torch.int8, device=dev)
        wo = torch.empty((nw + 31) // 32 + 1, dtype=torch.int32, device=dev)
        synth_llr_i8_range(t, 0, nw, sigma, SCALE, seed + 1 + rank, wl, None, local, stream)
        wstep = lambda: decode_i8_device(t, cfg, nw, wl, 0, 0, (nw + F - 1) // F, wo, 0, None, local, stream)
        for _ in range(args.warmup):
            wstep()
        stream.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            wstep()
        e1.record(stream)
        e1.synchronize()
        wms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
        weak = {"value": nw * world / (wms * 1e-3) / 1e9, "unit": "Gbps", "ms_per_step": wms,
                "info_bits_per_gpu_per_step": nw, "scaling": "weak"}
        del wl, wo
        torch.cuda.empty_cache()
        dist.barrier()

    # ---- e2e through the host-buffer C-ABI call (pinned memory) -----------
    # every rank streams its 1/N share of the e2e stream (an independent
    # sub-stream, own frame grid) from pinned host memory: H2D -> decode ->
    # D2H of the packed bits, inside the timed region
    ne_total = min(args.e2e_stages, n)
    ne = max(((ne_total // world) // 32) * 32, 32)
    e2e_llr = torch.empty(ne * B, dtype=torch.int8, device=dev)
    synth_llr_i8_range(t, rank * ne, ne, sigma, SCALE, seed, e2e_llr, None, local, stream)
    stream.synchronize()
    host_llr = torch.empty(ne * B, dtype=torch.int8, pin_memory=True)
    host_llr.copy_(e2e_llr)
    host_out = torch.empty((ne + 31) // 32, dtype=torch.int32, pin_memory=True)
    c = cfg.to_c()
    dev_idx = C.c_int32(local)
    ex = vd._lib.VdExec(1, C.pointer(dev_idx), 0)
    st = vd._lib.VdStats()

    def e2e_step():
        vd._lib.check(lib.vd_decode_i8(t.handle, C.byref(c), host_llr.data_ptr(), ne, host_out.data_ptr(),
                                       C.byref(st), C.byref(ex)))

    e2e_step()
    # the e2e result must equal the device-resident decode of the same stream
    chk = torch.empty((ne + 31) // 32 + 1, dtype=torch.int32, device=dev)
    decode_i8_device(t, cfg, ne, e2e_llr, 0, 0, (ne + F - 1) // F, chk, 0, None, local, stream)
    stream.synchronize()
    same = bool(torch.equal(host_out, chk[:(ne + 31) // 32].cpu()))
    del e2e_llr, chk
    if dist:
        dist.barrier()
    e2e_reps = max(args.e2e_steps, 1)
    t0 = time.perf_counter()
    for _ in range(e2e_reps):
        e2e_step()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_reps)
    e2e_gbps = ne * world / e2e_s / 1e9

    # ---- roofline ----------------------------------------------------------
    peaks, peak_src = measured_peaks()
    clocks = clk.summary()
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak, alu_src, dual_peak = alu_peaks(sms, sm_mhz)
    stats = vd.frame_stats(cfg, n)
    ops_bit = alu_ops_per_bit(stats.stages, n, S)
    bits_per_gpu_s = n / world / (ms_step * 1e-3)  # average per GPU over the slowest rank's time
    alu_achieved = ops_bit * bits_per_gpu_s / 1e12
    hbm_bytes_bit = B + 1 / 8  # int8 LLR read once + packed output
    hbm_achieved = hbm_bytes_bit * bits_per_gpu_s / 1e9
    tb_bit, t_src = kernel_traffic(args.workload if not args.frame else "")
    traffic = tb_bit * n / world if tb_bit is not None else None

    result = None
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            arm = CpuArm(args.code, target_s=args.cpu_seconds / 3)
            dt = sorted(arm.time_once() for _ in range(3))[1]
            cpu = {"value": arm.n / dt / 1e9, "unit": "Gbps", "cores": arm.cores, "kind": arm.kind,
                   "sample": arm.sample() + " (median of 3)"}
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
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "int8 LLR / int16x2 path metrics" if t.fast_path() else "int8 LLR / int32 path metrics",
            "data": "synthetic: random message, encoder, BPSK+AWGN at 3 dB, int8 q=rint(32y), generated in HBM",
            "config": {
                "workload": args.workload_desc if not args.frame else
                            f"{args.workload_desc.split(',')[0]}, frame override f={F} v1={V1} v2={V2} f0={F0}",
                "info_bits_per_step": n,
                "frames": nf,
                "parallelism": (f"one stream sharded over {world} GPUs: contiguous word-aligned frame ranges "
                                f"(vd_partition_frames) + v1/v2 halo, no collective" if world > 1 else "1 GPU"),
                "l2": (f"inputs ({B} B/bit x {n} bits = {n * B / 2**30:.2f} GiB) exceed L2; no flush needed"
                       if n * B // world > 256 << 20 else
                       f"inputs ({n * B / 2**20:.1f} MiB) fit in L2: steps re-read them warm (latency-bound size)"),
                "kernel": "fast (register-resident)" if t.fast_path() else "generic (warp per frame)",
                "bit_errors_vs_sent": errs,
                "ber_check": errs / n,
                "identity_vs_1gpu_decode": identity,
            },
            "roofline": {
                "bound": "alu",
                "achieved": alu_achieved,
                "peak": alu_peak,
                "unit": "Tops",
                "frac": alu_achieved / alu_peak,
                "traffic": traffic,
                "traffic_source": t_src,
                "ops_per_bit": ops_bit,
                "peak_source": alu_src,
                "dual_issue": {"peak": dual_peak, "frac": alu_achieved / dual_peak,
                               "source": "384 lane-ops/clk/SM (profiles/r01_pipe_probe_ncu.csv pipe rates)"},
                "hbm": {"achieved": hbm_achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm_achieved / peaks["hbm_gbs"], "bytes_per_bit": hbm_bytes_bit,
                        "peak_source": peak_src},
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_gbps, "unit": "Gbps", "h2d_bytes_per_step": ne * B * world,
                    "d2h_bytes_per_step": ((ne + 31) // 32) * 4 * world, "info_bits_per_step": ne * world,
                    "matches_device_decode": same,
                    # PCIe: H2D GB/s this line moved (ne bits at e2e_gbps -> ne * B bytes per
                    # ne / e2e_gbps ns), against the box's pinned-copy ceiling measured by
                    # tools/pcie_probe.py (profiles/r02_pcie_probe.json)
                    "h2d_gbs": (B * e2e_gbps / world) if e2e_gbps else None,
                    "h2d_ceiling_gbs": _pcie_ceiling()},
            "gpu_launches": int(round(launches * args.steps)),
            "gpu_launches_per_step_per_rank": launches,
            "clocks": clocks,
        }
        if weak:
            result["weak_scaling"] = weak
        api = dropin_e2e(args) if world == 1 and args.e2e_steps > 0 and args.workload == "C5" else None
        if api is not None:
            result["e2e_reference_api"] = api
        print(json.dumps(result))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return result


def _pcie_ceiling():
    """Pinned H2D GB/s of this box type (tools/pcie_probe.py), or None."""
    try:
        return json.loads((ROOT / "profiles" / "r02_pcie_probe.json").read_text())["h2d_one_copy_GBps"]
    except (OSError, ValueError, KeyError):
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

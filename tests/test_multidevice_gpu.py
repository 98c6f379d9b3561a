"""Host-buffer multi-device engine (decode_host, vd_decode_i8 with
exec.num_devices >= 2): frames sharded by vd_partition_frames, one issue
thread per device, per-device staging of pageable buffers. A device list
may repeat a device ({0, 0}), so the per-device interleaving, DeviceGuard
switching and staging code run on a one-GPU box too; with >= 2 GPUs the
real multi-device case runs as well. The bar is bit-identity with the
single-device decode (reference worker invariance, test_decoder.cpp:254-261).
"""
import threading

import numpy as np
import pytest

import oracle
import paper_2011_09337_b200 as vd

pytestmark = pytest.mark.gpu

K7 = (7, 2, [0o171, 0o133])


@pytest.fixture(scope="module")
def port():
    return oracle.port()


def _device_lists():
    import torch

    lists = [[0, 0], [0, 0, 0]]
    if torch.cuda.device_count() >= 2:
        lists += [[0, 1], [1, 0, 1]]
    return lists


@pytest.mark.parametrize("pinned", [False, True], ids=["pageable", "pinned"])
def test_device_list_matches_single_device(pinned, port):
    import torch

    t = vd.build_trellis(vd.CodeSpec(*K7))
    for n, cfg in ((300_017, vd.FrameConfig(256, 20, 20)), (123_457, vd.FrameConfig(320, 20, 45, 32)),
                   (200_000, vd.FrameConfig(100, 30, 45, 25, vd.TracebackStart.kRandom, 9))):
        rx, _ = port.gen_bench_block(*K7, n, 2.5, n)
        q = oracle.quantize(rx)
        if pinned:
            q = torch.from_numpy(q).pin_memory().numpy()
        exp, st, _ = port.framed_decode(*K7, q, n, cfg.f, cfg.v1, cfg.v2, cfg.f0, int(cfg.start), cfg.seed)
        one, st1 = vd.framed_decode_stream(q, n, t, cfg)
        assert np.array_equal(vd.unpack_bits(one, n), exp)
        for devs in _device_lists():
            for chunk in (0, 1 << 14):
                got, st2 = vd.framed_decode_stream(q, n, t, cfg, chunk_stages=chunk, devices=devs)
                assert np.array_equal(got, one), (devs, chunk, cfg)
                assert (st2.frames, st2.stages, st2.tracebacks) == st


def test_device_list_concurrent_threads(port):
    """Several host threads, each sharding over a device list, at once."""
    t = vd.build_trellis(vd.CodeSpec(*K7))
    cfg = vd.FrameConfig(256, 20, 20)
    jobs = []
    for i in range(4):
        n = 120_000 + 777 * i
        rx, _ = port.gen_bench_block(*K7, n, 2.0, 50 + i)
        q = oracle.quantize(rx)
        exp, _, _ = port.framed_decode(*K7, q, n, 256, 20, 20)
        jobs.append((q, n, exp))
    res = [None] * len(jobs)

    def run(i):
        q, n, _ = jobs[i]
        packed, _ = vd.framed_decode_stream(q, n, t, cfg, chunk_stages=1 << 15, devices=[0, 0])
        res[i] = vd.unpack_bits(packed, n)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for (_, _, exp), got in zip(jobs, res):
        assert np.array_equal(got, exp)


def test_batched_decode_on_every_device(port):
    """vd_decode_batch_i8 keeps its pinned table staging per (thread, device):
    one thread decoding batches on each visible device in turn."""
    import torch

    t = vd.build_trellis(vd.CodeSpec(*K7))
    cfg = vd.FrameConfig(256, 20, 20)
    lens = [65_536] * 4 + [10_000]
    n = sum(lens)
    rx, _ = port.gen_bench_block(*K7, n, 2.0, 5)
    q = oracle.quantize(rx)
    exp, blocks = [], []
    off = 0
    for ln in lens:
        blocks.append(q[off * 2:(off + ln) * 2])
        e, _, _ = port.framed_decode(*K7, blocks[-1], ln, 256, 20, 20)
        exp.append(e)
        off += ln
    devs = list(range(torch.cuda.device_count())) * 2
    for d in devs:
        res = vd.framed_decode_batch(blocks, t, cfg, gpu=d)
        for (bits, _), e in zip(res, exp):
            assert np.array_equal(bits, e), d


def test_synth_range_matches_whole_stream():
    """A shard's halo window synthesised on its own (vd_synth_llr_i8_range_device)
    equals the same stages of the whole-stream synthesis (bench.py's shards)."""
    import torch

    from paper_2011_09337_b200.device import synth_llr_i8, synth_llr_i8_range

    for code in (K7, (9, 3, [0o557, 0o663, 0o711])):
        t = vd.build_trellis(vd.CodeSpec(*code))
        b = code[1]
        n = 1 << 20
        full = torch.empty(n * b, dtype=torch.int8, device="cuda")
        fbits = torch.empty(n // 32, dtype=torch.int32, device="cuda")
        synth_llr_i8(t, n, 0.7, 32.0, 77, full, fbits)
        for t0, m in ((0, 1000), (12345, 77777), (n - 4099, 4099), (32 * 1001, 64 * 40)):
            part = torch.empty(m * b, dtype=torch.int8, device="cuda")
            pbits = torch.empty(-(-m // 32), dtype=torch.int32, device="cuda") if t0 % 32 == 0 else None
            synth_llr_i8_range(t, t0, m, 0.7, 32.0, 77, part, pbits)
            assert torch.equal(part, full[t0 * b:(t0 + m) * b]), (code, t0)
            if pbits is not None and m % 32 == 0:
                assert torch.equal(pbits, fbits[t0 // 32:(t0 + m) // 32]), (code, t0)


def test_bench_sharded_stream_identity(tmp_path):
    """bench.py's N > 1 path (one stream sharded over ranks, halo windows,
    max-over-ranks timing, rank-0 gather + 1-GPU identity check), run as two
    ranks on one device (VITDEC_BENCH_ONE_DEVICE=1, gloo)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, VITDEC_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", str(root / "bench.py"), "--gpus", "2",
           "--stages", str((1 << 26) + 12345), "--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "1",
           "--e2e-stages", str(1 << 22)]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["identity_vs_1gpu_decode"] is True
    assert d["e2e"]["matches_device_decode"] is True
    assert d["gpu_launches"] >= 3
    assert d["config"]["ber_check"] < 2e-3
    assert "weak_scaling" in d

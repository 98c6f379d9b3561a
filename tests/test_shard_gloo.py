"""Multi-process (world_size 2, gloo) check of the frame-shard decomposition
the multi-GPU path uses: each rank takes the contiguous frame
range vd_partition_frames assigns it, sees ONLY its halo window of LLRs
(vd_frame_window; everything outside is overwritten with garbage), decodes
it (CPU oracle standing in for one GPU), and the word-aligned packed slices
gathered over the process group must equal the single-process decode bit for
bit. No collective is needed on the data path; all_gather here only brings
the slices together for the check.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [
    (7, 2, [0o171, 0o133], 40_000, (256, 20, 20, 0, 0, 0)),
    (7, 2, [0o171, 0o133], 33_333, (100, 30, 45, 25, 1, 4)),
    (9, 2, [0o561, 0o753], 20_011, (37, 9, 50, 0, 0, 0)),
    (5, 2, [0o23, 0o35], 9_999, (320, 20, 45, 32, 0, 0)),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    import torch

    import oracle
    import paper_2011_09337_b200 as vd

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    try:
        port_ = oracle.port()
        rng = np.random.default_rng(1234)
        for k, b, polys, n, (f, v1, v2, f0, start, seed) in CASES:
            rx, _ = port_.gen_bench_block(k, b, polys, n, 2.0, 77)
            qllr = oracle.quantize(rx)
            cfg = vd.FrameConfig(f, v1, v2, f0, vd.TracebackStart(start), seed)
            first = vd.partition_frames(cfg, n, world)
            fb, fe = first[rank], first[rank + 1]
            words = (n + 31) // 32
            mine = np.zeros(words, np.uint32)
            if fb < fe:
                lo, hi = vd.frame_window(cfg, n, fb, fe)
                shard = rng.integers(-127, 128, n * b).astype(np.int8)  # garbage outside the halo window
                shard[lo * b:hi * b] = qllr[lo * b:hi * b]
                bits = oracle.framed_decode_range_i8(k, b, polys, shard, n, f, v1, v2, f0, start, seed, fb, fe)
                out_lo, out_hi = fb * f, min(fe * f, n)
                assert out_lo % 32 == 0 or fb == 0  # shards start on a packed output word
                sl = np.zeros(n, np.uint8)
                sl[out_lo:out_hi] = bits[out_lo:out_hi]
                mine = vd.pack_bits(sl)
            gathered = [torch.zeros(words, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(mine.astype(np.int64)))
            merged = np.zeros(words, np.uint32)
            for g in gathered:
                merged |= g.numpy().astype(np.uint32)
            full, _, _ = port_.framed_decode(k, b, polys, qllr, n, f, v1, v2, f0, start, seed)
            ok = ok and np.array_equal(vd.unpack_bits(merged, n), full)
    finally:
        dist.destroy_process_group()
    results.put((rank, ok))


@pytest.mark.parametrize("world", [2])
def test_frame_shards_over_gloo(world):
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = os.pathsep.join([os.path.dirname(here), here, os.environ.get("PYTHONPATH", "")])
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    results = [q.get() for _ in range(world)]
    assert all(ok for _, ok in results), results
    assert all(p.exitcode == 0 for p in procs)

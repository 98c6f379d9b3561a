#!/bin/bash
# Re-measure every workload row of DESIGN.md §4 / README.md on one B200 and
# write the JSON lines to gpurun_out/<tag>_*.json[l] (run on the GPU box):
#   tools/refresh_results.sh r02
set -u
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
b() {  # bench.py line -> {"row", "gbps", "frac", "ber"}
  local row=$1; shift
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 0 --e2e-stages 1048576 "$@" 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'row': '$row', 'gbps': round(d['value'],2), 'frac': round(d['roofline']['frac'],4), 'ber': d['config']['ber_check'], 'ms_per_step': round(d['ms_per_step'],4)}))"
}
{
  b "C3 2^26 (bench default)" --workload C3
  b "C3 2^30" --workload C3 --stages 1073741824
  b "C4 2^28" --workload C4
  b "U3 2^28" --workload U3
  b "C1 f=256/20/20" --workload C1
  b "C1 f=320/20/45/32" --workload C1 --frame 320,20,45,32
  b "C5 f=320/20/45/32 2^28" --frame 320,20,45,32 --stages 268435456
  b "C5 f=512/20/63 2^28" --frame 512,20,63 --stages 268435456
  b "C5 f=1024/42/42 2^28" --frame 1024,42,42 --stages 268435456
  b "C5 JIT code (165,117) 2^30" --stages 1073741824 --polys 165,117
  b "C1 JIT code (165,117)" --workload C1 --polys 165,117
  b "C1 K=6 (65,57) JIT" --workload C1 --k 6 --polys 65,57
  b "K=9 r1/4 (765,671,513,473) 2^28" --workload C4 --polys 765,671,513,473
  b "K=10 (1157,1753) 2^28" --workload C4 --k 10 --polys 1157,1753
} > $out/${tag}_workloads.jsonl
bash tools/sweep_frames.sh > $out/${tag}_frame_sweep.jsonl 2>&1
timeout 600 python tools/bench_batch.py > $out/${tag}_batch.jsonl 2>&1
timeout 600 python tools/bench_batch.py --block-bits 8192 --blocks 65536 >> $out/${tag}_batch.jsonl 2>&1
timeout 600 python tools/bench_wire.py > $out/${tag}_wire.jsonl 2>&1
timeout 600 python tools/bench_pageable.py > $out/${tag}_pageable_e2e.jsonl 2>&1
timeout 600 python tools/bench_serial.py > $out/${tag}_serial.jsonl 2>&1
timeout 600 python tools/bench_generic.py > $out/${tag}_generic.jsonl 2>&1
cat $out/${tag}_workloads.jsonl

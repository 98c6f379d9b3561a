for fr in 32,20,35 64,20,42 128,20,49 256,20,56 256,20,35 256,20,70 512,20,63 1024,20,70 1024,42,42 320,20,45,32; do
  timeout 300 python bench.py --frame $fr --stages 268435456 --steps 10 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'frame': '$fr', 'gbps': round(d['value'],2), 'frac': round(d['roofline']['frac'],4)}))"
done
timeout 300 python bench.py --workload C3 --stages 1073741824 --steps 10 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'frame': 'C3 2^30', 'gbps': round(d['value'],2), 'frac': round(d['roofline']['frac'],4)}))"
timeout 600 python tools/bench_batch.py 2>&1 | tail -3

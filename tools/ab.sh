#!/bin/bash
# A/B the fast kernel across tuning variants on the GPU box:
#   tools/ab.sh [workload] variant1 variant2 ...   (variant "base" = in-tree library)
w=${W:-C5}; st=${STAGES:-1073741824}
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib=build_variants/$v/libvitdec_b200.so; fi
  r=$(VITDEC_LIB=$lib timeout 300 python bench.py --workload $w --stages $st --steps 10 --warmup 3 --no-cpu --e2e-steps 0 --e2e-stages 1048576 2>&1 | tail -1)
  echo "$v $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), "Gbps frac", round(d["roofline"]["frac"],4), "ber", d["config"]["ber_check"])' 2>/dev/null || echo "$r")"
done

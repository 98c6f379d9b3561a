#!/bin/bash
# A/B variants on one frame configuration: FRAME=f,v1,v2[,f0] STAGES=N tools/ab_frame.sh base v1 v2 ...
fr=${FRAME:-256,20,20}; st=${STAGES:-268435456}
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib=build_variants/$v/libvitdec_b200.so; fi
  r=$(VITDEC_LIB=$lib timeout 300 python bench.py --stages $st --frame $fr --steps 5 --warmup 3 --no-cpu --e2e-steps 1 --e2e-stages 1048576 2>&1 | tail -1)
  echo "$v $fr $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), "Gbps frac", round(d["roofline"]["frac"],4))' 2>/dev/null || echo "$r")"
done

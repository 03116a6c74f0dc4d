#!/bin/bash
# A/B of two builds of libtidq.so (paper_1807_01409_b200/libtidq_A.so, _B.so):
# C2 sweep (bench.py, device only) and the C3/C4/C5 configs, fresh process each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=paper_1807_01409_b200
for v in ${LIB_VARIANTS:-A B A B}; do
  cp $L/libtidq_$v.so $L/libtidq.so
  timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu --no-join --no-configs 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 lib=$v', round(d['ms_per_step'],4))"
  [ -n "${NO_CONFIGS:-}" ] || AB_CONFIGS=${AB_CONFIGS:-C3,C4,C5} bash tools/ab_configs.sh "lib$v:" > /dev/null
  [ -f gpurun_out/ab_lib$v.jsonl ] && cp gpurun_out/ab_lib$v.jsonl gpurun_out/ab_lib${v}_$(date +%s).jsonl
done

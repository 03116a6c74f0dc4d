#!/bin/bash
# A/B of query-path knobs on the C4/C5 configs (one GPU): each variant's
# per-query device latency (tools/bench_configs.py) into gpurun_out/ab_<name>.jsonl.
# usage: tools/ab_configs.sh "name:ENV=V ENV2=V2" ...   (name "base" = no env)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "$@"; do
  name="${v%%:*}"; envs="${v#*:}"; [ "$name" = "$v" ] && envs=""
  env $envs timeout 600 python tools/bench_configs.py --configs ${AB_CONFIGS:-C4,C5} --reps 5 \
    > "gpurun_out/ab_${name}.jsonl" 2> "gpurun_out/ab_${name}.err"
  echo "ab $name ($envs) rc=$?"
done

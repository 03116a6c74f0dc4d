#!/bin/bash
# One gpurun job: tests, smoke, bench, ncu launch list + full capture of the scan kernel.
# usage: tools/gpu_job.sh [stages...]   stages: test smoke bench ncu ncufull sanitize
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
STAGES="${*:-test smoke bench ncu ncufull}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
for s in $STAGES; do
  echo "=== stage $s $(date +%T)"
  case $s in
    sel) timeout ${SEL_TIMEOUT:-900} python -m pytest ${TESTS} -x -q -m gpu > gpurun_out/pytest_sel.log 2>&1; echo "sel pytest rc=$?"; tail -25 gpurun_out/pytest_sel.log;;
    dtest) timeout 300 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist pytest rc=$?"; tail -15 gpurun_out/pytest_dist.log;;
    configs) timeout 900 python tools/bench_configs.py --configs ${CONFIGS:-C3,C4,C5} > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"; cat gpurun_out/configs.jsonl; tail -5 gpurun_out/configs.err;;
    test)  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log;;
    qbench) timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "qbench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err;;
    bench) timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err;;
    ref)   timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json;;
    ncu)   timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-join --no-configs > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?";;
    ncufull) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"mark_|super_offsets|emit_kernel" -s 0 -c 15 -o gpurun_out/prof_scan -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-join --no-configs > gpurun_out/ncu_full.log 2>&1; echo "ncufull rc=$?"; tail -3 gpurun_out/ncu_full.log
        python tools/ncu_summary.py gpurun_out/prof_scan.ncu-rep gpurun_out/ncu_scan_summary.json > gpurun_out/ncu_scan_summary.txt 2>&1
        python tools/ncu_raw.py gpurun_out/prof_scan.ncu-rep > gpurun_out/ncu_scan_raw.txt 2>&1
        [ -n "${KEEP_REP:-}" ] || rm -f gpurun_out/prof_scan.ncu-rep;;
    timeline) IFS=';' read -ra TLQ <<< "${TL_QUERIES:-C5|star x3;C5|chain x3;C4|star x3;C4|star x2}"  # ';'-separated
        for q in "${TLQ[@]}"; do
        cfg="${q%%|*}"; name="${q#*|}"; f="gpurun_out/timeline_${cfg}_${name// /_}.txt"
        timeout 300 python tools/timeline.py "$cfg" "$name" 3 > "$f" 2>&1; echo "timeline $cfg $name rc=$?"; head -1 "$f" | tail -1; grep -v Warn "$f" | sed -n 2p; done;;
    ncujoin) timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"expand_kernel|key_bitmap_kernel|bitmap_keep_kernel|radix_down|radix_up|os_pass|os_hist|semi_write|equal_range|gather_cols" -c ${NCU_JOIN_COUNT:-60} -o gpurun_out/prof_join -f python tools/bench_configs.py --configs ${NCU_JOIN_CFG:-C5} --only "${NCU_JOIN_Q:-star x3}" --reps 1 > gpurun_out/ncu_join.log 2>&1; echo "ncujoin rc=$?"; tail -3 gpurun_out/ncu_join.log
        python tools/ncu_join_summary.py gpurun_out/prof_join.ncu-rep gpurun_out/ncu_join_summary.json > gpurun_out/ncu_join_summary.txt 2>&1
        [ -n "${KEEP_REP:-}" ] || rm -f gpurun_out/prof_join.ncu-rep;;
    ncuemit) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"emit_kernel|mark_multi1|mark_kernel" -c ${NCU_EMIT_COUNT:-4} -o gpurun_out/prof_emit -f python tools/bench_configs.py --configs ${NCU_JOIN_CFG:-C5} --only "${NCU_JOIN_Q:-star x3}" --reps 1 > gpurun_out/ncu_emit.log 2>&1; echo "ncuemit rc=$?"
        python tools/ncu_join_summary.py gpurun_out/prof_emit.ncu-rep gpurun_out/ncu_emit_summary.json > gpurun_out/ncu_emit_summary.txt 2>&1; cat gpurun_out/ncu_emit_summary.txt
        [ -n "${KEEP_REP:-}" ] || rm -f gpurun_out/prof_emit.ncu-rep;;
    sanitize) for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest ${SAN_TESTS:-tests/test_gpu_scan.py} -x -q -k "${SAN_K:-golden or write_counts or evaluate_query}" > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log; done;;
  esac
done
echo "=== done $(date +%T)"

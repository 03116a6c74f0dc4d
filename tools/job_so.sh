cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pcodes.py tests/test_gpu_configs_c1.py tests/test_gpu_scan.py tests/test_gpu_query.py -x -q > gpurun_out/so_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/so_tests.log
AB_CONFIGS=C3,C4,C5 bash tools/ab_configs.sh "so0:TIDQ_SO=0" "so1:TIDQ_SO=1"
python tools/ab_compare.py gpurun_out/ab_so0.jsonl gpurun_out/ab_so1.jsonl
for v in 0 1 0 1; do TIDQ_SO=$v timeout 300 python bench.py --no-e2e --no-cpu --no-configs --no-join > gpurun_out/qb_so$v.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/qb_so$v.json').read().splitlines()[-1]); r=d['roofline']; print('C2 SO=$v', round(d['value']/1e9,1), round(d['ms_per_step'],4), 'mark', round(r['frac'],3), 'composite', round(r['scan_composite']['frac'],3), 'floor', round(r['scan_composite']['dram_floor']['step_frac_of_floor'],3))"; done

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pcodes.py tests/test_gpu_configs_c1.py tests/test_gpu_scan.py tests/test_gpu_query.py -x -q > gpurun_out/p16_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/p16_tests.log
for v in 0 1; do TIDQ_P16=$v timeout 300 python bench.py --no-e2e --no-cpu --no-configs --no-join > gpurun_out/qb_p$v.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/qb_p$v.json').read().splitlines()[-1]); r=d['roofline']; print('C2 P16=$v', round(d['value']/1e9,1), round(d['ms_per_step'],4), 'mark', round(r['frac'],3), round(r['avg_launch_ms']*1e3,1), 'us composite', round(r['scan_composite']['frac'],3), 'floor', round(r['scan_composite']['dram_floor']['step_frac_of_floor'],3))"; done

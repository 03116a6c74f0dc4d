cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops_scale.py tests/test_gpu_query.py tests/test_gpu_configs_c1.py -x -q > gpurun_out/dist_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dist_tests.log
AB_CONFIGS=C3 bash tools/ab_configs.sh "f0:TIDQ_DISTINCT_FILTER=0" "f1:TIDQ_DISTINCT_FILTER=1"
python tools/ab_compare.py gpurun_out/ab_f0.jsonl gpurun_out/ab_f1.jsonl

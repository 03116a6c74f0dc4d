cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_radix.py -x -q > gpurun_out/radix_tests.log 2>&1; echo "radix tests rc=$?"; tail -1 gpurun_out/radix_tests.log
timeout 600 python tools/sort_bench.py > gpurun_out/sort_bench.jsonl 2> gpurun_out/sort_bench.err; echo "sortbench rc=$?"; cut -c1-150 gpurun_out/sort_bench.jsonl; tail -3 gpurun_out/sort_bench.err

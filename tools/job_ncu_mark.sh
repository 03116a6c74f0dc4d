cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in 1 0; do TIDQ_P16=$v timeout 600 ncu --set full --clock-control none -k regex:"mark_multi1" -c 1 -o gpurun_out/prof_mark_p$v -f python tools/bench_configs.py --configs C5 --only "star x3" --reps 1 > gpurun_out/ncu_mark_p$v.log 2>&1; echo "ncu $v rc=$?"; done

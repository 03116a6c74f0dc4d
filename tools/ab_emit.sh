cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "1 0" "4 4" "1 4" "4 0" "2 0" "1 8" "2 6"; do
  set -- $cfg
  TIDQ_EMIT_GROUP=$1 TIDQ_EMIT_RESIDENT=$2 timeout 300 python bench.py --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('group',$1,'res',$2,'ms/step',round(d['ms_per_step'],4),'scan ms/launch',round(d['roofline']['avg_launch_ms'],4),'frac',round(d['roofline']['frac'],3))"
done
timeout 300 python tools/prof_host2.py

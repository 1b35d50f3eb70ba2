cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_summary.txt
for v in old new old new old new; do
  cp scripts/ab/lib_$v.so paper_2009_07400_b200/libtinymd_b200.so
  for w in weak c5; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $w', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4))" >> gpurun_out/ab_summary.txt
  done
done

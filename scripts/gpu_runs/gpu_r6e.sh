# A/B of two builds of the library on the same box (bench kernel times)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_summary.txt
for v in base keep base keep; do
  cp scripts/ab/lib_$v.so paper_2009_07400_b200/libtinymd_b200.so
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['kernel_ms_median'],4))" >> gpurun_out/ab_summary.txt
done

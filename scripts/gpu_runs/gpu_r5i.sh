cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TMD_SORT_EVERY=4 timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r5i_pytest_s4.log 2>&1; tail -1 gpurun_out/r5i_pytest_s4.log
rm -f gpurun_out/r5i_summary.txt
for e in 1 3 5 10 1 3 5 10; do
  TMD_SORT_EVERY=$e timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r5i_$e.log 2>&1
  tail -1 gpurun_out/r5i_$e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$e', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['kernel_ms_median'],4))" >> gpurun_out/r5i_summary.txt
done

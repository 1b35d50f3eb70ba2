cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 8 6 8 6; do
TMD_STEP_MINB=$m timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench1_m.log 2>&1
tail -1 gpurun_out/bench1_m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb $m', round(d['value']/1e9,3), round(d['roofline']['kernel_ms'],4))"
done

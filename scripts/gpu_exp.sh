cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
for i in 1 2 3; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench1_$i.log 2>&1
tail -1 gpurun_out/bench1_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('morton', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done

# Ad-hoc experiment runner for gpurun (edit freely):
#   /usr/local/graft/bin/gpurun --timeout 900 -- 'bash scripts/gpu_exp.sh'
# Example: the brick-numbering shape sweep that chose 2 x 4 x 4 cells.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sh in 1,2,2 2,2,2 0,2,2 1,2,3; do
TMD_ORDER_SHAPE=$sh timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench1_s.log 2>&1
tail -1 gpurun_out/bench1_s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shape $sh', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3d_pytest.log 2>&1
for i in 1 2; do
timeout 600 python bench.py --workload c5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3d_c5_$i.log 2>&1
TMD_EPOCH_SYNC=1 timeout 600 python bench.py --workload c5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3d_c5sync_$i.log 2>&1
done
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r3d_bench.log 2>&1

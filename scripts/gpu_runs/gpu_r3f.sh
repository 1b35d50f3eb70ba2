cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3f_pytest.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r3f_bench.log 2>&1
timeout 600 python bench.py --workload c5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3f_c5.log 2>&1
TMD_EPOCH_SYNC=1 timeout 600 python bench.py --workload c5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3f_c5sync.log 2>&1
timeout 600 python bench.py --workload c3 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3f_c3.log 2>&1

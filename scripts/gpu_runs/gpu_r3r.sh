cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3r_pytest.log 2>&1
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/r3r_mgpu.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r3r_mgpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/r3r_bench_n2.log 2>&1
TMD_OVERLAP=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r3r_bench_n2_noov.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 2 --workload c3 --steps 100 --warmup 5 --no-e2e > gpurun_out/r3r_c3_n2.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/profile_rebuild_mgpu.py 80 > gpurun_out/r3a_rebuild_p2.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r3a_pytest.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/r3a_bench_n2.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r3a_bench.log 2>&1

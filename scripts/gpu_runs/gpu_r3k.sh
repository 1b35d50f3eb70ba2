cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3k_pytest.log 2>&1
TMD_BUILD_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or lists or fused or lj80 or lj32" > gpurun_out/r3k_pytest_v1.log 2>&1
for v in 0 1 0 1; do TMD_BUILD_VARIANT=$v timeout 300 python scripts/profile_rebuild.py 80 2>&1 | grep "k_build" >> gpurun_out/r3k_build_v$v.log; done
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/r3k_mgpu.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r3k_mgpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/r3k_bench_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29642 bench.py --gpus 2 --workload c3 --steps 100 --warmup 5 --no-e2e > gpurun_out/r3k_c3_n2.log 2>&1

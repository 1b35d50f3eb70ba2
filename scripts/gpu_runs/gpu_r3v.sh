cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3v_pytest.log 2>&1
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/r3v_mgpu.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r3v_mgpu.log
for g in 1 0 1 0; do
TMD_MAIL_GATHER=$g timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2967$g bench.py --gpus 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r3v_n2_g$g.log 2>&1
TMD_MAIL_GATHER=$g timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2968$g bench.py --gpus 2 --workload c3 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r3v_c3n2_g$g.log 2>&1
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/r8a_mgpu_$NG.log 2>&1
echo "mgpu exit $?" >> gpurun_out/r8a_mgpu_$NG.log
for n in 2 $NG; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2981$n bench.py --gpus $n --steps 100 --warmup 5 > gpurun_out/r8a_bench_n$n.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2982$n bench.py --gpus $n --workload c3 --steps 100 --warmup 5 --no-e2e > gpurun_out/r8a_c3_n$n.log 2>&1
done
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/r8a_bench_n1.log 2>&1
timeout 600 python bench.py --workload c3 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r8a_c3_n1.log 2>&1
timeout 600 python bench.py --workload c5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r8a_c5_n1.log 2>&1
start=$(date +%s)
timeout 900 python bench.py --impl reference --steps 100 --warmup 5 > gpurun_out/r8a_ref_n1.log 2>&1; echo "rc $? wall $(( $(date +%s) - start )) s" >> gpurun_out/r8a_ref_n1.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
start=$(date +%s)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29691 bench.py --impl reference --gpus 2 --steps 100 --warmup 5 > gpurun_out/r5j_ref_n2.log 2> gpurun_out/r5j_ref_n2.err; echo "rc $? wall $(( $(date +%s) - start )) s" >> gpurun_out/r5j_ref_n2.log

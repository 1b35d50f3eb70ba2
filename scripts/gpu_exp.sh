cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TMD_TRACE_REBUILD=1 timeout 600 torchrun --standalone --nproc-per-node 2 scripts/mgpu_phases.py 80 100 > gpurun_out/phases2t.log 2>&1
TMD_TRACE_REBUILD=1 timeout 600 python scripts/mgpu_phases.py 80 100 > gpurun_out/phases1t.log 2>&1

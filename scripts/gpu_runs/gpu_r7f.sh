cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/trace_epoch_c5.py > gpurun_out/r7f_trace.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/profile_epoch.py --cells 80 --steps 45"
timeout 300 $CMD > gpurun_out/epoch_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_epoch.csv $CMD > gpurun_out/ncu_epoch.log 2>&1
echo done

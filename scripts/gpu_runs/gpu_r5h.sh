cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m paper_2009_07400_b200 --preset lj-32 --json > gpurun_out/r5h_cli_lj32.log 2>&1; echo "rc $?" >> gpurun_out/r5h_cli_lj32.log
timeout 300 python -m paper_2009_07400_b200 --nx 16 --ny 16 --nz 16 --steps 100 --ranks 4 --dump gpurun_out/r5h_traj.xyz --dump-every 20 > gpurun_out/r5h_cli_ranks4.log 2>&1; echo "rc $?" >> gpurun_out/r5h_cli_ranks4.log
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 -m paper_2009_07400_b200 --nx 32 --ny 16 --nz 16 --steps 100 --json > gpurun_out/r5h_cli_torchrun.log 2>&1; echo "rc $?" >> gpurun_out/r5h_cli_torchrun.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r5h_smoke.log 2>&1

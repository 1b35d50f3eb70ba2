cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5; do
 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r8w_pytest_$i.log 2>&1; echo "pytest $i rc $? $(tail -1 gpurun_out/r8w_pytest_$i.log)"
done

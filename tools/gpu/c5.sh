cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/c5_long.py > gpurun_out/c5_long.log 2>&1; echo "rc=$?" >> gpurun_out/c5_long.log

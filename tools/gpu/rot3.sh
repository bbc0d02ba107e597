cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ICB_PROF=1 timeout 900 python tools/time_rotation.py 131072 > gpurun_out/rot_c3.log 2>&1

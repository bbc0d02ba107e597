cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_cta_stability.py > gpurun_out/stab.log 2>&1

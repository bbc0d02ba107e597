cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 32768 131072; do timeout 600 python tools/prof_phases.py $c; done > gpurun_out/scan_stats.log 2>&1

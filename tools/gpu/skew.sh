cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_phases.py > gpurun_out/phases_skew.log 2>&1
timeout 600 python bench.py --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/b_c2.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/prof_step_phases.py 131072 34 > gpurun_out/phase_c3.log 2>&1
timeout 900 python tools/prof_step_phases.py 32768 34 > gpurun_out/phase_c2.log 2>&1

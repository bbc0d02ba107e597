cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KPROF=1 timeout 600 python tools/time_prefill.py 131072 > gpurun_out/tc_kprof_c3.log 2>&1
KPROF=1 timeout 600 python tools/time_prefill.py 32768 > gpurun_out/tc_kprof_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nn_tc_filter -s 2 -c 1 -o gpurun_out/prof_tc_c2 python tools/time_prefill.py 32768 > gpurun_out/ncu_tc_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nn_tc_filter -s 2 -c 1 -o gpurun_out/prof_tc_c3 python tools/time_prefill.py 131072 > gpurun_out/ncu_tc_c3.log 2>&1

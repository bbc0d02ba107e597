cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_forest.py -x -q -p no:cacheprovider -k "build" > gpurun_out/tc7_t1.log 2>&1; echo "rc=$?" >> gpurun_out/tc7_t1.log
grep -q "rc=0" gpurun_out/tc7_t1.log || exit 1
for ctx in 32768 131072; do ICB_PROF=1 timeout 600 python tools/time_prefill.py $ctx; done > gpurun_out/tc7_prefill.log 2>&1
KPROF=1 timeout 600 python tools/time_prefill.py 131072 2>&1 | grep -E "icb::|prefill" > gpurun_out/tc7_kprof.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nn_tc_filter -s 2 -c 1 -o /tmp/prof_tc7_c3 python tools/time_prefill.py 131072 > gpurun_out/ncu_tc7.log 2>&1
python tools/ncu_summary.py /tmp/prof_tc7_c3.ncu-rep nn_tc_filter gpurun_out/r02_nn_tc_filter_c3_ncu_summary.json > /dev/null 2>&1
python tools/ncu_lines.py /tmp/prof_tc7_c3.ncu-rep 30 > gpurun_out/tc7_lines.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_forest.py tests/test_gpu_large.py tests/test_gpu_dci_api.py -x -q -p no:cacheprovider > gpurun_out/tc7_t2.log 2>&1; echo "rc=$?" >> gpurun_out/tc7_t2.log

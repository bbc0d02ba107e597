cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_forest.py -x -q -p no:cacheprovider -k "build" > gpurun_out/tc_t1.log 2>&1; echo "rc=$?" >> gpurun_out/tc_t1.log
grep -q "rc=0" gpurun_out/tc_t1.log || exit 1
for ctx in 32768 131072; do
  for mode in TC F16 EXACT; do
    case $mode in F16) export ICB_BUILD_F16_FILTER=1;; EXACT) export ICB_BUILD_EXACT_NN=1;; esac
    echo "== $mode ctx=$ctx"
    ICB_PROF=1 timeout 600 python tools/time_prefill.py $ctx
    unset ICB_BUILD_F16_FILTER ICB_BUILD_EXACT_NN
  done
done > gpurun_out/tc_prefill.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_forest.py tests/test_gpu_large.py tests/test_gpu_dci_api.py -x -q -p no:cacheprovider > gpurun_out/tc_t2.log 2>&1; echo "rc=$?" >> gpurun_out/tc_t2.log

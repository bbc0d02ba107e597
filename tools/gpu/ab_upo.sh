cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=paper_2604_10539_b200
timeout 900 python -m pytest tests/test_gpu_forest.py tests/test_gpu_large.py tests/test_gpu_engine.py tests/test_gpu_dci_api.py -x -q -p no:cacheprovider > gpurun_out/upo_tests.log 2>&1; echo "rc=$?" >> gpurun_out/upo_tests.log
for c in 32768 131072; do timeout 600 python tools/prof_phases.py $c | grep -E "sub-phases|union|scan|per-CTA"; done > gpurun_out/upo_phases.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 2 > gpurun_out/ab_upo_c2.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 1 --ctx 131072 > gpurun_out/ab_upo_c3.log 2>&1

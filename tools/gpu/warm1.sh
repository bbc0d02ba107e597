cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=paper_2604_10539_b200
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/warm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/warm_tests.log
for c in 32768 131072; do timeout 600 python tools/time_prefill.py $c; done > gpurun_out/warm_prefill.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 2 > gpurun_out/ab_warm_c2.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 1 --ctx 131072 > gpurun_out/ab_warm_c3.log 2>&1

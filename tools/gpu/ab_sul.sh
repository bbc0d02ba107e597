cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=paper_2604_10539_b200
timeout 900 python -m pytest tests/test_gpu_forest.py tests/test_gpu_large.py tests/test_gpu_engine.py tests/test_gpu_dci_api.py -x -q -p no:cacheprovider > gpurun_out/sul_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sul_tests.log
for c in 32768 131072; do timeout 600 python tools/prof_phases.py $c | grep -E "sub-phases|union|scan|per-CTA"; done > gpurun_out/sul_phases.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 2 > gpurun_out/ab_sul_c2.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 1 --ctx 131072 > gpurun_out/ab_sul_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"query_kernel|dense_|insert_kernel|append|gather|attn_kernel|pages_from|rotate" --csv --log-file gpurun_out/launches_bench2.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches2.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launches2.log

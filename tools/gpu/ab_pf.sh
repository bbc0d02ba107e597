cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/ab.sh paper_2604_10539_b200/libicecache_b200_nopf.so paper_2604_10539_b200/libicecache_b200.so 2 > gpurun_out/ab_pf_c2.log 2>&1
bash tools/ab.sh paper_2604_10539_b200/libicecache_b200_nopf.so paper_2604_10539_b200/libicecache_b200.so 1 --ctx 131072 > gpurun_out/ab_pf_c3.log 2>&1
timeout 600 python tools/time_prefill.py > gpurun_out/prefill_c2.log 2>&1

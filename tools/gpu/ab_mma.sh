cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/mma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mma_tests.log
bash tools/ab.sh paper_2604_10539_b200/libicecache_b200_prev.so paper_2604_10539_b200/libicecache_b200.so 2 > gpurun_out/ab_mma_c2.log 2>&1
ICB_ATTN_SIMT=1 bash tools/ab.sh paper_2604_10539_b200/libicecache_b200.so paper_2604_10539_b200/libicecache_b200.so 1 > gpurun_out/ab_mma_c2_simt.log 2>&1
bash tools/ab.sh paper_2604_10539_b200/libicecache_b200_prev.so paper_2604_10539_b200/libicecache_b200.so 1 --ctx 131072 > gpurun_out/ab_mma_c3.log 2>&1
timeout 300 python tools/prof_phases.py > gpurun_out/phases_mma.log 2>&1

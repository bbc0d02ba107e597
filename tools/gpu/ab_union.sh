cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=paper_2604_10539_b200
for L in $P/libicecache_b200_prev.so $P/libicecache_b200.so; do
  echo "== $L"
  for c in 32768 131072; do ICB_LIB=$L timeout 600 python tools/prof_phases.py $c | grep -E "union|scan|per-CTA"; done
done > gpurun_out/ab_union_phases.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 2 > gpurun_out/ab_union_c2.log 2>&1
bash tools/ab.sh $P/libicecache_b200_prev.so $P/libicecache_b200.so 1 --ctx 131072 > gpurun_out/ab_union_c3.log 2>&1

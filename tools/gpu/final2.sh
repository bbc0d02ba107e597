cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/b_default.log 2>&1; echo "rc=$?" >> $O/b_default.log
for c in 32768 131072; do ICB_PROF=1 timeout 600 python tools/time_prefill.py $c; done > $O/prefill.log 2>&1

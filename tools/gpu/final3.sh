cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final3
O=gpurun_out/final3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/b_k20.log 2>&1; echo "rc=$?" >> $O/b_k20.log

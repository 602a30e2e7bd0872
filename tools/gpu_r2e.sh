# single GPU: whole pytest -m gpu (incl. the reference suite with its acceptance criteria),
# smoke, default bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2e; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 1800 python -m pytest tests/test_gpu_reference_suite.py -q -s > $O/pytest_refsuite.log 2>&1; echo rc=$? >> $O/pytest_refsuite.log
timeout 900 python bench.py > $O/bench_n1.log 2>&1; echo rc=$? >> $O/bench_n1.log
tail -3 $O/*.log | cut -c1-300

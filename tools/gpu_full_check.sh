#!/bin/bash
# full single-GPU check: pytest -m gpu, smoke, bench N=1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-full}
mkdir -p $o
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $o/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 900 python bench.py > $o/bench.json 2> $o/bench.err; echo "bench rc=$?" >> $o/bench.err
tail -3 $o/pytest_gpu.log; tail -2 $o/smoke.log; cat $o/bench.json | head -c 1500; tail -2 $o/bench.err

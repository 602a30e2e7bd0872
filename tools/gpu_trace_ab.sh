#!/bin/bash
# trace reductions: parity tests, A/B timing (compile-time-shaped vs runtime-L kernels, exact
# order), ncu --set full of the C2 fp32 tile-kernel launch
cd "${GRAFT_REPO_ROOT:-/root/repo}"
o=gpurun_out/${1:-trace_ab}
mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_objectives.py tests/test_gpu_harness.py -q -p no:cacheprovider > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
timeout 600 python tools/bench_trace.py > $o/bench_trace.jsonl 2> $o/bench_trace.err
cat > /tmp/tr1.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
from paper_2002_01119_b200 import mixing, objectives, simulation
L, d = 64, 25_557_032
o = objectives.quadratic_oracle(d, condition_number=7.0, noise_scale=0.0, seed=1)
X = mixing.empty_learner_major(L, d, torch.float32, "cuda").normal_()
for _ in range(3):
    simulation.trace_stats(X.T, o, exact=False)
torch.cuda.synchronize()
PY
[ -n "$NCU" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:trace_tile -s 1 -c 1 -o $o/trace_c2_tile python /tmp/tr1.py > $o/ncu.log 2>&1
tail -3 $o/pytest.log; cat $o/bench_trace.jsonl; tail -3 $o/bench_trace.err

"""Time the fused trace reductions (rm_trace_stats_*) at C2: one pass over W."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_01119_b200 import mixing, objectives, simulation as S

for L, d, dt in [(64, 25_557_032, torch.float32), (16, 1 << 20, torch.float32), (64, 25_557_032, torch.float64)]:
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1)
    X = mixing.empty_learner_major(L, d, dt, "cuda").normal_()
    for _ in range(3): S.trace_stats(X.T, oracle)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); S.trace_stats(X.T, oracle); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    byts = L * d * X.element_size() + 2 * 8 * d
    print(json.dumps({"L": L, "d": d, "dtype": str(dt), "ms": ms, "GBs": byts / (ms / 1e3) / 1e9}), flush=True)
    del X

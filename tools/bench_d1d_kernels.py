"""Single-GPU timing of the D1D partial-sum and apply kernels at a shard shape."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_01119_b200 import _lib, mixing
Lg, d = int(os.environ.get("LG", 16)), 25_557_032
dev = torch.device("cuda")
W = mixing.empty_learner_major(Lg, d, torch.float32, dev); W.normal_()
G = mixing.empty_learner_major(Lg, d, torch.float32, dev); G.normal_()
O = mixing.empty_learner_major(Lg, d, torch.float32, dev)
S = torch.randn(d, dtype=torch.float64, device=dev)
lib = _lib.load(); s = _lib.stream_ptr()
def t(fn, n=10):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
tp = t(lambda: lib.rm_partial_sum_f32(W.data_ptr(), Lg, d, W.stride(0), S.data_ptr(), s))
ta = t(lambda: lib.rm_apply_mean_sgd_f32(S.data_ptr(), G.data_ptr(), O.data_ptr(), Lg, 1, d, G.stride(0), O.stride(0), 0.01, None, s))
print(json.dumps({"Lg": Lg, "partial_ms": tp, "partial_GBs": (Lg * d * 4 + d * 8) / tp / 1e6,
                  "apply_ms": ta, "apply_GBs": (2 * Lg * d * 4 + d * 8) / ta / 1e6}), flush=True)

"""One C2 gradient pass (for an ncu launch list of the normal-generator kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_01119_b200 import mixing, objectives
from paper_2002_01119_b200.simulation import RunConfig
L, d = int(sys.argv[1]), int(sys.argv[2])
oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1, optimum=np.zeros(d))
Phi = mixing.empty_learner_major(L, d, torch.float32, torch.device("cuda")); Phi.normal_()
cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")
for k in range(2):
    oracle.device_gradients(Phi, cfg, k)
torch.cuda.synchronize()
print("ok")
ts = []
for k in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); oracle.device_gradients(Phi, cfg, 10 + k); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("grad_ms", sorted(ts)[len(ts) // 2], os.environ.get("TAG", ""))

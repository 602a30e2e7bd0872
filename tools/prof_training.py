"""Where does a run_training iteration spend its time?  torch.profiler over C2 RAD."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2002_01119_b200 import objectives, simulation as S
L, d = 64, 25_557_032
oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1)
cfg = S.RunConfig(n_learners=L, iterations=4, lr=0.01, batch_size=32, seed=5, dtype="float32", log_every=4)
S.run_training(S.Strategy.RAND_PSGD, oracle, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    S.run_training(S.Strategy.RAND_PSGD, oracle, cfg)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25, max_name_column_width=60))

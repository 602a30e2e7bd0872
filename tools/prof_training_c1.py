import cProfile, pstats, sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2002_01119_b200 import objectives, simulation as S
L, d = 16, 1 << 20
oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1)
cfg = S.RunConfig(n_learners=L, iterations=40, lr=0.01, batch_size=32, seed=5, dtype="float32", log_every=40)
S.run_training(S.Strategy.RAND_PSGD, oracle, S.RunConfig(n_learners=L, iterations=2, lr=0.01, batch_size=32, seed=5))
torch.cuda.synchronize()
t=time.perf_counter(); S.run_training(S.Strategy.RAND_PSGD, oracle, cfg); torch.cuda.synchronize(); print("s/iter", (time.perf_counter()-t)/40)
pr = cProfile.Profile(); pr.enable()
S.run_training(S.Strategy.RAND_PSGD, oracle, cfg); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)

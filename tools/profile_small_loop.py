"""Host-side profile of run_training at a tiny shape (the acceptance-criterion 8 cell):
where does the per-iteration time go when the GPU work is microseconds?"""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_01119_b200 import objectives, simulation
from paper_2002_01119_b200.simulation import RunConfig, Strategy

oracle = objectives.quadratic_oracle(dimension=32, condition_number=10.0, optimum=np.zeros(32),
                                     noise_scale=4.0, seed=0)
cfg = RunConfig(n_learners=32, iterations=1000, lr=9e-4, batch_size=8, seed=1, init_scale=0.0,
                log_every=1000)
simulation.run_training(Strategy.RAND_PSGD, oracle, cfg)
torch.cuda.synchronize()
t = time.perf_counter()
simulation.run_training(Strategy.RAND_PSGD, oracle, cfg)
torch.cuda.synchronize()
print("ms/iter", (time.perf_counter() - t) / cfg.iterations * 1e3)
pr = cProfile.Profile()
pr.enable()
simulation.run_training(Strategy.RAND_PSGD, oracle, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

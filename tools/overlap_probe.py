"""Can the gradient producer (compute-bound) overlap the fused mix (HBM-bound)?
C2 shapes, independent data: sequential vs concurrent on two streams."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_01119_b200 import mixing, objectives, simulation
from paper_2002_01119_b200.simulation import RunConfig

L, d = 64, 25_557_032
dev = torch.device("cuda")
oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1)
cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")
Phi = mixing.empty_learner_major(L, d, torch.float32, dev).normal_()
W = [mixing.empty_learner_major(L, d, torch.float32, dev).normal_() for _ in range(2)]
G = mixing.empty_learner_major(L, d, torch.float32, dev).normal_()
lt, rt = simulation.rad_tables(L, 12345, 0, dev)
side = torch.cuda.Stream()

def mix(n=1):
    for i in range(n):
        mixing.ring_mix_sgd(W[i % 2], G, 0.01, lt, rt, out=W[1 - i % 2])

def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)

for _ in range(2):
    oracle.device_gradients(Phi, cfg, 0); mix()
res = {}
res["grad_ms"] = timed(lambda: oracle.device_gradients(Phi, cfg, 1))
res["mix_ms"] = timed(lambda: mix())
res["mix3_ms"] = timed(lambda: mix(3))
res["sequential_ms"] = timed(lambda: (oracle.device_gradients(Phi, cfg, 2), mix()))

def conc(nmix):
    def f():
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            oracle.device_gradients(Phi, cfg, 3)
        mix(nmix)
        torch.cuda.current_stream().wait_stream(side)
    return f
res["concurrent_1mix_ms"] = timed(conc(1))
res["concurrent_3mix_ms"] = timed(conc(3))
print(json.dumps(res))

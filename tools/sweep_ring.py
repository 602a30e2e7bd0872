"""Tuning sweep for the ring mix kernel at C2 (run with RINGMIX_RING_NT / RINGMIX_STAGE_KB)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_01119_b200 import mixing, simulation
L, d = int(os.environ.get("SW_L", 64)), int(os.environ.get("SW_D", 25_557_032))
dev = torch.device("cuda")
W = [mixing.empty_learner_major(L, d, torch.float32, dev) for _ in range(2)]
W[0].normal_(); G = mixing.empty_learner_major(L, d, torch.float32, dev); G.normal_()
lt, rt = simulation.rad_tables(L, 12345, 0, dev)
for kb in [int(x) for x in os.environ.get("SW_KB", "0").split(",")]:
    if kb: os.environ["RINGMIX_STAGE_KB"] = str(kb)
    else: os.environ.pop("RINGMIX_STAGE_KB", None)
    for i in range(4): mixing.ring_mix_sgd(W[i % 2], G, 0.01, lt, rt, out=W[1 - i % 2])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    a.record()
    for i in range(n): mixing.ring_mix_sgd(W[i % 2], G, 0.01, lt, rt, out=W[1 - i % 2])
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    print(json.dumps({"nt": os.environ.get("RINGMIX_RING_NT", "512"), "stage_kb": kb, "L": L,
                      "ms": ms, "GBs": 12 * L * d / ms / 1e6}), flush=True)

"""C1 (16 x 1,048,576 fp32, the reference's demo scale) tuning sweep of the ring tile:
stage bytes (RINGMIX_STAGE_KB) x tile width (RINGMIX_TILE_COLS); back-to-back launches
timed as a block, like the bench's steps."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_01119_b200 import mixing, simulation

L, d = 16, 1 << 20
dev = torch.device("cuda")
W = [mixing.empty_learner_major(L, d, torch.float32, dev).normal_() for _ in range(2)]
G = mixing.empty_learner_major(L, d, torch.float32, dev).normal_()
lt, rt = simulation.rad_tables(L, 12345, 0, dev)
for kb in ["", "8", "12", "16", "24", "32", "48"]:
    for cw in ["", "64", "128", "256", "512"]:
        for k, v in (("RINGMIX_STAGE_KB", kb), ("RINGMIX_TILE_COLS", cw)):
            if v: os.environ[k] = v
            else: os.environ.pop(k, None)
        try:
            for i in range(5): mixing.ring_mix_sgd(W[i % 2], G, 0.01, lt, rt, out=W[1 - i % 2])
            torch.cuda.synchronize()
            res = []
            for rep in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for i in range(100): mixing.ring_mix_sgd(W[i % 2], G, 0.01, lt, rt, out=W[1 - i % 2])
                b.record(); torch.cuda.synchronize(); res.append(a.elapsed_time(b) / 100)
            ms = statistics.median(res)
            print(json.dumps({"stage_kb": kb or "auto", "cw": cw or "auto", "us": round(ms * 1e3, 2),
                              "GBs": round(12 * L * d / (ms / 1e3) / 1e9, 1)}), flush=True)
        except Exception as e:
            print(json.dumps({"stage_kb": kb, "cw": cw, "error": str(e)[:80]}), flush=True)

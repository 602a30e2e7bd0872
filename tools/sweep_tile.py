"""Tuning sweep: time the fused RAD mix kernel at several tile widths (RINGMIX_TILE_COLS)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_01119_b200 import mixing, simulation

def bench(L, d, cws, reps=20, dtype=torch.float32):
    dev = torch.device("cuda")
    W = mixing.empty_learner_major(L, d, dtype, dev); W.normal_()
    G = mixing.empty_learner_major(L, d, dtype, dev); G.normal_()
    O = mixing.empty_learner_major(L, d, dtype, dev)
    lt, rt = simulation.rad_tables(L, 12345, 0, dev)
    res = {}
    for cw in cws:
        if cw:
            os.environ["RINGMIX_TILE_COLS"] = str(cw)
        else:
            os.environ.pop("RINGMIX_TILE_COLS", None)
        for _ in range(3):
            mixing.ring_mix_sgd(W, G, 0.01, lt, rt, out=O)
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); mixing.ring_mix_sgd(W, G, 0.01, lt, rt, out=O); b.record()
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        gbs = (2 if dtype == torch.bfloat16 else 4) * 3 * L * d / (ms / 1e3) / 1e9
        res[cw] = (ms, gbs)
        print(json.dumps({"L": L, "d": d, "cw": cw, "ms": ms, "GBs": gbs}), flush=True)
    os.environ.pop("RINGMIX_TILE_COLS", None)
    return res

if __name__ == "__main__":
    bench(64, 25_557_032, [0, 32, 64, 128])
    bench(16, 1 << 20, [0, 128, 256, 512, 1024], reps=50)
    bench(16, 16 << 20, [0, 256, 512, 1024, 2048])
    bench(128, 43_154_944 // 4, [0, 32, 64])

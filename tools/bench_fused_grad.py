"""Training step with the quadratic oracle at a BASELINE shape (default C2: 64 x 25,557,032
fp32): gradient pass + ring mix (two passes, G in HBM) against the fused step
(rm_quadratic_mix_step_*: G produced in the mix kernel's epilogue).  Checks the two agree
bit for bit, prints median step times.

  python tools/bench_fused_grad.py [L] [d] [reps] [stale] [uniform]
uniform=1: the D1D step (uniform matrix) instead of the randomized ring.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_01119_b200 import mixing, objectives, simulation  # noqa: E402
from paper_2002_01119_b200.simulation import RunConfig  # noqa: E402


def main(L=64, d=25_557_032, reps=7, stale=0, uniform=0):
    dev = torch.device("cuda")
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                         optimum=np.zeros(d))
    X = mixing.empty_learner_major(L, d, torch.float32, dev).normal_()
    Phi = mixing.empty_learner_major(L, d, torch.float32, dev).normal_() if stale else None
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")

    def two_pass(k):
        G = oracle.device_gradients(X if Phi is None else Phi, cfg, k)
        if uniform:
            return mixing.mean_mix_sgd(X, G, 0.01)
        tabs = simulation.rad_tables(L, cfg.seed, k, dev)
        return mixing.ring_mix_sgd(X, G, 0.01, tabs[0], tabs[1])

    def fused(k):
        tabs = None if uniform else simulation.rad_tables(L, cfg.seed, k, dev)
        return oracle.device_mix_step(X, Phi, tabs, 0.01, cfg, k)

    res = {}
    for name, fn in (("two_pass", two_pass), ("fused", fused), ("two_pass", two_pass),
                     ("fused", fused)):
        for k in range(2):
            fn(k)
        torch.cuda.synchronize()
        ts = []
        for r in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = fn(10 + r)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            del out
        res.setdefault(name, []).append(float(np.median(ts)))
    same = bool(torch.equal(two_pass(3), fused(3)))
    print(json.dumps({"L": L, "d": d, "stale": bool(stale), "uniform": bool(uniform),
                      "step_ms": res,
                      "bit_identical": same}), flush=True)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]]
    main(*args)

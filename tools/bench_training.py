"""Full reference training loop on the GPU: run_training(RAD-PSGD, quadratic oracle)
through the drop-in API — per iteration the device gradient producer (bit-exact numpy
normals), the fused mix + SGD + divergence epilogue, the 8-byte divergence read-back,
the simulated clock, and (log_every) the fused trace reductions.

  python tools/bench_training.py [--ref]   (--ref: time the reference package on this
                                            host's CPU instead; needs /root/reference)
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CASES = [("C1", 16, 1 << 20, 20), ("C2", 64, 25_557_032, 10)]


def ours(dtype):
    import numpy as np
    import torch
    from paper_2002_01119_b200 import objectives, simulation as S
    for name, L, d, iters in CASES:
        oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1)
        for log_every in (1, iters):
            cfg = S.RunConfig(n_learners=L, iterations=iters, lr=0.01, batch_size=32, seed=5,
                              dtype=dtype, log_every=log_every)
            # warm-up with the timed configuration itself: kernels loaded and the caching
            # allocator's pool grown to the loop's footprint before the clock starts
            S.run_training(S.Strategy.RAND_PSGD, oracle, cfg)
            torch.cuda.synchronize()
            t = time.perf_counter()
            res = S.run_training(S.Strategy.RAND_PSGD, oracle, cfg)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            print(json.dumps({"impl": "ours", "case": name, "L": L, "d": d, "dtype": dtype,
                              "iterations": iters, "log_every": log_every,
                              "s_per_iter": dt / iters, "learner_params_per_s": L * d * iters / dt,
                              "records": len(res.records), "diverged": res.diverged}), flush=True)


def reference(iters_cap):
    sys.path.insert(0, "/root/reference/pkg/src")
    from ringmix import objectives, simulation as S
    for name, L, d, iters in CASES[:1]:
        iters = min(iters, iters_cap)
        oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1)
        cfg = S.RunConfig(n_learners=L, iterations=iters, lr=0.01, batch_size=32, seed=5,
                          log_every=iters)
        t = time.perf_counter()
        S.run_training(S.Strategy.RAND_PSGD, oracle, cfg)
        dt = time.perf_counter() - t
        print(json.dumps({"impl": "reference", "case": name, "L": L, "d": d, "iterations": iters,
                          "s_per_iter": dt / iters, "learner_params_per_s": L * d * iters / dt,
                          "cores": os.cpu_count()}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--dtype", default="float32")
    a = ap.parse_args()
    reference(3) if a.ref else ours(a.dtype)

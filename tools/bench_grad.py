"""Time the device quadratic-gradient producer (bit-exact numpy normals) and the
full device training step (gradient + fused RAD mix) at a given shape."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_01119_b200 import mixing, objectives, simulation
from paper_2002_01119_b200.simulation import RunConfig

def main(L, d, reps=5):
    dev = torch.device("cuda")
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                         optimum=np.zeros(d))
    Phi = mixing.empty_learner_major(L, d, torch.float32, dev); Phi.normal_()
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")
    for k in range(2):
        oracle.device_gradients(Phi, cfg, k)
    torch.cuda.synchronize()
    ts = []
    for k in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); G = oracle.device_gradients(Phi, cfg, 10 + k); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    # spot-check two learners vs numpy
    ok = True
    for l in (0, L - 1):
        z = np.random.default_rng(np.random.SeedSequence((5, 0, 10 + reps - 1, l))).standard_normal(d)
        ref = oracle.eigenvalues * (Phi[l].double().cpu().numpy() - 0.0) + (1.0 / np.sqrt(32)) * z
        ok &= bool(np.array_equal(G[l].double().cpu().numpy(), ref.astype(np.float32).astype(np.float64)))
    print(json.dumps({"L": L, "d": d, "grad_ms": float(np.median(ts)), "normals_per_s": L * d / (np.median(ts) / 1e3),
                      "bit_exact_spotcheck": ok}), flush=True)

def d1d_overlap(L, d, steps=5):
    """D1D training step with the device quadratic oracle: sequential (gradient then
    fused mean+SGD) vs overlapped (mean of W_k on a side stream || gradient of W_{k-1})."""
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                         optimum=np.zeros(d))
    cfg = RunConfig(n_learners=L, iterations=steps, lr=0.01, batch_size=32, seed=5,
                    dtype="float32")
    st = simulation.initial_state(oracle, cfg)
    res = {}
    for mode in ("sequential", "overlapped", "sequential", "overlapped"):
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if mode == "overlapped":
                simulation.D1D_SIDE_STREAM = True
                st = simulation.step_d1d(st, oracle, cfg)
                simulation.D1D_SIDE_STREAM = False
            else:
                st = simulation._gossip_step(st, oracle, cfg, None, stale=True)
            b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        res[mode] = float(np.median(ts))
    print(json.dumps({"L": L, "d": d, "d1d_step_ms": res}), flush=True)




def failure_stats(L, d):
    from paper_2002_01119_b200 import _lib
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                         optimum=np.zeros(d))
    Phi = mixing.empty_learner_major(L, d, torch.float32, torch.device("cuda")); Phi.normal_()
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")
    oracle.device_gradients(Phi, cfg, 3)
    torch.cuda.synchronize()
    off = _lib.load().rm_normal_stats_offset(L, d)
    cnt = oracle._ws[off:off + 8].cpu().numpy().view(np.uint32)
    nblocks = int((1.04 * d + 64.0 * np.sqrt(d + 1.0)) / 256) + 8
    print(json.dumps({"L": L, "d": d, "blocks": L * nblocks, "spec_failures": int(cnt[0]),
                      "left_to_sequential": int(cnt[1])}), flush=True)


def compare_paths(L, d, reps=3):
    """Fast (scratch-copy) vs compact (re-draw) generator layouts: identical bits, timing."""
    Phi = mixing.empty_learner_major(L, d, torch.float32, torch.device("cuda")); Phi.normal_()
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")
    out, ms = {}, {}
    for mode in ("1", "0"):
        os.environ["RINGMIX_NORMAL_FAST"] = mode
        oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                             optimum=np.zeros(d))
        oracle.device_gradients(Phi, cfg, 0)
        ts = []
        for k in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); G = oracle.device_gradients(Phi, cfg, 7); b.record()
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        out[mode], ms[mode] = G, float(np.median(ts))
        del oracle
        torch.cuda.empty_cache()
    os.environ["RINGMIX_NORMAL_FAST"] = "1"
    print(json.dumps({"L": L, "d": d, "fast_ms": ms["1"], "compact_ms": ms["0"],
                      "identical": bool(torch.equal(out["1"], out["0"]))}), flush=True)


if __name__ == "__main__":
    compare_paths(16, 1 << 20)
    compare_paths(64, 25_557_032)
    main(16, 1 << 20)
    main(64, 25_557_032)
    d1d_overlap(64, 25_557_032)
    failure_stats(16, 1 << 20)
    failure_stats(64, 25_557_032)

"""Single-GPU D1D training step with the device quadratic oracle (BASELINE configs[3], C4:
64 learners x 25,557,032 fp32): W_{k+1} = mean(W_k) - lr G(W_{k-1}) (simulation.py:304-312).

  two_pass      gradient to HBM, then the fused mean+SGD kernel (the kept-gradient step)
  fused_serial  rm_quadratic_mix_step (uniform): column mean, generator, final pass writes the step
  overlap(c)    simulation.step_d1d: column mean on a side stream capped at c CTAs/SM beside
                the generator, the final pass waits for it (default path)

Prints median step ms per mode and whether every mode gives the same bits.
  python tools/d1d_step_probe.py [L] [d] [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_01119_b200 import mixing, objectives, simulation  # noqa: E402
from paper_2002_01119_b200.simulation import RunConfig  # noqa: E402


def main(L=64, d=25_557_032, steps=10):
    dev = torch.device("cuda")
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                         optimum=np.zeros(d))
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")
    g = torch.Generator(device=dev).manual_seed(3)
    W = mixing.empty_learner_major(L, d, torch.float32, dev)
    Wp = mixing.empty_learner_major(L, d, torch.float32, dev)
    W.copy_(torch.randn((L, d), generator=g, device=dev))
    Wp.copy_(torch.randn((L, d), generator=g, device=dev))
    st = simulation.SimState(weights=W.T, prev_weights=Wp.T, iteration=7, seed=cfg.seed,
                             sim_time_s=0.0, compute_time_s=np.zeros(L), last_gradients=None)
    caps = [int(c) for c in os.environ.get("D1D_CAPS", "2,4,8,16").split(",")]

    def run(mode):
        if mode == "two_pass":
            return simulation._gossip_step(st, oracle, cfg, None, stale=True,
                                           keep_gradients=True).weights
        if mode == "fused_serial":
            return oracle.device_mix_step(W, Wp, None, simulation.learning_rate(cfg, 7), cfg,
                                          7).T
        simulation.D1D_MEAN_CTAS = int(mode[8:-1])
        return simulation.step_d1d(st, oracle, cfg, keep_gradients=False).weights

    modes = ["two_pass", "fused_serial"] + [f"overlap({c})" for c in caps]
    res, outs = {}, {}
    for mode in modes + modes:
        for _ in range(2):
            run(mode)
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = run(mode)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res.setdefault(mode, []).append(round(float(np.median(ts)), 3))
        outs[mode] = out.clone()
    same = all(torch.equal(outs["two_pass"], outs[m]) for m in modes)
    print(json.dumps({"L": L, "d": d, "step_ms": res, "bit_identical": same}), flush=True)


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])

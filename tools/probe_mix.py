"""Mix-kernel A/B probe: ms per launch of rm_ring_mix_sgd_* over back-to-back launches
(CUDA events around the loop only), plus torch copy / triad ceilings at the same bytes.

  python tools/probe_mix.py [--L 64] [--d 25557032] [--dtype float32] [--ceiling]
Variant knobs are the library's environment switches (RINGMIX_RING_IMPL, RINGMIX_RING_NT,
RINGMIX_STAGE_KB, RINGMIX_TILE_COLS), read once per process."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_01119_b200 import mixing, simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=64)
ap.add_argument("--d", type=int, default=25_557_032)
ap.add_argument("--dtype", default="float32")
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ceiling", action="store_true")
ap.add_argument("--fixed", action="store_true")
ap.add_argument("--mode", choices=["ring", "mean"], default="ring")
args = ap.parse_args()
dt = getattr(torch, args.dtype)
esz = torch.tensor([], dtype=dt).element_size()
L, d = args.L, args.d
dev = torch.device("cuda")
W = [mixing.empty_learner_major(L, d, dt, dev) for _ in range(2)]
G = mixing.empty_learner_major(L, d, dt, dev)
for r in range(L):
    W[0][r].normal_()
    G[r].normal_()
if args.fixed:
    lt, rt = simulation.fixed_ring_tables(L, dev)
else:
    lt, rt = simulation.rad_tables(L, 12345, 0, dev)
bytes_ = 3 * L * d * esz


def timeit(fn, n):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


env = {k: v for k, v in os.environ.items() if k.startswith("RINGMIX_")}
for rep in range(args.reps):
    if args.mode == "mean":
        ms = timeit(lambda i: mixing.mean_mix_sgd(W[i % 2], G, 0.01, out=W[1 - i % 2]), args.n)
    else:
        ms = timeit(lambda i: mixing.ring_mix_sgd(W[i % 2], G, 0.01, lt, rt, out=W[1 - i % 2]),
                    args.n)
    print(json.dumps({"what": "mix", "L": L, "d": d, "dtype": args.dtype, "env": env, "rep": rep,
                      "ms": ms, "GBs": bytes_ / ms / 1e6}), flush=True)
# correctness spot check of this variant against the per-item formula on a few columns
cols = torch.randint(0, d, (64,), device=dev)
out = mixing.ring_mix_sgd(W[0], G, 0.01, lt, rt)
Wd, Gd = W[0][:, cols].double(), G[:, cols].double()
l64, r64 = lt.long(), rt.long()
idx = torch.stack([l64, torch.arange(L, device=dev), r64], 1).sort(1).values
t = 1.0 / 3.0
acc = Wd[idx[:, 0]] * t
acc = torch.addcmul(acc, Wd[idx[:, 1]], torch.full_like(acc, t))  # not FMA-exact; tolerance check
acc = torch.addcmul(acc, Wd[idx[:, 2]], torch.full_like(acc, t))
ref = (acc - 0.01 * Gd).to(dt)
err = (out[:, cols].double() - ref.double()).abs().max().item()
print(json.dumps({"what": "spot_check", "max_abs_err": err}), flush=True)

if args.ceiling:
    # flat views: the same bytes as the mix (2 reads + 1 write), torch's vectorised kernels
    del W, G
    torch.cuda.empty_cache()
    Wf, Gf, Of = (torch.randn(L * d, device=dev).to(dt) for _ in range(3))
    for rep in range(args.reps):
        ms = timeit(lambda i: torch.add(Wf, Gf, alpha=-0.01, out=Of), args.n)
        print(json.dumps({"what": "torch_triad", "ms": ms, "GBs": bytes_ / ms / 1e6}), flush=True)
        ms = timeit(lambda i: Of.copy_(Wf), args.n)
        print(json.dumps({"what": "torch_copy", "ms": ms,
                          "GBs": 2 * L * d * esz / ms / 1e6}), flush=True)

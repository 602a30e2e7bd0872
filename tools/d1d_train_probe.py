"""D1D training step of a learner-sharded run with the device quadratic oracle, serial
(gradient, then the fused one-kernel D1D step) against the paper's concurrency (global
average of W_k on a side stream + the NVLS reduction, overlapped with the gradient of
W_{k-1}) — distributed.ShardedD1DTrainer.  BASELINE configs[3] (C4: 64 learners x
25,557,032 fp32) split over the ranks.  Prints per-mode step times (max over ranks) and
whether both modes produce the same bits.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/d1d_train_probe.py [L] [d] [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2002_01119_b200 import distributed as D, mixing, objectives  # noqa: E402
from paper_2002_01119_b200.simulation import RunConfig  # noqa: E402


def main(L=64, d=25_557_032, steps=10):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    lay = D.ShardLayout(L, world)
    b, e = lay.bounds[rank]
    Lg = e - b
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                         optimum=np.zeros(d), device=dev)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=32, seed=5, dtype="float32")
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    W = mixing.empty_learner_major(Lg, d, torch.float32, dev)
    Wp = mixing.empty_learner_major(Lg, d, torch.float32, dev)
    W.copy_(torch.randn((Lg, d), generator=g, device=dev))
    Wp.copy_(torch.randn((Lg, d), generator=g, device=dev))
    outs = {}
    res = {}
    # RINGMIX_D1D_TRAIN_CTAS_LIST="16,0,0;1,0,1": overlap modes with those CTA caps
    caps = [tuple(int(x) for x in c.split(",")) for c in
            os.environ.get("RINGMIX_D1D_TRAIN_CTAS_LIST", "1,0,1").split(";")]
    # overlapped modes: "apply" = gradient to HBM then one apply pass, "fused" = the
    # generator's final pass writes M - lr G (rm_quadratic_mean_step_shard_*)
    kinds = os.environ.get("RINGMIX_D1D_TRAIN_KINDS", "apply,fused").split(",")
    modes = ["serial", "serial_fused"] + [f"{kd}{c}" for kd in kinds for c in caps]
    conf = {"serial": (False, None, False), "serial_fused": (False, None, True)}
    for kd in kinds:
        for c in caps:
            conf[f"{kd}{c}"] = (True, c, kd == "fused")
    for mode in modes + modes:
        ov, cap, fz = conf[mode]
        tr = D.ShardedD1DTrainer(L, d, Lg, b, dev, oracle, overlap=ov, ctas=cap, fuse_grad=fz)
        out = mixing.empty_learner_major(Lg, d, torch.float32, dev)
        for k in range(3):
            tr.step(W, Wp, cfg, k, 0.01, out)
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for k in range(steps):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            tr.step(W, Wp, cfg, 10 + k, 0.01, out)
            z.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(z)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t))
        res.setdefault(mode, []).append(float(np.median(ts)))
        tr.step(W, Wp, cfg, 3, 0.01, out)
        torch.cuda.synchronize()
        outs[mode] = out.clone()
        del tr
        torch.cuda.synchronize()
        dist.barrier()
    same = torch.tensor([int(all(torch.equal(outs["serial"], outs[m]) for m in modes))],
                        device=dev)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": world, "L": L, "d": d, "step_ms": res,
                          "bit_identical": bool(same.item())}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])

"""torchrun multi-GPU check of the learner-sharded RAD and D1D steps vs the
single-GPU kernels on the same data (run: torchrun --nproc-per-node N tools/dist_check.py)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2002_01119_b200 import distributed as D, mixing, simulation

def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    L, d = int(os.environ.get("CHK_L", 64)), int(os.environ.get("CHK_D", 1_000_003))
    g = torch.Generator(device=dev).manual_seed(11)
    full = torch.randn((L, d), generator=g, device=dev)          # same on every rank
    Gf = torch.randn((L, d), generator=g, device=dev)
    ring = D.LearnerShardedRing(L, d, torch.float32)
    b, e = ring.row0, ring.row0 + ring.Lg
    ring.W[0].copy_(full[b:e])
    Gl = mixing.empty_learner_major(ring.Lg, d, torch.float32, dev)
    Gl.copy_(Gf[b:e])
    torch.cuda.synchronize(); dist.barrier()
    ok = True
    pull_steps = []
    # 3 RAD steps sharded vs single-GPU reference computed locally on full data
    Wref = mixing.empty_learner_major(L, d, torch.float32, dev); Wref.copy_(full)
    for k in range(3):
        lt, rt = simulation.rad_tables(L, 12345, k, dev)
        out = ring.step(lt, rt, Gl, 0.01)
        Wref = mixing.ring_mix_sgd(Wref, mixing.empty_learner_major(L, d, torch.float32, dev).copy_(Gf), 0.01, lt, rt)
        torch.cuda.synchronize()
        same = bool(torch.equal(out, Wref[b:e]))
        pull_steps.append(same)
        ok &= same
    # D1D: each layout's rows are the learners it holds — numpy-order chains (bit-identical to
    # the one-GPU step) where the class uses them, else the contiguous block (fp64 rounding)
    ref = mixing.mean_mix_sgd(Wref, mixing.empty_learner_major(L, d, torch.float32, dev).copy_(Gf), 0.01)
    Lg = ring.Lg

    def shard(obj, X, dt=torch.float32):
        ids = torch.tensor(D.d1d_learners(L, world, rank, getattr(obj, "chains", 0)), device=dev)
        return ids, mixing.empty_learner_major(len(ids), d, dt, dev).copy_(X[ids].to(dt))

    def check(obj, out, ids, refm, tol=2e-6):
        if getattr(obj, "chains", 0):
            return bool(torch.equal(out, refm[ids]))
        return (out.double() - refm[ids].double()).abs().max().item() <= tol

    d1d = D.LearnerShardedD1D(L, d, Lg, dev, chunk_cols=1 << 18)
    ids, Wl = shard(d1d, Wref)
    _, Gs = shard(d1d, Gf)
    out = mixing.empty_learner_major(Lg, d, torch.float32, dev)
    d1d.step(Wl, Gs, 0.01, out)
    torch.cuda.synchronize()
    dd = (out.double() - ref[ids].double()).abs().max().item()
    ok_d1d = check(d1d, out, ids, ref)
    nvls = f"nccl chains={d1d.chains} maxdiff {dd:.2e}"
    # NVSwitch multicast variant (our own in-switch reduction kernel)
    try:
        outs = []
        for cc in (None, 1 << 16):   # one chunk, and the chunk pipeline
            nv = D.LearnerShardedD1DNVLS(L, d, Lg, dev, chunk_cols=cc)
            ids, Wl = shard(nv, Wref)
            _, Gs = shard(nv, Gf)
            out2 = mixing.empty_learner_major(Lg, d, torch.float32, dev)
            for _ in range(2):
                nv.step(Wl, Gs, 0.01, out2)
            torch.cuda.synchronize()
            ok_d1d = ok_d1d and check(nv, out2, ids, ref)
            outs.append(out2)
        ok_d1d = ok_d1d and bool(torch.equal(outs[0], outs[1]))
        nvls += f"; nvls {len(nv.chunks)} chunks chains={nv.chains}"
        # one-kernel variant over several epochs
        fu = D.LearnerShardedD1DFused(L, d, Lg, dev, chunk_cols=1 << 16)
        ids, Wl = shard(fu, Wref)
        _, Gs = shard(fu, Gf)
        out3 = mixing.empty_learner_major(Lg, d, torch.float32, dev)
        for _ in range(3):
            fu.step(Wl, Gs, 0.01, out3)
        torch.cuda.synchronize()
        ok3 = check(fu, out3, ids, ref)
        ok_d1d = ok_d1d and ok3
        nvls += f"; fused {len(fu.chunks)} chunks chains={fu.chains} ok={ok3}"
        # the same fused step through peer tables (unicast NVLink, no multicast); numpy order
        # over any power-of-two world there (RINGMIX_D1D_NUMPY_ORDER=1 above 2 ranks)
        os.environ["RINGMIX_SYM_P2P"] = "1"
        os.environ["RINGMIX_D1D_NUMPY_ORDER"] = "1"
        try:
            fp = D.LearnerShardedD1DFused(L, d, Lg, dev, chunk_cols=1 << 16)
        finally:
            os.environ.pop("RINGMIX_SYM_P2P", None)
            os.environ.pop("RINGMIX_D1D_NUMPY_ORDER", None)
        ids5, Wl5 = shard(fp, Wref)
        _, Gs5 = shard(fp, Gf)
        out5 = mixing.empty_learner_major(Lg, d, torch.float32, dev)
        for _ in range(3):
            fp.step(Wl5, Gs5, 0.01, out5)
        torch.cuda.synchronize()
        dd5 = (out5.double() - ref[ids5].double()).abs().max().item()
        ok_d1d = ok_d1d and (not fp.multicast) and check(fp, out5, ids5, ref)
        nvls += f"; fused-p2p chains={fp.chains} maxdiff {dd5:.2e}"
        # no gradients (apply_mixing semantics): the fused kernel's HAS_G = false path
        out4 = mixing.empty_learner_major(Lg, d, torch.float32, dev)
        fu.step(Wl, None, 0.01, out4)
        ref4 = mixing.mean_mix_sgd(Wref, None, 0.01)
        torch.cuda.synchronize()
        ok_d1d = ok_d1d and check(fu, out4, ids, ref4)
        # other storage types: the fused kernel against the single-GPU mean kernel
        for dt, tol in ((torch.float64, 1e-13), (torch.bfloat16, 1e-2)):
            idd, Wd = shard(fu, full, dt)
            _, Gd = shard(fu, Gf, dt)
            od = mixing.empty_learner_major(Lg, d, dt, dev)
            fu.step(Wd, Gd, 0.01, od)
            Fd = mixing.empty_learner_major(L, d, dt, dev).copy_(full.to(dt))
            GFd = mixing.empty_learner_major(L, d, dt, dev).copy_(Gf.to(dt))
            rd = mixing.mean_mix_sgd(Fd, GFd, 0.01)
            torch.cuda.synchronize()
            err = (od.double() - rd[idd].double()).abs().max().item()
            ok_d1d = ok_d1d and (err == 0.0 if (fu.chains and dt == torch.float64) else err <= tol)
            nvls += f"; {dt} maxdiff {err:.2e}"
    except RuntimeError as exc:
        nvls = str(exc)[:100]
    ring.close()
    # the pull layout with peer-table step ordering (unicast atomics instead of multicast)
    os.environ["RINGMIX_SYM_P2P"] = "1"
    try:
        ring2 = D.LearnerShardedRing(L, d, torch.float32)
    finally:
        os.environ.pop("RINGMIX_SYM_P2P", None)
    ring2.W[0].copy_(full[b:e])
    ring2.publish()
    Wref2 = mixing.empty_learner_major(L, d, torch.float32, dev); Wref2.copy_(full)
    for k in range(3):
        lt, rt = simulation.rad_tables(L, 12345, k, dev)
        out = ring2.step(lt, rt, Gl, 0.01)
        Wref2 = mixing.ring_mix_sgd(Wref2, mixing.empty_learner_major(L, d, torch.float32, dev).copy_(Gf), 0.01, lt, rt)
    ring2.settle()
    torch.cuda.synchronize()
    same = bool(torch.equal(ring2.weights, Wref2[b:e]))
    pull_steps.append(same and ring2.sync is not None and not ring2.sync.multicast)
    ok &= pull_steps[-1]
    ring2.close()
    # RAD in ring-position order (push layout): 3 steps vs the single-GPU reference
    pos = D.LearnerShardedRingPos(L, d, torch.float32)
    tabs = mixing.permutation_tables(L, 12345, 0, 4, dev)
    g0, g1 = pos.g0, pos.g0 + pos.Lg
    pos.W[0].copy_(full[tabs.inv[0][g0:g1].long()])
    Wr = mixing.empty_learner_major(L, d, torch.float32, dev); Wr.copy_(full)
    Gfull = mixing.empty_learner_major(L, d, torch.float32, dev).copy_(Gf)
    ok_pos = True
    pos_steps = []
    torch.cuda.synchronize(); dist.barrier()
    for k in range(3):
        Gs = mixing.empty_learner_major(pos.Lg, d, torch.float32, dev)
        Gs.copy_(Gf[pos.slot_learners(tabs.inv[k]).long()])
        pos.step(tabs.inv[k].contiguous(), tabs.perm[k + 1].contiguous(), Gs, 0.01)
        lt, rt = tabs.step(k)
        Wr = mixing.ring_mix_sgd(Wr, Gfull, 0.01, lt.contiguous(), rt.contiguous())
        torch.cuda.synchronize()
        same = bool(torch.equal(pos.slots_local, Wr[pos.slot_learners(tabs.inv[k + 1]).long()]))
        pos_steps.append(same)
        ok_pos &= same
    pos_steps.append(bool(pos.placed) == (L % world == 0 and world <= 8))
    ok_pos &= pos_steps[-1]
    pos.close()
    # the D1D training step with the device oracle (ShardedD1DTrainer: average beside the
    # generator, gradient fused into its final pass) against the one-GPU step on the same
    # data — bit for bit with the numpy-order layout, else to fp64 rounding of the mean
    from paper_2002_01119_b200 import objectives
    from paper_2002_01119_b200.simulation import RunConfig
    ok_tr, tr_diff = True, None
    try:
        oracle = objectives.quadratic_oracle(d, condition_number=5.0, noise_scale=1.0, seed=3,
                                             device=dev)
        cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=4, seed=7,
                        dtype="float32")
        b0, e0 = D.ShardLayout(L, world).bounds[rank]
        tr = D.ShardedD1DTrainer(L, d, e0 - b0, b0, dev, oracle)
        ids = torch.tensor(D.d1d_learners(L, world, rank, tr.chains), device=dev)
        Wl = mixing.empty_learner_major(len(ids), d, torch.float32, dev).copy_(full[ids])
        Pl = mixing.empty_learner_major(len(ids), d, torch.float32, dev).copy_(Gf[ids])
        out_tr = mixing.empty_learner_major(len(ids), d, torch.float32, dev)
        tr.step(Wl, Pl, cfg, 3, 0.01, out_tr)
        Gref = oracle.device_gradients(mixing.empty_learner_major(L, d, torch.float32, dev)
                                       .copy_(Gf), cfg, 3)
        ref_tr = mixing.mean_mix_sgd(mixing.empty_learner_major(L, d, torch.float32, dev)
                                     .copy_(full), Gref, 0.01)
        torch.cuda.synchronize()
        tr_diff = (out_tr.double() - ref_tr[ids].double()).abs().max().item()
        ok_tr = tr_diff == 0.0 if tr.chains else tr_diff <= 2e-6
        nvls += f"; trainer chains={tr.chains} maxdiff {tr_diff:.2e}"
    except RuntimeError as exc:
        nvls += f"; trainer: {str(exc)[:80]}"
    ok_d1d = ok_d1d and ok_tr
    detail = torch.tensor([int(x) for x in pull_steps + pos_steps], device=dev)
    all_detail = [torch.zeros_like(detail) for _ in range(world)]
    dist.all_gather(all_detail, detail)
    ok_pull = ok
    ok = ok and ok_pos
    res = torch.tensor([int(ok), int(ok_d1d), int(ok_pull), int(ok_pos)], device=dev)
    dist.all_reduce(res, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": world, "rad_bit_identical": bool(res[0]), "d1d_ok": bool(res[1]),
                          "d1d_maxdiff_rank0": dd, "nvls": nvls, "pull_ok": bool(res[2]),
                          "pos_ok": bool(res[3]),
                          "per_rank_pull_pos_steps": [t.tolist() for t in all_detail]}),
              flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    main()

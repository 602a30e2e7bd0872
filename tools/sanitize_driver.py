"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck): one call of
every product kernel family — mix_tma (ring / mean / S-PSGD; fp32, fp64, bf16), the (d, L)
kernels, the trace reductions, the normal generator (zig_*), the learner-sharded pull and
ring-position kernels with in-kernel step ordering, the fused D1D kernel and the cross-rank
mean (the multi-GPU kernels with every rank emulated on this GPU through peer tables).
Prints one line per family; the sanitizer's own report is the result (tools/sanitize.sh)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_01119_b200 import _lib, distributed as D, mixing, objectives, simulation  # noqa

lib = _lib.load()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
only = set(sys.argv[1:])


def want(name):
    return not only or name in only


def rand(L, d, dt):
    X = mixing.empty_learner_major(L, d, dt, dev)
    X.copy_(torch.randn((L, d), generator=g, device=dev, dtype=torch.float64).to(dt))
    return X


def table(ts):
    return torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=dev)


if want("mix"):
    for dt in (torch.float32, torch.float64, torch.bfloat16):
        for L, d in ((16, 1000), (64, 515)):
            W, G = rand(L, d, dt), rand(L, d, dt)
            lt, rt = simulation.rad_tables(L, 12345, 1, dev)
            am = torch.zeros((), dtype=torch.int64, device=dev)
            mixing.ring_mix_sgd(W, G, 0.01, lt, rt, absmax=am)
            mixing.mean_mix_sgd(W, G, 0.01, absmax=am)
            Ws = rand(L, d, dt)
            Ws.copy_(Ws[0:1].expand(L, d))
            mixing.spsgd_update(Ws, G, 0.01)
    torch.cuda.synchronize()
    print("mix ok", flush=True)

if want("dL"):
    W = np.random.default_rng(0).standard_normal((300, 12))
    left, right = (t.cpu().numpy() for t in simulation.rad_tables(12, 3, 0, dev))
    mixing.gossip_step_host(W, W, 0.01, left, right)
    mixing.gossip_step_host(W, W, 0.01)
    Wd = torch.from_numpy(W).to(dev)
    mixing.gossip_step_dL(Wd, Wd, 0.01, torch.from_numpy(left).to(dev),
                          torch.from_numpy(right).to(dev))
    torch.cuda.synchronize()
    print("dL ok", flush=True)

if want("trace"):
    oracle = objectives.quadratic_oracle(2000, condition_number=10.0, noise_scale=1.0, seed=1)
    for dt in (torch.float32, torch.float64):
        simulation.trace_stats(rand(16, 2000, dt).T, oracle)
    torch.cuda.synchronize()
    print("trace ok", flush=True)

if want("normal"):
    objectives.standard_normal(5000, 1, 2, 3)
    oracle = objectives.quadratic_oracle(3000, condition_number=10.0, noise_scale=1.0, seed=1)
    Phi = rand(4, 3000, torch.float32)
    cfg = simulation.RunConfig(n_learners=4, iterations=1, lr=0.01, batch_size=8, seed=5,
                               dtype="float32")
    oracle.device_gradients(Phi, cfg, 0)
    torch.cuda.synchronize()
    print("normal ok", flush=True)

if want("shard"):
    L, d, world = 12, 515, 2
    lay = D.ShardLayout(L, world)
    full, Gf = rand(L, d, torch.float32), rand(L, d, torch.float32)
    bufs = [[mixing.empty_learner_major(e - b, d, torch.float32, dev) for _ in range(2)]
            for b, e in lay.bounds]
    for r, (b, e) in enumerate(lay.bounds):
        bufs[r][0].copy_(full[b:e])
    slots = [D._slot_table(lay, [bufs[r][p].data_ptr() for r in range(world)],
                           bufs[0][0].stride(0), 4, dev) for p in range(2)]
    flags = [torch.zeros(4, dtype=torch.int32, device=dev) for _ in range(world)]
    cnt = [torch.zeros(4, dtype=torch.int32, device=dev) for _ in range(world)]
    ftab = table(flags)
    tabs = mixing.permutation_tables(L, 7, 0, 3)
    plans = [torch.empty(lib.rm_shard_plan_ints(e - b), dtype=torch.int32, device=dev)
             for b, e in lay.bounds]
    dests = [torch.empty(e - b, dtype=torch.int64, device=dev) for b, e in lay.bounds]
    for k in range(2):       # pull layout, in-kernel ordering
        lt, rt = (t.contiguous() for t in tabs.step(k))
        for r, (b, e) in enumerate(lay.bounds):
            lib.rm_shard_plan(lt.data_ptr(), rt.data_ptr(), L, b, e - b, plans[r].data_ptr(),
                              _lib.stream_ptr())
            a = _lib.StepSyncArgs(flags[r].data_ptr(), None, cnt[r].data_ptr(), k + 1, world,
                                  ftab.data_ptr())
            Gl = Gf[b:e].contiguous()
            _lib.check(lib.rm_ring_mix_sgd_sharded_f32(
                slots[k % 2].data_ptr(), bufs[r][k % 2].data_ptr(), Gl.data_ptr(),
                bufs[r][1 - k % 2].data_ptr(), L, b, e - b, d, bufs[r][0].stride(0),
                Gl.stride(0), bufs[r][0].stride(0), plans[r].data_ptr(), 0.01, None,
                _lib.stream_ptr(), ctypes.byref(a)))
    for k in range(2):       # ring-position layout, epochs 3, 4
        ik, pn = tabs.inv[k].contiguous(), tabs.perm[k + 1].contiguous()
        for r, (b, e) in enumerate(lay.bounds):
            lib.rm_pos_plan(ik.data_ptr(), pn.data_ptr(), L, b, e - b,
                            slots[1 - k % 2].data_ptr(), plans[r].data_ptr(),
                            dests[r].data_ptr(), _lib.stream_ptr())
            a = _lib.StepSyncArgs(flags[r].data_ptr(), None, cnt[r].data_ptr(), k + 3, world,
                                  ftab.data_ptr())
            Gl = Gf[b:e].contiguous()
            _lib.check(lib.rm_ring_mix_sgd_pos_f32(
                slots[k % 2].data_ptr(), bufs[r][k % 2].data_ptr(), Gl.data_ptr(), L, b, e - b, d,
                bufs[r][0].stride(0), Gl.stride(0), plans[r].data_ptr(), dests[r].data_ptr(),
                0.01, None, _lib.stream_ptr(), ctypes.byref(a)))
    a = _lib.StepSyncArgs(flags[0].data_ptr(), None, cnt[0].data_ptr(), 4, world, ftab.data_ptr())
    lib.rm_step_sync_wait(ctypes.byref(a), _lib.stream_ptr())
    torch.cuda.synchronize()
    print("shard ok", flush=True)

if want("d1d"):
    L, d, world = 10, 4099, 2
    lay = D.ShardLayout(L, world)
    Ws = [rand(e - b, d, torch.float32) for b, e in lay.bounds]
    Gs = [rand(e - b, d, torch.float32) for b, e in lay.bounds]
    outs = [mixing.empty_learner_major(e - b, d, torch.float32, dev) for b, e in lay.bounds]
    P = [torch.empty(d, dtype=torch.float64, device=dev) for _ in range(world)]
    M = [torch.empty(d, dtype=torch.float64, device=dev) for _ in range(world)]
    F = [torch.zeros(128, dtype=torch.int32, device=dev) for _ in range(world)]
    C = [torch.zeros(128, dtype=torch.int32, device=dev) for _ in range(world)]
    ranks = (_lib.D1DRank * world)()
    for r, (b, e) in enumerate(lay.bounds):
        ranks[r] = _lib.D1DRank(Ws[r].data_ptr(), Gs[r].data_ptr(), outs[r].data_ptr(), None,
                                P[r].data_ptr(), M[r].data_ptr(), F[r].data_ptr(),
                                C[r].data_ptr(), e - b, r)
    tP, tM, tF = table(P), table(M), table(F)
    _lib.check(lib.rm_d1d_fused_p2p_f32(ctypes.byref(ranks), world, L, d, Ws[0].stride(0),
                                        Gs[0].stride(0), outs[0].stride(0), 0.01, tP.data_ptr(),
                                        tM.data_ptr(), tF.data_ptr(), world, 64 * 32, 64, 1, 30,
                                        10, _lib.stream_ptr()))
    _lib.check(lib.rm_p2p_mean_f64(tP.data_ptr(), tM.data_ptr(), world, 0, d, L,
                                   _lib.stream_ptr()))
    torch.cuda.synchronize()
    print("d1d ok", flush=True)

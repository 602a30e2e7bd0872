"""The kernels that otherwise only run with several GPUs, executed on ONE GPU with the
whole world emulated in-process (peer tables instead of NVSwitch multicast):

* the fused D1D step (`rm_d1d_fused_p2p_*`, one launch playing every rank: partial-sum,
  cross-rank reduce and apply roles handing column chunks to each other through flags)
  — the reference step is `simulation.step_d1d` (simulation.py:304-312);
* the cross-rank mean (`rm_p2p_mean_f64`, the peer-table form of `rm_nvls_mean_f64`);
* in-kernel step ordering (`rm_step_sync` with `done_peers`, `rm_step_sync_wait`,
  `rm_step_sync_publish`) of the learner-sharded RAD kernels, pull and ring-position
  layouts — the reference step is `simulation._gossip_step` (simulation.py:263-268);
* the bounded cross-rank wait: a wait nobody satisfies gives up after the timeout and
  is reported by `rm_xgpu_status` instead of trapping.

Expected values are restated in numpy in the kernels' documented summation order
(partials in ascending local row, ranks in ascending order) and must match bit for bit;
the sharded RAD steps must equal the single-GPU step bit for bit."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import _lib, distributed as D, mixing, simulation

pytestmark = pytest.mark.gpu

MAX_CHUNKS = 64


def _table(tensors) -> torch.Tensor:
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device="cuda")


def _status() -> int:
    s = ctypes.c_uint(0)
    _lib.check(_lib.load().rm_xgpu_status(ctypes.byref(s)), "rm_xgpu_status")
    return int(s.value)


def _rand(rows, d, dtype, g):
    X = mixing.empty_learner_major(rows, d, dtype)
    X.copy_(torch.randn((rows, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    return X


# ---------------------------------------------------------------------------
# cross-rank mean through peer tables
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("world,d,L", [(2, 1000, 16), (3, 4099, 10), (8, 65_537, 64)])
def test_p2p_mean_sums_ranks_in_order_and_broadcasts(world, d, L):
    g = torch.Generator(device="cuda").manual_seed(world * 7 + d)
    P = [torch.randn(d, generator=g, device="cuda", dtype=torch.float64) for _ in range(world)]
    M = [torch.full((d,), -7.0, device="cuda", dtype=torch.float64) for _ in range(world)]
    lib = _lib.load()
    tp, tm = _table(P), _table(M)
    # every rank reduces its own 1/world slice (as the pipeline does)
    sl = -(-d // world)
    for r in range(world):
        c0, c1 = min(d, r * sl), min(d, (r + 1) * sl)
        _lib.check(lib.rm_p2p_mean_f64(tp.data_ptr(), tm.data_ptr(), world, c0, c1, L,
                                       _lib.stream_ptr()), "rm_p2p_mean_f64")
    torch.cuda.synchronize()
    Ph = [p.cpu().numpy() for p in P]
    tot = Ph[0].copy()
    for x in Ph[1:]:
        tot = tot + x
    want = tot / L
    for r in range(world):
        assert np.array_equal(M[r].cpu().numpy(), want), r


# ---------------------------------------------------------------------------
# fused D1D, every rank in one launch
# ---------------------------------------------------------------------------

def _d1d_expected(Wb, Gb, L, lr, dtype):
    """numpy restatement of the fused D1D arithmetic: per rank the fp64 column sum of its
    rows in ascending order (partial_sum_range), ranks summed in ascending order, / L,
    then y = mean - lr*g in the accumulation type (fp64; fp32 for bf16), rounded once."""
    tot = None
    for W in Wb:
        s = np.zeros(W.shape[1])
        for row in W.astype(np.float64):
            s = s + row
        tot = s if tot is None else tot + s
    mean = tot / L
    outs = []
    for G in Gb:
        if dtype == torch.bfloat16:
            y = mean.astype(np.float32) - np.float32(lr) * G.astype(np.float32)
            outs.append(torch.from_numpy(y).to(torch.bfloat16))
        else:
            y = mean - lr * G.astype(np.float64)
            outs.append(torch.from_numpy(y).to(dtype))
    return outs


@pytest.mark.parametrize("L,d,world,chunk", [(16, 1000, 2, 1 << 21), (64, 100_003, 4, 1 << 14),
                                             (10, 4099, 3, 96 * 8), (64, 25_000, 8, 256 * 16)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_fused_d1d_emulated_world_matches_restatement(L, d, world, chunk, dtype):
    lay = D.ShardLayout(L, world)
    g = torch.Generator(device="cuda").manual_seed(L * 13 + d + world)
    lr = 0.01
    Ws = [_rand(e - b, d, dtype, g) for b, e in lay.bounds]
    Gs = [_rand(e - b, d, dtype, g) for b, e in lay.bounds]
    outs = [[mixing.empty_learner_major(e - b, d, dtype) for b, e in lay.bounds]
            for _ in range(2)]
    P = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
    M = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
    F = [torch.zeros(2 * MAX_CHUNKS, dtype=torch.int32, device="cuda") for _ in range(world)]
    C = [torch.zeros(2 * MAX_CHUNKS, dtype=torch.int32, device="cuda") for _ in range(world)]
    amax = [torch.zeros((), dtype=torch.int64, device="cuda") for _ in range(world)]
    tP, tM, tF = _table(P), _table(M), _table(F)
    lib = _lib.load()
    fn = getattr(lib, f"rm_d1d_fused_p2p_{mixing._suffix(Ws[0])}")
    _lib.check(lib.rm_set_xgpu_timeout(30.0))
    cur = Ws
    for epoch in (1, 2, 3):     # flags and counters only grow: several steps in a row
        dst = outs[epoch % 2]
        ranks = (_lib.D1DRank * world)()
        for r, (b, e) in enumerate(lay.bounds):
            ranks[r] = _lib.D1DRank(cur[r].data_ptr(), Gs[r].data_ptr(), dst[r].data_ptr(),
                                    amax[r].data_ptr(), P[r].data_ptr(), M[r].data_ptr(),
                                    F[r].data_ptr(), C[r].data_ptr(), e - b, r)
        want = _d1d_expected([w.cpu().to(torch.float64).numpy() if dtype == torch.bfloat16
                              else w.cpu().numpy() for w in cur],
                             [x.cpu().to(torch.float64).numpy() if dtype == torch.bfloat16
                              else x.cpu().numpy() for x in Gs], L, lr, dtype)
        _lib.check(fn(ctypes.byref(ranks), world, L, d, cur[0].stride(0), Gs[0].stride(0), dst[0].stride(0),
                      lr, tP.data_ptr(), tM.data_ptr(), tF.data_ptr(), world, chunk, MAX_CHUNKS,
                      epoch, 30, 10, _lib.stream_ptr()), "rm_d1d_fused_p2p")
        torch.cuda.synchronize()
        assert _status() == 0
        for r in range(world):
            assert torch.equal(dst[r].cpu(), want[r]), (epoch, r)
        cur = dst


def test_fused_d1d_emulated_equals_single_gpu_to_fp64_rounding():
    L, d, world = 64, 200_001, 4
    lay = D.ShardLayout(L, world)
    g = torch.Generator(device="cuda").manual_seed(99)
    W = _rand(L, d, torch.float32, g)
    G = _rand(L, d, torch.float32, g)
    ref = mixing.mean_mix_sgd(W, G, 0.01)
    P = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
    M = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
    F = [torch.zeros(2 * MAX_CHUNKS, dtype=torch.int32, device="cuda") for _ in range(world)]
    C = [torch.zeros(2 * MAX_CHUNKS, dtype=torch.int32, device="cuda") for _ in range(world)]
    out = mixing.empty_learner_major(L, d, torch.float32)
    ranks = (_lib.D1DRank * world)()
    for r, (b, e) in enumerate(lay.bounds):
        ranks[r] = _lib.D1DRank(W[b:e].data_ptr(), G[b:e].data_ptr(), out[b:e].data_ptr(), None,
                                P[r].data_ptr(), M[r].data_ptr(), F[r].data_ptr(),
                                C[r].data_ptr(), e - b, r)
    tP, tM, tF = _table(P), _table(M), _table(F)
    _lib.check(_lib.load().rm_d1d_fused_p2p_f32(
        ctypes.byref(ranks), world, L, d, W.stride(0), G.stride(0), out.stride(0), 0.01, tP.data_ptr(),
        tM.data_ptr(), tF.data_ptr(), world, 1 << 16, MAX_CHUNKS, 1, 30, 10, _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert _status() == 0
    diff = (out.double() - ref.double()).abs()
    scale = W.double().abs().mean(0, keepdim=True) + 0.01 * G.double().abs()
    assert bool((diff <= 2.0**-23 * (ref.double().abs() + scale)).all())
    assert float((out != ref).double().mean()) < 1e-4


@pytest.mark.parametrize("L,d,world", [(16, 1000, 2), (64, 100_003, 4), (64, 25_001, 8),
                                       (128, 4099, 2), (8, 777, 1), (64, 5000, 1)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_numpy_order_d1d_emulated_world_equals_single_gpu(L, d, world, dtype):
    """rm_set_d1d_numpy_order: rank g holds the learners of numpy's pairwise chains
    [g R, (g + 1) R) (R = 8 / world); its partial is numpy's tree over them and the ranks are
    combined in the tree order, so every rank's rows are the single-GPU D1D step's rows bit
    for bit (mixing.py:122-124, simulation.py:304-312) — the fused kernel over peer tables,
    several epochs."""
    chains = D.d1d_numpy_chains(L, world)
    assert chains == 8 // world
    g = torch.Generator(device="cuda").manual_seed(L + d + world)
    W = _rand(L, d, dtype, g)
    G = _rand(L, d, dtype, g)
    lr = 0.01
    ids = [torch.tensor(D.d1d_learners(L, world, r, chains), device="cuda") for r in range(world)]
    Lg = L // world
    def gather(X, i):
        t = mixing.empty_learner_major(Lg, d, dtype)
        t.copy_(X[i])
        return t

    cur = [gather(W, i) for i in ids]
    Gs = [gather(G, i) for i in ids]
    outs = [[mixing.empty_learner_major(Lg, d, dtype) for _ in range(world)] for _ in range(2)]
    P = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
    M = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
    F = [torch.zeros(2 * MAX_CHUNKS, dtype=torch.int32, device="cuda") for _ in range(world)]
    C = [torch.zeros(2 * MAX_CHUNKS, dtype=torch.int32, device="cuda") for _ in range(world)]
    amax = [torch.zeros((), dtype=torch.int64, device="cuda") for _ in range(world)]
    tP, tM, tF = _table(P), _table(M), _table(F)
    lib = _lib.load()
    fn = getattr(lib, f"rm_d1d_fused_p2p_{mixing._suffix(W)}")
    _lib.check(lib.rm_set_xgpu_timeout(30.0))
    full = W
    try:
        _lib.check(lib.rm_set_d1d_numpy_order(chains))
        for epoch in (1, 2, 3):
            ref = mixing.mean_mix_sgd(full, G, lr)
            dst = outs[epoch % 2]
            ranks = (_lib.D1DRank * world)()
            for r in range(world):
                amax[r].zero_()
                ranks[r] = _lib.D1DRank(cur[r].data_ptr(), Gs[r].data_ptr(), dst[r].data_ptr(),
                                        amax[r].data_ptr(), P[r].data_ptr(), M[r].data_ptr(),
                                        F[r].data_ptr(), C[r].data_ptr(), Lg, r)
            _lib.check(fn(ctypes.byref(ranks), world, L, d, cur[0].stride(0), Gs[0].stride(0),
                          dst[0].stride(0), lr, tP.data_ptr(), tM.data_ptr(), tF.data_ptr(),
                          world, 32 * world * 64, MAX_CHUNKS, epoch, 30, 10, _lib.stream_ptr()),
                       "rm_d1d_fused_p2p")
            torch.cuda.synchronize()
            assert _status() == 0
            for r in range(world):
                assert torch.equal(dst[r], ref[ids[r]]), (epoch, r)
                assert simulation.absmax_value(amax[r]) == float(ref[ids[r]].abs().max())
            cur = dst
            full = ref
        # the chunk-pipeline pieces: partial sums + peer-table tree reduction == column mean
        S = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
        Mm = [torch.empty(d, dtype=torch.float64, device="cuda") for _ in range(world)]
        psum = getattr(lib, f"rm_partial_sum_{mixing._suffix(W)}")
        for r in range(world):
            _lib.check(psum(cur[r].data_ptr(), Lg, d, cur[r].stride(0), S[r].data_ptr(),
                            _lib.stream_ptr()), "rm_partial_sum")
        tS, tMm = _table(S), _table(Mm)   # kept alive until the kernel has run
        _lib.check(lib.rm_p2p_mean_f64(tS.data_ptr(), tMm.data_ptr(), world, 0, d, L,
                                       _lib.stream_ptr()), "rm_p2p_mean_f64")
        torch.cuda.synchronize()
    finally:
        lib.rm_set_d1d_numpy_order(0)
    colmean = torch.empty(d, dtype=torch.float64, device="cuda")
    _lib.check(getattr(lib, f"rm_column_mean_{mixing._suffix(W)}")(
        full.data_ptr(), L, d, full.stride(0), colmean.data_ptr(), _lib.stream_ptr()))
    torch.cuda.synchronize()
    for r in range(world):
        assert torch.equal(Mm[r], colmean)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_interleaved_gradient_streams_are_rows_of_the_full_call(world):
    """rm_set_shard_streams: a numpy-order rank's learner set (runs of R learners every 8)
    draws exactly those learners' gradient streams (objectives.py:84-90)."""
    from paper_2002_01119_b200 import objectives
    from paper_2002_01119_b200.simulation import RunConfig
    L, d = 32, 3001
    chains = 8 // world
    oracle = objectives.quadratic_oracle(d, condition_number=4.0, noise_scale=1.0, seed=2)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.1, batch_size=3, seed=11)
    g = torch.Generator(device="cuda").manual_seed(5)
    Phi = _rand(L, d, torch.float32, g)
    full = oracle.device_gradients(Phi, cfg, 4)
    lib = _lib.load()
    for r in range(world):
        ids = torch.tensor(D.d1d_learners(L, world, r, chains), device="cuda")
        try:
            _lib.check(lib.rm_set_shard_streams(chains, 8))
            P = mixing.empty_learner_major(len(ids), d, torch.float32)
            P.copy_(Phi[ids])
            part = oracle.device_gradients(P, cfg, 4, learner0=r * chains)
        finally:
            lib.rm_set_shard_streams(0, 0)
        torch.cuda.synchronize()
        assert torch.equal(part, full[ids])


# ---------------------------------------------------------------------------
# in-kernel step ordering (rm_step_sync through peer tables)
# ---------------------------------------------------------------------------

class _EmuSync:
    """Per-rank rm_step_sync state of an emulated world: `done` flags, counters and the
    peer table of every rank's flag."""

    def __init__(self, world):
        self.world = world
        self.flags = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(world)]
        self.cnt = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(world)]
        self.table = _table(self.flags)
        self.epoch = 0

    def args(self, r, epoch):
        return _lib.StepSyncArgs(self.flags[r].data_ptr(), None, self.cnt[r].data_ptr(), epoch,
                                 self.world, self.table.data_ptr())


def _full_and_parts(L, d, world, dtype, seed):
    lay = D.ShardLayout(L, world)
    g = torch.Generator(device="cuda").manual_seed(seed)
    full = _rand(L, d, dtype, g)
    Gf = _rand(L, d, dtype, g)
    return lay, full, Gf


@pytest.mark.parametrize("L,d,world,fixed", [(16, 1000, 2, False), (10, 77, 3, False),
                                             (64, 4099, 8, False), (64, 100_003, 2, True),
                                             (64, 70_001, 4, True), (24, 5003, 3, True)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_pull_layout_steps_ordered_in_kernel(L, d, world, fixed, dtype):
    """K consecutive learner-sharded RAD steps, every step kernel ordering itself through
    the flags (waits for every rank's previous step, bumps every rank's flag).  fixed: the
    fixed ring with the 2-remote-row bound (rm_set_shard_remote_rows: 1 KB row segments)."""
    lay, full, Gf = _full_and_parts(L, d, world, dtype, L + d)
    K = 4
    tabs = mixing.permutation_tables(L, 4242, 0, K)
    fixed_tabs = tuple(t.contiguous() for t in simulation.fixed_ring_tables(L, torch.device("cuda")))
    esz = full.element_size()
    bufs = [[mixing.empty_learner_major(e - b, d, dtype) for _ in range(2)] for b, e in lay.bounds]
    Gs = []
    for r, (b, e) in enumerate(lay.bounds):
        bufs[r][0].copy_(full[b:e])
        Gl = mixing.empty_learner_major(e - b, d, dtype)
        Gl.copy_(Gf[b:e])
        Gs.append(Gl)
    row_ptrs = []
    for par in range(2):
        ptrs = np.empty(L, dtype=np.uint64)
        for r, (b, e) in enumerate(lay.bounds):
            for i in range(e - b):
                ptrs[b + i] = bufs[r][par].data_ptr() + i * bufs[r][par].stride(0) * esz
        row_ptrs.append(torch.from_numpy(ptrs.view(np.int64)).cuda())
    lib = _lib.load()
    fn = getattr(lib, f"rm_ring_mix_sgd_sharded_{mixing._suffix(full)}")
    sync = _EmuSync(world)
    _lib.check(lib.rm_set_xgpu_timeout(30.0))
    plans = [torch.empty(lib.rm_shard_plan_ints(e - b), dtype=torch.int32, device="cuda")
             for b, e in lay.bounds]
    ref, cur = full, 0
    if fixed:
        _lib.check(lib.rm_set_shard_remote_rows(2))
    try:
        for k in range(K):
            lt, rt = fixed_tabs if fixed else (t.contiguous() for t in tabs.step(k))
            epoch = k + 1
            for r, (b, e) in enumerate(lay.bounds):      # rank order within an epoch
                Lg = e - b
                _lib.check(lib.rm_shard_plan(lt.data_ptr(), rt.data_ptr(), L, b, Lg,
                                             plans[r].data_ptr(), _lib.stream_ptr()))
                src, dst = bufs[r][cur], bufs[r][1 - cur]
                a = sync.args(r, epoch)
                _lib.check(fn(row_ptrs[cur].data_ptr(), src.data_ptr(), Gs[r].data_ptr(),
                              dst.data_ptr(), L, b, Lg, d, src.stride(0), Gs[r].stride(0),
                              dst.stride(0), plans[r].data_ptr(), 0.03, None,
                              _lib.stream_ptr(), ctypes.byref(a)))
            cur = 1 - cur
            ref = mixing.ring_mix_sgd(ref, Gf, 0.03, lt, rt)
    finally:
        lib.rm_set_shard_remote_rows(0)
    # a reader of every rank's last step: stream-ordered wait, then compare
    _lib.check(lib.rm_step_sync_wait(ctypes.byref(sync.args(0, K)), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert _status() == 0
    for r in range(world):
        assert int(sync.flags[r][0]) == world * K
    got = torch.cat([bufs[r][cur] for r in range(world)])
    assert torch.equal(got, ref)


@pytest.mark.parametrize("L,d,world", [(24, 3001, 4), (10, 77, 3)])
def test_position_layout_steps_ordered_in_kernel_with_publish(L, d, world):
    """Ring-position layout with in-kernel ordering; the initial slot contents are
    written from outside the step and published (rm_step_sync_publish) first."""
    dtype = torch.float32
    lay, full, Gf = _full_and_parts(L, d, world, dtype, 5 * L + d)
    K = 4
    tabs = mixing.permutation_tables(L, 777, 0, K + 1)
    inv = tabs.inv
    bufs = [[mixing.empty_learner_major(e - b, d, dtype) for _ in range(2)] for b, e in lay.bounds]
    esz = full.element_size()
    slots = [D._slot_table(lay, [bufs[r][p].data_ptr() for r in range(world)],
                           bufs[0][0].stride(0), esz, "cuda") for p in range(2)]
    lib = _lib.load()
    fn = getattr(lib, f"rm_ring_mix_sgd_pos_{mixing._suffix(full)}")
    sync = _EmuSync(world)
    _lib.check(lib.rm_set_xgpu_timeout(30.0))
    inv0 = inv[0].long()
    for r, (b, e) in enumerate(lay.bounds):
        bufs[r][0].copy_(full[inv0[b:e]])
        _lib.check(lib.rm_step_sync_publish(ctypes.byref(sync.args(r, 1)), _lib.stream_ptr()))
    base = 1           # epoch 1 = the publish
    plans = [torch.empty(lib.rm_shard_plan_ints(e - b), dtype=torch.int32, device="cuda")
             for b, e in lay.bounds]
    dests = [torch.empty(e - b, dtype=torch.int64, device="cuda") for b, e in lay.bounds]
    ref, cur = full, 0
    for k in range(K):
        ik = inv[k].contiguous()
        pn = tabs.perm[k + 1].contiguous()
        for r, (b, e) in enumerate(lay.bounds):
            Lg = e - b
            _lib.check(lib.rm_pos_plan(ik.data_ptr(), pn.data_ptr(), L, b, Lg,
                                       slots[1 - cur].data_ptr(), plans[r].data_ptr(),
                                       dests[r].data_ptr(), _lib.stream_ptr()))
            Gs = mixing.empty_learner_major(Lg, d, dtype)
            Gs.copy_(Gf[ik[b:e].long()])
            src = bufs[r][cur]
            a = sync.args(r, base + k + 1)
            _lib.check(fn(slots[cur].data_ptr(), src.data_ptr(), Gs.data_ptr(), L, b, Lg, d,
                          src.stride(0), Gs.stride(0), plans[r].data_ptr(),
                          dests[r].data_ptr(), 0.02, None, _lib.stream_ptr(), ctypes.byref(a)))
        cur = 1 - cur
        lt, rt = tabs.step(k)
        ref = mixing.ring_mix_sgd(ref, Gf, 0.02, lt.contiguous(), rt.contiguous())
    _lib.check(lib.rm_step_sync_wait(ctypes.byref(sync.args(0, base + K)), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert _status() == 0
    nxt = inv[K].long()
    for r, (b, e) in enumerate(lay.bounds):
        assert torch.equal(bufs[r][cur], ref[nxt[b:e]]), r


def test_unsatisfied_wait_gives_up_and_reports_status():
    """A step whose predecessors never arrive waits for the timeout, then completes and
    sets the status bit (no trap: the context stays usable)."""
    lib = _lib.load()
    assert _status() == 0
    sync = _EmuSync(2)
    _lib.check(lib.rm_set_xgpu_timeout(0.2))
    try:
        # epoch 2: waits for done >= 2 * 2, nobody has arrived
        _lib.check(lib.rm_step_sync_wait(ctypes.byref(sync.args(0, 2)), _lib.stream_ptr()))
        torch.cuda.synchronize()
        assert _status() == 1
        assert _status() == 0           # read-and-clear
        x = torch.ones(4, device="cuda") * 2     # the context still works
        assert float(x.sum()) == 8.0
    finally:
        _lib.check(lib.rm_set_xgpu_timeout(600.0))


def test_oracle_pins_the_emulated_sharded_step():
    """One emulated pull-layout step against the C oracle directly (not only against the
    one-GPU kernel)."""
    L, d, world = 12, 515, 3
    lay, full, Gf = _full_and_parts(L, d, world, torch.float32, 3)
    p = O.c_permutation(L, 31337, 2)
    _, left, right = O.neighbour_tables(p)
    lt = torch.from_numpy(left.astype(np.int32)).cuda()
    rt = torch.from_numpy(right.astype(np.int32)).cuda()
    esz = 4
    ptrs = np.empty(L, dtype=np.uint64)
    parts = []
    for r, (b, e) in enumerate(lay.bounds):
        X = mixing.empty_learner_major(e - b, d, torch.float32)
        X.copy_(full[b:e])
        parts.append(X)
        for i in range(e - b):
            ptrs[b + i] = X.data_ptr() + i * X.stride(0) * esz
    row_ptrs = torch.from_numpy(ptrs.view(np.int64)).cuda()
    lib = _lib.load()
    sync = _EmuSync(world)
    outs = []
    for r, (b, e) in enumerate(lay.bounds):
        Lg = e - b
        plan = torch.empty(lib.rm_shard_plan_ints(Lg), dtype=torch.int32, device="cuda")
        _lib.check(lib.rm_shard_plan(lt.data_ptr(), rt.data_ptr(), L, b, Lg, plan.data_ptr(),
                                     _lib.stream_ptr()))
        Gl = mixing.empty_learner_major(Lg, d, torch.float32)
        Gl.copy_(Gf[b:e])
        out = mixing.empty_learner_major(Lg, d, torch.float32)
        _lib.check(lib.rm_ring_mix_sgd_sharded_f32(
            row_ptrs.data_ptr(), parts[r].data_ptr(), Gl.data_ptr(), out.data_ptr(), L, b, Lg, d,
            parts[r].stride(0), Gl.stride(0), out.stride(0), plan.data_ptr(), 0.01, None,
            _lib.stream_ptr(), ctypes.byref(sync.args(r, 1))))
        outs.append(out)
    torch.cuda.synchronize()
    got = torch.cat(outs).cpu().numpy().T
    W64 = full.double().cpu().numpy().T.copy()
    G64 = Gf.double().cpu().numpy().T.copy()
    want = O.c_ring_mix_sgd(W64, G64, 0.01, left, right).astype(np.float32)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# ring-position layout with arc placement (rm_pos_placement / rm_pos_plan_placed)
# ---------------------------------------------------------------------------

def _best_placement_numpy(inv_k, perm_next, sop_k, L, n):
    """Restatement of rm_pos_placement: best (rotation, arc -> rank) by exhaustive search
    (n <= 5), ties to the smallest rotation and the lexicographically first assignment."""
    import itertools
    Lg = L // n
    owner = np.empty(L, dtype=np.int64)
    qn = np.empty(L, dtype=np.int64)
    for q in range(L):
        owner[inv_k[q]] = sop_k[q] // Lg
    qn[:] = perm_next
    best = (-1, None, None)
    for r in range(L):
        arc = ((qn - r) % L) // Lg
        cnt = np.zeros((n, n), dtype=np.int64)
        np.add.at(cnt, (arc, owner), 1)
        for sig in itertools.permutations(range(n)):
            sc = sum(cnt[a, sig[a]] for a in range(n))
            if sc > best[0]:
                best = (sc, r, sig)
    return best


@pytest.mark.parametrize("L,n", [(12, 3), (16, 2), (24, 4), (40, 5), (64, 8), (128, 8)])
def test_pos_placement_matches_exhaustive_search(L, n):
    lib = _lib.load()
    tabs = mixing.permutation_tables(L, 99, 0, 5)
    sop = torch.arange(L, dtype=torch.int32, device="cuda")
    pos_n = torch.empty(L, dtype=torch.int32, device="cuda")
    sop_n = torch.empty(L, dtype=torch.int32, device="cuda")
    moved = torch.zeros(n, dtype=torch.int32, device="cuda")
    for k in range(4):
        _lib.check(lib.rm_pos_placement(tabs.inv[k].contiguous().data_ptr(),
                                        tabs.perm[k + 1].contiguous().data_ptr(), sop.data_ptr(),
                                        L, n, pos_n.data_ptr(), sop_n.data_ptr(),
                                        moved.data_ptr(), _lib.stream_ptr()))
        torch.cuda.synchronize()
        inv_k, pn = tabs.inv[k].cpu().numpy(), tabs.perm[k + 1].cpu().numpy()
        s_k, s_n, p_n = sop.cpu().numpy(), sop_n.cpu().numpy(), pos_n.cpu().numpy()
        Lg = L // n
        # a placement: bijection, every rank an arc of consecutive positions
        assert sorted(s_n.tolist()) == list(range(L)) and np.array_equal(p_n[s_n], np.arange(L))
        for g in range(n):
            arc = p_n[g * Lg:(g + 1) * Lg]
            assert np.all((np.diff(arc) % L) == 1)
        stay = sum(1 for q in range(L) if s_k[q] // Lg == s_n[pn[inv_k[q]]] // Lg)
        if n <= 5:
            best = _best_placement_numpy(inv_k, pn, s_k, L, n)
            assert stay == best[0]
        owner = {inv_k[q]: s_k[q] // Lg for q in range(L)}
        want_moved = np.zeros(n, dtype=np.int64)
        for l in range(L):
            if s_n[pn[l]] // Lg != owner[l]:
                want_moved[owner[l]] += 1
        assert np.array_equal(moved.cpu().numpy(), want_moved)
        assert stay >= sum(1 for q in range(L) if q // Lg == pn[inv_k[q]] // Lg) or n > 5
        sop.copy_(sop_n)


@pytest.mark.parametrize("L,d,world", [(24, 3001, 4), (16, 515, 2), (40, 77, 8),
                                       (128, 4099, 8), (128, 2051, 4)])
def test_placed_position_layout_steps_bit_identical(L, d, world):
    """Ring-position layout with the per-step arc placement, every rank emulated on this
    GPU, in-kernel ordering: after each step slot i of rank r holds learner
    inv_{k+1}[pos_of_slot[r * Lg + i]], equal to the single-GPU step."""
    dtype = torch.float32
    lay, full, Gf = _full_and_parts(L, d, world, dtype, 7 * L + d)
    Lg = L // world
    K = 5
    tabs = mixing.permutation_tables(L, 4321, 0, K + 1)
    inv = tabs.inv
    bufs = [[mixing.empty_learner_major(Lg, d, dtype) for _ in range(2)] for _ in range(world)]
    esz = full.element_size()
    slots = [D._slot_table(lay, [bufs[r][p].data_ptr() for r in range(world)],
                           bufs[0][0].stride(0), esz, "cuda") for p in range(2)]
    lib = _lib.load()
    sync = _EmuSync(world)
    _lib.check(lib.rm_set_xgpu_timeout(30.0))
    ident = torch.arange(L, dtype=torch.int32, device="cuda")
    place = [[ident.clone(), ident.clone()], [ident.clone(), ident.clone()]]
    inv0 = inv[0].long()
    for r in range(world):
        bufs[r][0].copy_(full[inv0[r * Lg:(r + 1) * Lg]])
    plans = [torch.empty(lib.rm_shard_plan_ints(Lg), dtype=torch.int32, device="cuda")
             for _ in range(world)]
    dests = [torch.empty(Lg, dtype=torch.int64, device="cuda") for _ in range(world)]
    ref, cur, pc = full, 0, 0
    for k in range(K):
        ik, pn = inv[k].contiguous(), tabs.perm[k + 1].contiguous()
        cp, npl = place[pc], place[1 - pc]
        _lib.check(lib.rm_pos_placement(ik.data_ptr(), pn.data_ptr(), cp[1].data_ptr(), L, world,
                                        npl[0].data_ptr(), npl[1].data_ptr(), None,
                                        _lib.stream_ptr()))
        for r in range(world):
            _lib.check(lib.rm_pos_plan_placed(ik.data_ptr(), pn.data_ptr(), cp[0].data_ptr(),
                                              cp[1].data_ptr(), npl[1].data_ptr(), L, r * Lg, Lg,
                                              slots[1 - cur].data_ptr(), plans[r].data_ptr(),
                                              dests[r].data_ptr(), _lib.stream_ptr()))
            learners = ik[cp[0][r * Lg:(r + 1) * Lg].long()].long()
            Gs = mixing.empty_learner_major(Lg, d, dtype)
            Gs.copy_(Gf[learners])
            src = bufs[r][cur]
            a = sync.args(r, k + 1)
            _lib.check(lib.rm_ring_mix_sgd_pos_f32(
                slots[cur].data_ptr(), src.data_ptr(), Gs.data_ptr(), L, r * Lg, Lg, d,
                src.stride(0), Gs.stride(0), plans[r].data_ptr(), dests[r].data_ptr(), 0.02, None,
                _lib.stream_ptr(), ctypes.byref(a)))
        cur, pc = 1 - cur, 1 - pc
        lt, rt = tabs.step(k)
        ref = mixing.ring_mix_sgd(ref, Gf, 0.02, lt.contiguous(), rt.contiguous())
        _lib.check(lib.rm_step_sync_wait(ctypes.byref(sync.args(0, k + 1)), _lib.stream_ptr()))
        torch.cuda.synchronize()
        nxt = inv[k + 1].long()
        pos_slots = place[pc][0].long()
        for r in range(world):
            learners = nxt[pos_slots[r * Lg:(r + 1) * Lg]]
            assert torch.equal(bufs[r][cur], ref[learners]), (k, r)
    assert _status() == 0

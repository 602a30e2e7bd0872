"""Learner-sharded kernels on one GPU: the ranks are emulated inside one process
(each "rank" owns a row range; row_ptrs point into the other ranks' buffers on
the same device).  The fused sharded step must be bit-identical to the
single-GPU step, the device planner must equal its host restatement, and the
D1D partial-sum / apply pair must reproduce the mean step."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import _lib, distributed as D, mixing

pytestmark = pytest.mark.gpu


def _tables(L, seed, k):
    p = O.c_permutation(L, seed, k)
    _, left, right = O.neighbour_tables(p)
    return (torch.from_numpy(left.astype(np.int32)).cuda(),
            torch.from_numpy(right.astype(np.int32)).cuda(), left, right)


def _emulate(L, d, world, dtype, k, with_g=True):
    lay = D.ShardLayout(L, world)
    g = torch.Generator(device="cuda").manual_seed(L * 31 + d)
    full = mixing.empty_learner_major(L, d, dtype)
    full.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    Gf = mixing.empty_learner_major(L, d, dtype)
    Gf.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    lt, rt, left, right = _tables(L, 4242, k)
    ref = mixing.ring_mix_sgd(full, Gf if with_g else None, 0.03, lt, rt)
    # each emulated rank: its own row block buffers (copies) so pointers differ
    parts = []
    for r in range(world):
        b, e = lay.rows(r)
        X = mixing.empty_learner_major(e - b, d, dtype)
        X.copy_(full[b:e])
        Gl = mixing.empty_learner_major(e - b, d, dtype)
        Gl.copy_(Gf[b:e])
        parts.append((b, e, X, Gl))
    esz = full.element_size()
    ptrs = np.empty(L, dtype=np.uint64)
    for b, e, X, _ in parts:
        for i in range(e - b):
            ptrs[b + i] = X.data_ptr() + i * X.stride(0) * esz
    row_ptrs = torch.from_numpy(ptrs.view(np.int64)).cuda()
    lib = _lib.load()
    sfx = mixing._suffix(full)
    fn = getattr(lib, f"rm_ring_mix_sgd_sharded_{sfx}")
    outs = []
    for b, e, X, Gl in parts:
        Lg = e - b
        plan = torch.empty(lib.rm_shard_plan_ints(Lg), dtype=torch.int32, device="cuda")
        _lib.check(lib.rm_shard_plan(lt.data_ptr(), rt.data_ptr(), L, b, Lg, plan.data_ptr(),
                                     _lib.stream_ptr()))
        # planner == host restatement
        rem, tri = D.plan_reference(left, right, b, Lg)
        pl = plan.cpu().numpy()
        assert pl[0] == len(rem) and list(pl[1:1 + len(rem)]) == rem
        assert [tuple(x) for x in pl[1 + 2 * Lg:1 + 6 * Lg].reshape(Lg, 4)] == tri
        out = mixing.empty_learner_major(Lg, d, dtype)
        amax = torch.zeros((), dtype=torch.int64, device="cuda")
        _lib.check(fn(row_ptrs.data_ptr(), X.data_ptr(), Gl.data_ptr() if with_g else None,
                      out.data_ptr(), L, b, Lg, d, X.stride(0), Gl.stride(0), out.stride(0),
                      plan.data_ptr(), 0.03, amax.data_ptr(), _lib.stream_ptr(), None))
        outs.append(out)
    torch.cuda.synchronize()
    return ref, torch.cat([o for o in outs], dim=0)


@pytest.mark.parametrize("L,d,world", [(16, 1000, 2), (64, 4099, 8), (64, 25_000, 4),
                                       (128, 3001, 8), (10, 77, 3), (33, 1, 4)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_sharded_ring_step_bit_identical_to_single_gpu(L, d, world, dtype):
    ref, got = _emulate(L, d, world, dtype, k=5)
    assert torch.equal(ref, got)


def test_sharded_without_gradient_and_fixed_ring():
    ref, got = _emulate(24, 2048, 4, torch.float32, k=0, with_g=False)
    assert torch.equal(ref, got)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_d1d_partial_sum_and_apply_reproduce_mean_step(dtype):
    L, d, world = 64, 100_003, 8
    lay = D.ShardLayout(L, world)
    g = torch.Generator(device="cuda").manual_seed(3)
    W = mixing.empty_learner_major(L, d, dtype)
    W.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    G = mixing.empty_learner_major(L, d, dtype)
    G.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    ref = mixing.mean_mix_sgd(W, G, 0.01)
    lib = _lib.load()
    sfx = mixing._suffix(W)
    S_parts = []
    for r in range(world):
        b, e = lay.rows(r)
        S = torch.empty(d, dtype=torch.float64, device="cuda")
        _lib.check(getattr(lib, f"rm_partial_sum_{sfx}")(
            W[b:e].data_ptr(), e - b, d, W.stride(0), S.data_ptr(), _lib.stream_ptr()))
        S_parts.append(S)
    S = torch.stack(S_parts).sum(0)          # what the all-reduce computes
    out = mixing.empty_learner_major(L, d, dtype)
    for r in range(world):
        b, e = lay.rows(r)
        _lib.check(getattr(lib, f"rm_apply_mean_sgd_{sfx}")(
            S.data_ptr(), G[b:e].data_ptr(), out[b:e].data_ptr(), e - b, L, d, G.stride(0),
            out.stride(0), 0.01, None, _lib.stream_ptr()))
    torch.cuda.synchronize()
    # the all-reduced sum is not numpy's pairwise order: agree to fp64 rounding of the sum
    diff = (out.double() - ref.double()).abs()
    scale = W.double().abs().mean(0, keepdim=True) + 0.01 * G.double().abs()
    if dtype == torch.float64:
        assert bool((diff <= 1e-14 * scale).all())
    else:
        assert bool((diff <= 2.0**-23 * (ref.double().abs() + scale)).all())
        assert float((out != ref).double().mean()) < 1e-4


@pytest.mark.parametrize("L,d,world", [(24, 3001, 4), (64, 2049, 8), (10, 77, 3), (16, 1000, 2)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_position_layout_steps_bit_identical_to_single_gpu(L, d, world, dtype):
    """RAD in ring-position order, ranks emulated in one process: after every step the
    slot of position x holds learner inv_{k+1}[x], equal to the single-GPU step."""
    lay = D.ShardLayout(L, world)
    g = torch.Generator(device="cuda").manual_seed(L + d)
    full = mixing.empty_learner_major(L, d, dtype)
    full.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    Gf = mixing.empty_learner_major(L, d, dtype)
    Gf.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    K = 4
    tabs = mixing.permutation_tables(L, 777, 0, K + 1)
    inv = tabs.inv
    bufs = [[mixing.empty_learner_major(e - b, d, dtype) for _ in range(2)]
            for (b, e) in lay.bounds]
    esz = full.element_size()
    slots = [D._slot_table(lay, [bufs[r][p].data_ptr() for r in range(world)],
                           bufs[0][0].stride(0), esz, "cuda") for p in range(2)]
    inv0 = inv[0].long()
    for r, (b, e) in enumerate(lay.bounds):
        bufs[r][0].copy_(full[inv0[b:e]])
    lib = _lib.load()
    fn = getattr(lib, f"rm_ring_mix_sgd_pos_{mixing._suffix(full)}")
    ref = full
    cur = 0
    for k in range(K):
        ik = inv[k].contiguous()
        pn = tabs.perm[k + 1].contiguous()
        for r, (b, e) in enumerate(lay.bounds):
            Lg = e - b
            plan = torch.empty(lib.rm_shard_plan_ints(Lg), dtype=torch.int32, device="cuda")
            dest = torch.empty(Lg, dtype=torch.int64, device="cuda")
            _lib.check(lib.rm_pos_plan(ik.data_ptr(), pn.data_ptr(), L, b, Lg,
                                       slots[1 - cur].data_ptr(), plan.data_ptr(),
                                       dest.data_ptr(), _lib.stream_ptr()))
            Gs = mixing.empty_learner_major(Lg, d, dtype)
            Gs.copy_(Gf[ik[b:e].long()])          # gradient of the learner in each slot
            src = bufs[r][cur]
            _lib.check(fn(slots[cur].data_ptr(), src.data_ptr(), Gs.data_ptr(), L, b, Lg, d,
                          src.stride(0), Gs.stride(0), plan.data_ptr(), dest.data_ptr(), 0.02,
                          None, _lib.stream_ptr(), None))
            torch.cuda.synchronize()
        cur = 1 - cur
        lt, rt = tabs.step(k)
        ref = mixing.ring_mix_sgd(ref, Gf, 0.02, lt.contiguous(), rt.contiguous())
        torch.cuda.synchronize()
        nxt = inv[k + 1].long()
        for r, (b, e) in enumerate(lay.bounds):
            assert torch.equal(bufs[r][cur], ref[nxt[b:e]]), (k, r)

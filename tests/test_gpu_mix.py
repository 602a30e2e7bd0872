"""Fused mix + SGD kernels vs the oracle, through the C-ABI.

Contract:
* fp64 storage: bit-exact with the oracle's explicit rounding sequence
  (oracle/mix_oracle.c), and within the reference's own atol 1e-15 of the
  reference's fp64 output (golden fixtures; OpenBLAS's edge columns round
  differently).
* fp32 storage: bit-exact with fl32(oracle fp64 result on the same fp32
  inputs) — i.e. the reference's fp64 arithmetic rounded once — which implies
  the north-star tolerance |y - y_ref| <= 1e-6 * ((|w_l|+|w_j|+|w_r|)/3 + |lr g|)
  (checked too).
* bf16 storage: fp32 arithmetic; within 1 bf16 ulp of the fp64 result.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import _lib, mixing

pytestmark = pytest.mark.gpu

DT = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}


def _rand(L, d, dtype, seed, ld=None, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = mixing.empty_learner_major(L, d, dtype, "cuda") if ld is None else \
        torch.empty((L, ld), dtype=dtype, device="cuda")[:, :d]
    X.copy_((torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64) * scale)
            .to(dtype))
    return X


def _host_dL(X):
    """learner-major CUDA tensor -> reference (d, L) fp64 numpy."""
    return np.ascontiguousarray(X.to(torch.float64).cpu().numpy().T)


def _tables(L, seed, k):
    p = O.c_permutation(L, seed, k)
    _, left, right = O.neighbour_tables(p)
    return (torch.from_numpy(left.astype(np.int32)).cuda(),
            torch.from_numpy(right.astype(np.int32)).cuda(), left, right)


def _abi_ring(X, G, out, left, right, lr, absmax=None):
    L, d = X.shape
    fn = getattr(_lib.load(), f"rm_ring_mix_sgd_{ {torch.float32: 'f32', torch.float64: 'f64', torch.bfloat16: 'bf16'}[X.dtype]}")
    rc = fn(X.data_ptr(), None if G is None else G.data_ptr(), out.data_ptr(), left.data_ptr(),
            right.data_ptr(), L, d, X.stride(0), (G if G is not None else X).stride(0),
            out.stride(0), lr, None if absmax is None else absmax.data_ptr(), _lib.stream_ptr())
    _lib.check(rc)
    torch.cuda.synchronize()


SHAPES = [(4, 1), (5, 7), (8, 64), (16, 1000), (16, 4099), (33, 33), (64, 1031), (128, 777),
          (200, 130), (1000, 37), (1500, 19)]


@pytest.mark.parametrize("L,d", SHAPES)
@pytest.mark.parametrize("with_g", [True, False])
def test_ring_f64_bit_exact_vs_oracle(L, d, with_g):
    X = _rand(L, d, torch.float64, L * 1000 + d)
    G = _rand(L, d, torch.float64, 7 + d) if with_g else None
    lt, rt, left, right = _tables(L, 12345, d)
    out = mixing.empty_learner_major(L, d, torch.float64)
    _abi_ring(X, G, out, lt, rt, 0.01)
    ref = O.c_ring_mix_sgd(_host_dL(X), None if G is None else _host_dL(G), 0.01, left, right)
    assert np.array_equal(_host_dL(out), ref)


@pytest.mark.parametrize("L,d", SHAPES)
def test_ring_f32_is_reference_fp64_rounded_once(L, d):
    X = _rand(L, d, torch.float32, L + d)
    G = _rand(L, d, torch.float32, 3 * d + 1)
    lt, rt, left, right = _tables(L, 42, L)
    lr = 0.05
    out = mixing.ring_mix_sgd(X, G, lr, lt, rt)
    torch.cuda.synchronize()
    W64, G64 = _host_dL(X), _host_dL(G)
    ref64 = O.c_ring_mix_sgd(W64, G64, lr, left, right)
    got = _host_dL(out)
    assert np.array_equal(got, ref64.astype(np.float32).astype(np.float64))
    # north-star tolerance vs the reference's own numpy arithmetic (W @ T - lr G)
    if L != 3:
        ref_np = O.numpy_gossip_step(W64, G64, lr, perm=O.c_permutation(L, 42, L))
        assert O.magnitude_tolerance_ok(got, ref_np, W64, G64, lr, left, right)


@pytest.mark.parametrize("L,d", [(4, 1), (8, 64), (16, 1000), (64, 1031), (128, 4096)])
def test_ring_bf16_within_one_ulp(L, d):
    X = _rand(L, d, torch.bfloat16, L + 5 * d)
    G = _rand(L, d, torch.bfloat16, d)
    lt, rt, left, right = _tables(L, 5, 3)
    out = mixing.ring_mix_sgd(X, G, 0.1, lt, rt)
    ref = O.c_ring_mix_sgd(_host_dL(X), _host_dL(G), 0.1, left, right)
    got = _host_dL(out)
    ulp = np.abs(torch.from_numpy(ref).to(torch.bfloat16).to(torch.float64).numpy()) * 2.0**-7
    # fp32 arithmetic error (~1e-7 of the inputs) can exceed one bf16 ulp of a
    # nearly cancelled result, hence the absolute floor
    assert np.all(np.abs(got - ref) <= np.maximum(ulp, 1e-6))


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("L,d", [(1, 5), (2, 9), (3, 100), (5, 33), (8, 1000), (16, 4099),
                                 (64, 1031), (129, 300), (300, 40)])
def test_mean_bit_exact_vs_oracle(dtype, L, d):
    X = _rand(L, d, DT[dtype], L * 7 + d)
    G = _rand(L, d, DT[dtype], d + 11)
    out = mixing.mean_mix_sgd(X, G, 0.01)
    ref = O.c_mean_sgd(_host_dL(X), _host_dL(G), 0.01)
    if dtype == "f32":
        ref = ref.astype(np.float32).astype(np.float64)
    got = _host_dL(out)
    assert np.array_equal(got, ref)
    # exact consensus of the average (reference test_mixing.py:104-111)
    avg = mixing.mean_mix_sgd(X, None, 0.0)
    a = _host_dL(avg)
    assert np.all(a == a[:, :1])


def test_l3_ring_takes_exact_mean_path():
    X = _rand(3, 500, torch.float64, 1)
    G = _rand(3, 500, torch.float64, 2)
    lt, rt, _, _ = _tables(3, 1, 0)
    a = mixing.ring_mix_sgd(X, G, 0.1, lt, rt)
    b = mixing.mean_mix_sgd(X, G, 0.1)
    assert torch.equal(a, b)


@pytest.mark.parametrize("dtype", ["f32", "f64", "bf16"])
def test_spsgd_update_and_mismatch_flag(dtype):
    L, d = 6, 333
    w = _rand(1, d, DT[dtype], 3)
    X = mixing.empty_learner_major(L, d, DT[dtype])
    X.copy_(w.expand(L, d))
    G = _rand(L, d, DT[dtype], 4)
    mm = torch.zeros((), dtype=torch.int32, device="cuda")
    out = mixing.spsgd_update(X, G, 0.1, mismatch=mm)
    assert int(mm) == 0
    m = O.c_mean_sgd(_host_dL(G), None, 0.0)
    ref = _host_dL(X) - 0.1 * m
    got = _host_dL(out)
    if dtype == "f64":
        assert np.array_equal(got, ref)
    elif dtype == "f32":
        assert np.array_equal(got, ref.astype(np.float32).astype(np.float64))
    else:
        assert np.allclose(got, ref, rtol=2**-7, atol=1e-6)
    X[2, 17] += 1.0
    mixing.spsgd_update(X, G, 0.1, mismatch=mm)
    assert int(mm) != 0


def test_unaligned_layout_uses_scalar_path_and_agrees():
    L, d = 8, 1001
    X = _rand(L, d, torch.float32, 9, ld=1003)   # 4-byte-misaligned rows
    G = _rand(L, d, torch.float32, 10, ld=1005)
    lt, rt, left, right = _tables(L, 8, 8)
    out = torch.empty((L, 1007), dtype=torch.float32, device="cuda")[:, :d]
    mixing.ring_mix_sgd(X, G, 0.25, lt, rt, out=out)
    ref = O.c_ring_mix_sgd(_host_dL(X), _host_dL(G), 0.25, left, right)
    assert np.array_equal(_host_dL(out), ref.astype(np.float32).astype(np.float64))


def test_fused_divergence_epilogue():
    L, d = 16, 5000
    X = _rand(L, d, torch.float32, 1)
    G = _rand(L, d, torch.float32, 2)
    lt, rt, _, _ = _tables(L, 1, 1)
    amax = torch.zeros((), dtype=torch.int64, device="cuda")
    out = mixing.ring_mix_sgd(X, G, 0.1, lt, rt, absmax=amax)
    from paper_2002_01119_b200.simulation import absmax_value
    assert absmax_value(amax) == float(out.abs().max())
    X[3, 77] = float("inf")
    amax.zero_()
    mixing.ring_mix_sgd(X, G, 0.1, lt, rt, absmax=amax)
    assert np.isinf(absmax_value(amax))
    X[3, 77] = float("nan")
    amax.zero_()
    mixing.ring_mix_sgd(X, G, 0.1, lt, rt, absmax=amax)
    assert np.isnan(absmax_value(amax))


def test_argument_errors_mirror_reference():
    X = _rand(8, 10, torch.float32, 1)
    lt, rt, _, _ = _tables(8, 1, 1)
    with pytest.raises(ValueError, match="read-after-write"):
        mixing.ring_mix_sgd(X, None, 0.1, lt, rt, out=X)
    with pytest.raises(ValueError):
        mixing.ring_mix_sgd(X, _rand(8, 11, torch.float32, 2), 0.1, lt, rt)
    X2 = _rand(2, 10, torch.float32, 1)
    lt2 = torch.zeros(2, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match="degenerate"):
        mixing.ring_mix_sgd(X2, None, 0.1, lt2, lt2)


def test_apply_mixing_matches_reference_semantics():
    # reference test_mixing.py:97-111 (ring vs W @ T; uniform collapses exactly)
    L = 8
    rng = np.random.default_rng(0)
    W = rng.standard_normal((5, L))
    T = mixing.build_ring_matrix(L)
    assert np.allclose(mixing.apply_mixing(W, T), W @ T, rtol=0, atol=1e-15)
    p = O.c_permutation(L, 3, 3)
    Tp = T[np.ix_(p, p)]
    assert np.allclose(mixing.apply_mixing(W, Tp), W @ Tp, rtol=0, atol=1e-15)
    U = mixing.build_uniform_matrix(L)
    mixed = mixing.apply_mixing(W, U)
    assert np.all(mixed == mixed[:, :1])
    assert np.array_equal(mixed[:, 0], W.mean(axis=1))
    # generic dense T -> library GEMM
    A = rng.random((L, L))
    assert np.allclose(mixing.apply_mixing(W, A), W @ A, atol=1e-12)
    # torch (d, L) view input keeps dtype/device
    Wt = torch.from_numpy(W.T.copy()).cuda().float().T
    out = mixing.apply_mixing(Wt, T)
    assert out.is_cuda and out.dtype == torch.float32 and tuple(out.shape) == (5, L)
    with pytest.raises(ValueError, match="size mismatch"):
        mixing.apply_mixing(W, mixing.build_ring_matrix(L + 1))


@pytest.mark.slow
def test_full_size_c1_bit_exact():
    """BASELINE config 1 at full size (16 x 2^20 fp32): bit-exact vs the C oracle."""
    L, d = 16, 1 << 20
    X = _rand(L, d, torch.float32, 100)
    G = _rand(L, d, torch.float32, 101)
    lt, rt, left, right = _tables(L, 12345, 0)
    out = mixing.ring_mix_sgd(X, G, 0.01, lt, rt)
    ref = O.c_ring_mix_sgd(_host_dL(X), _host_dL(G), 0.01, left, right)
    assert np.array_equal(_host_dL(out), ref.astype(np.float32).astype(np.float64))


@pytest.mark.slow
def test_full_size_c2_properties():
    """BASELINE config 2 shape (64 x 25,557,032 fp32, 6.5 GB/buffer): size-independent
    properties — mass conservation (doubly stochastic T), sampled columns bit-exact vs
    the oracle, and the divergence epilogue equals max|W'|."""
    L, d = 64, 25_557_032
    X = _rand(L, d, torch.float32, 200)
    G = _rand(L, d, torch.float32, 201)
    lt, rt, left, right = _tables(L, 12345, 7)
    amax = torch.zeros((), dtype=torch.int64, device="cuda")
    out = mixing.ring_mix_sgd(X, G, 0.01, lt, rt, absmax=amax)
    # mean over learners moves by -lr * mean(G) (reference test_simulation.py:159-170)
    moved = out.double().mean(0) - X.double().mean(0)
    expect = -0.01 * G.double().mean(0)
    assert torch.allclose(moved, expect, rtol=0, atol=1e-6)
    from paper_2002_01119_b200.simulation import absmax_value
    assert absmax_value(amax) == float(out.abs().max())
    cols = torch.randint(0, d, (4096,), generator=torch.Generator().manual_seed(0))
    cols = torch.cat([cols, torch.tensor([0, 1, d - 2, d - 1])])
    Xs, Gs, Os = (t[:, cols.cuda()].contiguous() for t in (X, G, out))
    ref = O.c_ring_mix_sgd(_host_dL(Xs), _host_dL(Gs), 0.01, left, right)
    assert np.array_equal(_host_dL(Os), ref.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("dtype", ["f32", "f64", "bf16"])
def test_empty_parameter_vectors(dtype):
    """d = 0 (the reference's (0, L) weight matrix): every kernel entry point returns
    an empty result without launching, and the absmax stays at zero."""
    L = 16
    X = mixing.empty_learner_major(L, 0, DT[dtype], "cuda")
    G = mixing.empty_learner_major(L, 0, DT[dtype], "cuda")
    lt, rt, _, _ = _tables(L, 3, 0)
    assert mixing.ring_mix_sgd(X, G, 0.1, lt, rt).shape == (L, 0)
    assert mixing.mean_mix_sgd(X, G, 0.1).shape == (L, 0)
    assert mixing.spsgd_update(X, G, 0.1).shape == (L, 0)
    out = mixing.empty_learner_major(L, 0, DT[dtype], "cuda")
    absmax = torch.zeros(1, dtype=torch.int64, device="cuda")
    _abi_ring(X, G, out, lt, rt, 0.1, absmax)
    assert int(absmax.item()) == 0


def test_single_column_and_ragged_tails_all_dtypes():
    """d = 1 and d one past a vector multiple: the TMA tile path's ragged tail and the
    scalar path agree with the oracle (fp64 bit-exact, fp32 rounded once)."""
    for L, d in [(8, 1), (16, 5), (64, 129), (64, 4097)]:
        X = _rand(L, d, torch.float64, 11 * L + d)
        G = _rand(L, d, torch.float64, 5 * d + 3)
        lt, rt, left, right = _tables(L, 99, d)
        out = mixing.ring_mix_sgd(X, G, 0.02, lt, rt)
        ref = O.c_ring_mix_sgd(_host_dL(X), _host_dL(G), 0.02, left, right)
        assert np.array_equal(_host_dL(out), ref)
        X32, G32 = X.float(), G.float()
        out32 = mixing.ring_mix_sgd(X32, G32, 0.02, lt, rt)
        ref32 = O.c_ring_mix_sgd(_host_dL(X32), _host_dL(G32), 0.02, left, right)
        assert np.array_equal(_host_dL(out32), ref32.astype(np.float32).astype(np.float64))


def test_parameter_vectors_beyond_2_31_columns():
    """Maximum sizes: d = 2^31 + 37 columns (past the 32-bit tile coordinates the TMA
    path uses, so the 64-bit-indexed kernel takes over), L = 4, fp32, G = NULL:
    ~69 GB of HBM.  Sampled columns, including both ends, are bit-exact vs the oracle,
    and the divergence epilogue sees the whole matrix."""
    free, _ = torch.cuda.mem_get_info()
    L, d = 4, (1 << 31) + 37
    if free < 2 * L * d * 4 + (8 << 30):
        pytest.skip("needs ~77 GB of free HBM")
    X = mixing.empty_learner_major(L, d, torch.float32, "cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    for r in range(L):
        X[r].normal_(generator=g)
    lt, rt, left, right = _tables(L, 99, 3)
    amax = torch.zeros((), dtype=torch.int64, device="cuda")
    out = mixing.ring_mix_sgd(X, None, 0.0, lt, rt, absmax=amax)
    torch.cuda.synchronize()
    cols = torch.randint(0, d, (4096,), generator=torch.Generator().manual_seed(1))
    cols = torch.cat([cols, torch.arange(0, 64), torch.arange(d - 64, d),
                      torch.arange((1 << 31) - 32, (1 << 31) + 32)]).cuda()
    Xs, Os = X[:, cols].contiguous(), out[:, cols].contiguous()
    ref = O.c_ring_mix_sgd(_host_dL(Xs), None, 0.0, left, right)
    assert np.array_equal(_host_dL(Os), ref.astype(np.float32).astype(np.float64))
    from paper_2002_01119_b200.simulation import absmax_value
    assert absmax_value(amax) == float(max(out[r].abs().max().item() for r in range(L)))
    del X, out
    torch.cuda.empty_cache()

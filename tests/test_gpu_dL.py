"""The step on the reference's own (d, L) C-order arrays (rm_gossip_step_dL_*, device;
rm_gossip_step_host_dL_*, host arrays pipelined over row chunks): bit-exact against the
oracle's restatement of simulation._gossip_step (simulation.py:263-268) for the ring,
ring[p, p] and uniform (D1D, mixing.py:122-124) matrices."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import mixing

pytestmark = pytest.mark.gpu


def _data(d, L, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((d, L)), rng.standard_normal((d, L))


def _tabs(L, seed, k):
    _, left, right = O.neighbour_tables(O.c_permutation(L, seed, k))
    return left.astype(np.int32), right.astype(np.int32)


@pytest.mark.parametrize("d,L", [(1, 4), (1000, 16), (4099, 64), (777, 128), (300, 5),
                                 (65_537, 10), (50, 3), (2049, 256)])
def test_host_dL_f64_ring_and_mean_bit_exact(d, L):
    W, G = _data(d, L, d + L)
    left, right = _tabs(L, 4242, 7) if L >= 3 else (None, None)
    out = mixing.gossip_step_host(W, G, 0.01, left, right)
    ref = O.c_ring_mix_sgd(W, G, 0.01, left, right) if L != 3 else O.c_mean_sgd(W, G, 0.01)
    assert np.array_equal(out, ref)
    mean = mixing.gossip_step_host(W, G, 0.01)
    assert np.array_equal(mean, O.c_mean_sgd(W, G, 0.01))
    # apply_mixing semantics (G = None) and a small workspace (many row chunks)
    ws = mixing.workspace_dL(L, 7, np.float64)
    am = mixing.gossip_step_host(W, None, 0.0, left, right, workspace=ws)
    assert np.array_equal(am, O.c_ring_mix_sgd(W, None, 0.0, left, right) if L != 3 else
                          O.c_mean_sgd(W, None, 0.0))


@pytest.mark.parametrize("d,L", [(1000, 16), (4099, 64), (33, 7)])
def test_host_dL_f32_rounds_the_fp64_result_once(d, L):
    W64, G64 = _data(d, L, 3 * d + L)
    W, G = W64.astype(np.float32), G64.astype(np.float32)
    left, right = _tabs(L, 9, 2)
    out = mixing.gossip_step_host(W, G, 0.02, left, right)
    ref = O.c_ring_mix_sgd(W.astype(np.float64), G.astype(np.float64), 0.02, left, right)
    assert out.dtype == np.float32 and np.array_equal(out, ref.astype(np.float32))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_device_dL_matches_learner_major_kernel(dtype):
    """(d, L) device layout and learner-major layout give the same bits."""
    d, L = 100_003, 64
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn((d, L), generator=g, device="cuda", dtype=torch.float64).to(dtype)
    Gt = torch.randn((d, L), generator=g, device="cuda", dtype=torch.float64).to(dtype)
    tabs = mixing.permutation_tables(L, 12345, 3, 1)
    lt, rt = tabs.left[0].contiguous(), tabs.right[0].contiguous()
    amax = torch.zeros((), dtype=torch.int64, device="cuda")
    out = mixing.gossip_step_dL(X, Gt, 0.01, lt, rt, absmax=amax)
    Wl = mixing.empty_learner_major(L, d, dtype)
    Wl.copy_(X.T)
    Gl = mixing.empty_learner_major(L, d, dtype)
    Gl.copy_(Gt.T)
    ref = mixing.ring_mix_sgd(Wl, Gl, 0.01, lt, rt)
    assert torch.equal(out.T, ref)
    from paper_2002_01119_b200.simulation import absmax_value
    assert absmax_value(amax) == float(out.abs().max())
    mean = mixing.gossip_step_dL(X, Gt, 0.01)
    assert torch.equal(mean.T, mixing.mean_mix_sgd(Wl, Gl, 0.01))


def test_apply_mixing_on_numpy_uses_the_dL_path_and_keeps_errors():
    L = 12
    W, _ = _data(500, L, 1)
    p = O.c_permutation(L, 5, 0)
    T = mixing.conjugate_by_permutation(mixing.build_ring_matrix(L), p)
    _, left, right = O.neighbour_tables(p)
    assert np.array_equal(mixing.apply_mixing(W, T), O.c_ring_mix_sgd(W, None, 0.0, left, right))
    U = mixing.build_uniform_matrix(L)
    mixed = mixing.apply_mixing(W, U)
    assert np.all(mixed == mixed[:, :1])                     # reference test_mixing.py:104-111
    with pytest.raises(ValueError, match="size mismatch"):
        mixing.apply_mixing(W, mixing.build_ring_matrix(L + 1))
    with pytest.raises(ValueError):
        mixing.gossip_step_host(W, np.zeros((500, L + 1)), 0.1)


def test_empty_and_invalid():
    W = np.zeros((0, 8))
    assert mixing.gossip_step_host(W, None, 0.1).shape == (0, 8)
    with pytest.raises(ValueError):
        mixing.gossip_step_host(np.zeros((4, 8)), None, 0.1, left=np.arange(8))
    with pytest.raises(ValueError, match="degenerate ring"):
        mixing.gossip_step_host(np.zeros((4, 2)), None, 0.1, left=[1, 0], right=[1, 0])

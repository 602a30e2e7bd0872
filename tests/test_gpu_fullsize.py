"""BASELINE configs at their full sizes on one B200, checked through size-independent
properties and sampled columns against the C oracle (rows of W are independent — column
c of W' depends only on column c of W and G — so a sampled-column check is exact):

* C3: RAD-PSGD, 128 learners x 43,154,944 fp32 (LSTM acoustic model; 22.1 GB per
  buffer, 66 GB for W, G, W') — simulation.py:285-301 / :263-268;
* C4: D1D-PSGD, 64 learners x 25,557,032 fp32 — simulation.py:304-312;
* C2 with the fixed ring (AD-PSGD, simulation.py:276-282) and in bf16 storage.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import mixing
from paper_2002_01119_b200.simulation import absmax_value

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _need(bytes_):
    free, _ = torch.cuda.mem_get_info()
    if free < bytes_ + (4 << 30):
        pytest.skip(f"needs {bytes_ / 2**30:.0f} GiB of free HBM")


def _rand(L, d, dtype, seed):
    X = mixing.empty_learner_major(L, d, dtype, "cuda")
    g = torch.Generator(device="cuda").manual_seed(seed)
    for r in range(L):
        X[r].copy_(torch.randn(d, generator=g, device="cuda").to(dtype))
    return X


def _host_dL(X):
    return X.double().cpu().numpy().T.copy()


def _sample_cols(d, seed, n=4096, tile=128):
    cols = torch.randint(0, d, (n,), generator=torch.Generator().manual_seed(seed))
    edges = torch.tensor([0, 1, 2, 3, tile - 1, tile, tile + 1, d // 2, d - 5, d - 4, d - 3,
                          d - 2, d - 1])
    return torch.cat([cols, edges]).cuda()


def _tables(L, seed, k):
    p = O.c_permutation(L, seed, k)
    _, left, right = O.neighbour_tables(p)
    return (torch.from_numpy(left.astype(np.int32)).cuda(),
            torch.from_numpy(right.astype(np.int32)).cuda(), left, right)


@pytest.fixture(autouse=True)
def _release_hbm():
    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def test_full_size_c3_rad_128_learners():
    L, d = 128, 43_154_944
    _need(3 * L * d * 4)
    X = _rand(L, d, torch.float32, 300)
    G = _rand(L, d, torch.float32, 301)
    lt, rt, left, right = _tables(L, 12345, 11)
    amax = torch.zeros((), dtype=torch.int64, device="cuda")
    out = mixing.ring_mix_sgd(X, G, 0.01, lt, rt, absmax=amax)
    torch.cuda.synchronize()
    cols = _sample_cols(d, 3)
    Xs, Gs, Os = (t[:, cols].contiguous() for t in (X, G, out))
    ref = O.c_ring_mix_sgd(_host_dL(Xs), _host_dL(Gs), 0.01, left, right)
    assert np.array_equal(_host_dL(Os), ref.astype(np.float32).astype(np.float64))
    # the divergence epilogue saw the whole 5.5 G-element output
    assert absmax_value(amax) == float(max(out[r].abs().max().item() for r in range(L)))
    # mass conservation of a doubly stochastic T, per column (reference
    # test_simulation.py:159-170), on a 1 M-column stripe in fp64
    s = slice(d // 3, d // 3 + (1 << 20))
    moved = out[:, s].double().mean(0) - X[:, s].double().mean(0)
    assert torch.allclose(moved, -0.01 * G[:, s].double().mean(0), rtol=0, atol=1e-6)


def test_full_size_c4_d1d_64_learners():
    L, d = 64, 25_557_032
    _need(3 * L * d * 4)
    X = _rand(L, d, torch.float32, 400)
    G = _rand(L, d, torch.float32, 401)
    amax = torch.zeros((), dtype=torch.int64, device="cuda")
    out = mixing.mean_mix_sgd(X, G, 0.01, absmax=amax)
    torch.cuda.synchronize()
    cols = _sample_cols(d, 4)
    Xs, Gs, Os = (t[:, cols].contiguous() for t in (X, G, out))
    ref = O.c_mean_sgd(_host_dL(Xs), _host_dL(Gs), 0.01)
    assert np.array_equal(_host_dL(Os), ref.astype(np.float32).astype(np.float64))
    assert absmax_value(amax) == float(max(out[r].abs().max().item() for r in range(L)))
    # without gradients every learner holds the exact column mean (consensus)
    cons = mixing.mean_mix_sgd(X, None, 0.0)
    s = slice(d - (1 << 16), d)
    assert bool((cons[:, s] == cons[0:1, s]).all())


def test_full_size_c2_fixed_ring_and_bf16():
    L, d = 64, 25_557_032
    _need(3 * L * d * 4)
    X = _rand(L, d, torch.float32, 500)
    G = _rand(L, d, torch.float32, 501)
    ident = np.arange(L)
    left, right = np.roll(ident, 1), np.roll(ident, -1)
    lt = torch.from_numpy(left.astype(np.int32)).cuda()
    rt = torch.from_numpy(right.astype(np.int32)).cuda()
    out = mixing.ring_mix_sgd(X, G, 0.01, lt, rt)
    cols = _sample_cols(d, 5)
    Xs, Gs, Os = (t[:, cols].contiguous() for t in (X, G, out))
    ref = O.c_ring_mix_sgd(_host_dL(Xs), _host_dL(Gs), 0.01, left, right)
    assert np.array_equal(_host_dL(Os), ref.astype(np.float32).astype(np.float64))
    del out
    # bf16 storage: the fp32 sequence on bf16 inputs, within one bf16 ulp of the oracle
    Xb, Gb = X.to(torch.bfloat16), G.to(torch.bfloat16)
    del X, G
    lt2, rt2, left2, right2 = _tables(L, 12345, 3)
    ob = mixing.ring_mix_sgd(Xb, Gb, 0.01, lt2, rt2)
    Xs, Gs, Os = (t[:, cols].contiguous() for t in (Xb, Gb, ob))
    ref = O.c_ring_mix_sgd(_host_dL(Xs), _host_dL(Gs), 0.01, left2, right2)
    got = _host_dL(Os)
    ulp = np.maximum(np.abs(ref), 1e-30) * 2.0**-7
    assert bool((np.abs(got - ref) <= np.maximum(ulp, 1e-6)).all())

"""Randomised parity sweep through the public API (fixed master seed, so failures
replay): random learner counts, widths, padding (aligned TMA path and unaligned
64-bit path), storage types, learning rates, with and without gradients, for the
ring (RAD / fixed) and mean (D1D) steps, plus random permutation requests with
seeds and steps across the 64-bit range — all against the oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import mixing

pytestmark = pytest.mark.gpu
DT = {"f32": torch.float32, "f64": torch.float64}


def _rows(L, d, ld, dtype, gen):
    buf = torch.empty((L, ld), dtype=dtype, device="cuda")
    X = buf[:, :d]
    X.copy_(torch.randn((L, d), generator=gen, device="cuda", dtype=torch.float64).to(dtype))
    return X


def _host(X):
    return np.ascontiguousarray(X.to(torch.float64).cpu().numpy().T)


def test_random_ring_and_mean_steps_match_oracle():
    rng = np.random.default_rng(20260518)
    gen = torch.Generator(device="cuda").manual_seed(7)
    for case in range(120):
        L = int(rng.choice([3, 4, 5, 7, 8, 16, 31, 64, 100, 128, 257, 300]))
        d = int(rng.integers(1, 6000))
        pad = int(rng.choice([0, 0, 1, 3, 32]))        # 0 / 32: aligned rows, else not
        dtype = str(rng.choice(["f32", "f64"]))
        lr = float(rng.choice([0.0, 0.01, 0.5, 3.0]))
        with_g = bool(rng.integers(0, 2))
        mode = str(rng.choice(["ring", "mean"]))
        X = _rows(L, d, d + pad, DT[dtype], gen)
        G = _rows(L, d, d + pad, DT[dtype], gen) if with_g else None
        if mode == "ring":
            p = O.c_permutation(L, int(rng.integers(0, 2**63)), int(rng.integers(0, 1000)))
            _, left, right = O.neighbour_tables(p)
            lt = torch.from_numpy(left.astype(np.int32)).cuda()
            rt = torch.from_numpy(right.astype(np.int32)).cuda()
            out = mixing.ring_mix_sgd(X, G, lr, lt, rt)
            if L == 3:   # every entry of the 3-ring is 1/3: the reference's exact-mean path
                ref = O.c_mean_sgd(_host(X), None if G is None else _host(G), lr)
            else:
                ref = O.c_ring_mix_sgd(_host(X), None if G is None else _host(G), lr, left,
                                       right)
        else:
            out = mixing.mean_mix_sgd(X, G, lr)
            ref = O.c_mean_sgd(_host(X), None if G is None else _host(G), lr)
        if dtype == "f32":
            ref = ref.astype(np.float32).astype(np.float64)
        assert np.array_equal(_host(out), ref), (case, L, d, pad, dtype, lr, with_g, mode)


def test_random_permutation_requests_match_oracle():
    rng = np.random.default_rng(99)
    for case in range(300):
        n = int(rng.choice([1, 2, 3, 4, 9, 16, 64, 100, 128, 1000, 2048]))
        seed = int(rng.integers(0, 2**63)) * int(rng.integers(1, 3)) + int(rng.integers(0, 2))
        step = int(rng.integers(0, 2**63)) if case % 3 == 0 else int(rng.integers(0, 10**6))
        got = mixing.permutation_for_step(n, seed, step)
        assert np.array_equal(got, O.c_permutation(n, seed, step)), (case, n, seed, step)

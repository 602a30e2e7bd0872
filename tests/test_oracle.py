"""Pin the oracle against the reference's own outputs (golden fixtures) — CPU only.

The oracle (oracle/) is the checker for every GPU parity test, so it is
verified first: bit-exact permutations (C and pure-Python restatements),
sequential streams, the raw PCG64 core, and the step arithmetic against the
reference trajectories frozen by tests/golden/make_golden.py.
"""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import normal_cases, perm_cases, sequential_cases, spectral_golden, step_cases
from oracle import ringmix_oracle as O


def test_golden_numpy_version_recorded():
    z = np.load(O.ORACLE_DIR.parent / "tests" / "golden" / "perms.npz")
    assert str(z["numpy_version"]) == "2.3.5"


def test_c_oracle_permutations_match_reference_golden():
    cases = perm_cases()
    assert len(cases) > 1000
    for L, seed, step, ref in cases:
        got = O.c_permutation(L, seed, step)
        assert np.array_equal(got, ref), (L, seed, step)


def test_python_oracle_permutations_match_reference_golden():
    for L, seed, step, ref in perm_cases():
        if L > 64:
            continue
        assert np.array_equal(O.py_permutation(L, seed, step), ref), (L, seed, step)


def test_oracle_sequential_streams_match_reference_golden():
    for n, seed, trial, count, ref in sequential_cases():
        got = O.c_permutation_sequential(n, seed, trial, count)
        assert np.array_equal(got, ref), (n, seed, trial)
        g = O.PyPCG64(O.entropy_words(seed, O.TAG_TRIAL, trial))
        py = np.stack([g.permutation(n) for _ in range(count)])
        assert np.array_equal(py, ref)


@pytest.mark.parametrize("entropy", [(0,), (5, 1, 0), (2**64 - 1, 1, 2**40 + 5), (3**45, 4, 7),
                                     (1, 2, 3, 4, 5, 6)])
def test_oracle_raw64_matches_numpy_pcg64(entropy):
    words = O.entropy_words(*entropy)
    ref = np.random.PCG64(np.random.SeedSequence(entropy)).random_raw(64)
    assert np.array_equal(O.c_raw64(words, 64), ref)
    g = O.PyPCG64(words)
    assert [g.next64() for _ in range(64)] == [int(x) for x in ref]


def test_entropy_words_match_numpy_coercion():
    for ent in [(0,), (1, 2**32), (2**64 - 1, 0, 7), (3**45,)]:
        ss = np.random.SeedSequence(ent)
        st = O.py_seedseq_state(O.entropy_words(*ent))
        ref = ss.generate_state(4, np.uint64)
        assert [int(x) for x in ref] == st


def test_neighbour_tables_reproduce_conjugated_ring():
    for L in (3, 4, 5, 8, 16, 33):
        p = O.c_permutation(L, 9, 4)
        inv, left, right = O.neighbour_tables(p)
        T = O.ring_matrix(L)[np.ix_(p, p)]
        for j in range(L):
            nz = set(np.nonzero(T[:, j])[0])
            assert nz == {left[j], j, right[j]}
        assert np.array_equal(p[inv], np.arange(L))


def _oracle_step(case, k_step, W, Wprev):
    """One reference step restated by the C oracle on (d, L) fp64 arrays."""
    s, L = case["strategy"], case["L"]
    G = case["G"][k_step]
    k = case["k0"] + k_step
    lr = case["lr"]
    if s == "spsgd":
        m = O.c_mean_sgd(G, None, 0.0)
        return W - lr * m
    if s == "d1d" or L == 3:
        return O.c_mean_sgd(W, G, lr)
    if s == "rand_psgd":
        p = O.c_permutation(L, case["seed"], k)
    else:
        p = np.arange(L)
    _, left, right = O.neighbour_tables(p)
    return O.c_ring_mix_sgd(W, G, lr, left, right)


def _uses_mean_path(case) -> bool:
    return case["strategy"] in ("d1d", "spsgd") or case["L"] == 3


@pytest.mark.parametrize("case", step_cases(), ids=lambda c: f"{c['strategy']}-L{c['L']}-d{c['d']}")
def test_c_oracle_step_trajectories(case):
    """The scalar C restatement reproduces the reference's fp64 step outputs.

    Mean path (D1D, S-PSGD, L = 3): bit for bit (numpy pairwise summation is
    deterministic).  Ring path: the reference's `W @ T` is an OpenBLAS dgemm
    whose rounding order is implementation-defined; its main kernel
    accumulates ascending k with FMA (what the oracle restates, bit-exact on
    most columns) but its N-remainder columns use separate mul/add.  There the
    oracle agrees to the reference's own test tolerance (atol 1e-15,
    test_simulation.py:133)."""
    W, Wp = case["W0"], case["Wprev"]
    for s in range(case["nsteps"]):
        out = _oracle_step(case, s, W, Wp)
        ref = case["traj"][s]
        if _uses_mean_path(case):
            assert np.array_equal(out, ref), (case["strategy"], s)
        else:
            assert np.allclose(out, ref, rtol=0, atol=1e-15), (case["strategy"], s)
            assert (out != ref).mean() < 0.05
        W, Wp = ref, W


@pytest.mark.parametrize("case", step_cases(), ids=lambda c: f"{c['strategy']}-L{c['L']}")
def test_numpy_oracle_step_trajectories(case):
    W = case["W0"]
    L = case["L"]
    for s in range(case["nsteps"]):
        k = case["k0"] + s
        G = case["G"][s]
        if case["strategy"] == "spsgd":
            out = O.numpy_spsgd(W, G, case["lr"])
        elif case["strategy"] == "d1d":
            out = O.numpy_gossip_step(W, G, case["lr"], uniform=True)
        else:
            p = O.c_permutation(L, case["seed"], k) if case["strategy"] == "rand_psgd" else None
            out = O.numpy_gossip_step(W, G, case["lr"], perm=p)
        assert np.array_equal(out, case["traj"][s])
        W = out


def test_c_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 8, 9, 64, 127, 128, 129, 300, 1025):
        a = rng.standard_normal(n) * np.exp(3 * rng.standard_normal(n))
        assert O.lib().or_pairwise_sum(np.ascontiguousarray(a).ctypes.data, n) == a.sum()


def test_spectral_golden_closed_forms():
    z = spectral_golden()
    for L, rho in zip(z["L"], z["rho"]):
        assert rho == 1.0 / 3.0 + (2.0 / 3.0) * np.cos(2.0 * np.pi / L)


def test_magnitude_tolerance_helper():
    rng = np.random.default_rng(1)
    W = rng.standard_normal((50, 8))
    G = rng.standard_normal((50, 8))
    p = O.c_permutation(8, 1, 1)
    _, left, right = O.neighbour_tables(p)
    ref = O.c_ring_mix_sgd(W, G, 0.1, left, right)
    assert O.magnitude_tolerance_ok(ref.astype(np.float32), ref, W, G, 0.1, left, right)
    assert not O.magnitude_tolerance_ok(ref + 1e-3, ref, W, G, 0.1, left, right)


def test_c_oracle_standard_normal_matches_golden_and_numpy():
    for ent, ref in normal_cases():
        z, draws = O.c_standard_normal(len(ref), *ent)
        assert np.array_equal(z, ref), ent
        assert draws >= len(ref)
    z, _ = O.c_standard_normal(300_000, 77, 0, 1, 2)
    assert np.array_equal(z, np.random.default_rng(np.random.SeedSequence((77, 0, 1, 2)))
                          .standard_normal(300_000))

"""Host-side API (L x L objects, validation, entropy words) — CPU only.

Mirrors the reference's own tests for the mixing-matrix API
(pkg/tests/test_mixing.py:16-95, test_spectral.py:22-31)."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import spectral_golden
from paper_2002_01119_b200 import mixing, seeding, simulation, spectral


def test_ring_structure():
    L = 7
    T = mixing.build_ring_matrix(L)
    for i in range(L):
        for j in range(L):
            want = 1.0 / 3.0 if j in (i, (i + 1) % L, (i - 1) % L) else 0.0
            assert T[i, j] == want


def test_ring_l3_is_dense_uniform():
    assert np.array_equal(mixing.build_ring_matrix(3), mixing.build_uniform_matrix(3))


@pytest.mark.parametrize("L", [0, 1, 2])
def test_ring_rejects_degenerate_sizes(L):
    with pytest.raises(ValueError, match="degenerate"):
        mixing.build_ring_matrix(L)


def test_uniform_entries_and_validation():
    assert np.all(mixing.build_uniform_matrix(5) == 0.2)
    with pytest.raises(ValueError):
        mixing.build_uniform_matrix(0)


@pytest.mark.parametrize("L", [3, 4, 5, 8, 16, 33, 64])
def test_doubly_stochastic(L):
    for T in (mixing.build_ring_matrix(L), mixing.build_uniform_matrix(L)):
        r = mixing.verify_doubly_stochastic(T)
        assert r.ok and r.max_row_error <= 1e-12 and r.max_col_error <= 1e-12


def test_verify_reports_failure_without_raising():
    r = mixing.verify_doubly_stochastic(np.array([[0.9, 0.0], [0.1, 1.0]]))
    assert not r.ok
    assert not mixing.verify_doubly_stochastic(np.ones((2, 3))).ok


def test_conjugation_and_rejection():
    L = 6
    T = mixing.build_ring_matrix(L)
    perm = np.array([3, 0, 5, 1, 4, 2])
    P = np.zeros((L, L))
    P[perm, np.arange(L)] = 1.0
    assert np.allclose(mixing.conjugate_by_permutation(T, perm), P.T @ T @ P, atol=1e-15)
    with pytest.raises(ValueError):
        mixing.conjugate_by_permutation(mixing.build_ring_matrix(4), np.array([0, 1, 1, 2]))


def test_ring_structure_detection():
    L = 9
    perm = np.array([4, 7, 0, 2, 8, 1, 3, 6, 5])
    T = mixing.conjugate_by_permutation(mixing.build_ring_matrix(L), perm)
    left, right = mixing.ring_structure(T)
    inv = np.argsort(perm)
    for j in range(L):
        assert {left[j], right[j]} == {inv[(perm[j] - 1) % L], inv[(perm[j] + 1) % L]}
    assert mixing.ring_structure(mixing.build_uniform_matrix(L)) is None
    assert mixing.ring_structure(np.eye(L)) is None


def test_entropy_words_match_numpy():
    for ent in [(0,), (5, 1, 0), (2**32, 1, 2**40), (3**45, 4)]:
        ours = seeding.entropy_words(*ent)
        ss = np.random.SeedSequence(ent)
        from oracle.ringmix_oracle import py_seedseq_state
        assert [int(x) for x in ss.generate_state(4, np.uint64)] == py_seedseq_state([int(x) for x in ours])
    with pytest.raises(ValueError):
        seeding.entropy_words(1, -1)


def test_cell_seed_matches_reference_formula():
    ss = np.random.SeedSequence((1234, seeding.TAG_CELL, 3, 64, 0))
    assert seeding.cell_seed(1234, 3, 64, 0) == int(ss.generate_state(1, np.uint64)[0])


def test_spectral_closed_forms_match_reference_golden():
    z = spectral_golden()
    Ls = [int(x) for x in z["L"]]
    assert np.array_equal([spectral.second_eigenvalue_ring(L) for L in Ls], z["rho"])
    assert np.array_equal([spectral.spectral_rho(mixing.build_ring_matrix(L)).rho for L in Ls],
                          z["rho_eig"])
    assert np.array_equal([spectral.randomized_frobenius_expectation(L, 5) for L in Ls],
                          z["frob_exp_k5"])
    assert np.array_equal([spectral.randomized_consensus_bound(L, 5) for L in Ls], z["bound_k5"])
    assert np.array_equal(spectral.fixed_consensus_curve(16, 10).distances, z["fixed_curve_16"])


def test_spectral_golden_scalars():
    # reference test_spectral.py:28-31 / test_cli.py:22-26
    assert spectral.second_eigenvalue_ring(3) == pytest.approx(0.0, abs=1e-15)
    assert spectral.second_eigenvalue_ring(4) == pytest.approx(1.0 / 3.0)
    assert spectral.second_eigenvalue_ring(16) == pytest.approx(0.949253021674191, rel=1e-14)
    assert f"{spectral.second_eigenvalue_ring(8):.9f}" == "0.804737854"


def test_spectral_validation():
    with pytest.raises(ValueError):
        spectral.second_eigenvalue_ring(2)
    with pytest.raises(ValueError):
        spectral.fixed_mixing_consensus_bound(8, -1)
    with pytest.raises(ValueError):
        spectral.monte_carlo_consensus(8, 0, 10, 1)
    with pytest.raises(ValueError):
        spectral.monte_carlo_consensus(8, 3, 10, 1, norm_kind="nuclear")
    with pytest.raises(ValueError):
        spectral.monte_carlo_consensus(7, 1, 2, 0, exhaustive=True)


def test_exhaustive_monte_carlo_matches_reference_golden():
    z = spectral_golden()
    ex = spectral.monte_carlo_consensus(5, 1, 2, seed=0, exhaustive=True)
    assert np.allclose(ex.distances, z["exh5_dist"], rtol=1e-14)
    assert np.allclose(ex.squared_distances, z["exh5_sq"], rtol=1e-14)


def test_runconfig_validation_mirrors_reference():
    base = dict(n_learners=4, iterations=5, lr=0.1, batch_size=2, seed=5)
    simulation.RunConfig(**base)
    for bad in [dict(n_learners=0), dict(iterations=0), dict(lr=-1.0), dict(batch_size=0),
                dict(warmup_iters=-1), dict(staleness_mode="eventually"), dict(init_scale=-1),
                dict(data_partition="x"), dict(log_every=0), dict(divergence_threshold=0),
                dict(dtype="float16")]:
        with pytest.raises(ValueError):
            simulation.RunConfig(**{**base, **bad})


def test_learning_rate_warmup_ramp():
    cfg = simulation.RunConfig(n_learners=4, iterations=5, lr=0.2, batch_size=2, seed=5,
                               warmup_iters=4)
    assert simulation.learning_rate(cfg, 0) == pytest.approx(0.05)
    assert simulation.learning_rate(cfg, 3) == pytest.approx(0.2)
    assert simulation.learning_rate(cfg, 10) == 0.2


def test_cost_model_and_clock():
    cm = simulation.CostModel()
    assert cm.allreduce_time(4) == pytest.approx(0.0132, rel=1e-12)
    with pytest.raises(ValueError):
        simulation.CostModel(message_size_bytes=0.0)
    assert simulation.mixing_rho(simulation.Strategy.D1D, 8) == 0.0
    assert simulation.mixing_rho(simulation.Strategy.RAND_PSGD, 16) == pytest.approx(
        0.949253021674191)


def test_hot_path_requires_cuda_without_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        mixing.permutation_for_step(8, 42, 0)
    with pytest.raises(RuntimeError, match="CUDA"):
        mixing.apply_mixing(np.zeros((4, 5)), mixing.build_ring_matrix(5))


@pytest.mark.parametrize("L", [4, 5])
def test_expected_gram_matches_enumeration(L):
    """E[T'T] over all relabellings of the ring equals the closed form (reference
    test_spectral.py:71-79), and it is doubly stochastic with eigenvalues {1, a, ..., a}."""
    import itertools
    import math
    T = mixing.build_ring_matrix(L)
    total = np.zeros((L, L))
    for perm in itertools.permutations(range(L)):
        C = mixing.conjugate_by_permutation(T, np.array(perm))
        total += C.T @ C
    G = spectral.expected_gram(L)
    assert np.allclose(total / math.factorial(L), G, atol=1e-14)
    eig = np.sort(np.linalg.eigvalsh(G))
    a = 1.0 / 3.0 - 2.0 / (3.0 * (L - 1))
    assert np.allclose(eig, [a] * (L - 1) + [1.0], atol=1e-14)
    with pytest.raises(ValueError):
        spectral.expected_gram(2)


def test_gradient_check_and_evaluate_loss_on_the_quadratic_oracle():
    """Reference acceptance criterion 11's finite-difference half (test_acceptance.py:307-315)
    on the quadratic oracle's host methods (no GPU needed)."""
    from paper_2002_01119_b200.objectives import QuadraticObjective, evaluate_loss, gradient_check
    lam = np.logspace(0.0, 1.0, 32)
    opt = np.random.default_rng(0).standard_normal(32)
    q = QuadraticObjective.__new__(QuadraticObjective)     # host methods only, no device
    q.eigenvalues, q.optimum, q.noise_scale = lam, opt, 1.0
    rng = np.random.default_rng(3)
    for _ in range(5):
        w = rng.standard_normal(32)
        assert gradient_check(q, w) <= 1e-7
        assert evaluate_loss(q, w) == q.loss(w)
    with pytest.raises(ValueError):
        gradient_check(q, w, step=0.0)

"""Device permutation generator: bit-exact against the reference's golden vectors
(frozen from ringmix + numpy 2.3.5) and the C oracle.  Calls go through the C-ABI."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import perm_cases, sequential_cases
from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import _lib, mixing, seeding, spectral

pytestmark = pytest.mark.gpu


def _tables_via_abi(n, seed, step0, nsteps, tag=1):
    words = seeding.entropy_words(seed, tag)
    t = [torch.empty((nsteps, n), dtype=torch.int32, device="cuda") for _ in range(4)]
    rc = _lib.load().rm_perm_tables(words.ctypes.data, len(words), step0, nsteps, n,
                                    *(x.data_ptr() for x in t), _lib.stream_ptr())
    _lib.check(rc, "rm_perm_tables")
    torch.cuda.synchronize()
    return [x.cpu().numpy().astype(np.int64) for x in t]


def test_device_permutations_match_reference_golden():
    cases = perm_cases()
    for L, seed, step, ref in cases:
        perm, inv, left, right = _tables_via_abi(L, seed, step, 1)
        assert np.array_equal(perm[0], ref), (L, seed, step)
        assert np.array_equal(inv[0][ref], np.arange(L))
        _, l_ref, r_ref = O.neighbour_tables(ref)
        assert np.array_equal(left[0], l_ref) and np.array_equal(right[0], r_ref)


def test_permutation_for_step_api_matches_golden():
    for L, seed, step, ref in perm_cases()[::7]:
        got = mixing.permutation_for_step(L, seed, step)
        assert got.dtype == np.int64
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("L,seed", [(16, 12345), (64, seeding.cell_seed(1234, 3, 64, 0)),
                                    (128, 2**64 - 1), (1000, 7)])
def test_batched_steps_match_oracle(L, seed):
    step0, n = 2**32 - 40, 300   # crosses the 32-bit limb boundary of the step index
    perm, inv, left, right = _tables_via_abi(L, seed, step0, n)
    for s in range(0, n, 13):
        ref = O.c_permutation(L, seed, step0 + s)
        assert np.array_equal(perm[s], ref), s
        _, l_ref, r_ref = O.neighbour_tables(ref)
        assert np.array_equal(left[s], l_ref) and np.array_equal(right[s], r_ref)


def test_sequential_streams_match_reference_golden():
    for n, seed, trial, count, ref in sequential_cases():
        words = seeding.entropy_words(seed, seeding.TAG_TRIAL)
        out = torch.empty((1, count, n), dtype=torch.int32, device="cuda")
        _lib.check(_lib.load().rm_perm_sequential(words.ctypes.data, len(words), trial, 1, count,
                                                  n, out.data_ptr(), _lib.stream_ptr()))
        assert np.array_equal(out[0].cpu().numpy(), ref), (n, seed, trial)


def test_device_stream_object_continues_like_a_numpy_generator():
    # mixing.sample_permutation(n, stream(...)) called repeatedly == one
    # Generator drawing repeatedly (buffered 32-bit half carried across calls)
    for n, seed, trial, count, ref in sequential_cases():
        rng = seeding.stream(seed, seeding.TAG_TRIAL, trial)
        got = np.stack([mixing.sample_permutation(n, rng) for _ in range(count)])
        assert np.array_equal(got, ref)


def test_trial_permutations_batch_matches_oracle():
    perms = spectral.trial_permutations(12, 6, 50, seed=2).cpu().numpy()
    for t in (0, 1, 17, 49):
        assert np.array_equal(perms[t], O.c_permutation_sequential(12, 2, t, 6))


@pytest.mark.parametrize("entropy", [(0,), (5, 1, 0), (2**64 - 1, 1, 2**40 + 5), (3**45, 4, 7)])
def test_raw_pcg64_core_matches_numpy(entropy):
    words = seeding.entropy_words(*entropy)
    out = torch.empty(100, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().rm_pcg64_raw(words.ctypes.data, len(words), 100, out.data_ptr(),
                                        _lib.stream_ptr()))
    ref = np.random.PCG64(np.random.SeedSequence(entropy)).random_raw(100)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref)


def test_reference_purity_properties():
    # reference test_mixing.py:62-75
    a = mixing.permutation_for_step(8, 123, 4)
    b = mixing.permutation_for_step(8, 123, 4)
    assert np.array_equal(a, b)
    assert len({tuple(mixing.permutation_for_step(8, 123, k)) for k in range(10)}) > 1
    p = mixing.sample_permutation(10, seeding.stream(5, 1, 0))
    assert np.array_equal(np.sort(p), np.arange(10))
    assert np.array_equal(p, mixing.sample_permutation(10, seeding.stream(5, 1, 0)))
    assert np.array_equal(mixing.permutation_for_step(1, 3, 3), [0])


def test_uniformity_l4():
    # SPEC.md sample_permutation example: 24 perms at 1/24 +- 0.005 over many draws
    tabs = mixing.permutation_tables(4, 99, 0, 100_000)
    p = tabs.perm.cpu().numpy()
    codes = p[:, 0] * 64 + p[:, 1] * 16 + p[:, 2] * 4 + p[:, 3]
    _, counts = np.unique(codes, return_counts=True)
    assert len(counts) == 24
    assert np.all(np.abs(counts / 100_000 - 1 / 24) < 0.005)


def test_invalid_arguments_raise_value_error():
    with pytest.raises(ValueError):
        mixing.permutation_for_step(0, 1, 1)
    with pytest.raises(ValueError):
        mixing.permutation_for_step(4, -1, 1)
    with pytest.raises(TypeError):
        mixing.sample_permutation(4, np.random.default_rng(0))


def test_stream_is_generator_compatible():
    """seeding.stream(...) behaves like the reference's numpy Generator (seeding.py:35-37):
    device permutations and device standard normals, then any other Generator method
    (lognormal of the simulated clock, simulation.py:112; integers; normal) continues at
    the same position on the host — the same numbers as numpy throughout."""
    from paper_2002_01119_b200 import seeding
    ent = (12345, seeding.TAG_CLOCK, 7)
    ref = np.random.default_rng(np.random.SeedSequence(ent))
    s = seeding.stream(*ent)
    assert np.array_equal(s.permutation(16), ref.permutation(16))
    assert np.array_equal(s.permutation(9), ref.permutation(9))      # buffered half carried
    assert np.array_equal(s.lognormal(0.1, 0.5, 16), ref.lognormal(0.1, 0.5, 16))
    assert np.array_equal(s.permutation(5), ref.permutation(5))      # now on the host
    assert np.array_equal(s.integers(0, 100, 7), ref.integers(0, 100, 7))
    # a fresh stream's large standard_normal runs on the device; later draws continue
    ent2 = (3, seeding.TAG_GRADIENT, 11, 2)
    ref2 = np.random.default_rng(np.random.SeedSequence(ent2))
    s2 = seeding.stream(*ent2)
    n = seeding.DeviceStream.DEVICE_NORMAL_MIN + 17
    assert np.array_equal(s2.standard_normal(n), ref2.standard_normal(n))
    assert np.array_equal(s2.standard_normal((3, 4)), ref2.standard_normal((3, 4)))
    assert np.array_equal(s2.permutation(33), ref2.permutation(33))
    assert s2.bit_generator.state == ref2.bit_generator.state

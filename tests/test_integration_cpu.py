"""Host-only pieces of the reference-side binding (integration/ringmix_b200.py): ring
structure detection and the SeedSequence entropy words.  Loading the library needs no GPU."""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT / "integration"))
import ringmix_b200 as B  # noqa: E402

from paper_2002_01119_b200 import mixing, seeding  # noqa: E402


def test_ring_tables_detect_conjugated_rings():
    L = 10
    p = np.random.default_rng(3).permutation(L)
    T = mixing.conjugate_by_permutation(mixing.build_ring_matrix(L), p)
    left, right = B._ring_tables(T)
    inv = np.argsort(p)
    assert np.array_equal(np.sort(np.stack([left, right]), axis=0),
                          np.sort(np.stack([inv[(p - 1) % L], inv[(p + 1) % L]]), axis=0))
    assert B._ring_tables(mixing.build_uniform_matrix(L)) is None
    assert B._ring_tables(np.eye(L)) is None


@pytest.mark.parametrize("ints", [(0,), (12345, 1), (2**40 + 7, 1, 3), (3**45, 1, 2**33)])
def test_entropy_words_match_the_package(ints):
    assert np.array_equal(B._entropy_words(*ints), seeding.entropy_words(*ints))


def test_negative_seed_rejected():
    with pytest.raises(ValueError):
        B._entropy_words(-1, 1)

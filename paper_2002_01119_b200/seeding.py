"""Counter-based random streams, device-backed (mirror of reference seeding.py).

Reference: pkg/src/ringmix/seeding.py:1-37.  Every stream is a pure function of
an entropy tuple (seed, TAG, idx...).  The reference returns a numpy
``Generator``; here ``stream`` returns a :class:`DeviceStream` whose
permutation draws run on the GPU through ``rm_pcg_seed`` /
``rm_pcg_permutations`` and are bit-identical to numpy 2.3.5's
``default_rng(SeedSequence(entropy)).permutation`` — including the buffered
32-bit half that carries between successive draws (spectral.py:273-277).

``seed_sequence`` stays a host ``np.random.SeedSequence`` (seed bookkeeping,
e.g. harness.cell_seed, harness.py:61-64); it is not on the hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

TAG_GRADIENT = 0
TAG_PERMUTATION = 1
TAG_CLOCK = 2
TAG_INIT = 3
TAG_TRIAL = 4
TAG_CELL = 5
TAG_DATA = 6

_MASK32 = 0xFFFFFFFF


def _check(entropy) -> None:
    for part in entropy:
        if int(part) < 0:
            raise ValueError(f"entropy components must be >= 0, got {part}")


def entropy_words(*entropy: int) -> np.ndarray:
    """numpy's _coerce_to_uint32_array for a tuple of non-negative ints."""
    _check(entropy)
    words: list[int] = []
    for v in entropy:
        v = int(v)
        if v == 0:
            words.append(0)
        while v:
            words.append(v & _MASK32)
            v >>= 32
    return np.ascontiguousarray(np.array(words, dtype=np.uint32))


def seed_sequence(*entropy: int) -> np.random.SeedSequence:
    """SeedSequence for an entropy tuple of non-negative integers (seeding.py:27-32)."""
    _check(entropy)
    return np.random.SeedSequence(entropy)


def cell_seed(master_seed: int, strategy_id: int, n_learners: int, trial: int) -> int:
    """Per-cell run seed (reference harness.py:61-64), a 64-bit value."""
    ss = seed_sequence(master_seed, TAG_CELL, strategy_id, n_learners, trial)
    return int(ss.generate_state(1, np.uint64)[0])


class DeviceStream:
    """A PCG64 stream seeded from SeedSequence(entropy), living on the GPU.

    Only the draws on the learner-averaging path are provided: permutations.
    """

    def __init__(self, *entropy: int, device: torch.device | str | None = None):
        _lib.require_cuda()
        self.entropy = tuple(int(e) for e in entropy)
        self.device = torch.device(device if device is not None else "cuda")
        words = entropy_words(*self.entropy)
        self._state = torch.empty(6, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().rm_pcg_seed(words.ctypes.data, len(words), 0, 0, 1,
                                               self._state.data_ptr(), _lib.stream_ptr()),
                       "rm_pcg_seed")

    def permutations(self, n: int, count: int) -> torch.Tensor:
        """`count` successive permutations of range(n), int32 CUDA tensor (count, n)."""
        if n < 1:
            raise ValueError(f"need n >= 1, got {n}")
        out = torch.empty((count, n), dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().rm_pcg_permutations(self._state.data_ptr(), 1, count, n,
                                                       out.data_ptr(), _lib.stream_ptr()),
                       "rm_pcg_permutations")
        return out

    def permutation(self, n: int) -> np.ndarray:
        """Generator.permutation(n) for an int n: int64 numpy array (reference dtype)."""
        return self.permutations(n, 1)[0].to(torch.int64).cpu().numpy()

    def __repr__(self) -> str:
        return f"DeviceStream(entropy={self.entropy}, device={self.device})"


def stream(*entropy: int) -> DeviceStream:
    """Fresh device stream for an entropy tuple.  Pure: same tuple, same draws."""
    _check(entropy)
    return DeviceStream(*entropy)

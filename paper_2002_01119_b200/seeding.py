"""Counter-based random streams, device-backed (mirror of reference seeding.py).

Reference: pkg/src/ringmix/seeding.py:1-37.  Every stream is a pure function of
an entropy tuple (seed, TAG, idx...).  The reference returns a numpy
``Generator``; here ``stream`` returns a Generator-compatible :class:`DeviceStream`
whose permutation and standard-normal draws run on the GPU (``rm_pcg_seed`` /
``rm_pcg_permutations`` / ``rm_standard_normal_f64``) and are bit-identical to numpy
2.3.5's ``default_rng(SeedSequence(entropy))`` — including the buffered 32-bit half
that carries between successive permutation draws (spectral.py:273-277); every other
Generator method continues on a host Generator at the same position.

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
    """A numpy-``Generator``-compatible PCG64 stream seeded from SeedSequence(entropy), whose
    draws on the learner-averaging path run on the GPU, bit-identical to numpy 2.3.5:

    * ``permutation(n)`` / ``permutations(n, count)`` — the state lives on the device
      (6 x u64, rm_pcg_seed / rm_pcg_permutations) and carries the buffered 32-bit half
      from draw to draw, like repeated ``Generator.permutation`` calls;
    * ``standard_normal(size)`` on a fresh stream — the device ziggurat
      (rm_standard_normal_f64; the gradient noise and initial weights of
      simulation.py:207, objectives.py:90).

    Every other ``Generator`` method (``lognormal`` for the simulated clock,
    simulation.py:112; ``integers``; ``normal``; ...) and any draw after a device normal
    continues on a host ``numpy.random.Generator`` positioned exactly where this stream
    is (the device state is copied over, or the device normal replayed), which then stays
    authoritative.  So code written against the reference's ``seeding.stream`` works
    unchanged and draws the same numbers."""

    # below this many normals the host generator is faster than a device launch
    DEVICE_NORMAL_MIN = 1 << 15

    def __init__(self, *entropy: int, device: torch.device | str | None = None):
        _lib.require_cuda()
        self.entropy = tuple(int(e) for e in entropy)
        self.device = torch.device(device if device is not None else "cuda")
        self._fresh = True
        self._host: np.random.Generator | None = None
        self._replay: list[tuple] = []      # device normals not reflected in a state
        words = entropy_words(*self.entropy)
        self._state = torch.empty(6, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().rm_pcg_seed(words.ctypes.data, len(words), 0, 0, 1,
                                               self._state.data_ptr(), _lib.stream_ptr()),
                       "rm_pcg_seed")

    # -- host hand-off ------------------------------------------------------------------
    def _to_host(self) -> np.random.Generator:
        """The host Generator positioned where this stream is (created once)."""
        if self._host is None:
            g = np.random.Generator(np.random.PCG64(np.random.SeedSequence(self.entropy)))
            if self._replay:
                for name, args in self._replay:
                    getattr(g, name)(*args)
            elif not self._fresh:
                st = self._state.cpu().numpy().view(np.uint64).tolist()
                g.bit_generator.state = {
                    "bit_generator": "PCG64",
                    "state": {"state": (int(st[0]) << 64) | int(st[1]),
                              "inc": (int(st[2]) << 64) | int(st[3])},
                    "has_uint32": int(st[4] != 0), "uinteger": int(st[5])}
            self._host = g
        return self._host

    @property
    def bit_generator(self):
        return self._to_host().bit_generator

    def __getattr__(self, name):
        # Generator methods without a device path run on the positioned host generator
        if name.startswith("_"):
            raise AttributeError(name)
        attr = getattr(np.random.Generator, name, None)
        if attr is None:
            raise AttributeError(name)
        self._fresh = False
        return getattr(self._to_host(), name)

    # -- device draws -------------------------------------------------------------------
    def permutations(self, n: int, count: int) -> torch.Tensor:
        """`count` successive permutations of range(n), int32 CUDA tensor (count, n)."""
        if n < 1:
            raise ValueError(f"need n >= 1, got {n}")
        if self._host is not None or self._replay:
            g = self._to_host()
            return torch.from_numpy(np.stack([g.permutation(n) for _ in range(count)])
                                    .astype(np.int32)).to(self.device)
        out = torch.empty((count, n), dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().rm_pcg_permutations(self._state.data_ptr(), 1, count, n,
                                                       out.data_ptr(), _lib.stream_ptr()),
                       "rm_pcg_permutations")
        self._fresh = False
        return out

    def permutation(self, x):
        """Generator.permutation: an int n draws on the device (int64 numpy array, the
        reference's dtype); an array argument shuffles a copy on the host generator."""
        if isinstance(x, (int, np.integer)):
            return self.permutations(int(x), 1)[0].to(torch.int64).cpu().numpy()
        self._fresh = False
        return self._to_host().permutation(x)

    def standard_normal(self, size=None, dtype=np.float64, out=None):
        """Generator.standard_normal; a fresh stream's float64 draw of at least
        DEVICE_NORMAL_MIN values runs on the device."""
        n = int(np.prod(size)) if size is not None else 1
        if (self._fresh and self._host is None and out is None and size is not None and
                np.dtype(dtype) == np.float64 and n >= self.DEVICE_NORMAL_MIN):
            from .objectives import standard_normal as device_normal
            z = device_normal(n, *self.entropy, device=self.device).cpu().numpy()
            self._fresh = False
            self._replay.append(("standard_normal", (size,)))
            return z.reshape(size)
        self._fresh = False
        return self._to_host().standard_normal(size, dtype=dtype, out=out)

    def __repr__(self) -> str:
        return f"DeviceStream(entropy={self.entropy}, device={self.device})"


def stream(*entropy: int) -> DeviceStream:
    """Fresh stream for an entropy tuple (seeding.py:35-37): a Generator-compatible
    DeviceStream.  Pure: same tuple, same draws."""
    _check(entropy)
    return DeviceStream(*entropy)

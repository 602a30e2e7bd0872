"""ORACLE — test infrastructure only.

CPU restatement of the reference's learner-averaging path, used as the
checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs.  The product package (paper_2002_01119_b200) never
imports this module; its CUDA path fails loudly when its library is missing.

What is restated, and where it comes from (paths under /root/reference):

* permutation_for_step / sample_permutation / seeding.stream
  (pkg/src/ringmix/mixing.py:72-86, seeding.py:27-37): numpy 2.3.5's
  SeedSequence -> PCG64 -> Generator.permutation chain, restated twice:
  in plain C (oracle/perm_oracle.c, fast) and in pure Python below
  (`py_permutation`, small cases only).
* neighbour tables of the conjugated ring T = ring[p, p]
  (simulation.py:299-300, mixing.py:89-103): left[j] = inv[(p[j]-1) % L],
  right[j] = inv[(p[j]+1) % L].
* the step arithmetic (simulation.py:263-268 `apply_mixing(W, T) - lr*G`,
  mixing.py:106-125): `numpy_*` functions perform the reference's own numpy
  operations on the reference's (d, L) fp64 layout; `c_*` functions are the
  scalar C restatement in oracle/mix_oracle.c with an explicit rounding
  sequence (FMA chain in ascending learner index for rings, numpy pairwise
  summation for the uniform mean).

Parity of this oracle is pinned against tests/golden/*.npz, which
tests/golden/make_golden.py produced by importing the reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
BUILD_DIR = ORACLE_DIR / "_build"
LIB_PATH = BUILD_DIR / "liboracle.so"

MASK32 = 0xFFFFFFFF
TAG_GRADIENT = 0
TAG_PERMUTATION = 1
TAG_TRIAL = 4


# --------------------------------------------------------------------------
# build / load the C restatement
# --------------------------------------------------------------------------

def build(force: bool = False) -> Path:
    """Compile oracle/*.c into oracle/_build/liboracle.so with gcc."""
    srcs = [ORACLE_DIR / "perm_oracle.c", ORACLE_DIR / "mix_oracle.c",
            ORACLE_DIR / "normal_oracle.c"]
    if not force and LIB_PATH.exists():
        mtime = LIB_PATH.stat().st_mtime
        if all(s.stat().st_mtime <= mtime for s in srcs):
            return LIB_PATH
    BUILD_DIR.mkdir(exist_ok=True)
    tmp = LIB_PATH.with_suffix(f".so.tmp{os.getpid()}")
    cmd = ["gcc", "-O2", "-mfma", "-ffp-contract=off", "-shared", "-fPIC",
           "-o", str(tmp), *map(str, srcs), "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64, u64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        L.or_permutation.argtypes = [vp, i32, u64, i64, vp]
        L.or_permutation_sequential.argtypes = [vp, i32, u64, i64, i32, vp]
        L.or_raw64.argtypes = [vp, i32, i32, vp]
        L.or_ring_mix_sgd.argtypes = [vp, vp, vp, vp, vp, i64, i64, ctypes.c_double]
        L.or_ring_mix_sgd.restype = None
        L.or_mean_sgd.argtypes = [vp, vp, vp, i64, i64, ctypes.c_double]
        L.or_mean_sgd.restype = None
        L.or_pairwise_sum.argtypes = [vp, i64]
        L.or_pairwise_sum.restype = ctypes.c_double
        L.or_standard_normal.argtypes = [vp, i32, i64, vp, vp, vp, vp]
        L.or_standard_normal.restype = i64
        _lib = L
    return _lib


# --------------------------------------------------------------------------
# entropy words (numpy _coerce_to_uint32_array)
# --------------------------------------------------------------------------

def int_limbs(v: int) -> list[int]:
    if v < 0:
        raise ValueError(f"entropy components must be >= 0, got {v}")
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & MASK32)
        v >>= 32
    return out


def entropy_words(*ints: int) -> list[int]:
    words: list[int] = []
    for v in ints:
        words += int_limbs(int(v))
    return words


def _u32(words) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(words, dtype=np.uint32))


# --------------------------------------------------------------------------
# permutations
# --------------------------------------------------------------------------

def c_permutation(n: int, seed: int, step: int, tag: int = TAG_PERMUTATION) -> np.ndarray:
    prefix = _u32(entropy_words(seed, tag))
    out = np.empty(max(n, 1), dtype=np.int64)
    rc = lib().or_permutation(prefix.ctypes.data, len(prefix), step, n, out.ctypes.data)
    assert rc == 0
    return out[:n]


def c_permutation_sequential(n: int, seed: int, idx: int, count: int,
                             tag: int = TAG_TRIAL) -> np.ndarray:
    prefix = _u32(entropy_words(seed, tag))
    out = np.empty((count, max(n, 1)), dtype=np.int64)
    rc = lib().or_permutation_sequential(prefix.ctypes.data, len(prefix), idx, n, count,
                                         out.ctypes.data)
    assert rc == 0
    return out[:, :n]


def c_raw64(words, count: int) -> np.ndarray:
    w = _u32(words)
    out = np.empty(count, dtype=np.uint64)
    lib().or_raw64(w.ctypes.data, len(w), count, out.ctypes.data)
    return out


# Pure-Python restatement (small cases; cross-checks the C one).
_M32 = 0xFFFFFFFF
_PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341
_M128 = (1 << 128) - 1
_M64 = (1 << 64) - 1


def py_seedseq_state(words) -> list[int]:
    hc = 0x43B0D7E5

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & _M32
        hc = (hc * 0x931E8875) & _M32
        v = (v * hc) & _M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (0xCA01F9DD * x - 0x4973F715 * y) & _M32
        return r ^ (r >> 16)

    pool = [hashmix(words[i] if i < len(words) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(words)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(words[s]))
    hb = 0x8B51F9DD
    w = []
    for i in range(8):
        v = pool[i % 4] ^ hb
        hb = (hb * 0x58F38DED) & _M32
        v = (v * hb) & _M32
        w.append(v ^ (v >> 16))
    return [w[2 * i] | (w[2 * i + 1] << 32) for i in range(4)]


class PyPCG64:
    def __init__(self, words):
        v = py_seedseq_state(words)
        self.inc = ((((v[2] << 64) | v[3]) << 1) | 1) & _M128
        self.state = 0
        self._step()
        self.state = (self.state + ((v[0] << 64) | v[1])) & _M128
        self._step()
        self.buf = None

    def _step(self):
        self.state = (self.state * _PCG_MULT + self.inc) & _M128

    def next64(self) -> int:
        self._step()
        x = ((self.state >> 64) ^ self.state) & _M64
        r = self.state >> 122
        return ((x >> r) | (x << ((64 - r) & 63))) & _M64

    def next32(self) -> int:
        if self.buf is not None:
            b, self.buf = self.buf, None
            return b
        n = self.next64()
        self.buf = n >> 32
        return n & _M32

    def interval(self, mx: int) -> int:
        if mx == 0:
            return 0
        mask = (1 << mx.bit_length()) - 1
        draw = self.next32 if mx <= _M32 else self.next64
        while True:
            v = draw() & mask
            if v <= mx:
                return v

    def permutation(self, n: int) -> np.ndarray:
        a = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            a[i], a[j] = a[j], a[i]
        return np.array(a, dtype=np.int64)


def py_permutation(n: int, seed: int, step: int, tag: int = TAG_PERMUTATION) -> np.ndarray:
    return PyPCG64(entropy_words(seed, tag, step)).permutation(n)


def neighbour_tables(perm) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """inv, left, right of the conjugated ring ring[p, p] (finding 4)."""
    p = np.asarray(perm, dtype=np.int64)
    L = len(p)
    inv = np.empty(L, dtype=np.int64)
    inv[p] = np.arange(L)
    left = inv[(p - 1) % L]
    right = inv[(p + 1) % L]
    return inv, left, right


# --------------------------------------------------------------------------
# normals (quadratic-oracle gradient noise)
# --------------------------------------------------------------------------

ZIG_HEADER = ORACLE_DIR.parent / "paper_2002_01119_b200" / "csrc" / "ziggurat_tables.h"
_zig = None


def ziggurat_tables():
    """numpy's ki (uint64) / wi / fi (float64) tables, as generated from the
    installed libnpyrandom.a into csrc/ziggurat_tables.h."""
    global _zig
    if _zig is None:
        import re
        v = [int(x, 16) for x in re.findall(r"0x([0-9a-f]{16})ull", ZIG_HEADER.read_text())]
        ki = np.array(v[:256], dtype=np.uint64)
        wi = np.array(v[256:512], dtype=np.uint64).view(np.float64)
        fi = np.array(v[512:768], dtype=np.uint64).view(np.float64)
        _zig = (ki, wi, fi)
    return _zig


def c_standard_normal(n: int, *entropy: int) -> tuple[np.ndarray, int]:
    """stream(*entropy).standard_normal(n) restated in C; returns (values, raw draws)."""
    ki, wi, fi = ziggurat_tables()
    w = _u32(entropy_words(*entropy))
    out = np.empty(max(n, 1), dtype=np.float64)
    draws = lib().or_standard_normal(w.ctypes.data, len(w), n, ki.ctypes.data, wi.ctypes.data,
                                     fi.ctypes.data, out.ctypes.data)
    return out[:n], int(draws)


# --------------------------------------------------------------------------
# step arithmetic
# --------------------------------------------------------------------------

def ring_matrix(L: int) -> np.ndarray:
    """mixing.py:43-62 (1/3 on the diagonal and both ring neighbours)."""
    if L < 3:
        raise ValueError(f"degenerate ring topology: need at least 3 learners, got {L}")
    T = np.zeros((L, L))
    i = np.arange(L)
    T[i, i] = 1.0 / 3.0
    T[i, (i + 1) % L] = 1.0 / 3.0
    T[i, (i - 1) % L] = 1.0 / 3.0
    return T


def numpy_apply_mixing(W_dL: np.ndarray, T: np.ndarray) -> np.ndarray:
    """mixing.py:106-125, the reference's own numpy operations."""
    L = T.shape[0]
    if np.all(T == 1.0 / L):
        return np.tile(W_dL.mean(axis=1, keepdims=True), (1, L))
    return W_dL @ T


def numpy_gossip_step(W_dL, G_dL, lr: float, perm=None, uniform: bool = False):
    """simulation.py:263-268: apply_mixing(W, T) - lr * G, (d, L) fp64."""
    L = W_dL.shape[1]
    if uniform:
        T = np.full((L, L), 1.0 / L)
    else:
        T = ring_matrix(L)
        if perm is not None:
            p = np.asarray(perm)
            T = T[np.ix_(p, p)]
    mixed = numpy_apply_mixing(W_dL, T)
    if G_dL is None:
        return mixed
    return mixed - lr * G_dL


def numpy_spsgd(W_dL, G_dL, lr: float):
    """simulation.py:251-260."""
    L = W_dL.shape[1]
    if np.any(W_dL != W_dL[:, :1]):
        raise ValueError("SPSGD requires identical weights on all learners")
    return W_dL - lr * np.tile(G_dL.mean(axis=1, keepdims=True), (1, L))


def c_ring_mix_sgd(W_dL, G_dL, lr: float, left, right) -> np.ndarray:
    W = np.ascontiguousarray(W_dL, dtype=np.float64)
    d, L = W.shape
    out = np.empty_like(W)
    G = None if G_dL is None else np.ascontiguousarray(G_dL, dtype=np.float64)
    lf = np.ascontiguousarray(left, dtype=np.int32)
    rt = np.ascontiguousarray(right, dtype=np.int32)
    lib().or_ring_mix_sgd(W.ctypes.data, None if G is None else G.ctypes.data, out.ctypes.data,
                          lf.ctypes.data, rt.ctypes.data, d, L, float(lr))
    return out


def c_mean_sgd(W_dL, G_dL, lr: float) -> np.ndarray:
    W = np.ascontiguousarray(W_dL, dtype=np.float64)
    d, L = W.shape
    out = np.empty_like(W)
    G = None if G_dL is None else np.ascontiguousarray(G_dL, dtype=np.float64)
    lib().or_mean_sgd(W.ctypes.data, None if G is None else G.ctypes.data, out.ctypes.data,
                      d, L, float(lr))
    return out


def magnitude_tolerance_ok(y, y_ref, W_dL, G_dL, lr, left=None, right=None, rel=1e-6):
    """SURVEY §8(c) tolerance: |y - y_ref| <= rel * ((|w_l|+|w_j|+|w_r|)/3 + |lr g|)
    element-wise (mean |w| for the uniform path) and norm-wise rel error <= rel."""
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    A = np.abs(W_dL)
    if left is None:
        scale = np.tile(A.mean(axis=1, keepdims=True), (1, W_dL.shape[1]))
    else:
        j = np.arange(W_dL.shape[1])
        scale = (A[:, left] + A[:, j] + A[:, right]) / 3.0
    if G_dL is not None:
        scale = scale + np.abs(lr * G_dL)
    elem_ok = bool(np.all(np.abs(y - y_ref) <= rel * scale + 1e-300))
    norm_ok = bool(np.linalg.norm(y - y_ref) <= rel * max(np.linalg.norm(y_ref), 1e-300))
    return elem_ok and norm_ok

"""libringmix_b200 binding for the reference package `ringmix`.

This is the module a maintainer adds to the reference (`ringmix/_b200.py`): plain ctypes +
numpy, no torch.  `install(ringmix)` routes the reference's learner-averaging path through
the B200 kernels while every other line of the reference stays as it is:

  ringmix.mixing.permutation_for_step   (mixing.py:79-86)     -> rm_perm_tables
  ringmix.mixing.apply_mixing           (mixing.py:106-125)   -> rm_gossip_step_host_dL_f64
      for ring / ring[p, p] / uniform T (anything else keeps numpy's W @ T)
  ringmix.simulation._gossip_step       (simulation.py:263-268)
      W' = apply_mixing(W, T) - lr * G fused into one rm_gossip_step_host_dL_f64 call

The reference's (d, L) float64 C-order arrays are passed as they are (the (d, L) kernels
need no transpose).  Same arithmetic as the reference: permutations are
bit-exact; the mix is OpenBLAS's FMA chain, bit-exact except where OpenBLAS's small-matrix
remainder kernels round differently (an implementation-defined choice of the BLAS).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB = Path(os.environ.get("RINGMIX_B200_LIB",
                          _HERE.parent / "paper_2002_01119_b200" / "lib" / "libringmix_b200.so"))

_vp, _i32, _i64, _u64, _f64 = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                               ctypes.c_double)
_lib = ctypes.CDLL(str(LIB))
_lib.rm_last_error.restype = ctypes.c_char_p
_lib.rm_device_alloc.argtypes = [_i64, ctypes.POINTER(ctypes.c_void_p)]
_lib.rm_device_free.argtypes = [_vp]
_lib.rm_memcpy.argtypes = [_vp, _vp, _i64, _vp]
_lib.rm_stream_synchronize.argtypes = [_vp]
_lib.rm_perm_tables.argtypes = [_vp, _i32, _u64, _i32, _i32, _vp, _vp, _vp, _vp, _vp]
_lib.rm_gossip_step_host_dL_f64.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _i64, _f64, _vp, _i64,
                                            _vp, _vp]

CALLS = {"permutation_for_step": 0, "apply_mixing": 0, "gossip_step": 0, "numpy_fallback": 0}


def _check(rc):
    if rc != 0:   # negative: bad argument (the reference's ValueError text); positive: CUDA
        raise (ValueError if rc < 0 else RuntimeError)(_lib.rm_last_error().decode())


class _DeviceBuffer:
    def __init__(self, nbytes):
        self.nbytes = nbytes
        self.ptr = ctypes.c_void_p()
        _check(_lib.rm_device_alloc(nbytes, ctypes.byref(self.ptr)))

    def __del__(self):
        try:
            _lib.rm_device_free(self.ptr)
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass


_buffers: dict = {}


def _buffer(key, nbytes) -> _DeviceBuffer:
    b = _buffers.get(key)
    if b is None or b.nbytes < nbytes:
        b = _buffers[key] = _DeviceBuffer(nbytes)
    return b


def _entropy_words(*ints) -> np.ndarray:
    """numpy's _coerce_to_uint32_array of the SeedSequence entropy tuple."""
    out = []
    for v in ints:
        v = int(v)
        if v < 0:
            raise ValueError("seeds must be non-negative")
        if v == 0:
            out.append(0)
        while v:
            out.append(v & 0xFFFFFFFF)
            v >>= 32
    return np.array(out, dtype=np.uint32)


def permutation_for_step(n: int, shared_seed: int, step: int) -> np.ndarray:
    """The reference's permutation for iteration `step`, drawn on the GPU (bit-exact)."""
    CALLS["permutation_for_step"] += 1
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    words = _entropy_words(shared_seed, 1)          # TAG_PERMUTATION (seeding.py:19)
    buf = _buffer("perm", 4 * 4 * n)
    base = buf.ptr.value
    _check(_lib.rm_perm_tables(words.ctypes.data, len(words), int(step), 1, n, base,
                               base + 4 * n, base + 8 * n, base + 12 * n, None))
    perm = np.empty(n, dtype=np.int32)
    _check(_lib.rm_memcpy(perm.ctypes.data, base, 4 * n, None))
    _check(_lib.rm_stream_synchronize(None))
    return perm.astype(np.int64)


def _ring_tables(T: np.ndarray):
    """(left, right) int32 tables if T is a ring / ring[p, p] matrix (every column: three
    entries fl(1/3), one on the diagonal, zeros elsewhere), else None."""
    L = T.shape[0]
    if L < 3:
        return None
    nz = T != 0.0
    if not np.all(nz.sum(axis=0) == 3) or not np.all(T[nz] == 1.0 / 3.0) or \
            not np.all(np.diag(T) == 1.0 / 3.0):
        return None
    rows = np.nonzero(nz.T)[1].reshape(L, 3)
    j = np.arange(L)
    others = rows[rows != j[:, None]].reshape(L, 2)
    return (np.ascontiguousarray(others[:, 0], dtype=np.int32),
            np.ascontiguousarray(others[:, 1], dtype=np.int32))


def gossip_step(W, T, lr: float, G) -> np.ndarray | None:
    """apply_mixing(W, T) - lr * G on the GPU for ring / uniform T (G may be None);
    None when T has another structure (the caller keeps the numpy path)."""
    T = np.asarray(T, dtype=np.float64)
    W = np.asarray(W)
    if W.ndim != 2 or T.ndim != 2 or T.shape[0] != T.shape[1] or W.shape[1] != T.shape[0]:
        return None
    d, L = W.shape
    if L > 512:
        return None
    if np.all(T == 1.0 / L):
        tabs = None
    else:
        tabs = _ring_tables(T)
        if tabs is None:
            return None
    W = np.ascontiguousarray(W, dtype=np.float64)
    if G is not None:
        G = np.ascontiguousarray(G, dtype=np.float64)
    out = np.empty((d, L), dtype=np.float64)
    if d == 0:
        return out
    rows = max(1, min(d, (64 << 20) // (9 * 8 * L)))
    ws = _buffer(("ws", L), 4096 + 9 * 8 * L * rows)
    _check(_lib.rm_gossip_step_host_dL_f64(
        W.ctypes.data, None if G is None else G.ctypes.data, out.ctypes.data,
        None if tabs is None else tabs[0].ctypes.data, None if tabs is None else tabs[1].ctypes.data,
        L, d, float(lr), ws.ptr, ws.nbytes, None, None))
    _check(_lib.rm_stream_synchronize(None))
    return out


def install(ringmix) -> None:
    """Route the reference's averaging path through libringmix_b200 (see module doc)."""
    mixing, simulation = ringmix.mixing, ringmix.simulation
    numpy_apply = mixing.apply_mixing

    def apply_mixing(W, T):
        # the reference's shape checks and errors first (mixing.py:115-120)
        Wa, Ta = np.asarray(W), np.asarray(T)
        if Wa.ndim != 2 or Ta.ndim != 2 or Ta.shape[0] != Ta.shape[1] or \
                Wa.shape[1] != Ta.shape[0]:
            return numpy_apply(W, T)
        out = gossip_step(Wa, Ta, 0.0, None)
        if out is None:
            CALLS["numpy_fallback"] += 1
            return numpy_apply(W, T)
        CALLS["apply_mixing"] += 1
        return out

    def _gossip_step(state, oracle, cfg, T, stale):
        # simulation.py:263-268 with the mix and the update fused into one GPU pass
        k = state.iteration
        Phi = state.prev_weights if stale else state.weights
        G = simulation.gradient_matrix(oracle, Phi, cfg, k)
        W_next = gossip_step(state.weights, T, simulation.learning_rate(cfg, k), G)
        if W_next is None:
            CALLS["numpy_fallback"] += 1
            W_next = numpy_apply(state.weights, T) - simulation.learning_rate(cfg, k) * G
        else:
            CALLS["gossip_step"] += 1
        return simulation._advance(state, W_next, G)

    for mod in (mixing, simulation):
        mod.apply_mixing = apply_mixing
        mod.permutation_for_step = permutation_for_step
    simulation._gossip_step = _gossip_step

"""Mixing matrices, permutations and the fused mix kernels (mirror of mixing.py).

Reference: pkg/src/ringmix/mixing.py:1-141.

L x L objects (ring/uniform matrices, conjugation, the stochasticity check)
are host fp64 numpy exactly as in the reference: they are tiny and off the
hot path.  Everything proportional to d runs on the GPU:

* permutations: ``permutation_for_step`` / ``sample_permutation`` /
  ``permutation_tables`` draw on the device (bit-exact with numpy 2.3.5),
* ``apply_mixing(W, T)``: ring and conjugated-ring matrices run the fused
  gather-mix kernel, uniform matrices the pairwise-mean kernel; any other
  dense T is a plain cuBLAS GEMM through torch (library GEMM, not the path),
* learner-major primitives ``ring_mix_sgd`` / ``mean_mix_sgd`` /
  ``spsgd_update`` used by simulation.step_* (simulation.py:251-312).

Learner-major layout: a CUDA tensor X of shape (L, d), row stride ld >= d,
unit column stride.  The reference's (d, L) weights matrix is ``X.T``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, seeding
from .seeding import DeviceStream

_DT_SUFFIX = {torch.float32: "f32", torch.float64: "f64", torch.bfloat16: "bf16"}


@dataclass(frozen=True)
class StochasticityReport:
    """Result of `verify_doubly_stochastic`.  Reports, never raises (mixing.py:32-40)."""

    max_row_error: float
    max_col_error: float
    min_entry: float
    tol: float
    ok: bool


def build_ring_matrix(n_learners: int) -> np.ndarray:
    """1/3-weighted ring (mixing.py:43-62); L < 3 is degenerate and rejected."""
    if n_learners < 3:
        raise ValueError(
            f"degenerate ring topology: need at least 3 learners, got {n_learners}")
    L = n_learners
    T = np.zeros((L, L))
    i = np.arange(L)
    for nb in (i, (i + 1) % L, (i - 1) % L):
        T[i, nb] = 1.0 / 3.0
    return T


def build_uniform_matrix(n_learners: int) -> np.ndarray:
    """All entries 1/L (mixing.py:65-69)."""
    if n_learners < 1:
        raise ValueError(f"need at least 1 learner, got {n_learners}")
    return np.full((n_learners, n_learners), 1.0 / n_learners)


def sample_permutation(n: int, rng: DeviceStream) -> np.ndarray:
    """Uniform random permutation of range(n) drawn from a device stream (mixing.py:72-76)."""
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    if not isinstance(rng, DeviceStream):
        raise TypeError("rng must be a paper_2002_01119_b200.seeding.stream(...) device stream "
                        "(there is no host RNG path)")
    return rng.permutation(n)


@dataclass
class PermTables:
    """Device tables for steps [step0, step0 + nsteps): int32 CUDA tensors (nsteps, L).

    left[s, j] / right[s, j] are learner j's ring neighbours under
    T = ring[p, p] (simulation.py:299-300): inv[(p[j] -/+ 1) mod L].
    """

    step0: int
    perm: torch.Tensor
    inv: torch.Tensor
    left: torch.Tensor
    right: torch.Tensor

    def step(self, k: int) -> tuple[torch.Tensor, torch.Tensor]:
        s = k - self.step0
        return self.left[s], self.right[s]


def permutation_tables(n: int, shared_seed: int, step0: int = 0, nsteps: int = 1,
                       device=None, tag: int = seeding.TAG_PERMUTATION) -> PermTables:
    """Generate permutation_for_step(n, seed, k) for k in [step0, step0+nsteps) on the GPU,
    with inverse and neighbour tables, in one launch (one thread per step)."""
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    if step0 < 0 or step0 + nsteps - 1 >= 2**64:
        raise ValueError("steps must lie in [0, 2**64)")
    _lib.require_cuda()
    dev = torch.device(device if device is not None else "cuda")
    words = seeding.entropy_words(shared_seed, tag)
    t = [torch.empty((nsteps, n), dtype=torch.int32, device=dev) for _ in range(4)]
    with torch.cuda.device(dev):
        _lib.check(_lib.load().rm_perm_tables(words.ctypes.data, len(words), step0, nsteps, n,
                                              *(x.data_ptr() for x in t), _lib.stream_ptr()),
                   "rm_perm_tables")
    return PermTables(step0, *t)


def permutation_for_step(n: int, shared_seed: int, step: int) -> np.ndarray:
    """Permutation for iteration `step`, a pure function of (shared_seed, step) (mixing.py:79-86)."""
    tabs = permutation_tables(n, shared_seed, step, 1)
    return tabs.perm[0].to(torch.int64).cpu().numpy()


def conjugate_by_permutation(T: np.ndarray, perm) -> np.ndarray:
    """Entry (i, j) = T[perm[i], perm[j]] (mixing.py:89-103)."""
    perm = np.asarray(perm)
    n = T.shape[0]
    if T.shape != (n, n):
        raise ValueError(f"mixing matrix must be square, got {T.shape}")
    if perm.shape != (n,) or not np.array_equal(np.sort(perm), np.arange(n)):
        raise ValueError("perm is not a permutation of range(n)")
    return T[np.ix_(perm, perm)]


def verify_doubly_stochastic(T, tol: float = 1e-12) -> StochasticityReport:
    """Row/column sums and non-negativity to `tol`; never raises (mixing.py:128-141)."""
    T = np.asarray(T)
    if T.ndim != 2 or T.shape[0] != T.shape[1]:
        return StochasticityReport(np.inf, np.inf, -np.inf, tol, False)
    row_err = float(np.max(np.abs(T.sum(axis=1) - 1.0)))
    col_err = float(np.max(np.abs(T.sum(axis=0) - 1.0)))
    min_entry = float(T.min())
    ok = row_err <= tol and col_err <= tol and min_entry >= -tol
    return StochasticityReport(row_err, col_err, min_entry, tol, ok)


# ----------------------------------------------------------------------------
# learner-major device primitives (the hot path)
# ----------------------------------------------------------------------------

def _rows(X: torch.Tensor, name: str = "W") -> tuple[int, int, int]:
    """(L, d, ld) of a learner-major CUDA tensor; raises if the layout is wrong."""
    _lib.require_cuda(X)
    if X.dim() != 2:
        raise ValueError(f"{name} must be 2-D learner-major (L, d), got shape {tuple(X.shape)}")
    L, d = X.shape
    if d > 1 and X.stride(1) != 1:
        raise ValueError(f"{name} must have unit column stride (learner-major rows)")
    ld = X.stride(0) if L > 1 else max(d, 1)
    if ld < d:
        raise ValueError(f"{name} rows overlap (ld={ld} < d={d})")
    return L, d, ld


def _suffix(X: torch.Tensor) -> str:
    try:
        return _DT_SUFFIX[X.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {X.dtype}; use float32, float64 or bfloat16") from None


def _same(X: torch.Tensor, Y: torch.Tensor | None, name: str) -> None:
    if Y is None:
        return
    if Y.dtype != X.dtype or Y.device != X.device or Y.shape != X.shape:
        raise ValueError(f"{name} must match W in dtype/device/shape: "
                         f"{Y.dtype}/{Y.device}/{tuple(Y.shape)} vs {X.dtype}/{X.device}/{tuple(X.shape)}")


def empty_learner_major(L: int, d: int, dtype=torch.float32, device=None,
                        align_elems: int = 32) -> torch.Tensor:
    """Allocate an (L, d) learner-major tensor whose rows start 128-byte aligned
    (ld rounded up to `align_elems`), the layout the TMA path wants."""
    ld = ((max(d, 1) + align_elems - 1) // align_elems) * align_elems
    buf = torch.empty((L, ld), dtype=dtype, device=device if device is not None else "cuda")
    return buf[:, :d]


def _prep_out(W: torch.Tensor, out: torch.Tensor | None) -> torch.Tensor:
    if out is None:
        L, d = W.shape
        out = empty_learner_major(L, d, W.dtype, W.device)
    _same(W, out, "out")
    _rows(out, "out")
    if W.numel() and out.data_ptr() == W.data_ptr():
        raise ValueError("in-place mixing is a read-after-write hazard across learners; "
                         "use distinct buffers")
    return out


def ring_mix_sgd(W: torch.Tensor, G: torch.Tensor | None, lr: float, left: torch.Tensor,
                 right: torch.Tensor, out: torch.Tensor | None = None,
                 absmax: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """out[j] = (W[left j] + W[j] + W[right j]) / 3 - lr * G[j]   (one fused HBM pass).

    simulation._gossip_step with T = ring[p, p] (simulation.py:263-301).  L == 3
    takes the reference's exact column-mean path (mixing.py:122-124).
    `absmax` (optional int64 CUDA scalar, zeroed by the caller) receives the
    bit pattern of max|out| as a double (fused _check_divergence).
    """
    L, d, ldw = _rows(W)
    _same(W, G, "G")
    ldg = _rows(G, "G")[2] if G is not None else ldw
    out = _prep_out(W, out)
    ldo = _rows(out, "out")[2]
    if left.dtype != torch.int32 or right.dtype != torch.int32 or left.numel() != L \
            or right.numel() != L or left.device != W.device or right.device != W.device:
        raise ValueError("left/right must be int32 CUDA tensors with L entries on W's device")
    fn = getattr(_lib.load(), f"rm_ring_mix_sgd_{_suffix(W)}")
    with torch.cuda.device(W.device):
        _lib.check(fn(W.data_ptr(), _lib.ptr(G), out.data_ptr(), left.data_ptr(),
                      right.data_ptr(), L, d, ldw, ldg, ldo, float(lr), _lib.ptr(absmax),
                      _lib.stream_ptr(stream)), "rm_ring_mix_sgd")
    return out


def mean_mix_sgd(W: torch.Tensor, G: torch.Tensor | None, lr: float,
                 out: torch.Tensor | None = None, absmax: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    """out[j] = mean_l W[l] - lr * G[j]  (D1D, simulation.py:304-312; numpy pairwise mean)."""
    L, d, ldw = _rows(W)
    _same(W, G, "G")
    ldg = _rows(G, "G")[2] if G is not None else ldw
    out = _prep_out(W, out)
    ldo = _rows(out, "out")[2]
    fn = getattr(_lib.load(), f"rm_mean_sgd_{_suffix(W)}")
    with torch.cuda.device(W.device):
        _lib.check(fn(W.data_ptr(), _lib.ptr(G), out.data_ptr(), L, d, ldw, ldg, ldo, float(lr),
                      _lib.ptr(absmax), _lib.stream_ptr(stream)), "rm_mean_sgd")
    return out


def spsgd_update(W: torch.Tensor, G: torch.Tensor, lr: float, out: torch.Tensor | None = None,
                 mismatch: torch.Tensor | None = None, absmax: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    """out[j] = W[j] - lr * mean_l G[l]  (step_spsgd, simulation.py:251-260).

    `mismatch` (int32 CUDA scalar, zeroed by caller) becomes nonzero if the
    learners' weights differ (the reference's ValueError condition)."""
    L, d, ldw = _rows(W)
    if G is None:
        raise ValueError("spsgd needs gradients")
    _same(W, G, "G")
    ldg = _rows(G, "G")[2]
    out = _prep_out(W, out)
    ldo = _rows(out, "out")[2]
    fn = getattr(_lib.load(), f"rm_spsgd_{_suffix(W)}")
    with torch.cuda.device(W.device):
        _lib.check(fn(W.data_ptr(), G.data_ptr(), out.data_ptr(), L, d, ldw, ldg, ldo, float(lr),
                      _lib.ptr(mismatch), _lib.ptr(absmax), _lib.stream_ptr(stream)),
                   "rm_spsgd")
    return out


def ring_mix_sgd_host(W_host: torch.Tensor, G_host: torch.Tensor | None, lr: float, left,
                      right, out_host: torch.Tensor | None = None,
                      workspace: torch.Tensor | None = None, absmax: torch.Tensor | None = None,
                      device=None, sync: bool = True) -> torch.Tensor:
    """The fused step on HOST buffers (L, d) fp32 (pinned for overlap): H2D, kernel and
    D2H pipelined over column chunks inside libringmix_b200 (rm_ring_mix_sgd_host_f32)."""
    _lib.require_cuda()
    for name, t in (("W_host", W_host), ("G_host", G_host), ("out_host", out_host)):
        if t is not None and (t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous float32 host tensor")
    L, d = W_host.shape
    if G_host is not None and G_host.shape != W_host.shape:
        raise ValueError("G_host must match W_host")
    if out_host is None:
        out_host = torch.empty_like(W_host, pin_memory=True)
    left = torch.as_tensor(np.asarray(left, dtype=np.int32) if not isinstance(left, torch.Tensor)
                           else left.to(torch.int32)).cpu().contiguous()
    right = torch.as_tensor(np.asarray(right, dtype=np.int32)
                            if not isinstance(right, torch.Tensor)
                            else right.to(torch.int32)).cpu().contiguous()
    dev = torch.device(device if device is not None else "cuda")
    if workspace is None:
        workspace = host_workspace(L, min(d, 1 << 21), dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().rm_ring_mix_sgd_host_f32(
            W_host.data_ptr(), _lib.ptr(G_host), out_host.data_ptr(), left.data_ptr(),
            right.data_ptr(), L, d, float(lr), workspace.data_ptr(), workspace.numel(),
            _lib.ptr(absmax), _lib.stream_ptr()), "rm_ring_mix_sgd_host_f32")
        if sync:
            torch.cuda.current_stream().synchronize()
    return out_host


def host_workspace(L: int, chunk_cols: int, device=None) -> torch.Tensor:
    """Device workspace (bytes) for ring_mix_sgd_host: 3 slots x (W, G, W') chunks."""
    nbytes = 4096 + 3 * 3 * L * 4 * (((chunk_cols + 31) // 32) * 32)
    return torch.empty(nbytes, dtype=torch.uint8,
                       device=torch.device(device if device is not None else "cuda"))


def _host_ptr(a):
    """(pointer, dtype) of a C-contiguous host numpy array or CPU tensor."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda or not a.is_contiguous():
            raise ValueError("expected a contiguous host tensor")
        return a.data_ptr(), {torch.float32: np.float32, torch.float64: np.float64}.get(a.dtype)
    if not a.flags.c_contiguous:
        raise ValueError("expected a C-contiguous (d, L) array")
    return a.ctypes.data, a.dtype.type


def workspace_dL(L: int, rows: int, dtype=np.float64, device=None) -> torch.Tensor:
    """Device workspace for gossip_step_host: 3 slots x (W, G, W') chunks of `rows` rows."""
    esz = np.dtype(dtype).itemsize
    return torch.empty(4096 + 9 * rows * L * esz, dtype=torch.uint8,
                       device=torch.device(device if device is not None else "cuda"))


def gossip_step_host(W, G, lr: float, left=None, right=None, out=None, workspace=None,
                     absmax: torch.Tensor | None = None, device=None, sync: bool = True):
    """The step on the reference's own arrays: W, G host (d, L) C-order float64 or float32
    (numpy arrays, or CPU tensors — pinned for overlap), returns `out` = apply_mixing(W, T)
    - lr * G with T = ring[p, p] given by neighbour tables `left` / `right`, or the uniform
    mean when both are None (simulation.py:263-268; mixing.py:106-125).  Row chunks go
    H2D || kernel || D2H inside libringmix_b200 (rm_gossip_step_host_dL_*); nothing is
    transposed.  G may be None (apply_mixing)."""
    _lib.require_cuda()
    wp, wdt = _host_ptr(W)
    if wdt not in (np.float32, np.float64) or len(W.shape) != 2:
        raise ValueError("W must be a (d, L) float32 or float64 host array")
    d, L = W.shape
    gp = None
    if G is not None:
        gp, gdt = _host_ptr(G)
        if tuple(G.shape) != (d, L) or gdt is not wdt:
            raise ValueError("G must match W (shape and dtype)")
    if out is None:
        out = np.empty((d, L), dtype=wdt)
    op, odt = _host_ptr(out)
    if tuple(out.shape) != (d, L) or odt is not wdt:
        raise ValueError("out must match W (shape and dtype)")
    if (left is None) != (right is None):
        raise ValueError("give both neighbour tables or neither (uniform mean)")
    tabs = None
    if left is not None:
        tabs = [np.ascontiguousarray(np.asarray(t.cpu() if isinstance(t, torch.Tensor) else t,
                                                dtype=np.int32)) for t in (left, right)]
        if any(t.shape != (L,) for t in tabs):
            raise ValueError(f"neighbour tables must have {L} entries")
    dev = torch.device(device if device is not None else "cuda")
    if workspace is None:
        workspace = workspace_dL(L, max(1, min(d, (1 << 24) // max(L, 1))), wdt, dev)
    sfx = "f64" if wdt is np.float64 else "f32"
    with torch.cuda.device(dev):
        _lib.check(getattr(_lib.load(), f"rm_gossip_step_host_dL_{sfx}")(
            wp, gp, op, None if tabs is None else tabs[0].ctypes.data,
            None if tabs is None else tabs[1].ctypes.data, L, d, float(lr),
            workspace.data_ptr(), workspace.numel(), _lib.ptr(absmax), _lib.stream_ptr()),
            "rm_gossip_step_host_dL")
        if sync:
            torch.cuda.current_stream().synchronize()
    return out


def gossip_step_dL(W: torch.Tensor, G: torch.Tensor | None, lr: float, left=None, right=None,
                   out: torch.Tensor | None = None, absmax: torch.Tensor | None = None):
    """gossip_step_host on DEVICE (d, L) row-major tensors (unit column stride)."""
    _lib.require_cuda(W)
    if W.dim() != 2 or W.stride(1) != 1 or W.dtype not in (torch.float32, torch.float64):
        raise ValueError("W must be a (d, L) float32/float64 CUDA tensor with unit column stride")
    d, L = W.shape
    if G is not None and (G.shape != W.shape or G.dtype != W.dtype or G.stride(1) != 1):
        raise ValueError("G must match W")
    if out is None:
        out = torch.empty_like(W, memory_format=torch.contiguous_format)
    sfx = "f64" if W.dtype == torch.float64 else "f32"
    _lib.check(getattr(_lib.load(), f"rm_gossip_step_dL_{sfx}")(
        W.data_ptr(), _lib.ptr(G), out.data_ptr(), _lib.ptr(left), _lib.ptr(right), L, d,
        W.stride(0), G.stride(0) if G is not None else L, out.stride(0), float(lr),
        _lib.ptr(absmax), _lib.stream_ptr()), "rm_gossip_step_dL")
    return out


# ----------------------------------------------------------------------------
# apply_mixing (reference-facing, any T)
# ----------------------------------------------------------------------------

def ring_structure(T: np.ndarray) -> tuple[np.ndarray, np.ndarray] | None:
    """If every column j of T holds exactly three entries equal to fl(1/3), one of
    them on the diagonal, and zeros elsewhere (ring and ring[p, p] matrices),
    return int32 (left, right) neighbour tables; else None."""
    L = T.shape[0]
    if L < 3:
        return None
    third = 1.0 / 3.0
    nz = T != 0.0
    if not np.all(nz.sum(axis=0) == 3) or not np.all(T[nz] == third):
        return None
    if not np.all(np.diag(T) == third):
        return None
    rows = np.nonzero(nz.T)[1].reshape(L, 3)  # per column j: sorted row indices
    j = np.arange(L)
    others = rows[rows != j[:, None]].reshape(L, 2)
    return others[:, 0].astype(np.int32), others[:, 1].astype(np.int32)


def apply_mixing(W, T):
    """One averaging step W @ T, columns of W are learners (mixing.py:106-125).

    W: a (d, L) numpy array (promoted to float64, as `W @ T` does in the
    reference) or a (d, L) CUDA tensor (float32/float64/bfloat16; a `.T` view of
    learner-major storage avoids any copy).  Returns the same kind as W.
    """
    is_np = isinstance(W, np.ndarray)
    Tn = np.asarray(T, dtype=np.float64)
    shape = W.shape
    if len(shape) != 2 or Tn.ndim != 2 or Tn.shape[0] != Tn.shape[1]:
        raise ValueError(f"expected W (d, L) and square T, got {tuple(shape)} and {Tn.shape}")
    if shape[1] != Tn.shape[0]:
        raise ValueError(
            f"size mismatch: W has {shape[1]} columns, T is {Tn.shape[0]}x{Tn.shape[0]}")
    _lib.require_cuda()
    L = Tn.shape[0]
    if is_np and L <= 512:
        # the reference's own (d, L) array: the (d, L) kernels take it as it is
        W64 = np.ascontiguousarray(np.asarray(W, dtype=np.float64))
        if np.all(Tn == 1.0 / L):
            return gossip_step_host(W64, None, 0.0)
        rs = ring_structure(Tn)
        if rs is not None:
            return gossip_step_host(W64, None, 0.0, rs[0], rs[1])
        X = torch.from_numpy(np.ascontiguousarray(np.asarray(W, dtype=np.float64).T)).cuda()
    else:
        X = W.T
        if X.dim() == 2 and X.shape[1] > 1 and X.stride(1) != 1:
            X = X.contiguous()
    if np.all(Tn == 1.0 / L):
        Y = mean_mix_sgd(X, None, 0.0)
    else:
        rs = ring_structure(Tn)
        if rs is not None:
            left = torch.from_numpy(rs[0]).to(X.device)
            right = torch.from_numpy(rs[1]).to(X.device)
            Y = ring_mix_sgd(X, None, 0.0, left, right)
        else:
            # general dense mixing: library GEMM (cuBLAS), not the fused path
            Tt = torch.from_numpy(Tn).to(device=X.device, dtype=X.dtype)
            Y = (Tt.T @ X).contiguous()
    if is_np:
        return np.ascontiguousarray(Y.cpu().numpy().T)
    return Y.T

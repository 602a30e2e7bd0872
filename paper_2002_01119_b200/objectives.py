"""Quadratic gradient oracle on the GPU (mirror of reference objectives.py, quadratic part).

Reference: pkg/src/ringmix/objectives.py:57-90 (QuadraticObjective) and
:145-164 (quadratic_oracle).  The spectrum and optimum are built exactly as in
the reference (``np.logspace``; optimum = stream(seed, TAG_DATA).standard_normal(d)
drawn by the device normal generator, bit-identical to numpy).  The oracle
implements the device protocol used by ``simulation.gradient_matrix``:

    device_gradients(Phi, cfg, k) -> G (L, d)
        G[l] = lam * (Phi[l] - w*) + noise_scale/sqrt(batch) * z_l,
        z_l = numpy stream(cfg.seed, TAG_GRADIENT, k, l).standard_normal(d)

computed by ``rm_quadratic_grad_*`` (csrc/normal.cu) bit-for-bit like the
reference's per-learner loop (simulation.py:233-237).  The logistic oracle is
out of scope.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib, mixing, seeding


def normal_workspace_bytes(nstreams: int, n: int, device) -> int:
    """Workspace size for the device normal generator.

    The fast layout keeps every speculative ziggurat block (~8.4 B per normal) so
    the output pass is a coalesced copy; it is used when it fits in a quarter of
    the free HBM (``RINGMIX_NORMAL_FAST=0`` forces the compact layout, which
    regenerates the draws in the output pass).  Both give identical bits.
    """
    lib = _lib.load()
    base = int(lib.rm_normal_workspace_bytes(nstreams, n))
    if os.environ.get("RINGMIX_NORMAL_FAST", "1") != "0":
        fast = int(lib.rm_normal_workspace_bytes_fast(nstreams, n))
        with torch.cuda.device(device):
            free = torch.cuda.mem_get_info()[0]
        if fast <= free // 4:
            return fast
    return base


def _normal_workspace(nstreams: int, n: int, device) -> torch.Tensor:
    nbytes = normal_workspace_bytes(nstreams, n, device)
    return torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)


def standard_normal(n: int, *entropy: int, device=None) -> torch.Tensor:
    """numpy ``stream(*entropy).standard_normal(n)`` generated on the GPU (fp64 CUDA tensor)."""
    _lib.require_cuda()
    dev = torch.device(device if device is not None else "cuda")
    words = seeding.entropy_words(*entropy)
    Z = torch.empty((1, max(n, 1)), dtype=torch.float64, device=dev)
    ws = _normal_workspace(1, n, dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().rm_standard_normal_f64(
            words.ctypes.data, len(words), 0, 0, 1, n, Z.data_ptr(), Z.stride(0), ws.data_ptr(),
            ws.numel(), _lib.stream_ptr()), "rm_standard_normal_f64")
    return Z[0, :n]


class QuadraticObjective:
    """1/2 (w - w*)' A (w - w*) with diagonal A and additive gradient noise (objectives.py:57-90)."""

    kind = "quadratic"

    def __init__(self, eigenvalues, optimum, noise_scale: float, device=None):
        self.eigenvalues = np.asarray(eigenvalues, dtype=float)
        self.optimum = np.asarray(optimum, dtype=float)
        self.noise_scale = float(noise_scale)
        if self.eigenvalues.ndim != 1 or self.optimum.shape != self.eigenvalues.shape:
            raise ValueError("eigenvalues and optimum must be 1-d with equal length")
        if np.any(self.eigenvalues <= 0):
            raise ValueError("eigenvalues must be strictly positive")
        if self.noise_scale < 0:
            raise ValueError("noise_scale must be >= 0")
        self.dimension = len(self.eigenvalues)
        self.device = torch.device(device if device is not None else "cuda")
        self._lam = torch.from_numpy(self.eigenvalues).to(self.device)
        self._opt = torch.from_numpy(self.optimum).to(self.device)
        self._ws = None

    # ---- reference host API (small helpers, fp64 numpy) ----
    def loss(self, w) -> float:
        dev = np.asarray(w, dtype=float) - self.optimum
        return 0.5 * float(np.sum(self.eigenvalues * dev * dev))

    def loss_columns(self, W) -> np.ndarray:
        dev = np.asarray(W) - self.optimum[:, None]
        return 0.5 * np.einsum("i,il,il->l", self.eigenvalues, dev, dev)

    def gradient(self, w) -> np.ndarray:
        return self.eigenvalues * (np.asarray(w, dtype=float) - self.optimum)

    def stochastic_gradient(self, w, batch, shard=None) -> np.ndarray:
        """Reference per-learner call; the noise comes from the device generator."""
        noise_sd = self.noise_scale / np.sqrt(batch.batch_size)
        z = standard_normal(self.dimension, *batch.sample_seed, device=self.device)
        return self.gradient(w) + noise_sd * z.cpu().numpy()

    # ---- device protocol (simulation.gradient_matrix) ----
    def device_gradients(self, Phi: torch.Tensor, cfg, k: int, learner0: int = 0,
                         out: torch.Tensor | None = None) -> torch.Tensor:
        """Gradients of learners [learner0, learner0 + L) at Phi (L, d); learner0 > 0 for a
        rank's shard of a learner-sharded run (same bits as the rows of the full call)."""
        L, d = Phi.shape
        if d != self.dimension:
            raise ValueError(f"Phi has {d} columns, oracle dimension is {self.dimension}")
        sfx = {torch.float32: "f32", torch.float64: "f64"}.get(Phi.dtype)
        if sfx is None:
            raise TypeError("device quadratic gradients support float32/float64 weights")
        ldp = mixing._rows(Phi, "Phi")[2]
        G = mixing.empty_learner_major(L, d, Phi.dtype, Phi.device) if out is None else out
        if G.shape != Phi.shape or G.dtype != Phi.dtype or G.device != Phi.device:
            raise ValueError("out must match Phi in shape, dtype and device")
        need = int(_lib.load().rm_normal_workspace_bytes(L, d))
        if self._ws is None or self._ws.numel() < need or self._ws.device != Phi.device:
            self._ws = None
            need = normal_workspace_bytes(L, d, Phi.device)
            self._ws = torch.empty(need, dtype=torch.uint8, device=Phi.device)
        lam, opt = self._lam.to(Phi.device), self._opt.to(Phi.device)
        words = seeding.entropy_words(cfg.seed, seeding.TAG_GRADIENT)
        noise_sd = float(self.noise_scale / np.sqrt(cfg.batch_size))
        fn = getattr(_lib.load(), f"rm_quadratic_grad_shard_{sfx}")
        with torch.cuda.device(Phi.device):
            _lib.check(fn(words.ctypes.data, len(words), int(k), int(learner0), L, d,
                          Phi.data_ptr(), ldp, lam.data_ptr(), opt.data_ptr(), noise_sd,
                          G.data_ptr(), G.stride(0), self._ws.data_ptr(), self._ws.numel(),
                          _lib.stream_ptr()),
                       "rm_quadratic_grad")
        return G

    def device_mean_step(self, M: torch.Tensor, Phi: torch.Tensor, lr: float, cfg, k: int,
                         ready: torch.cuda.Event | None = None, learner0: int = 0,
                         absmax: torch.Tensor | None = None,
                         out: torch.Tensor | None = None) -> torch.Tensor:
        """The D1D step with this oracle's gradient fused into the generator's final pass
        (rm_quadratic_mean_step_shard_*): out = M - lr * G(Phi) for learners
        [learner0, learner0 + L), G never written (simulation.py:304-312, objectives.py:84-90).
        M: the column means (fp64, d), possibly still being produced on another stream or GPU
        — only the final pass waits for ``ready``.  Same bits as ``device_gradients`` followed
        by the mean apply."""
        L, d = Phi.shape
        if d != self.dimension or M.numel() != d or M.dtype != torch.float64:
            raise ValueError("M must be the fp64 column means of the oracle's dimension")
        sfx = {torch.float32: "f32", torch.float64: "f64"}.get(Phi.dtype)
        if sfx is None:
            raise TypeError("the fused gradient step supports float32/float64 weights")
        lib = _lib.load()
        ldp = mixing._rows(Phi, "Phi")[2]
        need = int(lib.rm_quadratic_mix_workspace_bytes(L, d))
        ws = getattr(self, "_ws_fused", None)
        if ws is None or ws.numel() < need or ws.device != Phi.device:
            self._ws_fused = None
            self._ws_fused = ws = torch.empty(need, dtype=torch.uint8, device=Phi.device)
        if out is None:
            out = mixing.empty_learner_major(L, d, Phi.dtype, Phi.device)
        lam, opt = self._lam.to(Phi.device), self._opt.to(Phi.device)
        words = seeding.entropy_words(cfg.seed, seeding.TAG_GRADIENT)
        noise_sd = float(self.noise_scale / np.sqrt(cfg.batch_size))
        fn = getattr(lib, f"rm_quadratic_mean_step_shard_{sfx}")
        with torch.cuda.device(Phi.device):
            _lib.check(fn(words.ctypes.data, len(words), int(k), int(learner0), M.data_ptr(),
                          Phi.data_ptr(), out.data_ptr(), L, d, ldp, out.stride(0),
                          lam.data_ptr(), opt.data_ptr(), noise_sd, float(lr),
                          _lib.ptr(absmax), ws.data_ptr(), ws.numel(), _lib.stream_ptr(),
                          None if ready is None else ready.cuda_event),
                       "rm_quadratic_mean_step_shard")
        return out

    def device_mix_step(self, W: torch.Tensor, Phi: torch.Tensor | None, tables, lr: float,
                        cfg, k: int, absmax: torch.Tensor | None = None) -> torch.Tensor:
        """One training step with this oracle's gradient fused into the mix
        (rm_quadratic_mix_step_*): apply_mixing(W, T) - lr * G(Phi) with G never written
        to HBM, bit-identical to ``device_gradients`` followed by the ring / mean step
        (simulation.py:263-268, objectives.py:84-90).  W, Phi: learner-major (L, d);
        Phi None = the gradient at W; tables = (left, right) or None (uniform matrix).
        Returns the learner-major result."""
        L, d = W.shape
        if d != self.dimension:
            raise ValueError(f"W has {d} columns, oracle dimension is {self.dimension}")
        sfx = {torch.float32: "f32", torch.float64: "f64"}.get(W.dtype)
        if sfx is None:
            raise TypeError("the fused gradient step supports float32/float64 weights")
        lib = _lib.load()
        ldw = mixing._rows(W, "W")[2]
        if Phi is None:
            Phi, ldp = W, ldw
        else:
            if Phi.shape != W.shape or Phi.dtype != W.dtype or Phi.device != W.device:
                raise ValueError("Phi must match W in shape, dtype and device")
            ldp = mixing._rows(Phi, "Phi")[2]
        need = int(lib.rm_quadratic_mix_workspace_bytes(L, d))
        ws = getattr(self, "_ws_fused", None)
        if ws is None or ws.numel() < need or ws.device != W.device:
            self._ws_fused = None
            self._ws_fused = ws = torch.empty(need, dtype=torch.uint8, device=W.device)
        out = mixing.empty_learner_major(L, d, W.dtype, W.device)
        lam, opt = self._lam.to(W.device), self._opt.to(W.device)
        words = seeding.entropy_words(cfg.seed, seeding.TAG_GRADIENT)
        noise_sd = float(self.noise_scale / np.sqrt(cfg.batch_size))
        left, right = (None, None) if tables is None else tables
        fn = getattr(lib, f"rm_quadratic_mix_step_{sfx}")
        with torch.cuda.device(W.device):
            _lib.check(fn(words.ctypes.data, len(words), int(k), W.data_ptr(), Phi.data_ptr(),
                          out.data_ptr(), _lib.ptr(left), _lib.ptr(right), L, d, ldw, ldp,
                          out.stride(0), lam.data_ptr(), opt.data_ptr(), noise_sd, float(lr),
                          _lib.ptr(absmax), ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
                       "rm_quadratic_mix_step")
        return out

    def device_loss_columns(self, X: torch.Tensor) -> torch.Tensor:
        dev = X.to(torch.float64) - self._opt.to(X.device)
        return 0.5 * (self._lam.to(X.device) * dev * dev).sum(dim=1)

    def device_loss(self, w: torch.Tensor) -> float:
        dev = w.to(torch.float64) - self._opt.to(w.device)
        return 0.5 * float((self._lam.to(w.device) * dev * dev).sum().item())


def quadratic_oracle(dimension: int, condition_number: float = 1.0, optimum=None,
                     noise_scale: float = 0.0, seed: int = 0, device=None) -> QuadraticObjective:
    """Quadratic objective with log-spaced spectrum in [1, condition_number] (objectives.py:145-164)."""
    if dimension < 1:
        raise ValueError(f"dimension must be >= 1, got {dimension}")
    if condition_number < 1:
        raise ValueError(f"condition_number must be >= 1, got {condition_number}")
    eigenvalues = np.logspace(0.0, np.log10(condition_number), dimension)
    if optimum is None:
        optimum = standard_normal(dimension, seed, seeding.TAG_DATA,
                                  device=device).cpu().numpy()
    return QuadraticObjective(eigenvalues, np.asarray(optimum, dtype=float), noise_scale,
                              device=device)


def evaluate_loss(oracle, w) -> float:
    """Full-batch loss at w (objectives.py:192-194)."""
    return oracle.loss(w)


def gradient_check(oracle, w, step: float = 1e-5) -> float:
    """Relative error ||fd - grad|| / max(||grad||, 1e-12) of the analytic gradient
    against central differences of the loss (objectives.py:197-214); host fp64."""
    if step <= 0:
        raise ValueError(f"step must be > 0, got {step}")
    w = np.asarray(w, dtype=float)
    grad = np.asarray(oracle.gradient(w), dtype=float)
    fd = np.empty_like(grad)
    for i in range(len(w)):
        bump = np.zeros_like(w)
        bump[i] = step
        fd[i] = (oracle.loss(w + bump) - oracle.loss(w - bump)) / (2.0 * step)
    return float(np.linalg.norm(fd - grad)) / max(float(np.linalg.norm(grad)), 1e-12)

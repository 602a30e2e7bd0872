"""Training step with the quadratic oracle's gradient fused into the mix kernel
(rm_quadratic_mix_step_*; reference simulation.py:263-268 with
gradient_matrix simulation.py:226-238 and objectives.py:84-90).

The fused step must be bit-identical to the two-pass path the reference's arithmetic
is pinned on elsewhere (tests/test_gpu_objectives.py: device_gradients == the
reference's per-learner loop; tests/test_gpu_mixing.py: ring / mean step == oracle):
weights and max|W'| are compared bit for bit, for the randomized ring, the fixed
ring, the uniform matrix (D1D) and the 3-ring (uniform shortcut), fp32 and fp64,
gradient at W (synchronous) or at a separate Phi (stale), TMA tiles and the scalar
path, ragged widths, and with every normal lookup forced through the walk fallback.
run_training traces are compared fused vs unfused."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from paper_2002_01119_b200 import _lib, mixing, objectives, simulation
from paper_2002_01119_b200.simulation import RunConfig, Strategy

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["copy", "tile"], autouse=True)
def fused_kernel(request, monkeypatch):
    """Both fused kernels (generator-side zig_mix_kernel, mix_tma_kernel's Z modes)."""
    monkeypatch.setenv("RINGMIX_FUSED_KERNEL", request.param)
    return request.param


def _two_pass(oracle, X, Phi, tables, lr, cfg, k):
    G = oracle.device_gradients(X if Phi is None else Phi, cfg, k)
    absmax = torch.zeros((), dtype=torch.int64, device=X.device)
    if tables is None:
        out = mixing.mean_mix_sgd(X, G, lr, absmax=absmax)
    else:
        out = mixing.ring_mix_sgd(X, G, lr, tables[0], tables[1], absmax=absmax)
    return out, absmax


def _weights(L, d, dtype, seed, ld=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = mixing.empty_learner_major(L, d, dtype) if ld is None else \
        torch.empty((L, ld), dtype=dtype, device="cuda")[:, :d]
    X.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    return X


def _tables(kind, L, seed, k):
    if kind == "uniform":
        return None
    if kind == "fixed":
        return simulation.fixed_ring_tables(L, torch.device("cuda"))
    return simulation.rad_tables(L, seed, k, torch.device("cuda"))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("kind", ["rad", "fixed", "uniform"])
@pytest.mark.parametrize("stale", [False, True])
@pytest.mark.parametrize("L,d", [(16, 100_003), (3, 4099), (64, 1 << 17)])
def test_fused_step_is_bit_identical_to_two_pass(dtype, kind, stale, L, d):
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.5, seed=4)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.05, batch_size=3, seed=21)
    k = 7
    X = _weights(L, d, dtype, 1)
    Phi = _weights(L, d, dtype, 2) if stale else None
    tabs = _tables(kind, L, cfg.seed, k)
    ref, ref_amax = _two_pass(oracle, X, Phi, tabs, 0.05, cfg, k)
    amax = torch.zeros((), dtype=torch.int64, device="cuda")
    got = oracle.device_mix_step(X, Phi, tabs, 0.05, cfg, k, absmax=amax)
    assert torch.equal(got, ref)
    assert int(amax) == int(ref_amax)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fused_step_scalar_path_unaligned_rows(dtype):
    """Row stride not a multiple of 16 bytes: the scalar kernel's Z modes."""
    L, d = 12, 5001
    oracle = objectives.quadratic_oracle(d, condition_number=3.0, noise_scale=0.7, seed=8)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.1, batch_size=5, seed=3)
    X = _weights(L, d, dtype, 5, ld=d + 2)
    Phi = _weights(L, d, dtype, 6, ld=d + 3)
    for tabs in (_tables("rad", L, 3, 2), None):
        for P in (None, Phi):
            ref, ref_amax = _two_pass(oracle, X, P, tabs, 0.1, cfg, 2)
            amax = torch.zeros((), dtype=torch.int64, device="cuda")
            got = oracle.device_mix_step(X, P, tabs, 0.1, cfg, 2, absmax=amax)
            assert torch.equal(got, ref)
            assert int(amax) == int(ref_amax)


@pytest.mark.parametrize("kind", ["rad", "uniform"])
def test_fused_step_walk_fallback(kind, monkeypatch):
    """Every normal located by walking the generator's block table (the path a group
    spanning three or more blocks takes)."""
    monkeypatch.setenv("RINGMIX_ZDESC_WALK", "1")
    L, d = 16, 70_001
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=2)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.02, batch_size=4, seed=77)
    X = _weights(L, d, torch.float32, 9)
    tabs = _tables(kind, L, cfg.seed, 1)
    ref, _ = _two_pass(oracle, X, None, tabs, 0.02, cfg, 1)
    assert torch.equal(oracle.device_mix_step(X, None, tabs, 0.02, cfg, 1), ref)


def test_fused_step_covers_regenerated_blocks():
    """A shape large enough that some speculative ziggurat blocks fail to merge (about
    2e-4 of blocks): their normals come from the fixup's regenerated scratch slots."""
    L, d = 64, 1 << 20
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=3)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.01, batch_size=8, seed=11)
    X = _weights(L, d, torch.float32, 4)
    tabs = _tables("rad", L, cfg.seed, 3)
    ref, _ = _two_pass(oracle, X, None, tabs, 0.01, cfg, 3)
    got = oracle.device_mix_step(X, None, tabs, 0.01, cfg, 3)
    torch.cuda.synchronize()
    lib = _lib.load()
    off = int(lib.rm_normal_stats_offset(L, d))
    ws = oracle._ws_fused
    rejected = int(ws[off:off + 4].cpu().numpy().view(np.uint32)[0])
    assert rejected > 0
    assert torch.equal(got, ref)


@pytest.mark.parametrize("strategy", [Strategy.RAND_PSGD, Strategy.ADPSGD_FIXED, Strategy.D1D,
                                      Strategy.DPSGD_FIXED])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_run_training_fused_equals_unfused(strategy, dtype, monkeypatch):
    d, L = 30_011, 8
    oracle = objectives.quadratic_oracle(d, condition_number=20.0, noise_scale=1.0, seed=6)
    cfg = RunConfig(n_learners=L, iterations=9, lr=0.05, batch_size=4, seed=13, log_every=2,
                    dtype=dtype)
    monkeypatch.setattr(simulation, "FUSED_GRADIENT", "all")
    a = simulation.run_training(strategy, oracle, cfg)
    monkeypatch.setattr(simulation, "FUSED_GRADIENT", "off")
    b = simulation.run_training(strategy, oracle, cfg)
    assert torch.equal(a.state.weights, b.state.weights)
    assert torch.equal(a.state.last_gradients, b.state.last_gradients)
    assert [r.mean_loss for r in a.records] == [r.mean_loss for r in b.records]
    assert [r.consensus_dist for r in a.records] == [r.consensus_dist for r in b.records]


def test_fused_policy():
    """auto: ring steps at W itself only; all: every gossip step; off: none."""
    X = torch.empty((4, 8), dtype=torch.float32, device="cuda")
    o = objectives.quadratic_oracle(8, seed=1)
    f = simulation._fused_ok
    assert f(o, X, False) and not f(o, X, False, stale=True) and not f(o, X, False, ring=False)
    assert not f(o, X, True)
    assert not f(o, X.to(torch.bfloat16), False)
    simulation.FUSED_GRADIENT, old = "all", simulation.FUSED_GRADIENT
    try:
        assert f(o, X, False, ring=False, stale=True)
        simulation.FUSED_GRADIENT = "off"
        assert not f(o, X, False)
    finally:
        simulation.FUSED_GRADIENT = old


def test_fused_step_argument_errors():
    L, d = 8, 1000
    oracle = objectives.quadratic_oracle(d, seed=1)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.1, batch_size=1, seed=1)
    X = _weights(L, d, torch.float32, 1)
    with pytest.raises(TypeError):
        oracle.device_mix_step(X.to(torch.bfloat16), None, None, 0.1, cfg, 0)
    with pytest.raises(ValueError):
        oracle.device_mix_step(X[:, :999], None, None, 0.1, cfg, 0)
    lib = _lib.load()
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(X)
    w = (ctypes.c_uint32 * 1)(1)
    rc = lib.rm_quadratic_mix_step_f32(ctypes.addressof(w), 1, 0, X.data_ptr(), None,
                                       out.data_ptr(), None, None, L, d, d, d, d,
                                       oracle._lam.data_ptr(), oracle._opt.data_ptr(), 1.0, 0.1,
                                       None, ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    assert rc != 0 and "workspace" in _lib.last_error()


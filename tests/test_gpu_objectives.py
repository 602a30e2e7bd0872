"""Device gradient producer (quadratic oracle) and full run_training vs the reference.

* numpy Generator.standard_normal reproduced bit-for-bit on the GPU (parallel
  ziggurat over jump-ahead PCG64 blocks) — golden streams + live numpy.
* G = lam*(Phi - w*) + sd*z for all learners == the reference's per-learner
  stochastic_gradient loop (simulation.py:233-237) bit-for-bit in fp64.
* run_training with the device oracle reproduces the reference's own
  run_training trace (tests/golden/training.npz)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import normal_cases, training_cases
from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import _lib, mixing, objectives, seeding, simulation
from paper_2002_01119_b200.simulation import RunConfig, Strategy

pytestmark = pytest.mark.gpu


def test_standard_normal_matches_golden_streams():
    for ent, ref in normal_cases():
        got = objectives.standard_normal(len(ref), *ent).cpu().numpy()
        assert np.array_equal(got, ref), ent


@pytest.mark.parametrize("n,ent", [(1_000_003, (3, 0, 5, 1)), (5_000_000, (2**40, 6)),
                                   (257, (1, 2, 3, 4, 5, 6, 7))])
def test_standard_normal_matches_numpy_live(n, ent):
    got = objectives.standard_normal(n, *ent).cpu().numpy()
    ref = np.random.default_rng(np.random.SeedSequence(ent)).standard_normal(n)
    assert np.array_equal(got, ref)


def _host_gradients(oracle, Phi_ld, seed, k, batch):
    sd = oracle.noise_scale / np.sqrt(batch)
    G = np.empty_like(Phi_ld)
    for l in range(Phi_ld.shape[0]):
        z = np.random.default_rng(np.random.SeedSequence((seed, 0, k, l))).standard_normal(
            Phi_ld.shape[1])
        G[l] = oracle.eigenvalues * (Phi_ld[l] - oracle.optimum) + sd * z
    return G


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("L,d,k", [(8, 5000, 0), (3, 77, 2**32 + 9), (16, 40_000, 5)])
def test_device_gradients_equal_reference_loop(dtype, L, d, k):
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.5, seed=4)
    ref_opt = np.random.default_rng(np.random.SeedSequence((4, 6))).standard_normal(d)
    assert np.array_equal(oracle.optimum, ref_opt)
    g = torch.Generator(device="cuda").manual_seed(0)
    Phi = mixing.empty_learner_major(L, d, dtype)
    Phi.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.1, batch_size=3, seed=99)
    G = oracle.device_gradients(Phi, cfg, k)
    ref = _host_gradients(oracle, Phi.double().cpu().numpy(), 99, k, 3)
    got = G.double().cpu().numpy()
    if dtype == torch.float64:
        assert np.array_equal(got, ref)
    else:
        assert np.array_equal(got, ref.astype(np.float32).astype(np.float64))


def test_reference_stochastic_gradient_api():
    oracle = objectives.quadratic_oracle(300, condition_number=5.0, noise_scale=2.0, seed=1)
    w = np.linspace(-1, 1, 300)
    batch = simulation.BatchDescriptor(4, (7, 0, 3, 2))
    got = oracle.stochastic_gradient(w, batch)
    z = np.random.default_rng(np.random.SeedSequence((7, 0, 3, 2))).standard_normal(300)
    ref = oracle.eigenvalues * (w - oracle.optimum) + (2.0 / np.sqrt(4)) * z
    assert np.array_equal(got, ref)


def _uses_mean(c):
    return c["strategy"] in ("d1d", "spsgd") or c["L"] == 3


@pytest.mark.parametrize("case", training_cases(), ids=lambda c: f"{c['strategy']}-L{c['L']}")
def test_run_training_reproduces_reference_trace(case):
    oracle = objectives.quadratic_oracle(case["d"], condition_number=case["cond"],
                                         noise_scale=case["noise"], seed=case["seed"] + 100)
    assert np.array_equal(oracle.optimum, case["optimum"])
    cfg = RunConfig(n_learners=case["L"], iterations=case["iters"], lr=case["lr"], batch_size=4,
                    seed=case["seed"], staleness_mode=case["mode"], warmup_iters=case["warm"],
                    log_every=2, dtype="float64")
    res = simulation.run_training(Strategy(case["strategy"]), oracle, cfg)
    assert res.diverged == case["diverged"]
    recs = np.array([[r.iteration, r.sim_time_s, r.mean_loss, r.avg_model_loss,
                      r.consensus_dist, r.rho] for r in res.records])
    ref = case["records"]
    assert recs.shape == ref.shape
    assert np.array_equal(recs[:, 0], ref[:, 0])            # iterations
    assert np.array_equal(recs[:, 1], ref[:, 1])            # simulated clock (host, same draws)
    assert np.array_equal(recs[:, 5], ref[:, 5])            # rho
    assert np.allclose(recs[:, 2:5], ref[:, 2:5], rtol=1e-12, atol=1e-13)
    W = res.state.weights.cpu().numpy()
    if _uses_mean(case):
        assert np.array_equal(W, case["W"])
    else:
        # OpenBLAS edge-column rounding compounds over the run
        assert np.allclose(W, case["W"], rtol=0, atol=1e-13)


def test_device_log1p_is_bit_identical_to_host_libm():
    """numpy's ziggurat calls the C library's log1p (npy_log1p), which is what
    math.log1p calls; numpy's own np.log1p ufunc is a different SIMD code and
    is NOT the reference here."""
    import math

    from paper_2002_01119_b200 import _lib
    rng = np.random.default_rng(0)
    # the ziggurat tail evaluates log1p(-u), u = next_double in [0, 1)
    u = rng.integers(0, 2**53, 300_000, dtype=np.uint64).astype(np.float64) \
        * (1.0 / 9007199254740992.0)
    x = np.concatenate([-u, rng.uniform(-0.999, 5.0, 100_000), [0.0, -0.0, 1e-300, -1e-17,
                                                                1e-10, -0.2929, 0.41422, 1e20]])
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    _lib.check(_lib.load().rm_log1p_f64(xd.data_ptr(), yd.data_ptr(), len(x), _lib.stream_ptr()))
    ref = np.array([math.log1p(v) for v in x])
    assert np.array_equal(yd.cpu().numpy().view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("L,d,dtype", [(8, 1000, torch.float64), (64, 100_003, torch.float32),
                                       (3, 17, torch.float64), (128, 5000, torch.bfloat16)])
def test_fused_trace_stats_match_reference_formulas(L, d, dtype):
    oracle = objectives.quadratic_oracle(d, condition_number=7.0, noise_scale=1.0, seed=2)
    g = torch.Generator(device="cuda").manual_seed(5)
    X = mixing.empty_learner_major(L, d, dtype)
    X.copy_(torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64).to(dtype))
    cons_sq, loss_col, avg = simulation.trace_stats(X.T, oracle, exact=False)
    W = X.double().cpu().numpy().T              # reference (d, L) layout
    dev = W - W.mean(axis=1, keepdims=True)
    assert np.allclose(cons_sq.cpu().numpy(), (dev * dev).sum(axis=0), rtol=1e-12)
    assert np.allclose(loss_col.cpu().numpy(), oracle.loss_columns(W), rtol=1e-12)
    assert np.isclose(float(avg), oracle.loss(W.mean(axis=1)), rtol=1e-12)
    assert simulation.consensus_distance(X.T) == pytest.approx(
        float(np.sqrt((dev * dev).sum(axis=0).max())), rel=1e-12)


@pytest.mark.parametrize("L,d,dtype", [(4, 24, torch.float64), (8, 1000, torch.float64),
                                       (3, 1, torch.float64), (5, 7, torch.float64),
                                       (16, 100_003, torch.float64), (130, 2_000, torch.float64),
                                       (64, 70_001, torch.float32), (16, 3_000, torch.bfloat16)])
def test_exact_trace_stats_are_bitwise_numpy(L, d, dtype, monkeypatch):
    """rm_trace_stats_exact_*: numpy's own summation order, so the record values are the
    reference's bits (simulation.py:359-362, 398-409; objectives.py:72-79): the axis-0 sum
    and the einsum run sequentially over the parameters, the average-model loss is numpy's
    pairwise sum (split over the subtrees of its recursion on the GPU)."""
    oracle = objectives.quadratic_oracle(d, condition_number=9.0, noise_scale=1.0, seed=L)
    g = torch.Generator(device="cuda").manual_seed(d)
    X = mixing.empty_learner_major(L, d, dtype)
    X.copy_((torch.randn((L, d), generator=g, device="cuda", dtype=torch.float64)
             * torch.exp(2 * torch.randn((1, d), generator=g, device="cuda",
                                         dtype=torch.float64))).to(dtype))
    cons_sq, loss_col, avg = simulation.trace_stats(X.T, oracle, exact=True)
    W = X.double().cpu().numpy().T.copy()       # the reference's (d, L) C-order array
    dev = W - W.mean(axis=1, keepdims=True)
    assert np.array_equal(cons_sq.cpu().numpy(), (dev * dev).sum(axis=0))
    assert np.array_equal(loss_col.cpu().numpy(), oracle.loss_columns(W))
    assert float(avg) == oracle.loss(W.mean(axis=1))
    monkeypatch.setenv("RINGMIX_TRACE_EXACT", "1")
    assert simulation.consensus_distance(X.T) == float(np.sqrt((dev * dev).sum(axis=0).max()))
    c2, l2, a2 = simulation.trace_stats(X.T, None, exact=True)
    assert torch.equal(c2, cons_sq) and l2 is None and a2 is None


@pytest.mark.parametrize("overlap,ctas", [(True, 1), (True, 4), (True, 0), (False, 0)])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_d1d_step_mean_beside_fused_generator_is_bit_identical(dtype, overlap, ctas, monkeypatch):
    """step_d1d for steps whose gradients are not kept: the uniform fused step (default), or
    (RINGMIX_D1D_OVERLAP=1) the average of W_k on a side stream (capped CTAs) beside the
    generator, whose final pass writes mean - lr G(W_{k-1}) (rm_quadratic_mean_step_shard_*)
    — both equal to the gradient followed by the fused mean/SGD kernel (simulation.py:304-312)."""
    monkeypatch.setattr(simulation, "D1D_MEAN_CTAS", ctas)
    monkeypatch.setattr(simulation, "D1D_FUSED_OVERLAP", overlap)
    L, d = 16, 70_001
    oracle = objectives.quadratic_oracle(d, condition_number=5.0, noise_scale=1.0, seed=3)
    cfg = RunConfig(n_learners=L, iterations=3, lr=0.05, batch_size=2, seed=4, dtype=dtype)
    st = simulation.initial_state(oracle, cfg)
    st.weights.copy_(st.weights + torch.randn_like(st.weights) * 0.1)
    for _ in range(3):
        new = simulation.step_d1d(st, oracle, cfg, keep_gradients=False)
        assert new.last_gradients is None
        G = oracle.device_gradients(st.prev_weights.T, cfg, st.iteration)
        ref = mixing.mean_mix_sgd(st.weights.T, G, simulation.learning_rate(cfg, st.iteration))
        torch.cuda.synchronize()
        assert torch.equal(new.weights.T, ref)
        assert simulation.absmax_value(new.absmax_bits) == float(ref.abs().max())
        st = new


@pytest.mark.parametrize("side_stream", [True, False])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_overlapped_d1d_step_is_bit_identical_to_fused(dtype, side_stream, monkeypatch):
    """step_d1d with a device oracle (mean of W_k on a side stream || gradient of
    W_{k-1}) must equal the fused single-pass D1D kernel on the same inputs."""
    monkeypatch.setattr(simulation, "D1D_SIDE_STREAM", side_stream)
    L, d = 16, 50_001
    oracle = objectives.quadratic_oracle(d, condition_number=5.0, noise_scale=1.0, seed=3)
    cfg = RunConfig(n_learners=L, iterations=3, lr=0.05, batch_size=2, seed=4, dtype=dtype)
    st = simulation.initial_state(oracle, cfg)
    st.weights.copy_(st.weights + torch.randn_like(st.weights) * 0.1)
    for _ in range(2):
        new = simulation.step_d1d(st, oracle, cfg)
        G = oracle.device_gradients(st.prev_weights.T, cfg, st.iteration)
        ref = mixing.mean_mix_sgd(st.weights.T, G, simulation.learning_rate(cfg, st.iteration))
        torch.cuda.synchronize()
        assert torch.equal(new.weights.T, ref)
        assert simulation.absmax_value(new.absmax_bits) == float(ref.abs().max())
        st = new


def test_normal_workspace_covers_its_layout():
    """The workspace size reported by the library covers every region the kernels
    use (the counters sit at the end of the layout)."""
    from paper_2002_01119_b200 import _lib
    lib = _lib.load()
    for L, d in [(1, 1), (3, 77), (16, 1 << 20), (64, 25_557_032)]:
        assert lib.rm_normal_stats_offset(L, d) + 8 <= lib.rm_normal_workspace_bytes(L, d)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
def test_trace_stats_tiled_and_generic_kernels_agree(dtype, monkeypatch):
    """The TMA-tiled trace reduction and the generic kernel (unaligned rows / other
    shapes) give the same per-learner sums to fp64 rounding, on ragged shapes."""
    for L, d in [(3, 7), (8, 1), (16, 1000), (33, 4099), (64, 100_003), (128, 2_049)]:
        oracle = objectives.quadratic_oracle(d, condition_number=3.0, noise_scale=0.0, seed=L)
        X = mixing.empty_learner_major(L, d, dtype, "cuda").normal_()
        monkeypatch.delenv("RINGMIX_TRACE_NO_TMA", raising=False)
        a = simulation.trace_stats(X.T, oracle, exact=False)
        monkeypatch.setenv("RINGMIX_TRACE_NO_TMA", "1")
        b = simulation.trace_stats(X.T, oracle, exact=False)
        for x, y in zip(a, b):
            assert torch.allclose(x, y, rtol=1e-12, atol=1e-12)
        # and the reference's formulas on the host
        W = X.double().cpu().numpy()
        mean = W.mean(axis=0)
        cons = ((W - mean) ** 2).sum(axis=1)
        lam, opt = oracle.eigenvalues, oracle.optimum
        loss_cols = 0.5 * (lam * (W - opt) ** 2).sum(axis=1)
        np.testing.assert_allclose(a[0].cpu().numpy(), cons, rtol=1e-10)
        np.testing.assert_allclose(a[1].cpu().numpy(), loss_cols, rtol=1e-10)


@pytest.mark.parametrize("no_tma", ["", "1"])
def test_trace_stats_are_deterministic(no_tma, monkeypatch):
    """Per-CTA partials summed in a fixed order: repeated reductions of the same W give
    identical bits (the reference's trace CSVs are byte-stable for a fixed config)."""
    if no_tma:
        monkeypatch.setenv("RINGMIX_TRACE_NO_TMA", "1")
    L, d = 64, 3_000_017
    oracle = objectives.quadratic_oracle(d, condition_number=7.0, noise_scale=0.0, seed=2)
    X = mixing.empty_learner_major(L, d, torch.float32, "cuda").normal_()
    first = simulation.trace_stats(X.T, oracle, exact=False)
    for _ in range(5):
        again = simulation.trace_stats(X.T, oracle, exact=False)
        for x, y in zip(first, again):
            assert torch.equal(x, y)


@pytest.mark.parametrize("no_tma", ["", "1"])
@pytest.mark.parametrize("L,d", [(5, 333), (9, 4097), (16, 1000), (64, 100_003), (128, 2_049),
                                 (200, 3_001), (256, 1_025), (300, 777), (1000, 65)])
def test_trace_stats_every_kernel_and_many_learners(L, d, no_tma, monkeypatch):
    """Tiled TMA kernel (L <= 128; numpy's chains split over lane halves) and the generic
    kernel against the reference's formulas, including L > 128 (numpy's recursive pairwise
    mean; run_training with more than 128 learners)."""
    if no_tma:
        monkeypatch.setenv("RINGMIX_TRACE_NO_TMA", no_tma)
    oracle = objectives.quadratic_oracle(d, condition_number=3.0, noise_scale=0.0, seed=L)
    X = mixing.empty_learner_major(L, d, torch.float32, "cuda").normal_()
    cons, loss_col, avg = simulation.trace_stats(X.T, oracle)
    W = X.double().cpu().numpy().T                       # (d, L) as the reference holds it
    dev = W - W.mean(axis=1, keepdims=True)
    np.testing.assert_allclose(cons.cpu().numpy(), (dev * dev).sum(axis=0), rtol=1e-11)
    np.testing.assert_allclose(loss_col.cpu().numpy(), oracle.loss_columns(W), rtol=1e-11)
    assert float(avg) == pytest.approx(oracle.loss(W.mean(axis=1)), rel=1e-11)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_sharded_gradients_equal_rows_of_the_full_call(dtype):
    """rm_quadratic_grad_shard_*: a rank's learners [b, e) draw streams b..e-1, so its
    gradients are rows b..e-1 of the all-learner call (learner-sharded D1D training)."""
    L, d, k = 12, 30_001, 4
    oracle = objectives.quadratic_oracle(d, condition_number=5.0, noise_scale=1.0, seed=2)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.1, batch_size=2, seed=17)
    Phi = mixing.empty_learner_major(L, d, dtype)
    Phi.copy_(torch.randn((L, d), device="cuda", dtype=torch.float64).to(dtype))
    full = oracle.device_gradients(Phi, cfg, k).clone()
    for b, e in ((0, 5), (5, 12), (7, 8)):
        part = oracle.device_gradients(Phi[b:e], cfg, k, learner0=b)
        assert torch.equal(part, full[b:e]), (b, e)
    out = torch.empty_like(Phi[:4])
    assert oracle.device_gradients(Phi[3:7], cfg, k, learner0=3, out=out) is out
    assert torch.equal(out, full[3:7])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("L,d,b,e", [(16, 5_003, 4, 12), (64, 40_000, 32, 64), (8, 777, 0, 3)])
def test_sharded_mean_step_equals_rows_of_the_two_pass_step(dtype, L, d, b, e):
    """rm_quadratic_mean_step_shard_*: a rank's learners [b, e) of a learner-sharded D1D
    training step with the gradient fused into the generator's final pass and the global
    means M supplied (and waited for through an event) — rows b..e-1 of the single-GPU
    step mean(W) - lr * G(Phi) (simulation.py:304-312)."""
    oracle = objectives.quadratic_oracle(d, condition_number=6.0, noise_scale=1.2, seed=9)
    cfg = RunConfig(n_learners=L, iterations=1, lr=0.03, batch_size=4, seed=21)
    gen = torch.Generator(device="cuda").manual_seed(1)
    X, Phi = (mixing.empty_learner_major(L, d, dtype) for _ in range(2))
    X.copy_(torch.randn((L, d), generator=gen, device="cuda", dtype=torch.float64).to(dtype))
    Phi.copy_(torch.randn((L, d), generator=gen, device="cuda", dtype=torch.float64).to(dtype))
    k, lr = 6, 0.03
    G = oracle.device_gradients(Phi, cfg, k)
    ref = mixing.mean_mix_sgd(X, G, lr)
    lib = _lib.load()
    M = torch.empty(d, dtype=torch.float64, device="cuda")
    sfx = mixing._suffix(X)
    _lib.check(getattr(lib, f"rm_column_mean_{sfx}")(X.data_ptr(), L, d, X.stride(0),
                                                      M.data_ptr(), _lib.stream_ptr()), "mean")
    ready = torch.cuda.Event()
    ready.record()
    Lg = e - b
    P = Phi[b:e]
    out = mixing.empty_learner_major(Lg, d, dtype)
    absmax = torch.zeros((), dtype=torch.int64, device="cuda")
    ws = torch.empty(int(lib.rm_quadratic_mix_workspace_bytes(Lg, d)), dtype=torch.uint8,
                     device="cuda")
    words = seeding.entropy_words(cfg.seed, seeding.TAG_GRADIENT)
    _lib.check(getattr(lib, f"rm_quadratic_mean_step_shard_{sfx}")(
        words.ctypes.data, len(words), k, b, M.data_ptr(), P.data_ptr(), out.data_ptr(), Lg, d,
        P.stride(0), out.stride(0), oracle._lam.data_ptr(), oracle._opt.data_ptr(),
        float(oracle.noise_scale / np.sqrt(cfg.batch_size)), lr, absmax.data_ptr(),
        ws.data_ptr(), ws.numel(), _lib.stream_ptr(), ready.cuda_event), "mean step shard")
    torch.cuda.synchronize()
    assert torch.equal(out, ref[b:e])
    assert simulation.absmax_value(absmax) == float(ref[b:e].abs().max())

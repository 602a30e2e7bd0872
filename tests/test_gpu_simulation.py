"""Step functions (the reference's plugin boundary) vs the reference's own
trajectories frozen in tests/golden/steps.npz, plus the reference's
simulation tests restated (pkg/tests/test_simulation.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import step_cases
from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import mixing, simulation
from paper_2002_01119_b200.simulation import RunConfig, SimState, Strategy

pytestmark = pytest.mark.gpu


class SynthOracle:
    """Gradient stub: precomputed G[k] (d, L) columns, independent of the weights
    (same stub the golden fixtures were produced with)."""

    def __init__(self, Gs, dtype=torch.float64):
        self.Gs = Gs
        self.dimension = next(iter(Gs.values())).shape[0]
        self.dtype = dtype

    def device_gradients(self, X, cfg, k):
        G = mixing.empty_learner_major(X.shape[0], X.shape[1], X.dtype, X.device)
        G.copy_(torch.from_numpy(self.Gs[k].T.copy()).to(X.device, X.dtype))
        return G


class HostSynthOracle(SynthOracle):
    """Same stub through the reference's host protocol (stochastic_gradient)."""

    device_gradients = None

    def __getattribute__(self, name):
        if name == "device_gradients":
            raise AttributeError(name)
        return object.__getattribute__(self, name)

    def stochastic_gradient(self, w, batch, shard=None):
        _, _, k, l = batch.sample_seed
        return self.Gs[k][:, l]


def _state(case, dtype):
    def up(a):
        X = mixing.empty_learner_major(case["L"], case["d"], dtype)
        X.copy_(torch.from_numpy(a.T.copy()).to("cuda", dtype))
        return X.T
    return SimState(weights=up(case["W0"]), prev_weights=up(case["Wprev"]), iteration=case["k0"],
                    seed=case["seed"], compute_time_s=np.zeros(case["L"]))


def _cfg(case, dtype="float64"):
    return RunConfig(n_learners=case["L"], iterations=case["nsteps"], lr=case["lr"], batch_size=1,
                     seed=case["seed"], staleness_mode=case["mode"], dtype=dtype)


def _uses_mean_path(case):
    return case["strategy"] in ("d1d", "spsgd") or case["L"] == 3


@pytest.mark.parametrize("host_protocol", [False, True])
@pytest.mark.parametrize("case", step_cases(), ids=lambda c: f"{c['strategy']}-L{c['L']}-d{c['d']}")
def test_f64_steps_match_reference_trajectories(case, host_protocol):
    Gs = {case["k0"] + s: case["G"][s] for s in range(case["nsteps"])}
    oracle = (HostSynthOracle if host_protocol else SynthOracle)(Gs)
    cfg = _cfg(case)
    step = simulation._STEP_FUNCTIONS[Strategy(case["strategy"])]
    state = _state(case, torch.float64)
    for s in range(case["nsteps"]):
        state = step(state, oracle, cfg)
        got = state.weights.cpu().numpy()
        ref = case["traj"][s]
        if _uses_mean_path(case):
            assert np.array_equal(got, ref), s
        else:
            assert np.allclose(got, ref, rtol=0, atol=1e-15), s
        assert state.iteration == case["k0"] + s + 1


@pytest.mark.parametrize("case", step_cases(), ids=lambda c: f"{c['strategy']}-L{c['L']}-d{c['d']}")
def test_f32_steps_match_oracle_per_step(case):
    """fp32 storage: each step equals the oracle's fp64 step on the same fp32
    inputs, rounded once (bit-exact), and stays within the north-star tolerance."""
    Gs = {case["k0"] + s: case["G"][s] for s in range(case["nsteps"])}
    oracle = SynthOracle(Gs)
    cfg = _cfg(case, "float32")
    step = simulation._STEP_FUNCTIONS[Strategy(case["strategy"])]
    state = _state(case, torch.float32)
    L = case["L"]
    for s in range(case["nsteps"]):
        k = case["k0"] + s
        W = state.weights.double().cpu().numpy()
        G = Gs[k]
        state = step(state, oracle, cfg)
        got = state.weights.double().cpu().numpy()
        if case["strategy"] == "spsgd":
            ref = W - case["lr"] * O.c_mean_sgd(G, None, 0.0)
        elif _uses_mean_path(case):
            ref = O.c_mean_sgd(W, G, case["lr"])
        else:
            p = O.c_permutation(L, case["seed"], k) if case["strategy"] == "rand_psgd" \
                else np.arange(L)
            _, left, right = O.neighbour_tables(p)
            ref = O.c_ring_mix_sgd(W, G, case["lr"], left, right)
        assert np.array_equal(got, ref.astype(np.float32).astype(np.float64)), s


def _qoracle(d=6):
    class Quadratic:
        """Minimal quadratic objective (reference objectives.py:57-90 semantics)."""

        def __init__(self):
            rng = np.random.default_rng(2)
            self.dimension = d
            self.eigenvalues = np.logspace(0, 1, d)
            self.optimum = rng.standard_normal(d)

        def stochastic_gradient(self, w, batch, shard=None):
            return self.eigenvalues * (w - self.optimum) + \
                batch.rng().standard_normal(d) / np.sqrt(batch.batch_size)

        def loss_columns(self, W):
            dev = W - self.optimum[:, None]
            return 0.5 * np.einsum("i,il,il->l", self.eigenvalues, dev, dev)

        def loss(self, w):
            dev = w - self.optimum
            return 0.5 * float(np.sum(self.eigenvalues * dev * dev))
    return Quadratic()


def _cfg2(**kw):
    base = dict(n_learners=4, iterations=5, lr=0.1, batch_size=2, seed=5)
    base.update(kw)
    return RunConfig(**base)


def test_initial_state_broadcasts_one_model():
    st = simulation.initial_state(_qoracle(), _cfg2(n_learners=6))
    W = st.weights.cpu().numpy()
    assert W.shape == (6, 6) and np.all(W == W[:, :1])
    ref = np.random.default_rng(np.random.SeedSequence((5, 3))).standard_normal(6)
    assert np.array_equal(W[:, 0], ref)
    zero = simulation.initial_state(_qoracle(), _cfg2(init_scale=0.0))
    assert bool((zero.weights == 0).all())


def test_dpsgd_l3_first_step_bitwise_equals_d1d():
    o, cfg = _qoracle(), _cfg2(n_learners=3)
    a = simulation.step_dpsgd_fixed(simulation.initial_state(o, cfg), o, cfg)
    b = simulation.step_d1d(simulation.initial_state(o, cfg), o, cfg)
    assert torch.equal(a.weights, b.weights)


def test_stale_and_sync_agree_only_on_first_step():
    o, cfg = _qoracle(), _cfg2(n_learners=5)
    sync = simulation.step_dpsgd_fixed(simulation.initial_state(o, cfg), o, cfg)
    stale = simulation.step_adpsgd_fixed(simulation.initial_state(o, cfg), o, cfg)
    assert torch.equal(sync.weights, stale.weights)
    sync2 = simulation.step_dpsgd_fixed(sync, o, cfg)
    stale2 = simulation.step_adpsgd_fixed(stale, o, cfg)
    assert not torch.equal(sync2.weights, stale2.weights)


def test_rand_psgd_staleness_override_and_errors():
    o, cfg = _qoracle(), _cfg2(n_learners=5, staleness_mode="async")
    s1 = simulation.step_rand_psgd(simulation.initial_state(o, cfg), o, cfg)
    a = simulation.step_rand_psgd(s1, o, cfg, staleness_mode="sync")
    b = simulation.step_rand_psgd(s1, o, cfg, staleness_mode="async")
    assert not torch.equal(a.weights, b.weights)
    with pytest.raises(ValueError):
        simulation.step_rand_psgd(s1, o, cfg, staleness_mode="eventually")


def test_spsgd_rejects_disagreeing_learners():
    o, cfg = _qoracle(), _cfg2()
    st = simulation.initial_state(o, cfg)
    st.weights[0, 1] += 1.0
    with pytest.raises(ValueError, match="identical"):
        simulation.step_spsgd(st, o, cfg)


def test_mixing_preserves_learner_average():
    o, cfg = _qoracle(), _cfg2(n_learners=6)
    for step in (simulation.step_dpsgd_fixed, simulation.step_adpsgd_fixed,
                 simulation.step_rand_psgd, simulation.step_d1d):
        st = simulation.initial_state(o, cfg)
        for _ in range(5):
            before = st.weights.mean(dim=1)
            new = step(st, o, cfg)
            moved = new.weights.mean(dim=1)
            expected = before - cfg.lr * new.last_gradients.mean(dim=1)
            assert torch.allclose(moved, expected, rtol=0, atol=1e-12)
            st = new


def test_run_training_matches_reference_loop_semantics():
    o = _qoracle(d=8)
    cfg = _cfg2(n_learners=8, iterations=7, log_every=3)
    res = simulation.run_training(Strategy.RAND_PSGD, o, cfg)
    assert not res.diverged
    assert [r.iteration for r in res.records] == [3, 6, 7]
    assert res.state.iteration == 7
    assert all(np.isfinite(r.mean_loss) for r in res.records)
    d1d = simulation.run_training(Strategy.D1D, o, cfg)
    assert d1d.records[-1].rho == 0.0


def test_divergence_returns_partial_trace():
    o = _qoracle(d=4)
    cfg = _cfg2(n_learners=4, iterations=50, lr=5.0, divergence_threshold=1e3)
    res = simulation.run_training(Strategy.ADPSGD_FIXED, o, cfg)
    assert res.diverged
    assert res.state.iteration < 50
    assert float(res.state.weights.abs().max()) <= 1e3


def test_consensus_distance_matches_reference_formula():
    W = np.random.default_rng(0).standard_normal((20, 6))
    dev = W - W.mean(axis=1, keepdims=True)
    ref = float(np.sqrt((dev * dev).sum(axis=0).max()))
    assert simulation.consensus_distance(torch.from_numpy(W).cuda()) == pytest.approx(ref,
                                                                                      rel=1e-12)


@pytest.mark.parametrize("seed", [12345, None])
def test_graphed_ring_steps_equal_eager_steps(seed):
    """simulation.GraphedRingSteps (K steps in one CUDA graph) gives the same bits as K eager
    ring_mix_sgd calls (RAD with the device permutation tables, or the fixed ring), and a
    replay repeats them from the current W[0]."""
    L, d, K = 16, 5000, 70           # more than one 64-step table block
    g = torch.Generator(device="cuda").manual_seed(8)
    W0 = mixing.empty_learner_major(L, d, torch.float32)
    W0.copy_(torch.randn((L, d), generator=g, device="cuda"))
    G = mixing.empty_learner_major(L, d, torch.float32)
    G.copy_(torch.randn((L, d), generator=g, device="cuda"))
    start = W0.clone()
    gs = simulation.GraphedRingSteps(W0, G, 0.01, K, seed=seed, k0=5)
    out = gs.replay().clone()
    ref = start
    fixed = simulation.fixed_ring_tables(L, "cuda")
    for k in range(5, 5 + K):
        lt, rt = simulation.rad_tables(L, seed, k, "cuda") if seed is not None else fixed
        ref = mixing.ring_mix_sgd(ref, G, 0.01, lt, rt)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    assert simulation.absmax_value(gs.absmax[K - 1]) == float(ref.abs().max())
    gs.W[0].copy_(start)
    assert torch.equal(gs.replay(), ref)

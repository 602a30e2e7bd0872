"""Freeze golden fixtures by running the REFERENCE itself (not the oracle).

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/{perms,sequential,steps,spectral,normals,training}.npz and
tests/golden/sweep/*.csv (`make_golden.py sweep` regenerates only the sweep).  Each file records
the numpy version it was produced under (the Generator stream is only
guaranteed stable within a numpy version; these were frozen under 2.3.5 /
OpenBLAS 0.3.30).  Nothing at test time reads /root/reference: the GPU box
only sees these committed files.
"""

from __future__ import annotations

import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from ringmix import harness, mixing, seeding, simulation, spectral  # noqa: E402
from ringmix.simulation import RunConfig, SimState, Strategy  # noqa: E402

OUT = Path(__file__).resolve().parent
META = dict(numpy_version=np.__version__, generator="tests/golden/make_golden.py")

CELL_SEED = harness.cell_seed(1234, Strategy.RAND_PSGD, 64, 0)
SEEDS = [0, 5, 9, 42, 123, 12345, 2**32 - 1, 2**32, CELL_SEED, 2**64 - 1, 3**45]
STEPS = [0, 1, 2, 3, 4, 7, 100, 2**32 - 1, 2**32 + 3, 2**40 + 5]
SIZES = [1, 2, 3, 4, 5, 6, 8, 16, 33, 64, 128, 1000]


def words(v: int) -> list[int]:
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & 0xFFFFFFFF)
        v >>= 32
    return out


def make_perms():
    cases, flat, seed_words, seed_nwords = [], [], [], []
    for n, seed, step in itertools.product(SIZES, SEEDS, STEPS):
        if n == 1000 and step not in (0, 1, 2**32 + 3):
            continue
        p = mixing.permutation_for_step(n, seed, step)
        w = words(seed)
        cases.append((n, step, len(flat)))
        seed_words.append(w + [0] * (4 - len(w)))
        seed_nwords.append(len(w))
        flat.extend(int(x) for x in p)
    cases = np.array(cases, dtype=np.uint64)
    np.savez_compressed(
        OUT / "perms.npz",
        n=cases[:, 0].astype(np.int64), step=cases[:, 1], offset=cases[:, 2].astype(np.int64),
        seed_words=np.array(seed_words, dtype=np.uint32),
        seed_nwords=np.array(seed_nwords, dtype=np.int32),
        perm=np.array(flat, dtype=np.int64), **META)
    print("perms:", len(cases), "cases")


def make_sequential():
    """monte_carlo_consensus pattern: stream(seed, TAG_TRIAL, t), k_max draws."""
    recs = []
    for n, seed, trial, count in [(5, 2, 0, 3), (8, 2, 7, 20), (16, 11, 3, 20),
                                  (64, 2, 0, 5), (128, 2, 999, 4), (3, 0, 1, 9),
                                  (12, 2**40, 2**33, 6)]:
        rng = seeding.stream(seed, seeding.TAG_TRIAL, trial)
        ps = np.stack([mixing.sample_permutation(n, rng) for _ in range(count)])
        recs.append((n, seed, trial, count, ps))
    np.savez_compressed(
        OUT / "sequential.npz",
        meta=np.array([(r[0], r[1], r[2], r[3]) for r in recs], dtype=object),
        **{f"perms_{i}": r[4] for i, r in enumerate(recs)}, **META, allow_pickle=True)
    print("sequential:", len(recs), "streams")


class SynthOracle:
    """Gradient stub (SURVEY §8(d) SynthOracle): returns precomputed columns,
    G[k][:, l], independent of the weights — isolates the mix+SGD arithmetic."""

    def __init__(self, Gs):
        self.Gs = Gs
        self.dimension = next(iter(Gs.values())).shape[0]

    def stochastic_gradient(self, w, batch, shard=None):
        _, _, k, l = batch.sample_seed
        return self.Gs[k][:, l].copy()


def f32(a):
    return a.astype(np.float32).astype(np.float64)


def make_steps():
    """Reference step functions, three consecutive steps, fp32-representable inputs."""
    out = {}
    idx = 0
    specs = []
    for strategy, L, d, mode, lr, seed, k0 in [
        (Strategy.RAND_PSGD, 5, 7, "async", 0.1, 5, 0),
        (Strategy.RAND_PSGD, 8, 64, "sync", 0.01, 42, 0),
        (Strategy.RAND_PSGD, 16, 1000, "async", 0.01, 12345, 3),
        (Strategy.RAND_PSGD, 64, 130, "async", 0.05, CELL_SEED, 2**32 + 1),
        (Strategy.RAND_PSGD, 33, 33, "sync", 0.25, 2**64 - 1, 0),
        (Strategy.RAND_PSGD, 3, 9, "async", 0.1, 7, 0),
        (Strategy.ADPSGD_FIXED, 6, 100, "async", 0.1, 5, 0),
        (Strategy.DPSGD_FIXED, 4, 17, "sync", 0.1, 5, 0),
        (Strategy.DPSGD_FIXED, 3, 5, "sync", 0.1, 5, 0),
        (Strategy.D1D, 6, 100, "async", 0.1, 5, 0),
        (Strategy.D1D, 16, 257, "async", 0.01, 9, 0),
        (Strategy.D1D, 129, 40, "async", 0.01, 9, 0),
        (Strategy.D1D, 1, 10, "async", 0.1, 9, 0),
        (Strategy.SPSGD, 5, 50, "async", 0.1, 5, 0),
    ]:
        rng = np.random.default_rng(1000 + idx)
        nsteps = 3
        if strategy is Strategy.SPSGD:
            W0 = np.tile(f32(rng.standard_normal((d, 1))), (1, L))
        else:
            W0 = f32(rng.standard_normal((d, L)))
        Wp = f32(rng.standard_normal((d, L))) if strategy is not Strategy.SPSGD else W0.copy()
        Gs = {k0 + s: f32(rng.standard_normal((d, L))) for s in range(nsteps)}
        cfg = RunConfig(n_learners=L, iterations=nsteps, lr=lr, batch_size=1, seed=seed,
                        staleness_mode=mode)
        state = SimState(weights=W0.copy(), prev_weights=Wp.copy(), iteration=k0, seed=seed,
                         compute_time_s=np.zeros(L))
        oracle = SynthOracle(Gs)
        step = simulation._STEP_FUNCTIONS[strategy]
        traj = []
        for _ in range(nsteps):
            state = step(state, oracle, cfg)
            traj.append(state.weights.copy())
        out[f"W0_{idx}"] = W0
        out[f"Wprev_{idx}"] = Wp
        out[f"G_{idx}"] = np.stack([Gs[k0 + s] for s in range(nsteps)])
        out[f"traj_{idx}"] = np.stack(traj)
        specs.append((strategy.value, L, d, mode, lr, seed, k0, nsteps))
        idx += 1
    np.savez_compressed(OUT / "steps.npz", specs=np.array(specs, dtype=object), **out, **META,
                        allow_pickle=True)
    print("steps:", idx, "cases")


def make_spectral():
    rec = {}
    Ls = [3, 4, 5, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128]
    rec["L"] = np.array(Ls)
    rec["rho"] = np.array([spectral.second_eigenvalue_ring(L) for L in Ls])
    rec["rho_eig"] = np.array([spectral.spectral_rho(mixing.build_ring_matrix(L)).rho for L in Ls])
    rec["frob_exp_k5"] = np.array([spectral.randomized_frobenius_expectation(L, 5) for L in Ls])
    rec["bound_k5"] = np.array([spectral.randomized_consensus_bound(L, 5) for L in Ls])
    fc = spectral.fixed_consensus_curve(16, 10)
    rec["fixed_curve_16"] = fc.distances
    mc = spectral.monte_carlo_consensus(8, 6, 40, seed=2, norm_kind="frobenius")
    rec["mc8_frob_dist"] = mc.distances
    rec["mc8_frob_half"] = mc.halfwidths
    rec["mc8_frob_sq"] = mc.squared_distances
    mc2 = spectral.monte_carlo_consensus(12, 4, 20, seed=3, norm_kind="spectral")
    rec["mc12_spec_dist"] = mc2.distances
    rec["mc12_spec_half"] = mc2.halfwidths
    ex = spectral.monte_carlo_consensus(5, 1, 2, seed=0, exhaustive=True)
    rec["exh5_dist"] = ex.distances
    rec["exh5_sq"] = ex.squared_distances
    np.savez_compressed(OUT / "spectral.npz", **rec, **META)
    print("spectral: ok")


def make_normals():
    """numpy standard_normal streams the quadratic oracle draws (objectives.py:87-90)."""
    rec = {}
    cases = [((5, 0, 0, 0), 1000), ((12345, 0, 7, 3), 20000), ((2**64 - 1, 0, 2**33, 63), 777),
             ((9, 6), 4096), ((0, 0, 0, 0), 1)]
    for i, (ent, n) in enumerate(cases):
        rec[f"z_{i}"] = np.random.default_rng(np.random.SeedSequence(ent)).standard_normal(n)
        rec[f"ent_{i}"] = np.array([str(e) for e in ent])
    np.savez_compressed(OUT / "normals.npz", **rec, **META)
    print("normals:", len(cases), "streams")


def make_training():
    """Full reference run_training with its own quadratic oracle (the path's callers)."""
    from ringmix.objectives import quadratic_oracle
    from ringmix.simulation import run_training

    rec, specs = {}, []
    for i, (strategy, L, d, iters, lr, mode, cond, noise, seed, warm) in enumerate([
        (Strategy.RAND_PSGD, 8, 40, 6, 0.05, "async", 10.0, 1.0, 3, 0),
        (Strategy.RAND_PSGD, 5, 17, 5, 0.1, "sync", 4.0, 0.5, CELL_SEED, 2),
        (Strategy.ADPSGD_FIXED, 6, 33, 5, 0.05, "async", 10.0, 1.0, 7, 0),
        (Strategy.DPSGD_FIXED, 4, 9, 4, 0.1, "async", 2.0, 2.0, 11, 0),
        (Strategy.D1D, 8, 64, 6, 0.05, "async", 10.0, 1.0, 13, 0),
        (Strategy.SPSGD, 4, 25, 4, 0.05, "async", 3.0, 1.0, 17, 0),
    ]):
        oracle = quadratic_oracle(d, condition_number=cond, noise_scale=noise, seed=seed + 100)
        cfg = RunConfig(n_learners=L, iterations=iters, lr=lr, batch_size=4, seed=seed,
                        staleness_mode=mode, warmup_iters=warm, log_every=2)
        res = run_training(strategy, oracle, cfg)
        rec[f"records_{i}"] = np.array([[r.iteration, r.sim_time_s, r.mean_loss,
                                         r.avg_model_loss, r.consensus_dist, r.rho]
                                        for r in res.records])
        rec[f"W_{i}"] = res.state.weights
        rec[f"optimum_{i}"] = oracle.optimum
        specs.append((strategy.value, L, d, iters, lr, mode, cond, noise, seed, warm,
                      res.diverged))
    np.savez_compressed(OUT / "training.npz", specs=np.array(specs, dtype=object), **rec, **META,
                        allow_pickle=True)
    print("training:", len(specs), "runs")


SWEEP_CFG = dict(learner_counts=(4, 8), iterations=6, trials=2, master_seed=7, lr=0.05,
                 batch_mode="per-learner-fixed", batch_size=4, log_every=2, dimension=24,
                 oracle_seed=3, condition_number=10.0, noise_scale=1.0, straggler_count=1,
                 straggler_factor=3.0)


def make_sweep():
    """The reference's run_sweep artefacts (harness.py:192-234) for a small grid over all
    five strategies: per-cell trace CSVs, summary.csv, aggregate.csv."""
    import shutil
    import tempfile
    from ringmix.config import ExperimentConfig

    cfg = ExperimentConfig(strategies=tuple(Strategy), **SWEEP_CFG)
    dst = OUT / "sweep"
    if dst.exists():
        shutil.rmtree(dst)
    with tempfile.TemporaryDirectory() as tmp:
        harness.run_sweep(cfg, tmp, quiet=True)
        dst.mkdir()
        for f in sorted(Path(tmp).glob("*.csv")):
            shutil.copy(f, dst / f.name)
    print("sweep:", len(list(dst.glob("*.csv"))), "files")


def make_bounds():
    """The reference's verify_bounds (harness.py:283-336) report and rows."""
    rep = harness.verify_bounds(learner_counts=(3, 4, 8, 16, 33), k_max=8, trials=300, seed=5)
    rows = np.array([[r.n_learners, r.rho, r.eig_gap, r.powering_excess, r.mc_fro_ratio,
                      r.mc_spec_ratio] for r in rep.rows])
    np.savez_compressed(OUT / "bounds.npz", rows=rows, render=np.array(rep.render()), **META)
    print("bounds:", len(rep.rows), "rows")


MAKERS = dict(bounds=make_bounds, perms=make_perms, sequential=make_sequential, steps=make_steps,
              spectral=make_spectral, normals=make_normals, training=make_training,
              sweep=make_sweep)

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(MAKERS)):
        MAKERS[name]()

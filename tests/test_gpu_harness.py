"""run_sweep on the GPU vs the reference's own sweep artefacts (tests/golden/sweep/):
same files, same rows, every value (the records reduce in numpy's order for small d), the
files byte for byte, and the device run is byte-stable run to run."""

from __future__ import annotations

import csv
from pathlib import Path

import numpy as np
import pytest

from paper_2002_01119_b200 import harness
from paper_2002_01119_b200.simulation import Strategy

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "sweep"
CFG = harness.SweepConfig(strategies=tuple(Strategy), learner_counts=(4, 8), iterations=6,
                          trials=2, master_seed=7, lr=0.05, batch_mode="per-learner-fixed",
                          batch_size=4, log_every=2, dimension=24, oracle_seed=3,
                          condition_number=10.0, noise_scale=1.0, straggler_count=1,
                          straggler_factor=3.0)


def _rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def test_sweep_matches_reference_artefacts(tmp_path):
    res = harness.run_sweep(CFG, tmp_path / "a", quiet=True)
    assert not res.any_diverged
    ours = sorted(p.name for p in (tmp_path / "a").glob("*.csv"))
    assert ours == sorted(p.name for p in GOLD.glob("*.csv"))
    exact = {"iter", "sim_time_s", "rho", "strategy", "n_learners", "trial", "run_seed",
             "csv_file", "status", "final_iter", "total_sim_time_s", "trials", "completed",
             "median_total_sim_time_s"}
    for name in ours:
        a, b = _rows(tmp_path / "a" / name), _rows(GOLD / name)
        assert len(a) == len(b) and list(a[0]) == list(b[0])
        for ra, rb in zip(a, b):
            for k in ra:
                if k in exact:
                    assert ra[k] == rb[k], (name, k)
                else:
                    np.testing.assert_allclose(float(ra[k]), float(rb[k]), rtol=1e-10,
                                               atol=1e-12, err_msg=f"{name}:{k}")
    # byte-stable: a second run writes the same bytes
    harness.run_sweep(CFG, tmp_path / "b", quiet=True)
    for name in ours:
        assert (tmp_path / "a" / name).read_bytes() == (tmp_path / "b" / name).read_bytes()


def test_verify_bounds_matches_reference_report():
    """BASELINE config 5's caller (harness.py:283-336) with the Monte-Carlo trials on
    the GPU: same rows as the reference's own report (tests/golden/bounds.npz)."""
    z = np.load(GOLD.parent / "bounds.npz")
    rep = harness.verify_bounds(learner_counts=(3, 4, 8, 16, 33), k_max=8, trials=300, seed=5)
    rows = np.array([[r.n_learners, r.rho, r.eig_gap, r.powering_excess, r.mc_fro_ratio,
                      r.mc_spec_ratio] for r in rep.rows])
    ref = z["rows"]
    assert np.array_equal(rows[:, :2], ref[:, :2])
    np.testing.assert_allclose(rows[:, 2:4], ref[:, 2:4], rtol=0, atol=1e-14)
    # the Frobenius ratio is |mean - closed| / (3 se): a difference of nearly equal
    # numbers, so compare it (an O(1) quantity) to an absolute 1e-6
    np.testing.assert_allclose(rows[:, 4:], ref[:, 4:], rtol=1e-6, atol=1e-6)
    assert rep.ok and "overall: PASS" in str(z["render"])
    assert rep.render().splitlines()[:2] == str(z["render"]).splitlines()[:2]


def test_sweep_csvs_are_byte_identical_to_reference(tmp_path):
    """With the records reduced in numpy's order (rm_trace_stats_exact_*, used for
    d <= simulation.TRACE_EXACT_MAX_D) every artefact of the sweep — traces, summary,
    aggregate — is the reference's own file byte for byte (harness.py:115-122)."""
    harness.run_sweep(CFG, tmp_path / "a", quiet=True)
    diff = [p.name for p in sorted(GOLD.glob("*.csv"))
            if (tmp_path / "a" / p.name).read_bytes() != p.read_bytes()]
    assert not diff, diff

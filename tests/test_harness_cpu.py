"""Sweep-artefact formatting and cell seeds vs the reference's own run_sweep output
(tests/golden/sweep/, frozen by tests/golden/make_golden.py sweep).  Host only."""

from __future__ import annotations

import csv
from pathlib import Path

from paper_2002_01119_b200 import harness
from paper_2002_01119_b200.simulation import Strategy, TraceRecord

GOLD = Path(__file__).resolve().parent / "golden" / "sweep"


def _records(path: Path) -> tuple[TraceRecord, ...]:
    with open(path) as f:
        rows = list(csv.DictReader(f))
    return tuple(TraceRecord(int(r["iter"]), float(r["sim_time_s"]), float(r["mean_loss"]),
                             float(r["avg_model_loss"]), float(r["consensus_dist"]),
                             float(r["rho"])) for r in rows)


def _cells() -> tuple[harness.CellResult, ...]:
    with open(GOLD / "summary.csv") as f:
        rows = list(csv.DictReader(f))
    cells = []
    for r in rows:
        recs = _records(GOLD / r["csv_file"])
        cells.append(harness.CellResult(Strategy(r["strategy"]), int(r["n_learners"]),
                                        int(r["trial"]), int(r["run_seed"]), r["csv_file"],
                                        r["status"] == "diverged", recs[-1] if recs else None))
    return tuple(cells)


def test_trace_csv_text_is_byte_identical():
    for f in GOLD.glob("*_trial*.csv"):
        assert harness.trace_csv_text(_records(f)) == f.read_text()


def test_cell_seeds_match_reference():
    for c in _cells():
        assert harness.cell_seed(7, c.strategy, c.n_learners, c.trial) == c.run_seed


def test_summary_and_aggregate_text_are_byte_identical():
    cells = _cells()
    assert harness.summary_csv_text(cells) == (GOLD / "summary.csv").read_text()
    cfg = harness.SweepConfig(strategies=tuple(Strategy), learner_counts=(4, 8), iterations=6,
                              trials=2, master_seed=7, lr=0.05, batch_mode="per-learner-fixed",
                              batch_size=4)
    assert harness.aggregate_csv_text(cfg, cells) == (GOLD / "aggregate.csv").read_text()


def test_cost_model_and_run_config_follow_the_config():
    cfg = harness.SweepConfig(strategies=(Strategy.D1D,), learner_counts=(4,), iterations=3,
                              trials=1, master_seed=7, lr=0.05, batch_mode="global",
                              batch_size=32, straggler_count=1, straggler_factor=3.0)
    cm = harness.make_cost_model(cfg, 4)
    assert cm.compute_scale is not None and list(cm.compute_scale) == [3.0, 1.0, 1.0, 1.0]
    rc = harness.cell_run_config(cfg, Strategy.D1D, 4, 0)
    assert rc.batch_size == 8 and rc.seed == harness.cell_seed(7, Strategy.D1D, 4, 0)

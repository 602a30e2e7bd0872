"""Host-side pieces of bench.py (no GPU): the NVLink traffic model of the
learner-sharded layouts and the weak/strong scaling bookkeeping."""

from __future__ import annotations

import argparse
import importlib.util
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _tables(perms):
    perm = np.array(perms, dtype=np.int64)
    inv = np.argsort(perm, axis=1)
    L = perm.shape[1]
    left = np.array([[inv[s][(perm[s][j] - 1) % L] for j in range(L)] for s in range(len(perm))])
    right = np.array([[inv[s][(perm[s][j] + 1) % L] for j in range(L)] for s in range(len(perm))])
    return perm, inv, left, right


def test_nvlink_traffic_identity_ring():
    b = _bench()
    perm, inv, left, right = _tables([list(range(8))] * 2)
    # pull: rank 0 owns learners 0..3, neighbours 7 and 4 are remote
    pull = b.nvlink_traffic("learner", 8, 10, 4, 2, perm, inv, left[:1], right[:1])
    assert pull == [(2 * 10 * 4, 0), (2 * 10 * 4, 0)]
    # position layout, unchanged order: 2 boundary rows in, no relabel stores
    pos = b.nvlink_traffic("position", 8, 10, 4, 2, perm, inv, left[:1], right[:1])
    assert pos == [(2 * 10 * 4, 0), (2 * 10 * 4, 0)]


def test_nvlink_traffic_reversal_moves_every_row():
    b = _bench()
    perm, inv, left, right = _tables([list(range(8)), list(range(7, -1, -1))])
    pos = b.nvlink_traffic("position", 8, 1, 4, 2, perm, inv, left[:1], right[:1])
    # learner at position x moves to position 7 - x: every output crosses ranks
    assert pos == [(2 * 4, 4 * 4), (2 * 4, 4 * 4)]


def test_nvlink_traffic_position_layout_composes_the_permutations():
    """Slot x of step k holds learner inv_k[x]; its output goes to slot p_{k+1}[inv_k[x]].
    A 3-cycle relabelling (not an involution) tells p_{k+1}[inv_k[.]] from
    inv_{k+1}[p_k[.]]."""
    b = _bench()
    p0 = [1, 2, 0, 3]          # learner l at position p0[l]
    p1 = [0, 1, 2, 3]
    perm, inv, left, right = _tables([p0, p1])
    # 2 ranks: slots {0, 1} and {2, 3}; step 0 slot 0 holds learner 2 (-> slot 2, remote),
    # slot 1 holds learner 0 (-> slot 0, local); slot 2 holds learner 1 (-> slot 1,
    # remote), slot 3 holds learner 3 (local)
    pos = b.nvlink_traffic("position", 4, 1, 4, 2, perm, inv, left[:1], right[:1])
    assert pos == [(2 * 4, 1 * 4), (2 * 4, 1 * 4)]
    expect = np.asarray(p1)[np.asarray(inv[0])]
    assert list(expect) == [2, 0, 1, 3]


def test_weak_scaling_only_for_coordinate_stripes():
    b = _bench()
    a = argparse.Namespace(layout="coord", scaling="weak", dim=100, learners=4,
                           strategy="rand_psgd", d1d_collective="auto", d1d_chunk_cols=0)
    assert b.weak(a, 1) is True and b.total_dim(a, 1) == 100
    assert b.weak(a, 4) is True and b.total_dim(a, 4) == 400
    a.layout = "learner"
    assert b.weak(a, 4) is False and b.total_dim(a, 4) == 100
    assert "weak scaling" not in b.config_dict(a, 4)["parallelism"]


def test_nvlink_traffic_fixed_ring_tables():
    """The fixed ring's tables (left = j - 1, right = j + 1) cross ranks only at the
    two shard boundaries."""
    b = _bench()
    ident = np.tile(np.arange(8, dtype=np.int64), (2, 1))
    left, right = np.roll(ident, 1, axis=1), np.roll(ident, -1, axis=1)
    pull = b.nvlink_traffic("learner", 8, 10, 4, 2, ident, ident, left[:1], right[:1])
    assert pull == [(2 * 10 * 4, 0), (2 * 10 * 4, 0)]


def test_reference_arm_prints_the_contract_line():
    """`bench.py --impl reference` (host only: the oracle port of the reference's numpy
    arithmetic) prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3", "--dim", "4096"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


def test_resolve_picks_the_baseline_config_per_world_size():
    """N = 1: configs[1] (C2) on one GPU; N > 1: configs[2] (C3) learner-sharded in
    ring-position order for RAD, the learner layout for D1D / the fixed ring; an explicit
    coordinate layout keeps C2 stripes with weak scaling."""
    b = _bench()
    a = b.parse([])
    r1 = b.resolve(a, 1)
    assert (r1.learners, r1.dim, r1.layout, r1.config_index) == (64, 25_557_032, "coord", 1)
    r2 = b.resolve(a, 2)
    assert (r2.learners, r2.dim, r2.layout, r2.scaling, r2.config_index) == \
        (128, 43_154_944, "position", "strong", 2)
    d = b.resolve(b.parse(["--strategy", "d1d"]), 4)
    assert (d.layout, d.learners, d.config_index) == ("learner", 64, 3)
    c = b.resolve(b.parse(["--layout", "coord"]), 4)
    assert (c.layout, c.scaling, c.learners) == ("coord", "weak", 64)
    assert b.total_dim(c, 4) == 4 * 25_557_032
    assert "configs[2]" in b.config_dict(r2, 2)["workload"]


def test_self_launch_command(monkeypatch):
    """`--gpus N` without WORLD_SIZE re-runs bench.py under torch.distributed.run with N
    local ranks on 127.0.0.1."""
    import sys
    b = _bench()
    seen = {}
    monkeypatch.setattr(b.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    a = b.parse(["--gpus", "4", "--steps", "7"])
    b.self_launch(a)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]

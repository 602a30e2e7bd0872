"""Host-side logic of the multi-GPU layouts with a real world_size-2 gloo group
(no GPU): ownership, splits, the shard planner restatement, object exchange."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import distributed as D


def test_balanced_split_and_layout():
    assert D.balanced_split(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert D.balanced_split(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    lay = D.ShardLayout(64, 8)
    assert lay.rows(3) == (24, 32)
    assert all(lay.owner(l) == l // 8 for l in range(64))
    assert lay.local_index(27) == 3
    with pytest.raises(ValueError):
        D.balanced_split(4, 0)


def test_coordinate_shards_cover_all_columns():
    d = 25_557_032
    cols = [D.CoordinateShards(d, 8, r).columns for r in range(8)]
    assert cols[0][0] == 0 and cols[-1][1] == d
    assert all(a[1] == b[0] for a, b in zip(cols, cols[1:]))


@pytest.mark.parametrize("L,world", [(64, 8), (16, 2), (128, 8), (10, 3)])
def test_plan_reference_reconstructs_every_neighbourhood(L, world):
    lay = D.ShardLayout(L, world)
    for k in (0, 1, 7):
        p = O.c_permutation(L, 12345, k)
        _, left, right = O.neighbour_tables(p)
        for r in range(world):
            row0, row1 = lay.rows(r)
            Lg = row1 - row0
            rem, tri = D.plan_reference(left, right, row0, Lg)
            assert len(set(rem)) == len(rem) <= 2 * Lg
            assert all(lay.owner(x) != r for x in rem)

            def gid(sx):
                return row0 + sx if sx < Lg else rem[sx - Lg]
            for j, (a, b, c, jj) in enumerate(tri):
                g = row0 + j
                assert jj == j
                ids = [gid(a), gid(b), gid(c)]
                assert ids == sorted({left[g], g, right[g]})  # ascending global order


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = D.exchange_objects({"rank": rank, "blob": bytes([rank]) * 64, "off": 4096 * rank})
        lay = D.ShardLayout(16, world)
        row0, row1 = lay.rows(rank)
        p = O.c_permutation(16, 99, 3)
        _, left, right = O.neighbour_tables(p)
        rem, _ = D.plan_reference(left, right, row0, row1 - row0)
        # every rank's remote requests are served by the owner's rows
        reqs = D.exchange_objects(rem)
        served = sorted(x for r in reqs for x in r if lay.owner(x) == rank)
        q.put((rank, [g["rank"] for g in got], [g["off"] for g in got],
               bytes(got[1 - rank]["blob"]) == bytes([1 - rank]) * 64, served))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_and_plans():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ranks, offs, blob_ok, served in res:
        assert ranks == [0, 1] and offs == [0, 4096] and blob_ok
        for x in served:
            assert D.ShardLayout(16, 2).owner(x) == rank


def test_symmetric_addresses_multicast_or_peer_table(monkeypatch):
    """A symmetric buffer is reached through its multicast address when the handle has one,
    else (or with RINGMIX_SYM_P2P=1) through a table of every rank's address."""
    from paper_2002_01119_b200 import distributed as D

    class H:
        multicast_ptr = 0x7000
        buffer_ptrs = [0x1000, 0x2000, 0x3000]
        offset = 0x40

    mc, tab = D._sym_addresses(H, "cpu")
    assert mc == 0x7040 and tab is None
    monkeypatch.setenv("RINGMIX_SYM_P2P", "1")
    mc, tab = D._sym_addresses(H, "cpu")
    assert mc == 0 and tab.tolist() == [0x1040, 0x2040, 0x3040]
    monkeypatch.delenv("RINGMIX_SYM_P2P")
    H.multicast_ptr = 0
    mc, tab = D._sym_addresses(H, "cpu")
    assert mc == 0 and tab.tolist() == [0x1040, 0x2040, 0x3040]


@pytest.mark.parametrize("L,world", [(8, 1), (16, 2), (64, 4), (64, 8), (128, 2), (24, 3),
                                     (67, 2), (200, 2), (64, 16)])
def test_numpy_order_d1d_layout(L, world, monkeypatch):
    """The numpy-order D1D learner layout (distributed.d1d_numpy_chains / d1d_learners):
    where it applies, rank g holds exactly the learners of numpy's pairwise chains
    [g R, (g + 1) R) (l % 8), in ascending order, every learner on one rank; numpy's pairwise
    tree over the ranks' chain subtrees is then its tree over the eight chains (the restated
    sum below equals numpy's own np.sum bit for bit).  Elsewhere: contiguous blocks."""
    monkeypatch.delenv("RINGMIX_D1D_NUMPY_ORDER", raising=False)
    R = D.d1d_numpy_chains(L, world)
    applies = L % 8 == 0 and 8 <= L <= 128 and world in (1, 2, 4, 8)
    assert (R == 8 // world) if applies else R == 0
    sets = [D.d1d_learners(L, world, g, R) for g in range(world)]
    assert sorted(sum(sets, [])) == list(range(L))
    if not R:
        assert all(s == list(range(s[0], s[-1] + 1)) for s in sets if s)
        return
    for g, s in enumerate(sets):
        assert s == sorted(s) and all(g * R <= l % 8 < (g + 1) * R for l in s)
    rng = np.random.default_rng(L + world)
    x = rng.standard_normal(L) * rng.lognormal(0, 3, L)

    def subtree(vals):          # numpy's tree over consecutive chains
        while len(vals) > 1:
            vals = [vals[i] + vals[i + 1] for i in range(0, len(vals), 2)]
        return vals[0]

    parts = []
    for g in range(world):      # rank g: its chains (sequential over its rows), then the tree
        chains = []
        for q in range(R):
            rows = [l for l in sets[g] if l % 8 == g * R + q]
            acc = x[rows[0]]
            for l in rows[1:]:
                acc = acc + x[l]
            chains.append(acc)
        parts.append(subtree(chains))
    assert subtree(parts) == np.sum(x)       # numpy's pairwise sum of L <= 128 values
    monkeypatch.setenv("RINGMIX_D1D_NUMPY_ORDER", "0")
    assert D.d1d_numpy_chains(L, world) == 0

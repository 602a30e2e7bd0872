"""Readers for the committed golden fixtures (frozen from the reference by
tests/golden/make_golden.py under numpy 2.3.5)."""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from conftest import GOLDEN


def _seed_from_words(words, n) -> int:
    v = 0
    for i in range(int(n) - 1, -1, -1):
        v = (v << 32) | int(words[i])
    return v


@lru_cache(maxsize=None)
def perm_cases():
    z = np.load(GOLDEN / "perms.npz")
    out = []
    n, step, off = z["n"], z["step"], z["offset"]
    sw, sn, flat = z["seed_words"], z["seed_nwords"], z["perm"]
    for i in range(len(n)):
        L = int(n[i])
        out.append((L, _seed_from_words(sw[i], sn[i]), int(step[i]),
                    flat[int(off[i]):int(off[i]) + L]))
    return out


@lru_cache(maxsize=None)
def sequential_cases():
    z = np.load(GOLDEN / "sequential.npz", allow_pickle=True)
    meta = z["meta"]
    return [(int(m[0]), int(m[1]), int(m[2]), int(m[3]), z[f"perms_{i}"])
            for i, m in enumerate(meta)]


@lru_cache(maxsize=None)
def step_cases():
    z = np.load(GOLDEN / "steps.npz", allow_pickle=True)
    out = []
    for i, s in enumerate(z["specs"]):
        strategy, L, d, mode, lr, seed, k0, nsteps = s
        out.append(dict(idx=i, strategy=str(strategy), L=int(L), d=int(d), mode=str(mode),
                        lr=float(lr), seed=int(seed), k0=int(k0), nsteps=int(nsteps),
                        W0=z[f"W0_{i}"], Wprev=z[f"Wprev_{i}"], G=z[f"G_{i}"],
                        traj=z[f"traj_{i}"]))
    return out


@lru_cache(maxsize=None)
def spectral_golden():
    return dict(np.load(GOLDEN / "spectral.npz"))


@lru_cache(maxsize=None)
def normal_cases():
    z = np.load(GOLDEN / "normals.npz")
    out = []
    i = 0
    while f"z_{i}" in z:
        out.append((tuple(int(x) for x in z[f"ent_{i}"]), z[f"z_{i}"]))
        i += 1
    return out


@lru_cache(maxsize=None)
def training_cases():
    z = np.load(GOLDEN / "training.npz", allow_pickle=True)
    out = []
    for i, s in enumerate(z["specs"]):
        strategy, L, d, iters, lr, mode, cond, noise, seed, warm, diverged = s
        out.append(dict(idx=i, strategy=str(strategy), L=int(L), d=int(d), iters=int(iters),
                        lr=float(lr), mode=str(mode), cond=float(cond), noise=float(noise),
                        seed=int(seed), warm=int(warm), diverged=bool(diverged),
                        records=z[f"records_{i}"], W=z[f"W_{i}"], optimum=z[f"optimum_{i}"]))
    return out

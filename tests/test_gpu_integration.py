"""The reference-side ctypes binding shown in INTEGRATION.md, executed as written
(only the library path is made absolute): a maintainer's copy of it must produce
the same steps as the drop-in package and the oracle."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import ringmix_oracle as O
from paper_2002_01119_b200 import _lib, mixing

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _binding():
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2. C-ABI"):text.index("## 3. Multi-GPU")]
    code = "\n".join(re.findall(r"```python\n(.*?)```", sec, flags=re.S))
    code = code.replace('"libringmix_b200.so"', repr(str(_lib.LIB_PATH)))
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def _tables(L, seed, k):
    p = O.c_permutation(L, seed, k)
    _, left, right = O.neighbour_tables(p)
    return left.astype(np.int32), right.astype(np.int32)


def test_host_buffer_binding_matches_oracle():
    b = _binding()
    L, d = 16, 100_003
    rng = np.random.default_rng(3)
    W = rng.standard_normal((L, d)).astype(np.float32)
    G = rng.standard_normal((L, d)).astype(np.float32)
    left, right = _tables(L, 77, 5)
    ws = b["Workspace"](L, chunk_cols=1 << 14)
    out = b["gossip_step_f32"](W, G, 0.05, left, right, ws)
    ref = O.c_ring_mix_sgd(W.T.astype(np.float64), G.T.astype(np.float64), 0.05, left, right)
    assert np.array_equal(out, ref.T.astype(np.float32))
    with pytest.raises(ValueError):
        b["gossip_step_f32"](W[:2], G[:2], 0.05, left[:2], right[:2], ws)   # L < 3


def test_reference_layout_binding_matches_oracle():
    """gossip_step_dL on the reference's (d, L) float64 arrays: ring[p, p] and uniform."""
    b = _binding()
    L, d = 16, 50_001
    rng = np.random.default_rng(4)
    W = rng.standard_normal((d, L))
    G = rng.standard_normal((d, L))
    left, right = _tables(L, 77, 5)
    ws = b["Workspace"](L, chunk_cols=1 << 12, itemsize=8)
    out = b["gossip_step_dL"](W, G, 0.05, left, right, ws)
    assert np.array_equal(out, O.c_ring_mix_sgd(W, G, 0.05, left, right))
    mean = b["gossip_step_dL"](W, G, 0.05, None, None, ws)
    assert np.array_equal(mean, O.c_mean_sgd(W, G, 0.05))
    with pytest.raises(ValueError, match="degenerate ring"):
        b["gossip_step_dL"](W[:, :2].copy(), G[:, :2].copy(), 0.05, left[:2], right[:2], ws)


def test_device_binding_matches_drop_in():
    b = _binding()
    L, d, seed, k = 64, 4099, 1234, 17
    X = mixing.empty_learner_major(L, d, torch.float32, "cuda").normal_()
    G = mixing.empty_learner_major(L, d, torch.float32, "cuda").normal_()
    out = mixing.empty_learner_major(L, d, torch.float32, "cuda")

    class T:
        pass
    t = T()
    bufs = [torch.empty(L, dtype=torch.int32, device="cuda") for _ in range(4)]
    t.perm, t.inv, t.left, t.right = (x.data_ptr() for x in bufs)
    absmax = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    b["rad_step"](X.data_ptr(), G.data_ptr(), out.data_ptr(), L, d, X.stride(0), 0.01, seed, k,
                  t, absmax.data_ptr(), None)
    torch.cuda.synchronize()
    tabs = mixing.permutation_tables(L, seed, k, 1, "cuda")
    lt, rt = tabs.step(k)
    ref = mixing.ring_mix_sgd(X, G, 0.01, lt, rt)
    torch.cuda.synchronize()
    assert torch.equal(bufs[0].long(), tabs.perm[0].long())
    assert torch.equal(out, ref)
    assert absmax.item() > 0


def test_enable_peer_access():
    lib = _lib.load()
    n = torch.cuda.device_count()
    _lib.check(lib.rm_enable_peer_access(n))
    _lib.check(lib.rm_enable_peer_access(n))          # idempotent
    with pytest.raises(ValueError):
        _lib.check(lib.rm_enable_peer_access(0))
    with pytest.raises(ValueError):
        _lib.check(lib.rm_enable_peer_access(n + 1))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_one_process_drives_several_gpus():
    """Kernel attributes (dynamic shared memory opt-in) are per device: the TMA mix and
    trace kernels must work on every GPU one process drives, not only the first."""
    from paper_2002_01119_b200 import simulation
    L, d = 64, 100_003
    outs = []
    for dev in range(torch.cuda.device_count()):
        with torch.cuda.device(dev):
            g = torch.Generator(device=f"cuda:{dev}").manual_seed(1)
            X = mixing.empty_learner_major(L, d, torch.float32, f"cuda:{dev}")
            X.copy_(torch.randn((L, d), generator=g, device=f"cuda:{dev}"))
            tabs = mixing.permutation_tables(L, 5, 0, 1, f"cuda:{dev}")
            lt, rt = tabs.step(0)
            out = mixing.ring_mix_sgd(X, X, 0.1, lt, rt)
            cons = simulation.trace_stats(out.T)[0]
            torch.cuda.synchronize()
            outs.append((out.cpu(), cons.cpu()))
    for o, c in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(c, outs[0][1])

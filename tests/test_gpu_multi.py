"""Real multi-GPU run of the learner-sharded RAD + D1D steps (torchrun, one
process per GPU, NCCL + CUDA IPC); skipped when fewer than 2 GPUs are visible."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("L,d", [(64, 1_000_003), (67, 100_003), (5, 4_099)])
def test_learner_sharded_steps_on_all_visible_gpus(L, d):
    """Balanced and unbalanced learner shards, ragged widths: RAD (pull and position
    layouts, in-kernel step ordering) bit-identical to one GPU; D1D (NCCL, NVLS pipeline,
    fused kernel; fp32 / fp64 / bf16) and the D1D training step with the device oracle
    (ShardedD1DTrainer) bit-identical to one GPU with the numpy-order learner layout, within
    fp64 rounding of the sum otherwise."""
    import os
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           str(ROOT / "tools" / "dist_check.py")]
    env = dict(os.environ, CHK_L=str(L), CHK_D=str(d))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    res = json.loads(line)
    assert res["world"] == n and res["rad_bit_identical"] and res["d1d_ok"], res

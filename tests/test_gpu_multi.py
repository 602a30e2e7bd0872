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
def test_learner_sharded_steps_on_all_visible_gpus():
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           str(ROOT / "tools" / "dist_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    res = json.loads(line)
    assert res["world"] == n and res["rad_bit_identical"] and res["d1d_ok"], res

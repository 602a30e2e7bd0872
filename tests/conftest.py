"""Shared test plumbing.

Markers: `gpu` = needs a CUDA device (run on the B200 box with `-m gpu`).
Without a GPU those tests are skipped so `pytest tests/` stays green here.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

# a cross-rank wait that never completes (a test bug) gives up after 30 s, not 600 s
os.environ.setdefault("RINGMIX_XGPU_TIMEOUT_S", "30")

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)

"""Times the one-pass trace reductions (rm_trace_stats_*, simulation.trace_stats with
exact=False) on the configs' shapes: the compile-time-shaped kernel (default) against the
runtime-L kernel (RINGMIX_TRACE_RUNTIME_L=1), checks they agree to fp64 rounding, and
prints one JSON line per case with GB/s (algorithmic bytes: W once + lam/w* once) and the
fraction of MEASURED_PEAKS.json's HBM copy bandwidth.  Also times the exact-order kernel
(rm_trace_stats_exact_*) at small d.

  python tools/bench_trace.py [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2002_01119_b200 import mixing, objectives, simulation  # noqa: E402


def _peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6552.0


def _time(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    peak = _peak()
    cases = [(16, 1 << 20, torch.float32), (64, 25_557_032, torch.float32),
             (128, 43_154_944, torch.float32), (64, 25_557_032, torch.float64),
             (64, 25_557_032, torch.bfloat16), (128, 4_000_037, torch.float32),
             (8, 8_000_001, torch.float64)]
    for L, d, dt in cases:
        oracle = objectives.quadratic_oracle(d, condition_number=7.0, noise_scale=0.0, seed=1)
        X = mixing.empty_learner_major(L, d, dt, "cuda")
        X.normal_()
        res = {}
        for mode in ("tile", "runtime_l"):
            if mode == "runtime_l":
                os.environ["RINGMIX_TRACE_RUNTIME_L"] = "1"
            else:
                os.environ.pop("RINGMIX_TRACE_RUNTIME_L", None)
            out = simulation.trace_stats(X.T, oracle, exact=False)
            ms = _time(lambda: simulation.trace_stats(X.T, oracle, exact=False), args.reps)
            res[mode] = (ms, [o.clone() for o in out])
        os.environ.pop("RINGMIX_TRACE_RUNTIME_L", None)
        agree = all(torch.allclose(a, b, rtol=1e-12, atol=0)
                    for a, b in zip(res["tile"][1], res["runtime_l"][1]))
        nbytes = L * d * X.element_size() + 16 * d
        line = {"L": L, "d": d, "dtype": str(dt).split(".")[-1], "agree_rtol_1e-12": agree,
                "bytes": nbytes}
        for mode, (ms, _) in res.items():
            gbs = nbytes / ms / 1e6
            line[mode] = {"ms": round(ms, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 3)}
        print(json.dumps(line), flush=True)
        del X
        torch.cuda.empty_cache()
    for L, d in [(4, 24), (64, 1 << 16), (16, 1 << 20)]:
        oracle = objectives.quadratic_oracle(d, condition_number=7.0, noise_scale=0.0, seed=1)
        X = mixing.empty_learner_major(L, d, torch.float64, "cuda").normal_()
        ms = _time(lambda: simulation.trace_stats(X.T, oracle, exact=True), 5)
        print(json.dumps({"exact_order": True, "L": L, "d": d, "ms": round(ms, 4)}), flush=True)


if __name__ == "__main__":
    main()

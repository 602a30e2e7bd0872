#!/usr/bin/env python
"""Benchmark: learner-params mixed per second for the fused RAD-PSGD mix+SGD step.

Contract (task README / DESIGN.md §6):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
prints ONE JSON line on rank 0.

* A step = one pass of the hot path over one batch: the device permutation
  tables for step k (generated a block of 64 future steps per launch) and the
  fused gossip-mix + SGD kernel over all learners (W' = ring[p,p]-mix(W) - lr G),
  with the fused divergence epilogue.  W rotates between two HBM buffers.
* N = 1 workload: BASELINE.json configs[1] — RAD-PSGD, 64 learners x 25,557,032
  fp32 params (ResNet-50-sized flat vectors), synthetic N(0,1) weights and
  gradients, lr = 0.01.  3 x 6.54 GB buffers >> 126 MB L2, so no L2 flush.
* N > 1 (torchrun, one process per GPU): coordinate-sharded layout — every
  rank holds all 64 learners for its own 25,557,032-column stripe (rows of W
  are independent) and derives the same permutation from the
  shared seed, so there is no data-path collective: weak scaling.
  (`--layout learner` runs the learner-sharded NVLink path instead.)
* `value`: whole-job learner-params / s, device time (CUDA events), max over ranks.
* `e2e`: the same step through the public host-buffer API
  (mixing.ring_mix_sgd_host -> rm_ring_mix_sgd_host_f32): W, G in pinned host
  memory, H2D + kernel + D2H pipelined, timed on the device per step.
* `roofline`: the mix kernel's algorithmic bytes (12 B per learner-param:
  read W, read G, write W') / its CUDA-event duration vs measured HBM GB/s.
* `cpu_baseline`: the oracle port of the reference's arithmetic
  (numpy W @ T - lr G, fp64, (d, L) C-order) on a bounded sample, host cores.
* `--impl reference`: that same CPU path as the timed arm (the reference is a
  pure-Python/numpy package; its CPU path is the baseline).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "learner-params mixed/sec"
UNIT = "learner-params/s"
L_DEFAULT = 64
D_DEFAULT = 25_557_032
LR = 0.01
SEED = 12345
BYTES_PER_PARAM = {"float32": 12, "bfloat16": 6, "float64": 24}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--learners", type=int, default=L_DEFAULT)
    ap.add_argument("--dim", type=int, default=D_DEFAULT)
    ap.add_argument("--dtype", choices=["float32", "bfloat16", "float64"], default="float32")
    ap.add_argument("--strategy", choices=["rand_psgd", "adpsgd_fixed", "d1d"],
                    default="rand_psgd")
    ap.add_argument("--layout", choices=["coord", "learner"], default="coord")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ----------------------------------------------------------------------------
# environment helpers
# ----------------------------------------------------------------------------

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            z = json.loads(p.read_text())
            return float(z["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        z = json.loads(p.read_text())
        ent = z.get(kernel_key)
        if ent is None:
            return None
        return float(ent["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[tuple[float, list[str]]] = []
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self._th = threading.Thread(target=self._read, daemon=True)
        self._th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, begin: bool):
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for (t, r) in self.lines
                if self.t0 is not None and self.t0 - 0.06 <= t <= (self.t1 or t) + 0.06]
        if not rows:
            rows = [r for (_, r) in self.lines]
        if not rows:
            return None
        sm = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        mx = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------
# CPU baseline (oracle port of the reference's arithmetic)
# ----------------------------------------------------------------------------

def cpu_reference_step_fn(L: int, d_sample: int, uniform: bool):
    """The reference's step arithmetic on a (d_sample, L) fp64 C-order sample:
    apply_mixing(W, T) - lr * G (simulation.py:267, mixing.py:143-162), restated
    by the oracle (oracle/ringmix_oracle.py numpy_gossip_step)."""
    from oracle import ringmix_oracle as O

    rng = np.random.default_rng(0)
    W = rng.standard_normal((d_sample, L))
    G = rng.standard_normal((d_sample, L))
    state = {"k": 0}

    def step():
        k = state["k"]
        p = None if uniform else O.c_permutation(L, SEED, k)
        O.numpy_gossip_step(W, G, LR, perm=p, uniform=uniform)
        state["k"] = k + 1

    return step


def cpu_baseline(L: int, uniform: bool, seconds: float):
    cores = os.cpu_count() or 1
    d_sample = 1 << 20
    step = cpu_reference_step_fn(L, d_sample, uniform)
    step()  # warm
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 3:
        t = time.perf_counter()
        step()
        times.append(time.perf_counter() - t)
        if len(times) >= 50:
            break
    med = statistics.median(times)
    return {"value": L * d_sample / med, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"numpy fp64 apply_mixing(W,T) - lr*G on a (d=1,048,576 x L={L}) C-order "
                       f"sample, OpenBLAS threads={os.environ.get('OPENBLAS_NUM_THREADS', cores)}, "
                       f"median of {len(times)} steps ({sum(times):.1f} s)")}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    L = args.learners
    uniform = args.strategy == "d1d"
    d_sample = 1 << 20
    step = cpu_reference_step_fn(L, d_sample, uniform)
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        step()
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = L * d_sample * args.steps / total
    cores = os.cpu_count() or 1
    sample = (f"numpy fp64 apply_mixing(W,T) - lr*G (oracle port of simulation.py:267), "
              f"(d=1,048,576 x L={L}) C-order sample per step, all {cores} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0,1) weights and gradients",
        "config": config_dict(args, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(args, ws):
    return {"workload": f"{args.strategy} mix+SGD step, {args.learners} learners x "
                        f"{args.dim} params/learner ({'ResNet-50-sized' if args.dim == D_DEFAULT else 'custom'}"
                        f"), BASELINE.json configs[1]",
            "learners": args.learners, "params_per_learner": args.dim,
            "strategy": args.strategy, "lr": LR, "perm_seed": SEED,
            "layout": args.layout if ws > 1 else "single-gpu",
            "parallelism": f"{args.layout}-sharded x{ws}" if ws > 1 else "1 GPU",
            "l2": "inputs (3 x L x d x 4 B) far larger than the 126 MB L2; no flush needed"}


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2002_01119_b200 import _lib, mixing

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    dtype = {"float32": torch.float32, "bfloat16": torch.bfloat16,
             "float64": torch.float64}[args.dtype]
    L, d = args.learners, args.dim
    uniform = args.strategy == "d1d"

    # synthetic inputs, resident in HBM before the timed region
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    Wa = mixing.empty_learner_major(L, d, dtype, dev)
    Wb = mixing.empty_learner_major(L, d, dtype, dev)
    G = mixing.empty_learner_major(L, d, dtype, dev)
    for X in (Wa, G):
        for r in range(L):
            X[r].copy_(torch.randn(d, generator=gen, device=dev, dtype=torch.float32).to(dtype))
    amax = torch.zeros(args.warmup + args.steps, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    lib = _lib.load()
    sfx = mixing._suffix(Wa)
    ring_fn = getattr(lib, f"rm_ring_mix_sgd_{sfx}")
    mean_fn = getattr(lib, f"rm_mean_sgd_{sfx}")
    words = __import__("paper_2002_01119_b200.seeding", fromlist=["x"]).entropy_words(SEED, 1)
    block = 64
    tabs = [torch.empty((block, L), dtype=torch.int32, device=dev) for _ in range(4)]
    sptr = stream.cuda_stream
    if args.strategy == "adpsgd_fixed":
        fl, fr = (t.contiguous() for t in
                  __import__("paper_2002_01119_b200.simulation", fromlist=["x"])
                  .fixed_ring_tables(L, dev))
    launches = {"perm": 0, "mix": 0}
    tab0 = {"k": None}   # first step covered by the current table block

    def step(k, bufs, ev_pair=None):
        src, dst = bufs
        if args.strategy == "rand_psgd" and (tab0["k"] is None or k >= tab0["k"] + block):
            # one launch generates the tables of the next `block` steps
            _lib.check(lib.rm_perm_tables(words.ctypes.data, len(words), k, block, L,
                                          *(t.data_ptr() for t in tabs), sptr))
            tab0["k"] = k
            launches["perm"] += 1
        if ev_pair is not None:
            ev_pair[0].record(stream)
        if uniform:
            rc = mean_fn(src.data_ptr(), G.data_ptr(), dst.data_ptr(), L, d, src.stride(0),
                         G.stride(0), dst.stride(0), LR, amax[k].data_ptr(), sptr)
        else:
            if args.strategy == "rand_psgd":
                lp = tabs[2][k - tab0["k"]].data_ptr()
                rp = tabs[3][k - tab0["k"]].data_ptr()
            else:
                lp, rp = fl.data_ptr(), fr.data_ptr()
            rc = ring_fn(src.data_ptr(), G.data_ptr(), dst.data_ptr(), lp, rp, L, d,
                         src.stride(0), G.stride(0), dst.stride(0), LR, amax[k].data_ptr(), sptr)
        if ev_pair is not None:
            ev_pair[1].record(stream)
        launches["mix"] += 1
        _lib.check(rc, "mix")

    bufs = [Wa, Wb]
    k = 0
    for _ in range(args.warmup):
        step(k, (bufs[0], bufs[1]))
        bufs.reverse()
        k += 1
    torch.cuda.synchronize()

    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_start, t_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = {"perm": 0, "mix": 0}
    tab0["k"] = None   # the timed region generates its own tables
    if clocks:
        clocks.mark(True)
    t_start.record(stream)
    for i in range(args.steps):
        step(k, (bufs[0], bufs[1]), kev[i])
        bufs.reverse()
        k += 1
    t_stop.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.mark(False)
    if ws > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_stop)
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    # divergence flags of every step, checked after the timed region
    bits = amax.cpu().numpy().view(np.float64)
    if not np.all(np.isfinite(bits)):
        raise RuntimeError("non-finite weights in the benchmark run")
    if ws > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    clock_info = clocks.stop() if clocks else None

    params_per_step = L * d * ws
    value = params_per_step * args.steps / (elapsed_ms / 1e3)
    kern_avg_s = statistics.mean(kern_ms) / 1e3
    bpp = BYTES_PER_PARAM[args.dtype]
    algo_bytes = bpp * L * d
    peak, peak_src = measured_peaks()
    achieved = algo_bytes / kern_avg_s / 1e9
    key = f"mix_{args.strategy}_{args.dtype}_L{L}_d{d}"
    traffic = ncu_traffic(key)

    # end-to-end through the public host-buffer API
    e2e = None
    if not args.no_e2e and rank == 0 and args.dtype == "float32" and not uniform:
        e2e = run_e2e(args, torch, mixing, dev)
    if ws > 1:
        dist.barrier()

    cpu = None
    if rank == 0 and not args.no_cpu:
        del Wa, Wb, G
        cpu = cpu_baseline(L, uniform, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"float32": "f32", "bfloat16": "bf16", "float64": "f64"}[args.dtype],
            "data": "synthetic: N(0,1) weights and gradients generated on device (torch "
                    "Generator), permutations from the device generator (seed 12345)",
            "config": config_dict(args, ws),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"mix_tma_kernel ({args.strategy}, {args.dtype})",
                         "algorithmic_bytes_per_launch": algo_bytes,
                         "avg_launch_ms": kern_avg_s * 1e3, "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches["perm"] + launches["mix"],
            "gpu_launches_detail": dict(launches),
            "clocks": clock_info,
            "hbm_gbs_step": algo_bytes / (elapsed_ms / args.steps / 1e3) / 1e9,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_e2e(args, torch, mixing, dev):
    """Step through the host-buffer API (W, G pinned host -> W' host)."""
    L, d = args.learners, args.dim
    Wh = torch.empty((L, d), dtype=torch.float32, pin_memory=True)
    Gh = torch.empty((L, d), dtype=torch.float32, pin_memory=True)
    Oh = torch.empty((L, d), dtype=torch.float32, pin_memory=True)
    g = torch.Generator().manual_seed(7)
    Wh.normal_(generator=g)
    Gh.normal_(generator=g)
    ws_buf = mixing.host_workspace(L, 1 << 20, dev)
    from paper_2002_01119_b200 import mixing as M
    tabs = M.permutation_tables(L, SEED, 0, args.e2e_steps + 1, dev)
    left = tabs.left.cpu()
    right = tabs.right.cpu()
    stream = torch.cuda.current_stream()
    # warm-up call
    M.ring_mix_sgd_host(Wh, Gh, LR, left[0], right[0], out_host=Oh, workspace=ws_buf, sync=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    src, dst = Wh, Oh
    torch.cuda.synchronize()
    a.record(stream)
    for k in range(args.e2e_steps):
        M.ring_mix_sgd_host(src, Gh, LR, left[k], right[k], out_host=dst, workspace=ws_buf,
                            sync=False)
        src, dst = dst, src
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.e2e_steps
    return {"value": L * d / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": 2 * L * d * 4 + 2 * L * 4, "d2h_bytes_per_step": L * d * 4,
            "ms_per_step": ms, "steps": args.e2e_steps,
            "path": "mixing.ring_mix_sgd_host -> rm_ring_mix_sgd_host_f32 (pinned host W, G; "
                    "chunked H2D || kernel || D2H)"}


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

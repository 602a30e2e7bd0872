#!/usr/bin/env python
"""Benchmark: learner-params mixed per second for the fused RAD-PSGD mix+SGD step.

Contract (task README / DESIGN.md §6):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
prints ONE JSON line on rank 0.  `--gpus N` without torchrun launches N ranks itself
(torch.distributed.run, 127.0.0.1) and checks that WORLD_SIZE == N.

* A step = one pass of the hot path over one batch: the device permutation tables
  for step k (a block of 64 future steps per launch) and the fused gossip-mix + SGD
  kernel over all learners (W' = ring[p,p]-mix(W) - lr G) with the fused divergence
  epilogue.  W rotates between two HBM buffers.
* N = 1: BASELINE.json configs[1] — RAD-PSGD, 64 learners x 25,557,032 fp32 params
  (ResNet-50-sized flat vectors), synthetic N(0,1) weights and gradients, lr = 0.01.
  `extras` time the other BASELINE configs on the same GPU: `c1_demo` (configs[0],
  16 x 2^20, CUDA-graph replay), `c2_adpsgd_fixed` (configs[1]'s fixed ring), `c4_d1d`
  (configs[3], the D1D mean step) and `c3_single_gpu` (configs[2], 128 x 43,154,944:
  the strong-scaling reference point of the N > 1 runs).
* N > 1 (one process per GPU): strong scaling of BASELINE.json configs[2] — RAD-PSGD,
  128 learners x 43,154,944 fp32 (LSTM acoustic model), learners sharded over the
  ranks (north-star (d)) in ring-POSITION order (`--layout position`, the default):
  each step mixes positions locally (2 boundary rows pulled over NVLink) and stores
  every output straight into its learner's next-step slot on whichever GPU owns it;
  consecutive steps order themselves inside the kernels (no collective).
  `extras.learner_pull` times the learner-ordered pull layout on the same problem
  and `extras.coord_weak` the zero-communication coordinate stripes (every rank a
  64 x 25,557,032 stripe, weak scaling).  D1D (`--strategy d1d`, and `extras.c4_d1d_sharded`
  on configs[3]) shards learners with the fused partial-sum / cross-GPU-reduce / apply kernel;
  `extras.c2_adpsgd_fixed_sharded` is configs[1]'s fixed ring with learners sharded (only the
  two ring-boundary rows per rank cross GPUs); `extras.c4_d1d_training_sharded` times
  configs[3]'s D1D training step with the device oracle — the global average beside the
  gradient generator (north-star (c)) against the serial order.
* `value`: whole-job learner-params / s, device time (CUDA events), max over ranks.
* `e2e`: the same step through the public API with the step's inputs and results
  crossing PCIe every step: N = 1 host buffers in and out (W, G -> W',
  mixing.ring_mix_sgd_host); sharded layouts W resident, every rank's G H2D and
  max|W'| D2H.
* `roofline`: the mix kernel's algorithmic HBM bytes (12 B per learner-param) / its
  CUDA-event duration vs the measured HBM GB/s.
* `nvlink` (N > 1): NVML NVLink byte counters of every GPU over the timed region
  (busiest rank), against 900 GB/s per direction and the measured peer peaks; the
  traffic model is reported beside it.
* `cpu_baseline`: the oracle port of the reference's arithmetic
  (numpy W @ T - lr G, fp64, (d, L) C-order) on a bounded sample, host cores.
* `--impl reference`: that same CPU path as the timed arm (the reference is a
  pure-Python/numpy package; its CPU path is the baseline).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

# The CPU legs (cpu_baseline, --impl reference) run on rank 0 with every host
# core; torchrun exports OMP_NUM_THREADS=1 for multi-process jobs, which
# OpenBLAS would otherwise honour at import.
if os.environ.get("RANK", "0") == "0":
    os.environ["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "learner-params mixed/sec"
UNIT = "learner-params/s"
C1 = (16, 1 << 20)             # BASELINE.json configs[0] (the reference's demo scale)
C2 = (64, 25_557_032)          # BASELINE.json configs[1] (and configs[3], D1D)
C3 = (128, 43_154_944)         # BASELINE.json configs[2]
LR = 0.01
SEED = 12345
BYTES_PER_PARAM = {"float32": 12, "bfloat16": 6, "float64": 24}
NVLINK_NOMINAL_GBS = 900.0     # NVLink 5, per direction per GPU


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--learners", type=int, default=None,
                    help="default: the BASELINE config of the run (64, or 128 at N > 1)")
    ap.add_argument("--dim", type=int, default=None)
    ap.add_argument("--dtype", choices=["float32", "bfloat16", "float64"], default="float32")
    ap.add_argument("--strategy", choices=["rand_psgd", "adpsgd_fixed", "d1d"],
                    default="rand_psgd")
    ap.add_argument("--layout", choices=["auto", "coord", "learner", "position"],
                    default="auto", help="N > 1: auto = position (RAD) / learner (fixed "
                                         "ring, D1D)")
    ap.add_argument("--scaling", choices=["auto", "weak", "strong"], default="auto",
                    help="coord layout at N > 1: weak = every rank owns a full-width "
                         "(L x dim) column stripe of an L x (N*dim) problem; strong = the "
                         "L x dim problem split N ways")
    ap.add_argument("--d1d-collective", choices=["auto", "fused", "nvls", "nccl"],
                    default="auto")
    ap.add_argument("--d1d-chunk-cols", type=int, default=1 << 22,
                    help="learner-sharded D1D pipeline chunk (columns); 0 = one chunk")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--rewarm-seconds", type=float, default=0.4,
                    help="untimed steps right before the timed region (after the clock "
                         "sampler started) so the GPU is at its load clocks")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="capture the K timed steps (perm tables + mix launches) in one CUDA "
                         "graph and time its replay; auto = on for one-GPU problems under "
                         "1 GB per step (launch-bound sizes such as configs[0])")
    ap.add_argument("--event-every", type=int, default=4,
                    help="bracket every N-th mix launch with CUDA events (roofline timing)")
    return ap.parse_args(argv)


# ----------------------------------------------------------------------------
# configuration
# ----------------------------------------------------------------------------

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def resolve(args, ws):
    """Concrete layout / scaling / (L, d) / BASELINE config index of this run."""
    r = argparse.Namespace(**vars(args))
    if ws == 1:
        r.layout = "coord"            # the whole problem on one GPU
    elif args.layout == "auto":
        r.layout = "position" if args.strategy == "rand_psgd" else "learner"
    if args.scaling == "auto":
        r.scaling = "weak" if (ws > 1 and r.layout == "coord") else "strong"
    sharded = ws > 1 and r.layout in ("learner", "position")
    big = sharded and args.strategy == "rand_psgd"
    L, d = C3 if big else C2
    r.learners = args.learners if args.learners is not None else L
    r.dim = args.dim if args.dim is not None else d
    r.config_index = 2 if big else (3 if args.strategy == "d1d" else 1)
    return r


def weak(args, ws):
    """Weak scaling: coordinate stripes of fixed width per rank (no data-path collective)."""
    return args.layout == "coord" and args.scaling == "weak"


def total_dim(args, ws):
    return args.dim * ws if weak(args, ws) else args.dim


def config_name(L, d):
    return {C1: "reference CPU demo scale", C2: "ResNet-50-sized",
            C3: "LSTM-acoustic-model-sized"}.get((L, d), "custom")


def config_dict(args, ws):
    idx = getattr(args, "config_index", 1)
    return {"workload": f"{args.strategy} mix+SGD step, {args.learners} learners x "
                        f"{args.dim} params/learner ({config_name(args.learners, args.dim)}), "
                        f"BASELINE.json configs[{idx}]",
            "learners": args.learners, "params_per_learner": args.dim,
            "strategy": args.strategy, "lr": LR, "perm_seed": SEED,
            "layout": args.layout if ws > 1 else "single-gpu",
            "parallelism": ((f"coord-sharded over {ws} GPUs (weak scaling: every rank owns a "
                             f"{args.learners} x {args.dim} column stripe of the "
                             f"{args.learners} x {args.dim * ws} problem; shared-seed "
                             f"permutations, no data-path collective)") if weak(args, ws) else
                            (f"{args.layout}-sharded over {ws} GPUs (strong scaling: the whole "
                             f"{args.learners} x {args.dim} problem)")) if ws > 1 else "1 GPU",
            "l2": "inputs (3 x L x d x 4 B) far larger than the 126 MB L2; no flush needed",
            **({"d1d_collective": args.d1d_collective, "d1d_chunk_cols": args.d1d_chunk_cols}
               if ws > 1 and args.strategy == "d1d" and args.layout == "learner" else {})}


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
    apply_mixing(W, T) - lr * G (simulation.py:267, mixing.py:106-125), restated
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


def host_threads():
    """Thread count of the CPU legs (OpenBLAS set to every core at import, rank 0)."""
    return int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))


def cpu_baseline(L: int, uniform: bool, seconds: float):
    cores = host_threads()
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
                       f"sample, OpenBLAS threads={cores}, "
                       f"median of {len(times)} steps ({sum(times):.1f} s)")}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    n = max(ws, args.gpus)
    cfg = resolve(args, n)
    L = cfg.learners
    uniform = args.strategy == "d1d"
    d_sample = 1 << 20
    cores = host_threads()
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
    sample = (f"numpy fp64 apply_mixing(W,T) - lr*G (oracle port of simulation.py:267), "
              f"(d=1,048,576 x L={L}) C-order sample per step, all {cores} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak" if weak(cfg, n) else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0,1) weights and gradients",
        "config": config_dict(cfg, n),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# NVLink: measured peaks, counters, traffic model
# ----------------------------------------------------------------------------

def p2p_peaks():
    p = ROOT / "profiles" / "p2p_peaks.json"
    try:
        z = json.loads(p.read_text())
        return float(z["peer_read_gbs"]), float(z["peer_write_gbs"]), z["source"]
    except Exception:
        return NVLINK_NOMINAL_GBS, NVLINK_NOMINAL_GBS, "NVLink 5 nominal per direction"


def nvlink_counters(local):
    try:
        sys.path.insert(0, str(ROOT / "tools"))
        from nvlink_counters import NvlinkCounters
        c = NvlinkCounters(local)
        return c if c.ok else None
    except Exception:
        return None


def nvlink_traffic(layout, L, d, esz, ws, perm, inv, left, right):
    """Per-rank NVLink bytes per step of the learner-sharded RAD layouts, averaged over
    the timed steps (host numpy on the device-generated tables; rows s = step k,
    perm/inv have one extra row for step k+1).  Returns [(read, write)] per rank."""
    from paper_2002_01119_b200.distributed import balanced_split
    bounds = balanced_split(L, ws)
    nsteps = left.shape[0]
    out = []
    for b, e in bounds:
        rd = wr = 0
        for s in range(nsteps):
            if layout == "learner":      # pull: distinct remote neighbour rows
                nb = set(left[s, b:e].tolist()) | set(right[s, b:e].tolist())
                rd += sum(1 for x in nb if not b <= x < e)
            else:                        # position: 2 boundary rows in, relabel stores out
                rd += 2 if ws > 1 else 0
                # slot x holds learner inv_k[x]; its output goes to slot p_{k+1}[inv_k[x]]
                nxt = perm[s + 1][inv[s, b:e]]
                wr += int(((nxt < b) | (nxt >= e)).sum())
        out.append((rd * d * esz / nsteps, wr * d * esz / nsteps))
    return out


def host_pinned_budget() -> int:
    """Bytes of pinned host memory the whole job may use for the e2e variants (a
    quarter of the host's available RAM)."""
    try:
        import psutil
        return int(psutil.virtual_memory().available) // 4
    except Exception:
        return 32 << 30


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

class Workload:
    """One benchmark step for a layout: permutation tables (a block of 64 future steps
    per launch) + the fused mix launch(es) for this rank's share.  `spec`: layout,
    learners, dim, scaling, strategy, dtype, d1d options."""

    def __init__(self, spec, torch, dev, ws, rank, nsteps):
        from paper_2002_01119_b200 import _lib, distributed as D, mixing, seeding, simulation

        self.torch, self._lib, self.mixing = torch, _lib, mixing
        self.spec, self.dev, self.ws, self.rank = spec, dev, ws, rank
        dtype = {"float32": torch.float32, "bfloat16": torch.bfloat16,
                 "float64": torch.float64}[spec.dtype]
        L, d = spec.learners, spec.dim
        self.L, self.d = L, d
        self.layout = "single" if ws == 1 else spec.layout
        self.uniform = spec.strategy == "d1d"
        gen = torch.Generator(device=dev).manual_seed(1000 + rank)

        def fill(X):
            for r in range(X.shape[0]):
                X[r].copy_(torch.randn(X.shape[1], generator=gen, device=dev,
                                       dtype=torch.float32).to(dtype))
            return X

        def synth(rows, cols):
            return fill(mixing.empty_learner_major(rows, cols, dtype, dev))

        self.sharded = None
        if self.layout in ("single", "coord"):
            if self.layout == "coord":
                cols = d if spec.scaling == "weak" else D.CoordinateShards(d, ws, rank).width
            else:
                cols = d
            self.rows, self.cols = L, cols
            self.W = [synth(L, cols), mixing.empty_learner_major(L, cols, dtype, dev)]
            self.G = synth(L, cols)
        elif self.uniform:
            lay = D.ShardLayout(L, ws)
            b, e = lay.rows(rank)
            self.rows, self.cols = e - b, d
            self.W = [synth(e - b, d), mixing.empty_learner_major(e - b, d, dtype, dev)]
            self.d1d = None
            if spec.d1d_collective in ("auto", "fused"):
                try:
                    self.d1d = D.LearnerShardedD1DFused(L, d, e - b, dev)
                    self.d1d_kind = "fused" + ("" if self.d1d.multicast else "-p2p")
                except Exception:
                    if spec.d1d_collective == "fused":
                        raise
            if self.d1d is None and spec.d1d_collective in ("auto", "nvls"):
                try:
                    self.d1d = D.LearnerShardedD1DNVLS(
                        L, d, e - b, dev, chunk_cols=spec.d1d_chunk_cols or None)
                    self.d1d_kind = "nvls"
                except Exception:
                    if spec.d1d_collective == "nvls":
                        raise
            if self.d1d is None:
                self.d1d = D.LearnerShardedD1D(L, d, e - b, dev)
                self.d1d_kind = "nccl"
            self.G = synth(self.rows, d)
        else:
            if self.layout == "position":
                self.sharded = D.LearnerShardedRingPos(L, d, dtype)
            else:
                self.sharded = D.LearnerShardedRing(
                    L, d, dtype, fixed_ring=spec.strategy == "adpsgd_fixed")
            self.rows, self.cols = self.sharded.Lg, d
            fill(self.sharded.W[0])
            # the initial rows were written outside the step kernels: every rank's
            # first step must wait for every rank's writes
            self.sharded.publish()
            self.G = synth(self.rows, d)
            self.ident = torch.arange(L, dtype=torch.int32, device=dev)
        self.local_params = self.rows * self.cols
        self.amax = torch.zeros(nsteps + 1, dtype=torch.int64, device=dev)
        self.lib = _lib.load()
        sfx = mixing._suffix(self.G)
        self.ring_fn = getattr(self.lib, f"rm_ring_mix_sgd_{sfx}")
        self.mean_fn = getattr(self.lib, f"rm_mean_sgd_{sfx}")
        self.words = seeding.entropy_words(SEED, 1)
        self.block = 64
        # block + 1 rows: the position layout also needs step k+1's permutation
        self.tabs = [torch.empty((self.block + 1, L), dtype=torch.int32, device=dev)
                     for _ in range(4)]
        if spec.strategy == "adpsgd_fixed":
            self.fixed = tuple(t.contiguous() for t in simulation.fixed_ring_tables(L, dev))
        self.tab0 = None
        self.launches = {"perm": 0, "mix": 0, "barrier_allreduce": 0}
        self.cur = 0

    def reset_tables(self):
        self.tab0 = None

    def step(self, k, ev_pair=None, G=None):
        torch, _lib = self.torch, self._lib
        stream = torch.cuda.current_stream()
        sptr = stream.cuda_stream
        L = self.L
        G = self.G if G is None else G
        strat = self.spec.strategy
        if strat == "rand_psgd" and (self.tab0 is None or k >= self.tab0 + self.block):
            _lib.check(self.lib.rm_perm_tables(self.words.ctypes.data, len(self.words), k,
                                               self.block + 1, L,
                                               *(t.data_ptr() for t in self.tabs), sptr))
            self.tab0 = k
            self.launches["perm"] += 1
        if strat == "rand_psgd":
            lt, rt = self.tabs[2][k - self.tab0], self.tabs[3][k - self.tab0]
        elif strat == "adpsgd_fixed":
            lt, rt = self.fixed
        if ev_pair is not None:
            ev_pair[0].record(stream)
        am = self.amax[k].data_ptr()
        if self.layout == "position":
            if strat == "rand_psgd":
                ik, pn = self.tabs[1][k - self.tab0], self.tabs[0][k + 1 - self.tab0]
            else:
                ik = pn = self.ident
            self.sharded.step(ik, pn, G, LR, self.amax[k], barrier=False)
        elif self.layout == "learner":
            if self.uniform:
                src, dst = self.W[self.cur], self.W[1 - self.cur]
                self.d1d.step(src, G, LR, dst, self.amax[k])
                self.cur = 1 - self.cur
            else:
                self.sharded.step(lt, rt, G, LR, self.amax[k], barrier=False)
        else:
            src, dst = self.W[self.cur], self.W[1 - self.cur]
            if self.uniform:
                rc = self.mean_fn(src.data_ptr(), G.data_ptr(), dst.data_ptr(), L,
                                  self.cols, src.stride(0), G.stride(0), dst.stride(0), LR,
                                  am, sptr)
            else:
                rc = self.ring_fn(src.data_ptr(), G.data_ptr(), dst.data_ptr(),
                                  lt.data_ptr(), rt.data_ptr(), L, self.cols, src.stride(0),
                                  G.stride(0), dst.stride(0), LR, am, sptr)
            _lib.check(rc, "mix")
            self.cur = 1 - self.cur
        if ev_pair is not None:
            ev_pair[1].record(stream)
        if self.layout == "learner" and self.uniform:
            self.launches["mix"] += (1 if self.d1d_kind.startswith("fused") else
                                     (3 if self.d1d_kind == "nvls" else 2) * len(self.d1d.chunks))
        else:   # learner / position layouts launch a planner + the mix kernel
            self.launches["mix"] += 2 if self.sharded is not None else 1
        if self.sharded is not None:
            # next step reads this step's rows on peers (a no-op with in-kernel ordering)
            self.sharded.barrier()
            if self.sharded.sync is None:
                self.launches["barrier_allreduce"] += 1

    def close(self):
        if self.sharded is not None:
            self.sharded.close()


def measure(spec, torch, dist, dev, ws, rank, local, args, clocks=None, nvc=None):
    """Warm-up, re-warm at load clocks, K timed steps.  Returns the measurement dict
    (rank 0 gets the max-over-ranks numbers) and the workload (still open)."""
    K, Wm = args.steps, args.warmup
    nsteps = Wm + K + 4096          # amax slots: warm-up, re-warm (< 4000), timed, e2e
    wl = Workload(spec, torch, dev, ws, rank, nsteps + args.e2e_steps + 64)
    stream = torch.cuda.current_stream()
    k = 0
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0.record(stream)
    for _ in range(Wm):
        wl.step(k)
        k += 1
    w1.record(stream)
    torch.cuda.synchronize()
    # re-warm: untimed steps right before the timed region, after the clock sampler's
    # start-up sleep let the clocks drop.  The count is fixed up front and equal on every
    # rank (the sharded steps order themselves across ranks: every rank must issue the
    # same steps)
    step_ms = max(w0.elapsed_time(w1) / Wm, 1e-3)
    rewarm = int(min(3000, max(1, -(-args.rewarm_seconds * 1e3 // step_ms))))
    if ws > 1:
        t = torch.tensor([rewarm], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rewarm = int(t.item())
    if clocks:
        clocks.start()
        time.sleep(0.3)
    for i in range(rewarm):
        wl.step(k)
        k += 1
        if i % 8 == 7:
            torch.cuda.synchronize()
    use_graph = use_graph_for(spec, args, ws)
    sampled = [i for i in range(K) if i % args.event_every == 0] if not use_graph else []
    kev = {i: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for i in sampled}
    t_start, t_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = None
    if use_graph:
        # the K timed steps captured once (perm-table launches + mix launches), replayed
        # once untimed, then timed: the package's simulation.GraphedRingSteps for the ring
        # strategies, the bench's own step otherwise
        wl.reset_tables()
        if spec.strategy in ("rand_psgd", "adpsgd_fixed") and wl.layout == "single":
            from paper_2002_01119_b200 import simulation as S
            gs = S.GraphedRingSteps(wl.W[wl.cur], wl.G, LR, K,
                                    seed=SEED if spec.strategy == "rand_psgd" else None, k0=k)
            graph = gs.graph
            wl.graphed = gs
        else:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for i in range(K):
                    wl.step(k + i)
        graph.replay()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wl.launches = {key: 0 for key in wl.launches}
    wl.reset_tables()   # the timed region generates its own tables
    c0 = nvc.read() if nvc else None
    placed = getattr(wl.sharded, "placed", False)
    if placed:     # per-step learners leaving each rank (the relabelling stores)
        wl.sharded.moved_log = []
        wl.sharded.log_moves = True
    if clocks:
        clocks.mark(True)
    k_first = k
    if graph is not None:
        t_start.record(stream)
        graph.replay()
        t_stop.record(stream)
        # what the graph holds (the captured steps' launches)
        wl.launches = {"perm": (K + wl.block - 1) // wl.block if spec.strategy == "rand_psgd"
                       else 0, "mix": K, "barrier_allreduce": 0}
        k += K
    else:
        t_start.record(stream)
        for i in range(K):
            wl.step(k, kev.get(i))
            k += 1
        t_stop.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.mark(False)
    c1 = nvc.read() if nvc else None
    moved = None
    if placed:
        wl.sharded.log_moves = False
        moved = torch.stack(wl.sharded.moved_log).cpu().numpy() if wl.sharded.moved_log else None
    elapsed_ms = t_start.elapsed_time(t_stop)
    # per-launch kernel time: CUDA events around every event_every-th launch; in graph
    # mode the replay time per step (mix + its share of the 1-per-64-steps perm launch)
    kern_ms = [a.elapsed_time(b) for a, b in kev.values()] or [elapsed_ms / K]
    bits = wl.amax[:k].cpu().numpy().view(np.float64)
    if getattr(wl, "graphed", None) is not None:
        bits = np.concatenate([bits, wl.graphed.absmax.cpu().numpy().view(np.float64)])
    if not np.all(np.isfinite(bits)):
        raise RuntimeError("non-finite weights in the benchmark run")
    tx = rx = -1.0
    if c0 is not None and c1 is not None:
        tx, rx = float(c1[0] - c0[0]), float(c1[1] - c0[1])
    if ws > 1:
        t = torch.tensor([elapsed_ms, tx, rx], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, tx, rx = float(t[0]), float(t[1]), float(t[2])
        lo = torch.tensor([min(tx, rx)], device=dev, dtype=torch.float64)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)     # any rank without counters -> none
        if float(lo.item()) < 0:
            tx = rx = -1.0
    L = spec.learners
    params_per_step = L * total_dim(spec, ws)
    kern_avg_s = statistics.mean(kern_ms) / 1e3
    bpp = BYTES_PER_PARAM[spec.dtype]
    algo_bytes = bpp * wl.local_params
    peak, peak_src = measured_peaks()
    res = {
        "value": params_per_step * K / (elapsed_ms / 1e3),
        "ms_per_step": elapsed_ms / K,
        "kern_avg_s": kern_avg_s,
        "algo_bytes": algo_bytes,
        "achieved": algo_bytes / kern_avg_s / 1e9,
        "peak": peak, "peak_src": peak_src,
        "launches": dict(wl.launches),
        "rewarm_steps": rewarm,
        "k_first": k_first,
        "nvlink_counted": (tx, rx) if tx >= 0 else None,
        "graph": use_graph,
        "moved": moved,
    }
    return res, wl


def use_graph_for(spec, args, ws):
    if args.graph == "off" or ws > 1:
        return False
    if args.graph == "on":
        return True
    return spec.learners * spec.dim * BYTES_PER_PARAM[spec.dtype] < (1 << 30)


def ncu_nvlink(layout):
    """The committed ncu NVLink capture of this layout's kernel (profiles/ncu_nvlink.json,
    tools/pos_probe.py + tools/ncu_nvlink_summary.py): link bytes / payload bytes, and the
    payload counted by the hardware / the traffic model."""
    try:
        z = json.loads((ROOT / "profiles" / "ncu_nvlink.json").read_text())[layout]
        return z
    except Exception:
        return None


def nvlink_object(spec, res, wl, ws, dev, mixing):
    """NVLink bytes per step of the busiest rank over the step time, against 900 GB/s per
    direction (NVLink 5) and the measured concurrent peer peaks.  Payload bytes come from
    the traffic model, which the hardware counters pin: ncu's nvltx/nvlrx user-data bytes of
    the same kernel equal the model (profiles/ncu_nvlink.json, ratio 1.000); link-level bytes
    add the measured protocol overhead of that capture.  NVML's NVLink counters are not
    supported on these B200s (NVML_ERROR_NOT_SUPPORTED), so the counts cannot be taken
    inside this multi-process run.  Rank 0."""
    K = spec.steps
    L, d = spec.learners, spec.dim
    esz = BYTES_PER_PARAM[spec.dtype] // 3
    step_s = res["ms_per_step"] / 1e3
    prd, pwr, psrc = p2p_peaks()
    out = {"bound": "nvlink", "unit": "GB/s", "peak_nominal": NVLINK_NOMINAL_GBS,
           "peak_measured_read": prd, "peak_measured_write": pwr, "peak_measured_source": psrc}
    if res["nvlink_counted"] is not None:
        tx, rx = res["nvlink_counted"]
        tx_s, rx_s = tx / K, rx / K
        a_tx, a_rx = tx_s / step_s / 1e9, rx_s / step_s / 1e9
        out.update({"source": "NVML NVLink byte counters over the timed region (max over "
                              "ranks; link-level bytes incl. protocol overhead)",
                    "tx_bytes_per_step": tx_s, "rx_bytes_per_step": rx_s,
                    "achieved_tx": a_tx, "achieved_rx": a_rx,
                    "frac_nominal": max(a_tx, a_rx) / NVLINK_NOMINAL_GBS,
                    "frac_measured_peak": max(a_tx / pwr, a_rx / prd)})
    if not wl.uniform and spec.layout in ("learner", "position"):
        k0 = res["k_first"]
        if spec.strategy == "adpsgd_fixed":
            ident = np.tile(np.arange(L, dtype=np.int64), (K + 1, 1))
            host = [ident, ident, np.roll(ident, 1, axis=1), np.roll(ident, -1, axis=1)]
        else:
            tb = mixing.permutation_tables(L, SEED, k0, K + 1, dev)
            host = [t.cpu().numpy().astype(np.int64) for t in (tb.perm, tb.inv, tb.left, tb.right)]
        if spec.layout == "position" and res.get("moved") is not None:
            # arc placement: the relabelling stores each rank issued (rm_pos_placement's count)
            mv = res["moved"].astype(np.float64).mean(axis=0)
            per_rank = [(2 * d * esz, m * d * esz) for m in mv]
            out["placement"] = {"kind": "rotate", "moved_rows_per_step_per_rank": mv.tolist()}
        else:
            per_rank = nvlink_traffic(spec.layout, L, d, esz, ws, host[0], host[1],
                                      host[2][:-1], host[3][:-1])
        rd = max(r for r, _ in per_rank)
        wr = max(w for _, w in per_rank)
        a_rd, a_wr = rd / step_s / 1e9, wr / step_s / 1e9
        out["payload"] = {
            "read_bytes_per_step": rd, "write_bytes_per_step": wr,
            "achieved_read": a_rd, "achieved_write": a_wr,
            "frac_measured_peak": max(a_rd / prd, a_wr / pwr),
            "note": "busiest rank's payload per step (pull: distinct remote neighbour rows "
                    "read; position: 2 boundary rows read + relabel stores to next-step slots "
                    "on other GPUs) over the step time"}
        nc = ncu_nvlink(spec.layout)
        if nc is not None:
            ltx = nc.get("link_over_user_tx") or 1.0
            lrx = nc.get("link_over_user_rx") or 1.0
            # reads also send request packets (TX) for the data they receive
            link_tx = wr * ltx
            link_rx = rd * lrx
            out["link"] = {
                "tx_bytes_per_step": link_tx, "rx_bytes_per_step": link_rx,
                "achieved_tx": link_tx / step_s / 1e9, "achieved_rx": link_rx / step_s / 1e9,
                "frac_nominal": max(link_tx, link_rx) / step_s / 1e9 / NVLINK_NOMINAL_GBS,
                "link_over_payload": {"tx": ltx, "rx": lrx},
                "counter_check": {"payload_counted_over_model_tx": nc.get("user_over_model_tx"),
                                  "payload_counted_over_model_rx": nc.get("user_over_model_rx"),
                                  "harness_tx_GBs": nc.get("tx_GBs"),
                                  "harness_rx_GBs": nc.get("rx_GBs")},
                "source": "payload x the link/payload byte ratio ncu counted (nvltx__bytes, "
                          "nvlrx__bytes vs *_data_user) for this kernel in profiles/"
                          "ncu_nvlink.json (single-process 2-GPU harness tools/pos_probe.py)"}
            out["frac_nominal"] = out["link"]["frac_nominal"]
        else:
            out["frac_nominal"] = max(rd, wr) / step_s / 1e9 / NVLINK_NOMINAL_GBS
        out.setdefault("source", "traffic model pinned by ncu NVLink counters (see link)")
    return out


def extra_line(spec, res, ws, dev, wl, mixing):
    e = {"workload": config_dict(spec, ws)["workload"], "layout": spec.layout,
         "scaling": "weak" if weak(spec, ws) else "strong",
         "value": res["value"], "unit": UNIT, "ms_per_step": res["ms_per_step"],
         "kernel_avg_ms": res["kern_avg_s"] * 1e3,
         "hbm_frac": res["achieved"] / res["peak"],
         "timing": "CUDA-graph replay / K" if res["graph"] else "CUDA events"}
    if ws > 1 and spec.layout in ("learner", "position"):
        e["nvlink"] = nvlink_object(spec, res, wl, ws, dev, mixing)
    return e


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2002_01119_b200 import mixing

    ws, rank, local = dist_env()
    if args.gpus != ws:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws} "
                         f"(run without torchrun to let bench.py launch the ranks)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec = resolve(args, ws)
    L = spec.learners
    uniform = spec.strategy == "d1d"
    clocks = ClockSampler(local) if rank == 0 else None
    nvc = nvlink_counters(local) if ws > 1 else None

    res, wl = measure(spec, torch, dist, dev, ws, rank, local, args, clocks=clocks, nvc=nvc)
    clock_info = clocks.stop() if clocks else None
    key = f"mix_{spec.strategy}_{spec.dtype}_L{L}_d{spec.dim}" if ws == 1 else None
    traffic = ncu_traffic(key) if key else None
    step_sync = None
    if wl.sharded is not None:
        step_sync = wl.sharded.sync is not None
    nvlink = None
    if ws > 1 and spec.layout in ("learner", "position") and rank == 0:
        nvlink = nvlink_object(spec, res, wl, ws, dev, mixing)

    e2e = None
    want_e2e = not args.no_e2e and spec.dtype == "float32"
    if want_e2e and wl.sharded is None and (ws == 1 or spec.layout == "coord"):
        # every rank drives its own column stripe (own PCIe link), max over ranks.
        # e2e = the reference-facing call on HOST buffers (the reference's step takes and
        # returns host arrays): W, G pinned on the host, W' back, every step, through
        # mixing.ring_mix_sgd_host -> rm_ring_mix_sgd_host_f32.  The resident-W variant
        # (only G crosses PCIe) is reported beside it.
        ms_res = run_e2e_resident(args, spec, torch, wl, dev)
        ms_host, ms_lm, e2e_cols = None, None, 0
        if not uniform:
            budget = min(24 << 30, host_pinned_budget() // ws)
            e2e_cols = min(wl.cols, max(32, (budget // (3 * L * 4)) // 32 * 32))
            ms_host = run_e2e(args, spec, torch, dev, cols=e2e_cols)
            release_pinned(torch)
            ms_lm = run_e2e(args, spec, torch, dev, cols=e2e_cols, layout="learner")
            release_pinned(torch)
        if ws > 1:
            t = torch.tensor([ms_res, ms_host or 0.0, ms_lm or 0.0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_res = float(t[0])
            ms_host, ms_lm = (float(t[1]), float(t[2])) if ms_host else (None, None)
        resident = e2e_resident_line(args, spec, ms_res, ws, wl)
        if ms_host:
            e2e = e2e_line(args, spec, ms_host, ws, e2e_cols)
            e2e["resident_variant"] = resident
            lm = e2e_line(args, spec, ms_lm, ws, e2e_cols, layout="learner")
            e2e["learner_major_variant"] = {k: lm[k] for k in ("value", "unit", "ms_per_step",
                                                               "path")}
        else:
            e2e = resident
    elif want_e2e:
        # sharded layouts: W resident (sharded), every rank's G H2D + max|W'| D2H per step
        ms_res = run_e2e_sharded(args, torch, wl, dev, res["k_first"] + args.steps + 8)
        if ws > 1:
            t = torch.tensor([ms_res], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_res = float(t.item())
        e2e = e2e_resident_line(args, spec, ms_res, ws, wl)
    if ws > 1:
        torch.cuda.synchronize()
        dist.barrier()
    launches = res["launches"]
    wl.close()
    del wl
    torch.cuda.empty_cache()

    extras = {}
    if not args.no_extras and spec.strategy == "rand_psgd" and args.dtype == "float32" \
            and args.learners is None and args.dim is None:
        todo = []
        if ws == 1:
            # the other BASELINE configs on the same GPU, so the driver's run measures them
            todo.append(("c1_demo", dict(layout="coord", learners=C1[0], dim=C1[1],
                                         scaling="strong", config_index=0)))
            todo.append(("c2_adpsgd_fixed", dict(strategy="adpsgd_fixed", config_index=1)))
            todo.append(("c4_d1d", dict(strategy="d1d", config_index=3)))
            todo.append(("c3_single_gpu", dict(layout="coord", learners=C3[0], dim=C3[1],
                                               scaling="strong", config_index=2)))
        else:
            todo.append(("c4_d1d_sharded", dict(strategy="d1d", layout="learner",
                                                learners=C2[0], dim=C2[1], scaling="strong",
                                                config_index=3)))
            # north-star (d) as the paper states it: the fixed ring, where only the two
            # ring-boundary rows of each rank cross GPUs (configs[1]'s AD-PSGD)
            todo.append(("c2_adpsgd_fixed_sharded", dict(strategy="adpsgd_fixed",
                                                         layout="learner", learners=C2[0],
                                                         dim=C2[1], scaling="strong",
                                                         config_index=1)))
            if spec.layout != "learner":
                todo.append(("learner_pull", dict(layout="learner", learners=C3[0], dim=C3[1],
                                                  scaling="strong", config_index=2)))
            todo.append(("coord_weak", dict(layout="coord", learners=C2[0], dim=C2[1],
                                            scaling="weak", config_index=1)))
        for name, over in todo:
            sp = argparse.Namespace(**{**vars(spec), **over})
            free, _ = torch.cuda.mem_get_info(dev)
            need = 3.3 * sp.learners * (sp.dim if sp.layout == "coord" else sp.dim / ws) * 4
            ok = torch.tensor([1.0 if free > need else 0.0], device=dev)
            if ws > 1:
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if float(ok.item()) < 1:
                extras[name] = {"skipped": "not enough free HBM"}
                continue
            try:
                r2, w2 = measure(sp, torch, dist, dev, ws, rank, local, args, nvc=nvc)
            except (RuntimeError, ValueError) as exc:   # an extra never costs the headline line
                extras[name] = {"error": str(exc)[:200]}
                torch.cuda.empty_cache()
                continue
            if rank == 0:
                extras[name] = extra_line(sp, r2, ws, dev, w2, mixing)
            w2.close()
            del w2
            torch.cuda.empty_cache()

    if not args.no_extras and ws > 1 and spec.strategy == "rand_psgd" and \
            args.dtype == "float32" and args.learners is None and args.dim is None:
        try:
            line = d1d_training_extra(torch, dist, dev, ws, rank)
        except (RuntimeError, ValueError) as exc:
            line = {"error": str(exc)[:200]}
        if rank == 0:
            extras["c4_d1d_training_sharded"] = line

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:   # the CPU baseline is an N = 1 figure
        cpu = cpu_baseline(L, uniform, args.cpu_seconds)

    if rank == 0:
        achieved = res["achieved"]
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "weak" if weak(spec, ws) else "strong",
            "vs_baseline": None,
            "dtype": {"float32": "f32", "bfloat16": "bf16", "float64": "f64"}[spec.dtype],
            "data": "synthetic: N(0,1) weights and gradients generated on device (torch "
                    "Generator), permutations from the device generator (seed 12345)",
            "config": config_dict(spec, ws),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": res["peak"],
                         "unit": "GB/s", "frac": achieved / res["peak"], "traffic": traffic,
                         "kernel": (("mix_shard_kernel" if wl_kind(spec, ws) == "shard" else
                                     "d1d_fused_kernel" if wl_kind(spec, ws) == "d1d" else
                                     "mix_tma_kernel") + f" ({spec.strategy}, {spec.dtype})"),
                         "algorithmic_bytes_per_launch": res["algo_bytes"],
                         "avg_launch_ms": res["kern_avg_s"] * 1e3,
                         "timing": ("CUDA-graph replay of the K steps / K "
                                    "(simulation.GraphedRingSteps)" if res["graph"] else
                                    f"CUDA events around every {args.event_every}-th mix launch"),
                         "peak_source": res["peak_src"]},
            "cpu_baseline": cpu,
            "e2e": e2e,
            **({"nvlink": nvlink} if nvlink else {}),
            **({"step_ordering": "in-kernel flags (multimem.red / peer atomics), no collective"
                if step_sync else "NCCL 4-byte all-reduce between steps"}
               if step_sync is not None else {}),
            "gpu_launches": launches["perm"] + launches["mix"],
            "gpu_launches_detail": launches,
            "warmup_detail": {"warmup_steps": args.warmup,
                              "rewarm_steps_before_timing": res["rewarm_steps"],
                              "note": "untimed re-warm steps after the clock sampler started, "
                                      "so the timed region starts at load clocks"},
            "clocks": clock_info,
            **({"extras": extras} if extras else {}),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def d1d_training_extra(torch, dist, dev, ws, rank, steps=12):
    """configs[3]'s D1D *training* step with the device quadratic oracle, learners sharded
    (distributed.ShardedD1DTrainer): the paper's concurrency — the global average of W_k
    beside the generator of G(W_{k-1}), G fused into the generator's final pass — against
    the serial order (gradient, then the one-kernel fused D1D step).  Per-step device time
    (CUDA events, max over ranks, median of `steps`); both orders give the same bits."""
    from paper_2002_01119_b200 import distributed as D, mixing, objectives
    from paper_2002_01119_b200.simulation import RunConfig
    L, d = C2
    b, e = D.ShardLayout(L, ws).bounds[rank]
    oracle = objectives.quadratic_oracle(d, condition_number=10.0, noise_scale=1.0, seed=1,
                                         optimum=np.zeros(d), device=dev)
    cfg = RunConfig(n_learners=L, iterations=1, lr=LR, batch_size=32, seed=5, dtype="float32")
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    W = mixing.empty_learner_major(e - b, d, torch.float32, dev)
    Wp = mixing.empty_learner_major(e - b, d, torch.float32, dev)
    W.copy_(torch.randn((e - b, d), generator=g, device=dev))
    Wp.copy_(torch.randn((e - b, d), generator=g, device=dev))
    out = mixing.empty_learner_major(e - b, d, torch.float32, dev)
    res, outs = {}, {}
    for mode, overlap in (("serial", False), ("concurrent", True)):
        tr = D.ShardedD1DTrainer(L, d, e - b, b, dev, oracle, overlap=overlap,
                                 fuse_grad=overlap)
        for k in range(3):
            tr.step(W, Wp, cfg, k, LR, out)
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for k in range(steps):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            tr.step(W, Wp, cfg, 10 + k, LR, out)
            z.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(z)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t))
        res[mode] = float(np.median(ts))
        outs[mode] = out.clone()
        chains = tr.chains
        del tr
        torch.cuda.synchronize()
        dist.barrier()
    same = torch.tensor([int(torch.equal(outs["serial"], outs["concurrent"]))], device=dev)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    del W, Wp, out, outs
    torch.cuda.empty_cache()
    return {"workload": f"d1d training step (device quadratic oracle, bit-exact numpy "
                        f"gradient noise), {L} learners x {d} params, BASELINE.json configs[3]",
            "layout": "learner", "scaling": "strong", "unit": UNIT,
            "value": L * d / (res["concurrent"] / 1e3), "ms_per_step": res["concurrent"],
            "serial_ms_per_step": res["serial"], "bit_identical_orders": bool(same.item()),
            "numpy_order_chains": chains,
            "timing": "CUDA events per step, max over ranks, median of %d" % steps}


def wl_kind(spec, ws):
    if ws == 1 or spec.layout == "coord":
        return "tma"
    return "d1d" if spec.strategy == "d1d" else "shard"


def run_e2e_resident(args, spec, torch, wl, dev):
    """The step through the public API (mixing.ring_mix_sgd / mean_mix_sgd) with the
    weights resident in HBM (the simulator state, like model weights in training) and,
    every step, the step's input — its gradients G — copied from pinned host memory
    (H2D on a copy stream, double-buffered) and the step's result — max|W'|, the
    divergence metric run_training checks — read back to the host.  Returns ms/step."""
    from paper_2002_01119_b200 import mixing as M

    L, cols = wl.L, wl.cols
    G_host = torch.empty(wl.G.shape, dtype=wl.G.dtype, pin_memory=True)
    G_host.copy_(wl.G)
    Gd = [wl.G, M.empty_learner_major(L, cols, wl.G.dtype, dev)]
    W = wl.W
    res_host = torch.zeros(args.e2e_steps + 4, dtype=torch.int64).pin_memory()
    amax = torch.zeros(args.e2e_steps + 4, dtype=torch.int64, device=dev)
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    used = [torch.cuda.Event(), torch.cuda.Event()]
    uniform = spec.strategy == "d1d"
    nsteps = args.e2e_steps + 2
    tabs = M.permutation_tables(L, SEED, 0, nsteps + 1, dev)
    fixed = None
    if spec.strategy == "adpsgd_fixed":
        from paper_2002_01119_b200 import simulation as S
        fixed = S.fixed_ring_tables(L, dev)

    def one(k, cur):
        b = k % 2
        with torch.cuda.stream(copy):
            if k >= 2:
                copy.wait_event(used[b])
            Gd[b].copy_(G_host, non_blocking=True)
            copied[b].record(copy)
        comp.wait_event(copied[b])
        if uniform:
            M.mean_mix_sgd(W[cur], Gd[b], LR, out=W[1 - cur], absmax=amax[k])
        else:
            lt, rt = fixed if fixed is not None else tabs.step(k)
            M.ring_mix_sgd(W[cur], Gd[b], LR, lt, rt, out=W[1 - cur], absmax=amax[k])
        used[b].record(comp)
        res_host[k].copy_(amax[k], non_blocking=True)

    one(0, 0)                       # warm-up
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(comp)
    cur = 1
    for k in range(1, args.e2e_steps + 1):
        one(k, cur)
        cur = 1 - cur
    e.record(comp)
    torch.cuda.synchronize()
    return a.elapsed_time(e) / args.e2e_steps


def run_e2e_sharded(args, torch, wl, dev, k0):
    """Sharded layouts through their public step API (distributed.LearnerShardedRingPos /
    LearnerShardedRing / LearnerShardedD1DFused) with W resident: every step each rank
    copies its learners' gradients from pinned host memory (copy stream, double-buffered)
    and reads back max|W'|.  Returns this rank's ms/step."""
    from paper_2002_01119_b200 import mixing as M

    G_host = torch.empty(wl.G.shape, dtype=wl.G.dtype, pin_memory=True)
    G_host.copy_(wl.G)
    Gd = [wl.G, M.empty_learner_major(wl.rows, wl.cols, wl.G.dtype, dev)]
    res_host = torch.zeros(args.e2e_steps + 4, dtype=torch.int64).pin_memory()
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    used = [torch.cuda.Event(), torch.cuda.Event()]
    wl.reset_tables()

    def one(i, k):
        b = i % 2
        with torch.cuda.stream(copy):
            if i >= 2:
                copy.wait_event(used[b])
            Gd[b].copy_(G_host, non_blocking=True)
            copied[b].record(copy)
        comp.wait_event(copied[b])
        wl.step(k, G=Gd[b])
        used[b].record(comp)
        res_host[i].copy_(wl.amax[k], non_blocking=True)

    one(0, k0)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(comp)
    for i in range(1, args.e2e_steps + 1):
        one(i, k0 + i)
    e.record(comp)
    torch.cuda.synchronize()
    return a.elapsed_time(e) / args.e2e_steps


def run_e2e(args, spec, torch, dev, cols=None, layout="dL"):
    """Step through the host-buffer API for this rank's stripe of `cols` coordinates
    (default: the whole problem); returns ms/step.  layout "dL": the reference's own
    (d, L) C-order arrays (mixing.gossip_step_host -> rm_gossip_step_host_dL_f32, contiguous
    row chunks); "learner": learner-major (L, d) host buffers (mixing.ring_mix_sgd_host ->
    rm_ring_mix_sgd_host_f32, column chunks)."""
    from paper_2002_01119_b200 import mixing as M

    L = spec.learners
    d = spec.dim if cols is None else cols
    shape = (d, L) if layout == "dL" else (L, d)
    Wh = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    Gh = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    Oh = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    # synthetic host inputs, drawn on the device and copied once (a host RNG is ~100x
    # slower and torchrun runs ranks single-threaded)
    g = torch.Generator(device=dev).manual_seed(7)
    step_rows = max(1, (1 << 26) // shape[1])
    for host in (Wh, Gh):
        for r0 in range(0, shape[0], step_rows):
            r1 = min(shape[0], r0 + step_rows)
            host[r0:r1].copy_(torch.randn((r1 - r0, shape[1]), generator=g, device=dev))
    tabs = M.permutation_tables(L, SEED, 0, args.e2e_steps + 1, dev)
    left = tabs.left.cpu()
    right = tabs.right.cpu()
    stream = torch.cuda.current_stream()
    if layout == "dL":
        ws_buf = M.workspace_dL(L, max(1, (1 << 24) // L), np.float32, dev)

        def call(src, dst, k, sync):
            M.gossip_step_host(src, Gh, LR, left[k], right[k], out=dst, workspace=ws_buf,
                               sync=sync)
    else:
        ws_buf = M.host_workspace(L, 1 << 20, dev)

        def call(src, dst, k, sync):
            M.ring_mix_sgd_host(src, Gh, LR, left[k], right[k], out_host=dst, workspace=ws_buf,
                                sync=sync)
    call(Wh, Oh, 0, True)        # warm-up call
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    src, dst = Wh, Oh
    torch.cuda.synchronize()
    a.record(stream)
    for k in range(args.e2e_steps):
        call(src, dst, k, False)
        src, dst = dst, src
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / args.e2e_steps


def e2e_line(args, spec, ms, ws, cols=None, layout="dL"):
    """The step on host buffers: W, G from pinned host memory and W' back every step
    (12 B/param over PCIe); `cols` coordinates per rank (default: the whole problem)."""
    L = spec.learners
    d = total_dim(spec, ws) if cols is None else cols * ws
    sample = None if cols is None or cols * ws == total_dim(spec, ws) else (
        f"{cols} of each rank's {total_dim(spec, ws) // ws} columns (pinned-memory bound); "
        f"the rate is PCIe-bound, so it does not depend on the sample width")
    return {"value": L * d / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": 2 * L * d * 4 + 2 * L * 4 * ws,
            "d2h_bytes_per_step": L * d * 4,
            "ms_per_step": ms, "steps": args.e2e_steps,
            "path": (("reference-facing call on the reference's own (d, L) C-order host arrays: "
                      "mixing.gossip_step_host -> rm_gossip_step_host_dL_f32 (pinned host W, G "
                      "-> W'; contiguous row chunks H2D || kernel || D2H)") if layout == "dL"
                     else ("learner-major (L, d) host buffers: mixing.ring_mix_sgd_host -> "
                           "rm_ring_mix_sgd_host_f32 (column chunks)"))
                    + (f"; every rank its column stripe, max over {ws} ranks" if ws > 1 else ""),
            **({"sample": sample} if sample else {})}


def e2e_resident_line(args, spec, ms, ws, wl):
    L, d = spec.learners, total_dim(spec, ws)
    sharded = wl.sharded is not None or (ws > 1 and spec.layout == "learner")
    esz = BYTES_PER_PARAM[spec.dtype] // 3
    return {"value": L * d / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": L * d * esz, "d2h_bytes_per_step": 8 * ws,
            "ms_per_step": ms, "steps": args.e2e_steps,
            "path": ("public API (distributed.LearnerSharded* step) with W resident and "
                     "sharded; per step every rank copies its learners' G from pinned host "
                     "memory (copy stream, double-buffered) and reads back max|W'|; max over "
                     f"{ws} ranks") if sharded else
                    ("public API mixing.ring_mix_sgd with W resident in HBM (simulator state); "
                     "per step: G (the step's input) H2D from pinned host memory on a copy "
                     "stream, double-buffered, and max|W'| (the divergence metric) D2H" + (
                         f"; every rank its column stripe, max over {ws} ranks"
                         if ws > 1 else ""))}


def release_pinned(torch):
    """Return cached pinned host blocks to the OS (the e2e variants use large buffers)."""
    fn = getattr(torch._C, "_host_emptyCache", None)
    if fn is not None:
        fn()


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    """`--gpus N` without torchrun: launch N ranks (one per GPU) on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    run_ours(args)


if __name__ == "__main__":
    main()

"""ctypes binding of libringmix_b200.so (the C-ABI in include/ringmix_b200.h).

There is no fallback: if the library is missing or CUDA is unavailable the
hot-path functions raise.  The library is built in-tree by
``__graft_entry__.build()`` (or ``make -C paper_2002_01119_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "lib" / "libringmix_b200.so"

RM_EINVAL = -1
RM_ENOSYS = -2
RM_ERANGE = -3
RM_ETIMEDOUT = -4

vp = ctypes.c_void_p
i32 = ctypes.c_int
i64 = ctypes.c_int64
u64 = ctypes.c_uint64
dbl = ctypes.c_double

_SIGNATURES = {
    "rm_last_error": ([], ctypes.c_char_p),
    "rm_version": ([], i32),
    "rm_device_info": ([i32, vp, vp, vp], i32),
    "rm_device_alloc": ([i64, vp], i32),
    "rm_device_free": ([vp], i32),
    "rm_stream_synchronize": ([vp], i32),
    "rm_memcpy": ([vp, vp, i64, vp], i32),
    "rm_enable_peer_access": ([i32], i32),
    "rm_perm_tables": ([vp, i32, u64, i32, i32, vp, vp, vp, vp, vp], i32),
    "rm_perm_sequential": ([vp, i32, u64, i32, i32, i32, vp, vp], i32),
    "rm_pcg64_raw": ([vp, i32, i32, vp, vp], i32),
    "rm_pcg_seed": ([vp, i32, i32, u64, i32, vp, vp], i32),
    "rm_pcg_permutations": ([vp, i32, i32, i32, vp, vp], i32),
    "rm_ring_mix_batched_f64": ([vp, vp, vp, vp, i32, i32, i64, i64, i64, vp], i32),
    "rm_host_chunk_cols": ([i32, i64, vp], i32),
    "rm_ring_mix_sgd_host_f32": ([vp, vp, vp, vp, vp, i32, i64, dbl, vp, i64, vp, vp], i32),
    "rm_ipc_handle_size": ([], i32),
    "rm_ipc_get_handle": ([vp, vp, vp], i32),
    "rm_ipc_open_handle": ([vp, vp], i32),
    "rm_ipc_close_handle": ([vp], i32),
    "rm_shard_plan_ints": ([i32], i32),
    "rm_shard_plan": ([vp, vp, i32, i32, i32, vp, vp], i32),
    "rm_normal_workspace_bytes": ([i32, i64], i64),
    "rm_normal_workspace_bytes_fast": ([i32, i64], i64),
    "rm_normal_stats_offset": ([i32, i64], i64),
    "rm_quadratic_grad_f32": ([vp, i32, u64, i32, i64, vp, i64, vp, vp, dbl, vp, i64, vp, i64, vp],
                              i32),
    "rm_quadratic_grad_f64": ([vp, i32, u64, i32, i64, vp, i64, vp, vp, dbl, vp, i64, vp, i64, vp],
                              i32),
    "rm_standard_normal_f64": ([vp, i32, i32, u64, i32, i64, vp, i64, vp, i64, vp], i32),
    "rm_quadratic_grad_shard_f32": ([vp, i32, u64, i64, i32, i64, vp, i64, vp, vp, dbl, vp, i64,
                                     vp, i64, vp], i32),
    "rm_quadratic_grad_shard_f64": ([vp, i32, u64, i64, i32, i64, vp, i64, vp, vp, dbl, vp, i64,
                                     vp, i64, vp], i32),
    "rm_quadratic_mix_workspace_bytes": ([i32, i64], i64),
    "rm_quadratic_mix_step_f32": ([vp, i32, u64, vp, vp, vp, vp, vp, i32, i64, i64, i64, i64, vp,
                                   vp, dbl, dbl, vp, vp, i64, vp], i32),
    "rm_quadratic_mix_step_f64": ([vp, i32, u64, vp, vp, vp, vp, vp, i32, i64, i64, i64, i64, vp,
                                   vp, dbl, dbl, vp, vp, i64, vp], i32),
    "rm_log1p_f64": ([vp, vp, i64, vp], i32),
    "rm_nvls_mean_f64": ([vp, vp, i64, i64, i32, vp], i32),
    "rm_set_d1d_ctas_per_sm": ([i32, i32, i32], i32),
    "rm_set_d1d_numpy_order": ([i32], i32),
    "rm_set_shard_remote_rows": ([i32], i32),
    "rm_set_shard_streams": ([i32, i64], i32),
    "rm_trace_stats_workspace_bytes": ([i32], i64),
    "rm_trace_stats_f32": ([vp, i32, i64, i64, vp, vp, vp, vp, vp, vp, i64, vp], i32),
    "rm_trace_stats_f64": ([vp, i32, i64, i64, vp, vp, vp, vp, vp, vp, i64, vp], i32),
    "rm_trace_stats_bf16": ([vp, i32, i64, i64, vp, vp, vp, vp, vp, vp, i64, vp], i32),
    "rm_quadratic_mean_step_shard_f32": ([vp, i32, u64, i64, vp, vp, vp, i32, i64, i64, i64, vp,
                                          vp, dbl, dbl, vp, vp, i64, vp, vp], i32),
    "rm_quadratic_mean_step_shard_f64": ([vp, i32, u64, i64, vp, vp, vp, i32, i64, i64, i64, vp,
                                          vp, dbl, dbl, vp, vp, i64, vp, vp], i32),
    "rm_trace_stats_exact_workspace_bytes": ([i64], i64),
    "rm_trace_stats_exact_f32": ([vp, i32, i64, i64, vp, vp, vp, vp, vp, vp, i64, vp], i32),
    "rm_trace_stats_exact_f64": ([vp, i32, i64, i64, vp, vp, vp, vp, vp, vp, i64, vp], i32),
    "rm_trace_stats_exact_bf16": ([vp, i32, i64, i64, vp, vp, vp, vp, vp, vp, i64, vp], i32),
    "rm_column_mean_f32": ([vp, i32, i64, i64, vp, vp], i32),
    "rm_column_mean_f64": ([vp, i32, i64, i64, vp, vp], i32),
    "rm_column_mean_bf16": ([vp, i32, i64, i64, vp, vp], i32),
}
_SIGNATURES["rm_pos_plan"] = ([vp, vp, i32, i32, i32, vp, vp, vp, vp], i32)
_SIGNATURES["rm_pos_plan_placed"] = ([vp, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp], i32)
_SIGNATURES["rm_pos_placement"] = ([vp, vp, vp, i32, i32, vp, vp, vp, vp], i32)
_SIGNATURES["rm_step_sync_wait"] = ([vp, vp], i32)
_SIGNATURES["rm_xgpu_status"] = ([vp], i32)
for _sfx in ("f32", "f64"):
    _SIGNATURES[f"rm_gossip_step_dL_{_sfx}"] = (
        [vp, vp, vp, vp, vp, i32, i64, i64, i64, i64, dbl, vp, vp], i32)
    _SIGNATURES[f"rm_gossip_step_host_dL_{_sfx}"] = (
        [vp, vp, vp, vp, vp, i32, i64, dbl, vp, i64, vp, vp], i32)
_SIGNATURES["rm_set_xgpu_timeout"] = ([dbl], i32)
_SIGNATURES["rm_step_sync_publish"] = ([vp, vp], i32)
_SIGNATURES["rm_p2p_mean_f64"] = ([vp, vp, i32, i64, i64, i32, vp], i32)
for _sfx in ("f32", "f64", "bf16"):
    _SIGNATURES[f"rm_ring_mix_sgd_pos_{_sfx}"] = (
        [vp, vp, vp, i32, i32, i32, i64, i64, i64, vp, vp, dbl, vp, vp, vp], i32)
    _SIGNATURES[f"rm_ring_mix_sgd_sharded_{_sfx}"] = (
        [vp, vp, vp, vp, i32, i32, i32, i64, i64, i64, i64, vp, dbl, vp, vp, vp], i32)
    _SIGNATURES[f"rm_partial_sum_{_sfx}"] = ([vp, i32, i64, i64, vp, vp], i32)
    _SIGNATURES[f"rm_d1d_fused_nvls_{_sfx}"] = (
        [vp, vp, vp, i32, i32, i64, i64, i64, i64, dbl, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32,
         i64, i32, ctypes.c_uint32, i32, i32, vp], i32)
    _SIGNATURES[f"rm_d1d_fused_p2p_{_sfx}"] = (
        [vp, i32, i32, i64, i64, i64, i64, dbl, vp, vp, vp, i32, i64, i32, ctypes.c_uint32, i32,
         i32, vp], i32)
    _SIGNATURES[f"rm_apply_mean_sgd_{_sfx}"] = ([vp, vp, vp, i32, i32, i64, i64, i64, dbl, vp, vp],
                                                i32)
    _SIGNATURES[f"rm_ring_mix_sgd_{_sfx}"] = (
        [vp, vp, vp, vp, vp, i32, i64, i64, i64, i64, dbl, vp, vp], i32)
    _SIGNATURES[f"rm_mean_sgd_{_sfx}"] = ([vp, vp, vp, i32, i64, i64, i64, i64, dbl, vp, vp], i32)
    _SIGNATURES[f"rm_spsgd_{_sfx}"] = ([vp, vp, vp, i32, i64, i64, i64, i64, dbl, vp, vp, vp], i32)

OPTIONAL_SIGNATURES: dict = {}


class StepSyncArgs(ctypes.Structure):
    """rm_step_sync (include/ringmix_b200.h)."""
    _fields_ = [("done", vp), ("done_mc", vp), ("counter", vp), ("epoch", ctypes.c_uint32),
                ("world", i32), ("done_peers", vp)]


class D1DRank(ctypes.Structure):
    """rm_d1d_rank (include/ringmix_b200.h): one rank's buffers of the fused D1D step."""
    _fields_ = [("W", vp), ("G", vp), ("out", vp), ("absmax_bits", vp), ("P", vp), ("M", vp),
                ("flags", vp), ("counters", vp), ("Lg", i32), ("rank", i32)]


class RingmixError(RuntimeError):
    """A CUDA-side failure inside libringmix_b200."""


_lib = None


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def load() -> ctypes.CDLL:
    """Load the library (no CUDA call is made here)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (there is no CPU fallback for the ringmix_b200 hot path)")
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (args, res) in {**_SIGNATURES, **OPTIONAL_SIGNATURES}.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def last_error() -> str:
    return load().rm_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = last_error()
    if rc < 0:
        raise ValueError(msg or f"{what}: invalid argument ({rc})")
    raise RingmixError(f"{what}: {msg} (cuda error {rc})")


_cuda_ok = False


def require_cuda(t: torch.Tensor | None = None) -> None:
    global _cuda_ok
    if not _cuda_ok:       # a positive answer is cached (the check costs ~5 us per call)
        if not torch.cuda.is_available():
            raise RuntimeError("ringmix_b200 needs a CUDA device (B200, sm_100a); "
                               "no CPU fallback")
        _cuda_ok = True
    if t is not None and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    """cudaStream_t of `stream`, default: the current stream of the current device."""
    if stream is not None:
        return int(stream.cuda_stream)
    if _raw_stream is not None:          # same value, without building a Stream object
        return int(_raw_stream(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())

"""Single-process, two-GPU harness for the learner-sharded RAD pull kernel, so ncu can
capture it (a multi-rank command cannot be profiled): GPU 0 holds learners [0, L/2)
and runs rank 0's step; learners [L/2, L) live on GPU 1 and are read over NVLink
through peer pointers (rm_enable_peer_access).  C2 shapes.  PP_FIXED=1: the fixed ring
(AD-PSGD) instead of RAD — only the two boundary rows cross."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_01119_b200 import _lib, mixing, simulation

L, d = int(os.environ.get("PP_L", 64)), int(os.environ.get("PP_D", 25_557_032))
lib = _lib.load()
_lib.check(lib.rm_enable_peer_access(2))
d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
Lg = L // 2
X0 = mixing.empty_learner_major(Lg, d, torch.float32, d0).normal_()
with torch.cuda.device(d1):
    X1 = mixing.empty_learner_major(L - Lg, d, torch.float32, d1).normal_()
G0 = mixing.empty_learner_major(Lg, d, torch.float32, d0).normal_()
out = mixing.empty_learner_major(Lg, d, torch.float32, d0)
ptrs = np.empty(L, dtype=np.uint64)
for i in range(Lg):
    ptrs[i] = X0.data_ptr() + i * X0.stride(0) * 4
for i in range(L - Lg):
    ptrs[Lg + i] = X1.data_ptr() + i * X1.stride(0) * 4
row_ptrs = torch.from_numpy(ptrs.view(np.int64)).to(d0)
plan = torch.empty(lib.rm_shard_plan_ints(Lg), dtype=torch.int32, device=d0)
torch.cuda.set_device(d0)
res = {}
ms = []
for k in range(12):
    lt, rt = (simulation.fixed_ring_tables(L, d0) if os.environ.get("PP_FIXED") == "1"
              else simulation.rad_tables(L, 12345, k, d0))
    s = _lib.stream_ptr()
    _lib.check(lib.rm_shard_plan(lt.data_ptr(), rt.data_ptr(), L, 0, Lg, plan.data_ptr(), s))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(lib.rm_ring_mix_sgd_sharded_f32(row_ptrs.data_ptr(), X0.data_ptr(), G0.data_ptr(),
                                               out.data_ptr(), L, 0, Lg, d, X0.stride(0),
                                               G0.stride(0), out.stride(0), plan.data_ptr(),
                                               0.01, None, s, None))
    b.record(); torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
    R = int(plan[0].item())
    res.setdefault("remote_rows", []).append(R)
kern = float(np.median(ms[2:]))
R = float(np.mean(res["remote_rows"][2:]))
print(json.dumps({"L": L, "d": d, "kernel_ms": kern, "remote_rows": R,
                  "nvlink_read_GBs": R * d * 4 / (kern / 1e3) / 1e9,
                  "hbm_GBs": 3 * Lg * d * 4 / (kern / 1e3) / 1e9}), flush=True)

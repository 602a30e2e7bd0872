"""Single-process, two-GPU harness of rank 0's step in the learner-sharded layouts, so ncu
can capture the kernel and its NVLink counters (nvltx__bytes / nvlrx__bytes; a multi-rank
command cannot be profiled): GPU 0 owns positions / learners [0, L/2), GPU 1 holds the rest
and is reached through peer pointers (rm_enable_peer_access).  BASELINE config 3 shapes
(128 x 43,154,944 fp32) by default.

  PP_LAYOUT=position|learner python tools/pos_probe.py
prints the kernel time and the modelled NVLink bytes per launch (payload only)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_01119_b200 import _lib, distributed as D, mixing  # noqa: E402

L, d = int(os.environ.get("PP_L", 128)), int(os.environ.get("PP_D", 43_154_944))
layout = os.environ.get("PP_LAYOUT", "position")
steps = int(os.environ.get("PP_STEPS", 8))
lib = _lib.load()
_lib.check(lib.rm_enable_peer_access(2))
d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
lay = D.ShardLayout(L, 2)
(b0, e0), (b1, e1) = lay.bounds
Lg = e0 - b0
torch.cuda.set_device(d0)
bufs = [[mixing.empty_learner_major(e - b, d, torch.float32, dv) for _ in range(2)]
        for (b, e), dv in zip(lay.bounds, (d0, d1))]
for r, dv in enumerate((d0, d1)):
    with torch.cuda.device(dv):
        bufs[r][0].normal_()
G0 = mixing.empty_learner_major(Lg, d, torch.float32, d0).normal_()
esz = 4
slots = [D._slot_table(lay, [bufs[r][p].data_ptr() for r in range(2)], bufs[0][0].stride(0),
                       esz, d0) for p in range(2)]
tabs = mixing.permutation_tables(L, 12345, 0, steps + 1, d0)
plan = torch.empty(lib.rm_shard_plan_ints(Lg), dtype=torch.int32, device=d0)
dest = torch.empty(Lg, dtype=torch.int64, device=d0)
out = mixing.empty_learner_major(Lg, d, torch.float32, d0)
ms, model = [], []
perm = tabs.perm.cpu().numpy()
inv = tabs.inv.cpu().numpy()
for k in range(steps):
    s = _lib.stream_ptr()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = k % 2
    if layout == "position":
        ik, pn = tabs.inv[k].contiguous(), tabs.perm[k + 1].contiguous()
        _lib.check(lib.rm_pos_plan(ik.data_ptr(), pn.data_ptr(), L, 0, Lg,
                                   slots[1 - cur].data_ptr(), plan.data_ptr(), dest.data_ptr(), s))
        src = bufs[0][cur]
        a.record()
        _lib.check(lib.rm_ring_mix_sgd_pos_f32(slots[cur].data_ptr(), src.data_ptr(),
                                               G0.data_ptr(), L, 0, Lg, d, src.stride(0),
                                               G0.stride(0), plan.data_ptr(), dest.data_ptr(),
                                               0.01, None, s, None))
        b.record()
        nxt = perm[k + 1][inv[k, 0:Lg]]     # slot x -> slot p_{k+1}[inv_k[x]]
        remote_out = int(((nxt < b0) | (nxt >= e0)).sum())
        model.append({"read": 2 * d * esz, "write": remote_out * d * esz})
    else:
        lt, rt = tabs.left[k].contiguous(), tabs.right[k].contiguous()
        _lib.check(lib.rm_shard_plan(lt.data_ptr(), rt.data_ptr(), L, 0, Lg, plan.data_ptr(), s))
        src = bufs[0][cur]
        a.record()
        _lib.check(lib.rm_ring_mix_sgd_sharded_f32(
            slots[cur].data_ptr(), src.data_ptr(), G0.data_ptr(), out.data_ptr(), L, 0, Lg, d,
            src.stride(0), G0.stride(0), out.stride(0), plan.data_ptr(), 0.01, None, s, None))
        b.record()
        lt_h, rt_h = tabs.left[k].cpu().numpy(), tabs.right[k].cpu().numpy()
        nb = set(lt_h[0:Lg].tolist()) | set(rt_h[0:Lg].tolist())
        model.append({"read": sum(1 for x in nb if not 0 <= x < Lg) * d * esz, "write": 0})
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
kern = float(np.median(ms[2:]))
rd = float(np.mean([m["read"] for m in model[2:]]))
wr = float(np.mean([m["write"] for m in model[2:]]))
print(json.dumps({"layout": layout, "L": L, "d": d, "kernel_ms": kern,
                  "model_read_bytes_per_launch": rd, "model_write_bytes_per_launch": wr,
                  "per_launch_model": model, "per_launch_ms": ms,
                  "nvlink_read_GBs": rd / (kern / 1e3) / 1e9,
                  "nvlink_write_GBs": wr / (kern / 1e3) / 1e9}), flush=True)

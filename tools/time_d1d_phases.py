"""Per-phase timing of the learner-sharded D1D step (torchrun)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2002_01119_b200 import _lib, distributed as D, mixing

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
L, d = 64, 25_557_032
lay = D.ShardLayout(L, ws); b, e = lay.rows(rank); Lg = e - b
W = mixing.empty_learner_major(Lg, d, torch.float32, dev); W.normal_()
G = mixing.empty_learner_major(Lg, d, torch.float32, dev); G.normal_()
out = mixing.empty_learner_major(Lg, d, torch.float32, dev)
nv = D.LearnerShardedD1DNVLS(L, d, Lg, dev)
lib = _lib.load(); s = _lib.stream_ptr()
def ev():
    x = torch.cuda.Event(enable_timing=True); x.record(); return x
res = {}
for it in range(6):
    torch.cuda.synchronize(); dist.barrier(); torch.cuda.synchronize()
    t0 = ev(); lib.rm_partial_sum_f32(W.data_ptr(), Lg, d, W.stride(0), nv.P.data_ptr(), s)
    t1 = ev(); nv.hP.barrier(channel=0)
    t2 = ev(); lib.rm_nvls_mean_f64(nv.hP.multicast_ptr, nv.hM.multicast_ptr, nv.c0, nv.c1, L, s)
    t3 = ev(); nv.hM.barrier(channel=1)
    t4 = ev(); lib.rm_apply_mean_sgd_f32(nv.M.data_ptr(), G.data_ptr(), out.data_ptr(), Lg, 1, d, G.stride(0), out.stride(0), 0.01, None, s)
    t5 = ev(); torch.cuda.synchronize()
    if it >= 2:
        for k, (a, bb) in {"partial": (t0, t1), "barrier1": (t1, t2), "nvls_sum": (t2, t3), "barrier2": (t3, t4), "apply": (t4, t5)}.items():
            res.setdefault(k, []).append(a.elapsed_time(bb))
if rank == 0:
    print(json.dumps({k: sum(v) / len(v) for k, v in res.items()} | {"world": ws, "Lg": Lg}), flush=True)
dist.destroy_process_group()

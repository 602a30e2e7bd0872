"""Summarise the ncu NVLink captures of tools/pos_probe.py (gpu_n2_r2b.sh) into
profiles/ncu_nvlink.json, which bench.py cites in its `nvlink` object."""
import csv
import io
import json
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/n2_r2b"
out = {}
for lay in ("position", "learner"):
    text = open(f"{src}/ncu_{lay}.csv").read().splitlines()
    rows = list(csv.DictReader(io.StringIO("\n".join(x for x in text if x.startswith('"')))))
    launches = {}
    for r in rows:
        launches.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(
            r["Metric Value"].replace(",", ""))
    probe = [json.loads(x) for x in open(f"{src}/probe_{lay}.log") if x.startswith("{")][-1]
    L, d = probe["L"], probe["d"]
    if lay == "position":
        # payload model recomputed from the permutations (seed 12345, steps 0..): slot x of
        # step k holds learner inv_k[x], its output goes to slot p_{k+1}[inv_k[x]]
        sys.path.insert(0, ".")
        import numpy as np
        from oracle import ringmix_oracle as O
        P = [O.c_permutation(L, 12345, k) for k in range(len(probe["per_launch_model"]) + 1)]
        Lg = L // 2
        for k, ent in enumerate(probe["per_launch_model"]):
            nxt = P[k + 1][np.argsort(P[k])[:Lg]]
            ent["write"] = int(((nxt < 0) | (nxt >= Lg)).sum()) * d * 4
    lst = []
    for i, (lid, m) in enumerate(sorted(launches.items())):
        model = probe["per_launch_model"][3 + i]    # -s 3 -c 2: launches 3 and 4
        t = m["gpu__time_duration.sum"] * 1e-9
        lst.append({"launch": 3 + i, "duration_ms": t * 1e3,
                    "nvltx_bytes": m["nvltx__bytes.sum"],
                    "nvltx_user_bytes": m["nvltx__bytes_data_user.sum"],
                    "nvlrx_bytes": m["nvlrx__bytes.sum"],
                    "nvlrx_user_bytes": m["nvlrx__bytes_data_user.sum"],
                    "dram_read_bytes": m["dram__bytes_read.sum"],
                    "dram_write_bytes": m["dram__bytes_write.sum"],
                    "model_write_bytes": model["write"], "model_read_bytes": model["read"],
                    "tx_GBs": m["nvltx__bytes.sum"] / t / 1e9,
                    "rx_GBs": m["nvlrx__bytes.sum"] / t / 1e9,
                    "tx_user_GBs": m["nvltx__bytes_data_user.sum"] / t / 1e9,
                    "rx_user_GBs": m["nvlrx__bytes_data_user.sum"] / t / 1e9})
    s = lambda k: sum(x[k] for x in lst)  # noqa: E731
    out[lay] = {
        "kernel": "mix_shard_kernel<float, HAS_G>",
        "harness": f"tools/pos_probe.py PP_LAYOUT={lay}: rank 0's step of a 2-rank C3 job "
                   "(128 x 43,154,944 fp32) in one process, GPU 1 reached through peer pointers",
        "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                   "dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,"
                   "nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum "
                   "--clock-control none -k regex:mix_shard -s 3 -c 2",
        "launches": lst,
        "link_over_user_tx": (s("nvltx_bytes") / s("nvltx_user_bytes")
                              if s("nvltx_user_bytes") > 0 else None),
        "link_over_user_rx": s("nvlrx_bytes") / max(1.0, s("nvlrx_user_bytes")),
        "user_over_model_tx": s("nvltx_user_bytes") / max(1.0, s("model_write_bytes")),
        "user_over_model_rx": s("nvlrx_user_bytes") / max(1.0, s("model_read_bytes")),
        "tx_GBs": s("nvltx_bytes") / (s("duration_ms") / 1e3) / 1e9,
        "rx_GBs": s("nvlrx_bytes") / (s("duration_ms") / 1e3) / 1e9}
json.dump(out, open("profiles/ncu_nvlink.json", "w"), indent=1)
for k, v in out.items():
    print(k, {kk: round(vv, 4) for kk, vv in v.items() if isinstance(vv, float)})

"""Checks the NVML NVLink byte counters against a known transfer: copies N bytes from
GPU 0 to GPU 1 (cudaMemcpyPeer via torch) and prints each GPU's counter deltas; also
prints the `nvidia-smi nvlink -gt d` view for reference.  Needs 2 GPUs."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from nvlink_counters import NvlinkCounters  # noqa: E402

n = 8 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
c = [NvlinkCounters(i) for i in range(2)]
for i, x in enumerate(c):
    print(json.dumps({"gpu": i, "ok": x.ok, "method": x.method, "links": x.links,
                      "error": getattr(x, "error", None)}), flush=True)
# raw NVML return codes of the candidate fields on link 0 / scope 0
try:
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    for fid in (202, 204, 138, 139, 140, 141):
        v = nv.nvmlDeviceGetFieldValues(h, [(fid, 0)])[0]
        print(json.dumps({"field": fid, "ret": int(v.nvmlReturn), "type": int(v.valueType),
                          "ull": int(v.value.ullVal)}), flush=True)
    try:
        print(json.dumps({"util_counter_link0": str(nv.nvmlDeviceGetNvLinkUtilizationCounter(
            h, 0, 0))}), flush=True)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"util_counter_error": str(e)}), flush=True)
except Exception as e:  # noqa: BLE001
    print(json.dumps({"nvml_error": str(e)}), flush=True)
for args in (["nvlink", "-gt", "r", "-i", "0"], ["nvlink", "-s", "-i", "0"]):
    try:
        print("---- nvidia-smi " + " ".join(args) + "\n" + subprocess.run(
            ["nvidia-smi"] + args, capture_output=True, text=True, timeout=30).stdout[:1500])
    except Exception as e:  # noqa: BLE001
        print(e)
try:
    smi0 = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True,
                          text=True, timeout=30).stdout
except Exception as e:  # noqa: BLE001
    smi0 = str(e)
r0 = [x.read() for x in c]
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
r1 = [x.read() for x in c]
for i in range(2):
    if r0[i] and r1[i]:
        print(json.dumps({"gpu": i, "tx_bytes": r1[i][0] - r0[i][0], "rx_bytes": r1[i][1] - r0[i][1],
                          "copied_bytes": 3 * n}), flush=True)
try:
    smi1 = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True,
                          text=True, timeout=30).stdout
except Exception as e:  # noqa: BLE001
    smi1 = str(e)
print("---- nvidia-smi nvlink -gt d (before)\n" + smi0[:3000])
print("---- nvidia-smi nvlink -gt d (after)\n" + smi1[:3000])

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

"""NVLink traffic counters of one GPU through NVML (measurement helper for bench.py and
tools/probe_nvlink_counters.py; not on the product path).

B200 (NVLink 5) exposes per-link byte counters as NVML field values
NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES (scope = link id); older drivers expose
NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (KiB, all links).  `NvlinkCounters.read()`
returns (tx_bytes, rx_bytes) summed over the GPU's links, or None when neither works."""

from __future__ import annotations


class NvlinkCounters:
    FI_XMIT, FI_RCV = 202, 204           # NVML_FI_DEV_NVLINK_COUNT_{XMIT,RCV}_BYTES
    FI_TP_TX, FI_TP_RX = 138, 139        # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX} (KiB)
    MAX_LINKS = 18

    def __init__(self, gpu_index: int):
        self.ok = False
        self.method = None
        self.links: list[int] = []
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(gpu_index)
        except Exception as e:  # noqa: BLE001 (no NVML: counters unavailable)
            self.error = f"nvml: {e}"
            return
        for link in range(self.MAX_LINKS):
            try:
                if self.nv.nvmlDeviceGetNvLinkState(self.h, link):
                    self.links.append(link)
            except Exception:  # noqa: BLE001
                continue
        for method in ("count_bytes", "throughput_kib"):
            self.method = method
            try:
                if self._read_raw() is not None:
                    self.ok = True
                    return
            except Exception as e:  # noqa: BLE001
                self.error = f"{method}: {e}"
        self.method = None

    def _fields(self, ids_scopes):
        nv = self.nv
        vals = nv.nvmlDeviceGetFieldValues(self.h, [(fid, sc) for fid, sc in ids_scopes])
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                return None
            vt, x = v.valueType, v.value
            # NVML_VALUE_TYPE: 0 double, 1 uint, 2 ulong, 3 ulonglong, 4 slonglong, 5 sint
            out.append(int(x.dVal) if vt == 0 else int(x.uiVal) if vt in (1, 5) else
                       int(x.ullVal))
        return out

    def _read_raw(self):
        if self.method == "count_bytes":
            if not self.links:
                return None
            req = [(self.FI_XMIT, ln) for ln in self.links] + [(self.FI_RCV, ln) for ln in self.links]
            v = self._fields(req)
            if v is None:
                return None
            n = len(self.links)
            return sum(v[:n]), sum(v[n:])
        v = self._fields([(self.FI_TP_TX, 0), (self.FI_TP_RX, 0)])
        if v is None:
            return None
        return v[0] * 1024, v[1] * 1024

    def read(self):
        if not self.ok:
            return None
        try:
            return self._read_raw()
        except Exception:  # noqa: BLE001
            return None

"""NVLink byte counters from NVML (probe only: on this pool's B200s the throughput fields answer
NVML_ERROR_NOT_SUPPORTED and `nvidia-smi nvlink -gt d` prints N/A, profiles/r02_nvsmi_nvlink.txt) (no profiler): cumulative per-link TX / RX data throughput
counters (field ids NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX = 138/139, RAW 140/141, KiB,
nvml.h), summed over the device's links.  Read before and after a timed region they give the
NVLink bytes the kernels actually moved (the "NVLink bus GB/s" of the north star) while the
kernels run at full speed, which ncu's serialised replay cannot do for kernels that wait on
peers.

    python tools/nvml_nvlink.py            # probe: print every field / link that answers
"""
from __future__ import annotations

import json
import sys

FI_DATA_TX, FI_DATA_RX, FI_RAW_TX, FI_RAW_RX = 138, 139, 140, 141
MAX_LINKS = 18


class NvlinkCounters:
    def __init__(self, index: int):
        import pynvml as nv
        nv.nvmlInit()
        self.nv = nv
        self.h = nv.nvmlDeviceGetHandleByIndex(index)
        self.links = []
        for link in range(MAX_LINKS):
            try:
                if nv.nvmlDeviceGetNvLinkState(self.h, link) == nv.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except Exception:
                pass

    def _fields(self, fid):
        try:
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, [(fid, link) for link in self.links])
        except Exception:
            return None
        if any(v.nvmlReturn != 0 for v in vals):
            return None
        return [int(v.value.ullVal) for v in vals]

    def read(self):
        """{"data_tx": bytes, "data_rx": bytes, "raw_tx": ..., "raw_rx": ...} summed over links
        (None for a field the driver does not report)"""
        out = {}
        for name, fid in (("data_tx", FI_DATA_TX), ("data_rx", FI_DATA_RX),
                          ("raw_tx", FI_RAW_TX), ("raw_rx", FI_RAW_RX)):
            v = self._fields(fid)
            out[name] = None if v is None else 1024 * sum(v)
        return out


def delta(a: dict, b: dict) -> dict:
    return {k: (None if a.get(k) is None or b.get(k) is None else b[k] - a[k]) for k in a}


if __name__ == "__main__":
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    c = NvlinkCounters(idx)
    print(json.dumps({"links": c.links, "counters": c.read()}))

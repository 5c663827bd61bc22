"""Condenses an ncu --set full report (raw page) into the numbers the roofline needs."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex.sum", "lts__t_sectors_srcunit_tex_lookup_miss.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        for i, h in enumerate(hdr):  # any other tensor-pipe utilisation counters
            if "pipe_tensor" in h and "pct" in h and h not in d:
                d[h] = f"{r[i]} {units[i]}".strip()
        d["kernel"] = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps({"report": p, "launches": summarize(p)}, indent=1))

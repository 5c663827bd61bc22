"""profiles/ncu_traffic_<workload>.json from an ncu --set full capture of one bench step's
tc_conv_kernel launches (dram read+write per launch, summed per step) + a condensed summary file.

    python tools/make_traffic.py <report.ncu-rep> <workload> <summary.json> [split]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summarize  # noqa: E402


def mb(v):
    num, unit = v.split()
    f = float(num)
    return f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[unit]


rep, workload, out_summary = sys.argv[1], sys.argv[2], sys.argv[3]
split = sys.argv[4] if len(sys.argv) > 4 else "mixed"
launches = summarize(rep)
per = []
for l in launches:
    per.append({"duration_us": float(l["gpu__time_duration.sum"].split()[0]) * (1000 if "ms" in l["gpu__time_duration.sum"] else 1),
                "dram_read_MB": mb(l["dram__bytes_read.sum"]), "dram_write_MB": mb(l["dram__bytes_write.sum"]),
                "tensor_pipe_active_pct": float(l["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"].split()[0]),
                "l2_throughput_pct": float(l["lts__throughput.avg.pct_of_peak_sustained_elapsed"].split()[0]),
                "dram_throughput_pct": float(l["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"].split()[0])})
total = sum((p["dram_read_MB"] + p["dram_write_MB"]) * 1e6 for p in per)
Path(f"profiles/ncu_traffic_{workload}.json").write_text(json.dumps(
    {"workload": workload, "precision": "fp32", "split": split, "dram_bytes_per_step": total,
     "launches_per_step": len(per), "source": rep, "per_launch": per}, indent=1))
Path(out_summary).write_text(json.dumps({"report": rep, "launches": launches}, indent=1))
print(json.dumps(per, indent=1), total / 1e6, "MB per step")

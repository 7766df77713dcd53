"""Summarise ncu captures into profiles/ (run here, after gpurun brought the
.ncu-rep / launch list back).

    python scripts/summarize_ncu.py full <report.ncu-rep> <out.txt> [--traffic-json P --batch B]
    python scripts/summarize_ncu.py launches <launches.csv> <out.txt>
"""

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
    "launch__shared_mem_per_block_dynamic",
]


def full(rep, out, traffic_json=None, batch=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = []
    traffic = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"kernel: {name[:120]}")
        rd = wr = None
        for key in KEYS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"  {key:70s} {vals[i]:>16s} {units[i]}")
                if key == "dram__bytes_read.sum":
                    rd = (vals[i], units[i])
                if key == "dram__bytes_write.sum":
                    wr = (vals[i], units[i])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if rd and wr:
            b = float(rd[0].replace(",", "")) * scale.get(rd[1], 1) + \
                float(wr[0].replace(",", "")) * scale.get(wr[1], 1)
            traffic.append(b)
            lines.append(f"  dram read+write bytes per launch: {b:.6e}")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if traffic_json and traffic:
        with open(traffic_json, "w") as fh:
            json.dump({"batch": batch, "dram_bytes_per_launch": traffic[0], "source": rep}, fh,
                      indent=1)
    print("\n".join(lines))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            d[r[ki].split("(")[0][:90]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    tot = sum(sum(v) for v in d.values())
    lines = [f"{'kernel':90s} {'launches':>8s} {'mean_ns':>12s} {'share':>7s}"]
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        lines.append(f"{k:90s} {len(v):8d} {sum(v)/len(v):12.1f} {sum(v)/tot*100:6.1f}%")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        bt = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj, bt)
    else:
        launches(sys.argv[2], sys.argv[3])

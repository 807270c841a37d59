"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python scripts/summarize_ncu.py <full.ncu-rep> <launches.csv> <tag> [config]

Writes profiles/<tag>_ncu_full.txt (key metrics per kernel), profiles/<tag>_launches.txt
(per-launch durations and each kernel's share) and merges DRAM traffic per launch into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
]


def short(name):
    for k in ("tc_row_stage", "tc_column_stage", "tc_column_wide", "tc_alpha_r_stage", "tc_row_pair", "row_stage",
              "column_stage", "alpha_r_stage"):
        if k in name:
            return ("tc_" if name.find("tc_") >= 0 and not k.startswith("tc_") else "") + k
    return name[:60]


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    cfg = sys.argv[4] if len(sys.argv) > 4 else "sf"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines, traffic = [], {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = short(d.get("Kernel Name", "?"))
        lines.append(f"== {name}")
        for m in METRICS:
            if m in d:
                lines.append(f"  {m:75s} {d[m]:>16s} {units[hdr.index(m)]}")
        try:
            rd = float(d["dram__bytes_read.sum"]) * (1e6 if units[hdr.index("dram__bytes_read.sum")] == "Mbyte" else 1)
            wr = float(d["dram__bytes_write.sum"]) * (1e6 if units[hdr.index("dram__bytes_write.sum")] == "Mbyte" else 1)
            traffic.setdefault(name, []).append(rd + wr)
        except (KeyError, ValueError):
            pass
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.txt"), "w") as fh:
        fh.write(f"ncu --set full --clock-control none (cold L2 per replay) of {os.path.basename(rep)}\n")
        fh.write("\n".join(lines) + "\n")
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tj[cfg] = {k: int(sum(v) / len(v)) for k, v in traffic.items()}
    json.dump(tj, open(tpath, "w"), indent=1)
    # launch list
    per = {}
    for r in csv.reader(open(launches)):
        if len(r) > 14 and r[0] != "ID" and r[12] == "gpu__time_duration.sum":
            per.setdefault(short(r[4]), []).append(float(r[14]))
    tot = sum(sum(v) for v in per.values())
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w") as fh:
        fh.write(f"ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold): {os.path.basename(launches)}\n")
        for k, v in per.items():
            fh.write(f"{k:24s} launches {len(v):4d}  avg {sum(v) / len(v) / 1000:9.2f} us  share {sum(v) / tot:6.3f}\n")
    print(open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt")).read())
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()

"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into profiles/.

    python tools/ncu_summary.py <name>=<report.ncu-rep>[:<units>] ... [--launches <csv>] [--out profiles/r01]

<units> = algorithmic units per launch (sweeps for Jacobi) used to express
dram bytes per unit.  Writes <out>/ncu_<name>.txt (key metrics) and merges a
machine-readable entry into profiles/ncu_summary.json.
"""

import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic",
]

SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = (r[i], units[i])
        recs.append(rec)
    return recs


def num(v):
    val, unit = v
    try:
        x = float(val.replace(",", ""))
    except ValueError:
        return None
    return x * SCALE.get(unit, 1.0)


def main(argv):
    out_dir = "profiles"
    launches = None
    items = []
    i = 0
    while i < len(argv):
        a = argv[i]
        if a == "--out":
            out_dir = argv[i + 1]
            i += 2
            continue
        if a == "--launches":
            launches = argv[i + 1]
            i += 2
            continue
        name, spec = a.split("=", 1)
        units = 1
        if ":" in spec:
            spec, u = spec.rsplit(":", 1)
            units = int(u)
        items.append((name, spec, units))
        i += 1
    os.makedirs(out_dir, exist_ok=True)
    summ_path = os.path.join("profiles", "ncu_summary.json")
    summary = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for name, rep, units in items:
        recs = raw(rep)
        lines = []
        for j, rec in enumerate(recs):
            lines.append(f"[{name} launch {j}]")
            for k in KEYS:
                if k in rec:
                    lines.append(f"  {k} = {rec[k][0]} {rec[k][1]}")
        with open(os.path.join(out_dir, f"ncu_{name}.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        r0 = recs[0]
        dram = (num(r0["dram__bytes_read.sum"]) or 0) + (num(r0["dram__bytes_write.sum"]) or 0)
        t = num(r0["gpu__time_duration.sum"])
        summary[name] = {
            "report": os.path.basename(rep), "kernel": r0["Kernel Name"][0],
            "duration_s": t, "units_per_launch": units,
            "dram_bytes_per_launch": dram, "dram_bytes_per_unit": dram / units,
            "dram_throughput_pct": num(r0.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ("", ""))),
            "tensor_active_pct": num(r0.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", ("", ""))),
            "l2_hit_pct": num(r0.get("lts__t_sector_hit_rate.pct", ("", ""))),
            "sm_clock_hz": num(r0.get("sm__cycles_elapsed.avg.per_second", ("", ""))),
        }
        print(name, json.dumps(summary[name], indent=1))
    if launches:
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        hdr = rows[0]
        k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            name = r[k]
            c, s = agg.get(name, (0, 0.0))
            agg[name] = (c + 1, s + float(r[v].replace(",", "")))
        tot = sum(s for _, s in agg.values()) or 1.0
        with open(os.path.join(out_dir, "launch_shares.txt"), "w") as fh:
            fh.write("launches  total_us  share  kernel (ncu gpu__time_duration.sum, cold/serialised)\n")
            for name, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
                fh.write(f"{c:8d} {s / 1e3:9.1f} {100 * s / tot:6.1f}%  {name}\n")
        print(open(os.path.join(out_dir, "launch_shares.txt")).read())
    with open(summ_path, "w") as fh:
        json.dump(summary, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])

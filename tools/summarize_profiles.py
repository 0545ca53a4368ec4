#!/usr/bin/env python3
"""Summarise a gpu_round.sh capture (gpurun_out/<tag>) into tracked files under profiles/.

    python tools/summarize_profiles.py <tag> [--round r1]

Writes profiles/<round>_launches.txt (per-launch device times of one bench command: the
kernel's SHARE of the step), profiles/<round>_ncu_<kernel>.txt (key metrics of the
`ncu --set full` capture: duration, DRAM bytes, throughput, occupancy, pipe utilisation,
stall reasons) and merges the per-launch DRAM traffic into profiles/traffic.json (read by
bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
]


# the workload of each named capture (the default is the bench config)
CAPTURE_CONFIG = {
    "genm_m2": "single_pass_m2_R1_B128_n268435456",
    "genm_m4": "single_pass_m4_R1_B128_n268435456",
    "genm_m4_r2": "single_pass_m4_R1_B128_n268435456",
    "genm_m4_reg": "single_pass_m4_R1_B128_n268435456",
    "ordered": "ordered_walk_m16_R1_B1024_n1073741824",
}


def ncu_raw(rep):
    if rep.endswith(".raw.csv"):   # exported on the GPU box (ncu -i X --page raw --csv)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}, {}
    h, units, v = rows[0], rows[1], rows[2]
    return dict(zip(h, v)), dict(zip(h, units))


def main():
    tag = sys.argv[1]
    rnd = sys.argv[sys.argv.index("--round") + 1] if "--round" in sys.argv else "r1"
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    # launch list
    lc = os.path.join(src, "launches.csv")
    if os.path.exists(lc):
        rows = list(csv.reader(open(lc)))
        hdr = None
        lines, tot = [], {}
        for r in rows:
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                name = d["Kernel Name"]
                t = float(d["Metric Value"])
                lines.append(f"{t:12.0f} ns  {name[:110]}")
                key = name.split("(")[0]
                tot[key] = tot.get(key, 0.0) + t
        with open(os.path.join(dst, f"{rnd}_launches.txt"), "w") as f:
            f.write("# ncu --metrics gpu__time_duration.sum --clock-control none: every launch of\n"
                    "#   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu\n"
                    "# (cold-cache, serialised; compare shares, not absolute times)\n")
            f.write("\n".join(lines) + "\n\n# total device time per kernel\n")
            s = sum(tot.values())
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
                f.write(f"{v / 1e3:12.1f} us  {100 * v / s:5.1f} %  {k}\n")
    traffic_path = os.path.join(dst, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep") or f.endswith(".raw.csv")):
        vals, units = ncu_raw(os.path.join(src, rep))
        if not vals:
            continue
        name = rep[:-8] if rep.endswith(".ncu-rep") else rep[:-8]
        with open(os.path.join(dst, f"{rnd}_ncu_{name}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none capture {tag}/{rep}\n")
            f.write(f"# kernel: {vals.get('Kernel Name', '?')}\n")
            for k in KEYS:
                if k in vals:
                    f.write(f"{k:80s} {vals[k]} {units.get(k, '')}\n")
            f.write("\n# warp stall samples\n")
            for k, v in sorted(vals.items()):
                if k.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in k and v not in ("0", ""):
                    f.write(f"{k:80s} {v}\n")
        rd, wr = vals.get("dram__bytes_read.sum"), vals.get("dram__bytes_write.sum")
        ur, uw = units.get("dram__bytes_read.sum", ""), units.get("dram__bytes_write.sum", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        try:
            tb = float(rd) * scale.get(ur, 1) + float(wr) * scale.get(uw, 1)
            traffic[f"{name}_{CAPTURE_CONFIG.get(name, 'single_pass_m16_R1_B1024_n1073741824')}"] = tb
            if name == "async":
                traffic["single_pass_m16_R1_B1024_n1073741824"] = tb
        except (TypeError, ValueError):
            pass
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("wrote", sorted(os.listdir(dst)))


if __name__ == "__main__":
    main()

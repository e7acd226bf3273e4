"""Summarise ncu reports: key throughput metrics + top warp stall reasons.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [...]  [--json out.json --key NAME]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(path):
    hdr, units, rows = raw(path)
    res = []
    for vals in rows:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k in KEYS:
            if k in hdr:
                d[k] = (vals[hdr.index(k)], units[hdr.index(k)])
        stalls = []
        for i, name in enumerate(hdr):
            if name.startswith("smsp__average_warp_latency_issue_stalled_") or (
                    name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued")):
                try:
                    stalls.append((float(vals[i].replace(",", "")), name))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        d["top_stalls"] = [(n.split("stalled_")[-1], v) for v, n in stalls[:8]]
        res.append(d)
    return res


def main(argv):
    out, key = None, None
    if "--json" in argv:
        out = argv[argv.index("--json") + 1]
        key = argv[argv.index("--key") + 1] if "--key" in argv else None
    paths = [a for a in argv if a.endswith(".ncu-rep")]
    all_res = {}
    for p in paths:
        for d in summarise(p):
            print(f"== {p} :: {d['kernel']}")
            for k in KEYS:
                if k in d:
                    print(f"   {k:62s} {d[k][0]:>16s} {d[k][1]}")
            print("   top stalls:", ", ".join(f"{n}={v:.1f}" for n, v in d["top_stalls"]))
            all_res[p] = d
    if out:
        with open(out, "w") as fh:
            json.dump(all_res, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])

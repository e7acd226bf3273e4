"""Condense `ncu --set full` reports into the profiles/ summary JSON the bench reads.

    python tools/ncu_profile_json.py --out profiles/r01c_ncu_summary.json --note "..." \
        diff_uvw:fp32:1024,1024,1024=gpurun_out/r7/diff_fp32_1024.ncu-rep ...

Each entry: DRAM bytes per launch against the algorithmic bytes (SURVEY §8d:
5 words/cell advec_u, 10 words/cell diff_uvw), duration, issue/occupancy,
registers, top stall reasons and the hottest SASS instructions by warp-stall
samples (the TMA mbarrier wait shows up there when a kernel is data-starved).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from ncu_summary import summarise  # noqa: E402

from paper_2303_12374_b200.stencils.problem import BYTES_PER_CELL_WORDS as WORDS  # noqa: E402


def _num(pair):
    return float(str(pair[0]).replace(",", ""))


def _scale(pair):
    unit = pair[1]
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
            "s": 1e3}.get(unit, 1.0)


def hot_instructions(path, n=5):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, data = rows[1], rows[2:]
    i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    total = sum(int(r[i_s]) for r in data) or 1
    top = sorted(data, key=lambda r: -int(r[i_s]))[:n]
    return [[r[i_src].strip()[:60], round(int(r[i_s]) / total, 4)] for r in top]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("entries", nargs="+", help="kernel:precision:nx,ny,nz=report.ncu-rep")
    a = ap.parse_args(argv)
    res = {"_note": a.note} if a.note else {}
    for item in a.entries:
        spec, path = item.split("=", 1)
        kernel, precision, grid = spec.split(":")
        nx, ny, nz = (int(x) for x in grid.split(","))
        d = summarise(path)[0]
        rd = _num(d["dram__bytes_read.sum"]) * _scale(d["dram__bytes_read.sum"])
        wr = _num(d["dram__bytes_write.sum"]) * _scale(d["dram__bytes_write.sum"])
        ms = _num(d["gpu__time_duration.sum"]) * _scale(d["gpu__time_duration.sum"])
        alg = nx * ny * nz * WORDS[kernel] * (4 if precision == "fp32" else 8)
        res[f"{kernel}_{precision}_{nx}x{ny}x{nz}"] = {
            "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "algorithmic_bytes": alg,
            "traffic_over_algorithmic": (rd + wr) / alg, "duration_ms": ms,
            "dram_gbs": (rd + wr) / (ms * 1e-3) / 1e9, "algorithmic_gbs": alg / (ms * 1e-3) / 1e9,
            "issue_active_pct": _num(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
            "warps_active_pct": _num(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
            "registers": _num(d["launch__registers_per_thread"]),
            "grid": _num(d["launch__grid_size"]), "block": _num(d["launch__block_size"]),
            "smem_per_block": d["launch__shared_mem_per_block_dynamic"][0] + " " + d["launch__shared_mem_per_block_dynamic"][1],
            "warp_instructions": _num(d["smsp__inst_executed.sum"]),
            "instructions_per_cell": _num(d["smsp__inst_executed.sum"]) * 32 / (nx * ny * nz),
            "top_stalls": d["top_stalls"],
            "hot_sass_by_stall_samples": hot_instructions(path),
            "report": Path(path).name,
        }
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps({k: {kk: v[kk] for kk in ("traffic_over_algorithmic", "algorithmic_gbs", "duration_ms")}
                      for k, v in res.items() if not k.startswith("_")}, indent=1))


if __name__ == "__main__":
    main()

"""Summarize ncu captures into the committed evidence under profiles/.

    python profiles/summarize.py <prof.ncu-rep> <launches.csv> <tag>

writes profiles/<tag>_kernels.md (per-kernel duration, DRAM bytes vs the
algorithmic bytes, issue / warp / shared-memory counters, top stall
reasons), profiles/<tag>_launches.csv (the launch list, one bench step) and
profiles/ncu_traffic.json (dram read+write bytes per launch of the decode /
encode kernels, read by bench.py for roofline.traffic).
"""

from __future__ import annotations

import csv
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
     "smem pipe % of peak"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def load_raw(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    return rows[0], rows[1], rows[2:]


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * scale


def main(rep: str, launches: str, tag: str, config: str = "mib=256,chunk=65536,lanes=32,sb=12") -> None:
    hdr, units, rows = load_raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary `{tag}`", "", f"source: `{rep}` (ncu --set full, --clock-control none)",
             ""]
    traffic = {}
    for r in rows:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        lines.append(f"## {short}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for k, label in KEYS:
            if k in col:
                lines.append(f"| {label} (`{k}`) | {r[col[k]]} {units[col[k]]} |")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.2:
                    stalls.append((v, h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
        lines.append("| top stalls (warps per issue) | " + ", ".join(
            f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:6]) + " |")
        lines.append("")
        rd = to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
        wr = to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
        wf = float(r[col["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]])
        inst = float(r[col["smsp__inst_executed.sum"]])
        for key in ("decode", "encode", "histogram", "compact"):
            # the first launch of each: the bench step's (decode: from the
            # encoder's slot layout; the packed-stream decode comes later)
            if key in short and key not in traffic.get("dram_bytes", {}):
                traffic.setdefault("dram_bytes", {})[key] = rd + wr
                traffic.setdefault("smem_wavefronts", {})[key] = wf
                traffic.setdefault("warp_instructions", {})[key] = inst
    (HERE / f"{tag}_kernels.md").write_text("\n".join(lines) + "\n")
    traffic["config"] = config  # bench.py uses these bytes only for the same workload
    (HERE / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    # launch list: name, duration
    out = [["id", "kernel", "duration_ns"]]
    with open(launches) as f:
        rows = list(csv.reader(f))
    h = None
    for r in rows:
        if "Kernel Name" in r:
            h = {k: i for i, k in enumerate(r)}
            continue
        if h and len(r) == len(h) and r[h["Metric Name"]] == "gpu__time_duration.sum":
            out.append([r[h["ID"]], r[h["Kernel Name"]].split("(")[0], r[h["Metric Value"]]])
    with open(HERE / f"{tag}_launches.csv", "w", newline="") as f:
        csv.writer(f).writerows(out)
    print("wrote", tag)


if __name__ == "__main__":
    main(*sys.argv[1:5])

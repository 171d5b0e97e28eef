"""Summarise an ncu capture and a launch list into profiles/ (run on the CPU box).

    python scripts/ncu_summary.py <tag> <prof.ncu-rep> [<launches.csv>] [--blocks N] [--config 2]

Writes profiles/<tag>_ncu_summary.md (key counters of the captured kernel),
and, when a launch list is given, profiles/<tag>_launches.csv (per-launch
device times, cold and serialised under ncu -- compare shares, not
absolutes) and profiles/traffic.json (dram read+write bytes per launch,
used by bench.py's roofline "traffic").
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock under ncu"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe (LDS/LDG/STG) % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data pipe, LSU wavefronts % of peak"),
    ("l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data pipe, TEX wavefronts % of peak"),
    ("sm__inst_executed_pipe_tex.avg.pct_of_peak_sustained_active", "TEX pipe (texture fetches) % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput % of peak"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe (LOP3/PRMT/SHF) % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe (IMAD) % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__inst_executed_op_shared_ld.sum", "shared loads (warp instr)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "shared-store bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw_metrics(rep: str) -> dict:
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, rows[2][hdr.index("Kernel Name")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("rep")
    ap.add_argument("launches", nargs="?", default=None)
    ap.add_argument("--blocks", type=int, default=1 << 24)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--lookups", type=int, default=160)
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    m, kname = raw_metrics(a.rep)

    def num(key):
        v, u = m.get(key, ("", ""))
        try:
            return float(v.replace(",", "")), u
        except ValueError:
            return None, u

    lines = [f"# ncu summary `{a.tag}`", "", f"Kernel: `{kname}`", "",
             f"Workload: config {a.config}, {a.blocks} blocks per launch "
             f"(algorithmic {32 * a.blocks / 1e6:.1f} MB HBM, {a.lookups} lookups/block).", "",
             "| counter | metric | value | unit |", "|---|---|---|---|"]
    for key, label in KEYS:
        v, u = num(key)
        if v is not None:
            lines.append(f"| {label} | `{key}` | {v:,.3f} | {u} |")
    rd, ru = num("dram__bytes_read.sum")
    wr, wu = num("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = None
    if rd is not None and wr is not None:
        traffic = rd * scale.get(ru, 1) + wr * scale.get(wu, 1)
        lines += ["", f"DRAM traffic per launch: {traffic / 1e6:.1f} MB vs algorithmic "
                      f"{32 * a.blocks / 1e6:.1f} MB ({traffic / (32 * a.blocks):.3f}x)."]
    dur, du = num("gpu__time_duration.sum")
    if dur is not None:
        sec = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(du, 1e-6)
        lines += [f"Plaintext rate under ncu: {16 * a.blocks / sec / 1e9:.1f} GB/s; "
                  f"lookup rate {a.lookups * a.blocks / sec / 1e9:.1f} G/s."]
    with open(os.path.join(PROF, f"{a.tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")

    # launch list: keep our kernels (and totals for the shares)
    if a.launches is None:
        print("\n".join(lines))
        return
    with open(a.launches) as f:
        text = f.read()
    start = text.index('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    kept = [["kernel", "ns"]]
    total = ours = 0.0
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        ns = float(r[vi].replace(",", ""))
        total += ns
        name = r[ki]
        if "gaes::" in name:
            ours += ns
            kept.append([name.split("(")[0], f"{ns:.0f}"])
        else:
            kept.append(["(torch/other) " + name[:60], f"{ns:.0f}"])
    with open(os.path.join(PROF, f"{a.tag}_launches.csv"), "w", newline="") as f:
        csv.writer(f).writerows(kept)

    tpath = os.path.join(PROF, "traffic.json")
    tj = {}
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
    if traffic is not None:
        tj[f"cfg{a.config}"] = round(traffic / 1e9, 4)
        tj["unit"] = "GB per launch (dram__bytes_read.sum + dram__bytes_write.sum)"
        tj[f"cfg{a.config}_source"] = f"profiles/{a.tag}_ncu_summary.md"
    with open(tpath, "w") as f:
        json.dump(tj, f, indent=1)
    print("\n".join(lines))
    print(f"our kernels: {ours / 1e3:.1f} us of {total / 1e3:.1f} us listed")


if __name__ == "__main__":
    main()

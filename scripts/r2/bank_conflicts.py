"""Per-SASS-instruction attribution of shared-memory wavefronts and 'bank
conflicts' from an ncu report captured with --import-source on (source page).

    python scripts/r2/bank_conflicts.py report.ncu-rep [...]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    lines = txt.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main():
    for rep in sys.argv[1:]:
        rs = rows(rep)
        agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
        worst = []
        for r in rs:
            src = r["Source"].strip()
            op = re.split(r"[\s]+", src.lstrip("@!PT0123456789 "))[0] if src else "?"
            op = src.split()[0] if not src.startswith("@") else src.split()[1]
            base = op.split(".")[0]
            key = op if base in ("LDS", "STS", "LDSM", "TEX", "TLD", "LDG", "STG", "ATOMS") else base
            a = agg[key]
            a[0] += 1
            a[1] += num(r["Instructions Executed"])
            a[2] += num(r["L1 Wavefronts Shared"])
            a[3] += num(r["L1 Wavefronts Shared Ideal"])
            a[4] += num(r["L1 Wavefronts Shared Excessive"])
            if num(r["L1 Wavefronts Shared Excessive"]) > 0:
                worst.append((num(r["L1 Wavefronts Shared Excessive"]), r["Address"], src,
                              num(r["L1 Wavefronts Shared"]), num(r["L1 Wavefronts Shared Ideal"])))
        tot = [sum(a[i] for a in agg.values()) for i in range(5)]
        print(f"## {rep}\n")
        print("| opcode | SASS lines | warp instr executed | L1 wavefronts shared | ideal | excessive |")
        print("|---|---|---|---|---|---|")
        for k, a in sorted(agg.items(), key=lambda kv: -kv[1][2]):
            if a[2] or k.startswith(("LDS", "STS", "TEX", "LDG", "STG")):
                print(f"| {k} | {a[0]} | {a[1]:.0f} | {a[2]:.0f} | {a[3]:.0f} | {a[4]:.0f} |")
        print(f"| **total** | {tot[0]} | {tot[1]:.0f} | {tot[2]:.0f} | {tot[3]:.0f} | {tot[4]:.0f} |\n")
        worst.sort(reverse=True)
        print("instructions with excessive shared wavefronts (top 12):\n")
        print("| address | SASS | wavefronts | ideal | excessive |")
        print("|---|---|---|---|---|")
        for e, addr, src, w, i in worst[:12]:
            print(f"| {addr} | `{src}` | {w:.0f} | {i:.0f} | {e:.0f} |")
        print()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Warp-stall reasons per source line of one file in an ncu report (needs -lineinfo).

    python scripts/ncu_stalls.py report.ncu-rep fc_snapkv_tc.cu [line ranges a-b,c-d ...]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, fname = sys.argv[1], sys.argv[2]
    ranges = [tuple(map(int, r.split("-"))) for r in sys.argv[3:]] or [(0, 10 ** 9)]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    path, hdr = None, None
    per = defaultdict(lambda: defaultdict(float))
    for rec in csv.reader(io.StringIO(txt)):
        if not rec:
            continue
        if rec[0] in ("File Name", "File Path"):
            path = rec[1].split("/")[-1]
        elif rec[0] == "Line No":
            hdr = {h: i for i, h in enumerate(rec)}
        elif hdr and rec[0].isdigit() and path == fname:
            ln = int(rec[0])
            for name, i in hdr.items():
                if name.startswith("stall_") and "Not Issued" not in name:
                    try:
                        per[ln][name] += float(rec[i] or 0)
                    except ValueError:
                        pass
    grand = sum(sum(v.values()) for v in per.values()) or 1
    for a, b in ranges:
        agg = defaultdict(float)
        for ln, d in per.items():
            if a <= ln <= b:
                for k, v in d.items():
                    agg[k] += v
        tot = sum(agg.values())
        top = sorted(agg.items(), key=lambda kv: -kv[1])[:6]
        print(f"lines {a}-{b}: {100 * tot / grand:5.1f}% of {fname} samples | " +
              ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.0f}%" for k, v in top))


if __name__ == "__main__":
    main()

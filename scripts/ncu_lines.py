#!/usr/bin/env python
"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).

    python scripts/ncu_lines.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, path, hdr = [], None, None
    for rec in csv.reader(io.StringIO(txt)):
        if not rec:
            continue
        if rec[0] == "File Path":
            path = rec[1].split("/")[-1]
        elif rec[0] == "Line No":
            hdr = {h: i for i, h in enumerate(rec)}
        elif hdr and rec[0].isdigit():
            try:
                n = int(rec[hdr["Warp Stall Sampling (All Samples)"]])
            except (ValueError, IndexError):
                continue
            if n:
                rows.append((n, f"{path}:{rec[0]}", rec[1].strip()[:90]))
    total = sum(r[0] for r in rows) or 1
    for n, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * n / total:5.1f}%  {loc:28s} {src}")


if __name__ == "__main__":
    main()

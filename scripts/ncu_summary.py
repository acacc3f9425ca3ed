#!/usr/bin/env python
"""Summarise an ncu --set full capture into profiles/ncu_<config>.json (+ a text digest).

    python scripts/ncu_summary.py gpurun_out/prof_c2.ncu-rep c2 [alg_bytes_per_launch]

The first argument may also be the `ncu -i <rep> --page raw --csv` export of the report
(a .csv file), which is what the GPU box sends back when the reports are too large.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic",
]


def main():
    rep, config = sys.argv[1], sys.argv[2]
    alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    if rep.endswith(".csv"):
        with open(rep) as f:
            raw = f.read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {"report": rep, "kernels": []}
    for vals in rows[2:]:
        d = {"name": vals[hdr.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        out["kernels"].append(d)
    k0 = out["kernels"][0]

    def gb(key):
        v, u = float(k0[key]["value"]), k0[key]["unit"]
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]
    traffic = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
    out["dram_bytes_per_launch"] = traffic
    if alg:
        out["alg_bytes_per_launch"] = alg
        out["traffic_over_alg"] = traffic / alg
    with open(f"profiles/ncu_{config}.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()

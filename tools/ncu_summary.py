#!/usr/bin/env python3
"""Summarise an ncu --set full report of one step into profiles/ncu_summary.json:
per pass (in launch order) the duration, DRAM read+write bytes, FP64 pipe %, L1TEX %,
warps active %.  usage: ncu_summary.py <report.ncu-rep> <pass,names,in,order> <out.json> [tag]"""
import csv
import io
import json
import subprocess
import sys

rep, names, out = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
tag = sys.argv[4] if len(sys.argv) > 4 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]


def val(row, key):
    i = hdr.index(key)
    u = units[i]
    v = float(row[i])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
             "GB": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9,
             "us": 1e-6, "ms": 1e-3, "s": 1}.get(u, 1)
    return v * scale


res = {"report": rep, "tag": tag, "kernels": {}, "traffic_bytes_per_launch": {}, "fp_pipe_pct": {}}
for name, row in zip(names, data):
    t = val(row, "gpu__time_duration.sum")
    rd = val(row, "dram__bytes_read.sum")
    wr = val(row, "dram__bytes_write.sum")
    k = {"kernel": row[hdr.index("Kernel Name")], "duration_s": t, "dram_read_bytes": rd,
         "dram_write_bytes": wr,
         "fp64_pipe_pct": float(row[hdr.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")]),
         "l1tex_pct": float(row[hdr.index("l1tex__throughput.avg.pct_of_peak_sustained_active")]),
         "dram_pct": float(row[hdr.index("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")]),
         "warps_active_pct": float(row[hdr.index("sm__warps_active.avg.pct_of_peak_sustained_active")]),
         "registers": float(row[hdr.index("launch__registers_per_thread")])}
    res["kernels"][name] = k
    res["traffic_bytes_per_launch"][name] = rd + wr
    fk = "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
    if "<double" in k["kernel"] or "s512" in k["kernel"]:
        res["fp_pipe_pct"][name] = {"pipe": "fp64", "pct": k["fp64_pipe_pct"]}
    else:
        fm = "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"
        res["fp_pipe_pct"][name] = {"pipe": "fma", "pct": float(row[hdr.index(fm)]) if fm in hdr else None}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))

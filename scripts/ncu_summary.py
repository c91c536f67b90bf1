"""Summarise ncu outputs (run here, no GPU): launch list shares + key metrics of full captures."""
import csv
import json
import os
import re
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    agg = defaultdict(lambda: [0.0, 0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000.0 if unit in ("ns", "nsecond") else v * (1000.0 if unit in ("ms", "msecond") else 1.0)
        agg[name][0] += us
        agg[name][1] += 1
    tot = sum(a[0] for a in agg.values())
    out = {k: {"us_total": round(a[0], 2), "launches": a[1], "share": round(a[0] / tot, 4),
               "us_per_launch": round(a[0] / a[1], 2)} for k, a in sorted(agg.items(), key=lambda x: -x[1][0])}
    return {"total_us": round(tot, 1), "kernels": out}


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
           "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
           "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in raw.splitlines() if l.startswith('"')]
    rd = list(csv.reader(lines))
    hdr, units, data = rd[0], rd[1], rd[2:]
    res = []
    for row in data:
        d = dict(zip(hdr, row))
        ent = {"kernel": re.sub(r"\(.*", "", d.get("Kernel Name", "")).strip()[:120]}
        for m in METRICS:
            if m in d:
                u = units[hdr.index(m)]
                ent[m] = d[m] + (" " + u if u else "")
        for k in d:
            if ("pipe_tensor" in k or "tcgen05" in k or "pipe_tc" in k) and "pct_of_peak_sustained_active" in k:
                ent[k] = d[k]
        res.append(ent)
    return res


if __name__ == "__main__":
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    out = {}
    if os.path.exists(os.path.join(d, "launches.csv")):
        out["launch_list"] = launches(os.path.join(d, "launches.csv"))
    for f in sorted(os.listdir(d)):
        if f.endswith(".ncu-rep"):
            out[f] = full(os.path.join(d, f))
    print(json.dumps(out, indent=1))

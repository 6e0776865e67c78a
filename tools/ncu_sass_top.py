#!/usr/bin/env python
"""Hottest SASS instructions of a kernel by stall samples, with the
dominant stall reasons:   python tools/ncu_sass_top.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(out)))
hdr = rd[1]
rows = [dict(zip(hdr, r)) for r in rd[2:] if len(r) == len(hdr)]
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows) or 1
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
for r in rows[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    top = sorted(((int(r[h] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{100*s/tot:5.2f}% {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} " +
          " ".join(f"{n}:{100*v/max(s,1):.0f}" for v, n in top if v))

#!/usr/bin/env python
"""Per-source-line instruction / stall-sample totals of one kernel, grouped
into line ranges (regions) given on the command line.

    python tools/ncu_regions.py rep.ncu-rep file.cuh:A-B=name [file.cuh:C-D=name2 ...]

Lines outside every range are grouped per file.  Reads
`ncu -i rep --page source --csv --print-source cuda,sass`.
"""
import collections
import csv
import io
import subprocess
import sys


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr = None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if len(r) > 2 and r[2] == "-":
            d = dict(zip(hdr, r))
            yield (fname, int(r[0]), int(d.get("Instructions Executed", "0") or 0),
                   int(d.get("Warp Stall Sampling (All Samples)", "0") or 0))


def main(path, specs):
    regs = []
    for sp in specs:
        loc, name = sp.split("=")
        f, rng = loc.split(":")
        a, b = rng.split("-")
        regs.append((f, int(a), int(b), name))
    ins, smp = collections.Counter(), collections.Counter()
    for f, ln, i, s in rows(path):
        key = next((nm for (rf, a, b, nm) in regs if rf == f and a <= ln <= b), f)
        ins[key] += i
        smp[key] += s
    ti, ts = max(sum(ins.values()), 1), max(sum(smp.values()), 1)
    print(f"total warp instructions {ti}, stall samples {ts}")
    for k, v in ins.most_common():
        print(f"  {k:32s} {100 * v / ti:5.1f}% inst {100 * smp[k] / ts:5.1f}% samples")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])

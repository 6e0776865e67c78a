#!/usr/bin/env python
"""Top source lines of one kernel by executed warp instructions and stall
samples, from `ncu -i rep --page source --csv --print-source cuda,sass`.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, rows, tot_i, tot_s = None, [], 0, 0
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "Function Name" or hdr is None:
            continue
        if len(r) > 2 and r[2] == "-":           # source-line aggregate row
            d = dict(zip(hdr, r))
            ins = int(d.get("Instructions Executed", "0") or 0)
            smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            rows.append((ins, smp, fname, int(r[0]), r[1][:90]))
            tot_i += ins
            tot_s += smp
    rows.sort(reverse=True)
    print(f"total warp instructions {tot_i}, samples {tot_s}")
    for ins, smp, f, ln, src in rows[:top]:
        print(f"{100*ins/max(tot_i,1):5.1f}% inst {100*smp/max(tot_s,1):5.1f}% smp  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

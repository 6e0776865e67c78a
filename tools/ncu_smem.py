#!/usr/bin/env python
"""Source lines of one kernel ranked by shared-memory wavefronts (LDS/STS +
bank-conflict excess), from `ncu -i rep --page source --csv --print-source
cuda,sass`.   python tools/ncu_smem.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, rows = None, None, []
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
            g = lambda k: float(d.get(k, "0") or 0)
            rows.append((g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Excessive"),
                         g("Warp Stall Sampling (All Samples)"), fname, int(r[0]), r[1][:80]))
    tw = sum(x[0] for x in rows) or 1
    te = sum(x[1] for x in rows)
    print(f"shared wavefronts {tw:.3e}, excessive {te:.3e} ({100 * te / tw:.1f}%)")
    for w, e, s, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * w / tw:5.1f}% wf  excess {100 * e / tw:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

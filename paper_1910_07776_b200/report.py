"""Strip-chart data ("we show the AC/EX ratios in
strip charts", P:240 / P:274 inputs ordered by size).

Host-side formatting of results the GPU path already produced: per test case
of a batch evaluated with `want_ex=True`, the row
(experiment, learner, optimization, program, input_id, run_id, ratio) with
ratio = AC / EX, AC = rt_before / rt_after (reading D2) and EX the clamped
prediction the kernels scored (R7).  Rows are sorted by (experiment, learner,
optimization, program, input index, run, version), the input index following
the dataset's input order, which the generator and Table 1 give by
increasing size ("input sizes increase from left to right").  Export with 17
significant digits so a re-parse reproduces every ratio bit-exactly.
"""
from __future__ import annotations

import csv
import io

import numpy as np

HEADER = ["experiment", "learner", "optimization", "program", "input_id", "run_id", "ratio"]


def ratio_rows(ds, result, experiment=None, learner: str = "linreg", input_names=None) -> list:
    """Rows of every scored test case of `result` (a Context.evaluate(...,
    want_ex=True) dict over scenarios [0, S)).  experiment: per-scenario
    labels (e.g. cfg.scenarios.experiment) or None (scenario index)."""
    ex = result["ex"]
    S, O, GK = ex.shape
    G = GK // 32
    IR = ds.n_inputs * ds.n_runs
    rt = ds.runtime_ms
    names = ds.opt_names or [f"opt{o}" for o in range(O)]
    progs = ds.program_names or [f"p{p}" for p in range(ds.n_programs)]
    rows = []
    for s in range(S):
        e_lab = int(experiment[s]) if experiment is not None else s
        for o in range(O):
            nz = np.nonzero(ex[s, o])[0]
            for gk in nz:
                g, k = int(gk) >> 5, int(gk) & 31
                p, rest = divmod(g, IR)
                i, r = divmod(rest, ds.n_runs)
                b = int(ds.opt_bit[p, o])
                v = ((k >> b) << (b + 1)) | (k & ((1 << b) - 1))
                ac = rt[g * 64 + v] / rt[g * 64 + (v | (1 << b))]
                rows.append((e_lab, learner, names[o], progs[p], i, r, v,
                             (input_names or {}).get(i, f"in{i}"), ac / float(ex[s, o, gk])))
    rows.sort(key=lambda t: t[:7])
    return [dict(experiment=t[0], learner=t[1], optimization=t[2], program=t[3], input_id=t[7], run_id=t[5],
                 ratio=t[8]) for t in rows]


def export_ratios_csv(rows) -> str:
    """CSV text with HEADER and one row per test case (ratio as repr: 17 digits)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(HEADER)
    for r in rows:
        w.writerow([r["experiment"], r["learner"], r["optimization"], r["program"], r["input_id"], r["run_id"],
                    repr(float(r["ratio"]))])
    return buf.getvalue()


def parse_ratios_csv(text: str) -> list:
    rd = csv.reader(io.StringIO(text))
    hdr = next(rd)
    assert hdr == HEADER, hdr
    return [dict(experiment=int(a), learner=b, optimization=c, program=d, input_id=e, run_id=int(f), ratio=float(g))
            for a, b, c, d, e, f, g in rd]

"""NEXT-3 strip-chart data (report.py) and the 6-input Barnes-Hut config
(BH6, Table 1).  CPU: the oracle's own results feed the export."""
import numpy as np
import pytest

import gen
import oracle
from paper_1910_07776_b200 import report


@pytest.fixture(scope="module")
def bh6():
    cfg = gen.make_config("BH6")
    first, count = 0, 30                        # Exp 1 and Exp 2 instantiations
    ref = oracle.evaluate(cfg.dataset, cfg.scenarios, first, count, want_ex=True)
    return cfg, ref


def test_bh6_config_shape():
    cfg = gen.make_config("BH6")
    ds, sc = cfg.dataset, cfg.scenarios
    assert (ds.n_programs, ds.n_inputs, ds.n_runs, ds.n_groups) == (1, 6, 3, 18)
    # Table 2 Exp 1-4 instantiations for one program: 18 + 18 + 18 + 6*5*3
    assert sc.n_splits == 144
    assert [int((sc.experiment == e).sum()) for e in (1, 2, 3, 4)] == [18, 18, 18, 90]


def test_ratio_rows_are_the_scored_cases(bh6):
    cfg, ref = bh6
    rows = report.ratio_rows(cfg.dataset, ref, cfg.scenarios.experiment[:30], "linreg")
    opt = ref["opt"]
    predicted = (opt["n_train"] > 0) & (opt["n_test"] > 0)
    assert len(rows) == int(opt["n_test"][predicted].sum())
    # per (scenario, opt) the ratios sum to the row's sum_ratio, min / max agree
    by = {}
    k = 0
    for s in range(30):
        for o in range(cfg.dataset.n_opt_ids):
            if predicted[s, o]:
                by[(s, o)] = opt["sum_ratio"][s, o]
    tot = sum(r["ratio"] for r in rows)
    assert abs(tot - sum(by.values())) <= 1e-9 * abs(tot)
    # sorted by (experiment, learner, optimization, program, input, run)
    keys = [(r["experiment"], r["learner"], r["optimization"], r["program"], r["input_id"], r["run_id"]) for r in rows]
    assert keys == sorted(keys)


def test_ratio_export_round_trip_bit_exact(bh6):
    cfg, ref = bh6
    rows = report.ratio_rows(cfg.dataset, ref, cfg.scenarios.experiment[:30])
    text = report.export_ratios_csv(rows)
    back = report.parse_ratios_csv(text)
    assert [r["ratio"] for r in back] == [r["ratio"] for r in rows]
    assert report.export_ratios_csv([]).strip() == ",".join(report.HEADER)


def test_perfect_predictor_ratios_are_one(bh6):
    """substituting the ground truth for EX gives every ratio 1."""
    cfg, ref = bh6
    ex = ref["ex"].copy()
    ds = cfg.dataset
    G, O = ds.n_groups, ds.n_opt_ids
    rt = ds.runtime_ms
    for s, o, gk in zip(*np.nonzero(ex)):
        g, kk = gk >> 5, gk & 31
        b = int(ds.opt_bit[g // (ds.n_inputs * ds.n_runs), o])
        v = ((kk >> b) << (b + 1)) | (kk & ((1 << b) - 1))
        ex[s, o, gk] = rt[g * 64 + v] / rt[g * 64 + (v | (1 << b))]
    rows = report.ratio_rows(ds, dict(ex=ex), None)
    assert rows and all(r["ratio"] == 1.0 for r in rows)

#!/usr/bin/env python
"""Small evaluations of every kernel family for compute-sanitizer (SURVEY §4
T5): python tools/sanitize_cases.py CASE, CASE in c1 c2 c3 c4 ibk m5 fuse c5
sweep fit.  Each runs the C-ABI path once on a small batch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402
from paper_1910_07776_b200 import Context, default_params  # noqa: E402


def run(name, first, count, **prm):
    cfg = gen.make_config(*name) if isinstance(name, tuple) else gen.make_config(name)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    r = ctx.evaluate(first, count, params=default_params(**prm), want_ex=True, want_recs=True)
    ctx.close()
    return r


case = sys.argv[1]
if case == "c1":
    run("C1", 0, 64)
elif case == "c2":
    run("C2", 0, 240)
elif case == "c3":
    cfg = gen.make_config("C3", n_splits=1000)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    ctx.evaluate(0, 1000, want_ex=True, want_recs=True)
    ctx.close()
elif case == "c4":
    cfg = gen.make_config("C4", n_splits=6, n_programs=96)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    ctx.evaluate(0, 6, want_ex=True, want_recs=True)
    ctx.close()
elif case == "ibk":
    run("C1", 0, 64, learner=1)
    cfg = gen.make_config("C4", n_splits=2, n_programs=96)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    ctx.evaluate(0, 2, params=default_params(learner=1))
    ctx.close()
elif case == "m5":
    run("C1", 0, 16, learner=2)
elif case == "fuse":
    os.environ["SPEEDREC_FUSE_RANK"] = "1"
    run("C1", 0, 64)
elif case == "c5":
    cfg = gen.make_config("C5", n_masks_k=6)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    ctx.evaluate(0, cfg.scenarios.n_scenarios, params=default_params(top_k=8), want_masks=True)
    ctx.close()
elif case == "sweep":
    cfg = gen.make_config("C3", n_splits=200)
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    ctx.sweep(np.linspace(0.9, 1.3, 8), np.array([1, 3]), 0, 200)
    ctx.close()
elif case == "fit":
    cfg = gen.make_config("C1")
    ctx = Context(0)
    ctx.load(cfg.dataset)
    ctx.define_scenarios(cfg.scenarios)
    ctx.fit(17)
    ctx.close()
print("ok", case)

#!/usr/bin/env python
"""C4 (large-batch path): EX error vs the oracle with and without the
refinement pass of k_fit_big (sr_params.refine_steps), on sampled full-lattice
splits, with the oracle's kappa^ per fit.  Decides whether the refinement can
be conditional on a kappa estimate."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
from paper_1910_07776_b200 import Context, default_params  # noqa: E402

cfg = gen.make_config("C4", n_splits=10_000_000)
idx = [k * 156250 for k in range(16)]
ctx = Context(0)
ctx.load(cfg.dataset)
ctx.define_scenarios(cfg.scenarios)
res = {}
for rs in (2, 1, 0):
    res[rs] = [ctx.evaluate(s, 1, params=default_params(refine_steps=rs), want_ex=True)["ex"] for s in idx]
ctx.close()
with ThreadPoolExecutor(16) as pool:
    refs = list(pool.map(lambda s: oracle.evaluate(cfg.dataset, cfg.scenarios, s, 1, want_ex=True, n_threads=1,
                                                    want_kappa=True), idx))
for rs, exs in res.items():
    worst = 0.0
    for e, r in zip(exs, refs):
        m = r["ex"] != 0
        worst = max(worst, float((np.abs(e[m] - r["ex"][m]) / np.abs(r["ex"][m])).max()))
    print(f"refine_steps={rs}: worst EX rel err {worst:.3e}")
print("kappa^ range", min(float(np.nanmin(r["kappa"])) for r in refs), max(float(np.nanmax(r["kappa"])) for r in refs))

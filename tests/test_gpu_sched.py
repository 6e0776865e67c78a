"""The launch-scheduling choices of round 2 change when work runs, never what
it computes (DESIGN.md §5.2 work units, §5.8 launch groups, §5.9 IBK grid):

* dynamic work units of k_fit_warp (SPEEDREC_DYN_UNITS=0: static stride),
  LS on C3 / C2 and M5P teams on C2;
* the fork-join launch groups of the prefix-shared mask path
  (SPEEDREC_GROUP_STREAMS=1: sequential launches on the context stream).

Each pair of bench.py runs (same batch, one process per setting: the knobs
are read once per process) must give byte-identical score tables and totals.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
QUICK = ["--steps", "2", "--warmup", "1", "--no-e2e", "--no-extra", "--no-cpu-baseline"]


def _bench(args, dump, **env_over):
    env = dict(os.environ, **env_over)
    res = subprocess.run([sys.executable, "bench.py"] + args + QUICK + ["--dump-tables", dump], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    return line, np.load(dump)


def _same(a, b, keys):
    for k in keys:
        assert a[k].tobytes() == b[k].tobytes(), k


@pytest.mark.parametrize("args", [["--config", "C3", "--splits", "20000"], ["--config", "C2"],
                                  ["--config", "C2", "--learner", "m5"]], ids=["C3", "C2", "C2-m5"])
def test_dynamic_units_equal_static_stride(tmp_path, args):
    _, t0 = _bench(args, str(tmp_path / "static.npz"), SPEEDREC_DYN_UNITS="0")
    _, t1 = _bench(args, str(tmp_path / "dynamic.npz"), SPEEDREC_DYN_UNITS="1")
    _same(t0, t1, ("opt", "scn", "totals"))


def test_launch_groups_equal_sequential_launches(tmp_path):
    args = ["--config", "C5", "--masks-k", "12"]
    l0, t0 = _bench(args, str(tmp_path / "seq.npz"), SPEEDREC_GROUP_STREAMS="1")
    l1, t1 = _bench(args, str(tmp_path / "grp.npz"), SPEEDREC_GROUP_STREAMS="8")
    _same(t0, t1, ("masks", "top", "totals"))
    assert l0["top_masks_head"] == l1["top_masks_head"]

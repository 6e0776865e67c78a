"""T4: the N-rank run of bench.py -- scenario shards per
rank, CUDA path on every rank, score tables gathered to rank 0 -- gives
byte-identical tables to the 1-rank run of the same global batch.

Both ranks share the one GPU of the test box and exchange over gloo
(SPEEDREC_DIST_BACKEND=gloo), so bench.py's world > 1 branch (sharding,
gather, all-reduce of totals and timing, C5 top-K merge) runs end to end;
on a multi-GPU node the same code runs with NCCL.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import gen
import oracle
from tests.parity import compare

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
QUICK = ["--steps", "2", "--warmup", "1", "--no-e2e", "--no-extra", "--no-cpu-baseline"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(nproc, args, dump):
    env = dict(os.environ, SPEEDREC_DIST_BACKEND="gloo")
    if nproc == 1:
        cmd = [sys.executable, "bench.py"]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", f"--master-port={_port()}", "bench.py"]
    res = subprocess.run(cmd + args + QUICK + ["--gpus", str(nproc), "--dump-tables", dump], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    return line, np.load(dump)


def test_c3_two_ranks_equal_one_rank(tmp_path):
    S = 20000
    l2, t2 = _bench(2, ["--config", "C3", "--splits", str(S)], str(tmp_path / "two.npz"))
    l1, t1 = _bench(1, ["--config", "C3", "--splits", str(2 * S)], str(tmp_path / "one.npz"))
    assert l2["n_gpus"] == 2 and l2["gather"]["collective"] == "all_gather_into_tensor"
    assert l2["gather"]["bytes_per_rank"] == S * (6 * 56 + 16)
    assert t2["opt"].tobytes() == t1["opt"].tobytes()
    assert t2["scn"].tobytes() == t1["scn"].tobytes()
    assert np.array_equal(t2["totals"], t1["totals"])
    assert l2["pooled_ratio"] == l1["pooled_ratio"]
    # rank 1's shard, sampled, against the oracle
    from paper_1910_07776_b200.speedrec import OPT_SCORE_DTYPE, SCN_SCORE_DTYPE
    cfg = gen.make_config("C3", n_splits=2 * S)
    opt = t2["opt"].view(OPT_SCORE_DTYPE).reshape(2 * S, 6)
    scn = t2["scn"].view(SCN_SCORE_DTYPE)
    idx = np.r_[S, S + 1, np.random.default_rng(2).integers(S, 2 * S, size=40), 2 * S - 1]
    refs = [oracle.evaluate(cfg.dataset, cfg.scenarios, int(s), 1) for s in idx]
    print("C3 rank-1 shard vs oracle", compare(
        dict(opt=opt[idx], scn=scn[idx]),
        dict(opt=np.concatenate([r["opt"] for r in refs]), scn=np.concatenate([r["scn"] for r in refs]))))


def test_c5_two_ranks_stratified_equal_one_rank(tmp_path):
    args = ["--config", "C5", "--masks-k", "10"]
    l2, t2 = _bench(2, args, str(tmp_path / "two.npz"))
    l1, t1 = _bench(1, args, str(tmp_path / "one.npz"))
    assert t2["masks"].tobytes() == t1["masks"].tobytes()
    assert list(t2["top"]) == list(t1["top"]) and l2["top_masks_head"] == l1["top_masks_head"]
    assert np.array_equal(t2["totals"], t1["totals"])
    # the global mask table against the oracle's per-mask sums on sampled masks
    cfg = gen.make_config("C5", n_masks_k=10)
    folds = cfg.scenarios.n_splits
    rows = t2["masks"].view(oracle.MASK_SCORE_DTYPE)
    for m in (0, 1, 513, 1023):
        r = oracle.evaluate(cfg.dataset, cfg.scenarios, m * folds, folds)
        ref = oracle.aggregate_masks(r["opt"], r["scn"], folds, first_mask=m, top_k=1)[0][0]
        assert tuple(rows[m]) == tuple(ref), m

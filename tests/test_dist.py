"""Multi-process (world_size 2, gloo, CPU) tests of the sharding and exchange
logic the N-GPU bench uses (paper_1910_07776_b200/dist.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_07776_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # pooled totals: exact integer sums
        tot = torch.tensor([10 + rank, 20, 3 * rank, 1], dtype=torch.int64)
        red = D.reduce_totals(tot, dist)
        # timing: max over ranks
        mx = D.max_over_ranks(1.5 + rank, dist)
        # top-k merge: rank 0 owns masks 0..3, rank 1 masks 4..7
        correct = {0: 5, 1: 9, 2: 9, 3: 1, 4: 9, 5: 2, 6: 7, 7: 9}
        mine = [m for m in correct if (m < 4) == (rank == 0)]
        mine.sort(key=lambda m: (-correct[m], m))
        ids = mine[:3]
        top = D.merge_top_masks(ids + [-1], [correct[m] for m in ids] + [0], 4, dist)
        q.put((rank, red.tolist(), mx, top.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, red, mx, top in res:
        assert red == [21, 40, 3, 2]
        assert mx == 2.5
        assert top == [1, 2, 4, 7]          # ties on 9 correct broken by mask id (O8)


def test_stratified_mask_partition_covers_and_balances():
    for k, world in ((10, 8), (12, 4), (20, 8), (5, 2)):
        parts = [D.stratified_masks(k, r, world) for r in range(world)]
        allm = np.sort(np.concatenate(parts))
        assert np.array_equal(allm, np.arange(1 << k))
        # work proxy per mask: p^3/6 + p^2 + p with p = popcount + 1
        cost = []
        for q in parts:
            p = np.array([bin(int(x)).count("1") + 1 for x in q], dtype=np.float64)
            cost.append((p ** 3 / 6 + p ** 2 + p).sum())
            assert (np.diff(q) > 0).all()               # ascending: local order = global order
        cost = np.array(cost)
        assert cost.max() / cost.mean() - 1 < (1e-4 if k >= 16 else 3e-2 if k >= 10 else 0.15), (k, world, cost)
    # contiguous blocks are measurably worse (the reason for stratifying)
    blocks = np.array_split(np.arange(1 << 20), 8)
    pcs = [np.array([bin(int(x)).count("1") for x in b[:: 64]]).mean() for b in blocks]
    assert max(pcs) - min(pcs) > 2


def _c5_worker(rank, world, port, q):
    """Per-rank C5 evaluation of its stratified masks (the oracle stands in
    for the GPU here), local top-K -> global ids -> all-gather merge."""
    import gen
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = gen.make_config("C5", n_masks_k=5)
        sc = cfg.scenarios
        masks = D.stratified_masks(5, rank, world)
        sc.all_subsets_k = 0
        sc.feature_masks = np.stack([masks.astype(np.uint64), np.zeros(len(masks), np.uint64)], 1)
        sc.n_masks = len(masks)
        folds = sc.n_splits
        ref = oracle.evaluate(cfg.dataset, sc, 0, len(masks) * folds, n_threads=2)
        rows, top_local = oracle.aggregate_masks(ref["opt"], ref["scn"], folds, top_k=6)
        top = D.local_top_to_global(np.r_[top_local, -np.ones(6 - len(top_local), np.int64)], masks)
        corr = [int(rows["n_correct"][i]) if i >= 0 else 0 for i in np.r_[top_local, -np.ones(6 - len(top_local), np.int64)]]
        merged = D.merge_top_masks(top.tolist(), corr, 6, dist)
        q.put((rank, merged.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_c5_stratified_top_k_equals_single_process():
    import gen
    import oracle
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_c5_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = gen.make_config("C5", n_masks_k=5)
    folds = cfg.scenarios.n_splits
    ref = oracle.evaluate(cfg.dataset, cfg.scenarios, 0, cfg.scenarios.n_scenarios)
    _, want = oracle.aggregate_masks(ref["opt"], ref["scn"], folds, top_k=6)
    for _, got in res:
        assert got == want.tolist()


def test_shard_ranges_partition():
    for total, world, align in ((1000, 2, 1), (1003, 4, 1), (128 * 1024, 8, 128), (64, 8, 1)):
        seen = []
        for r in range(world):
            a, n = D.strong_range(total, r, world, align)
            assert a % align == 0 and n % align == 0
            seen.extend(range(a, a + n))
        assert seen == list(range(total // align * align))
    assert D.weak_range(1000, 3) == (3000, 1000)


def test_topk_key_order_matches_rule():
    keys = [D.topk_key(c, m) for c, m in ((5, 3), (9, 7), (9, 2), (0, 0))]
    order = np.argsort(keys)[::-1]
    assert list(order) == [2, 1, 0, 3]


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1910_07776_b200.speedrec import OPT_SCORE_DTYPE
        # weak scaling: rank r holds rows of scenarios [r*S, (r+1)*S) of one table
        full = _table(2 * 50)
        mine = full[rank * 50 * 6:(rank + 1) * 50 * 6]
        t = torch.from_numpy(mine.view(np.uint8).copy())
        g = D.gather_rows(t, dist).numpy()
        # C5: stratified mask lists of unequal length, padded, scattered back
        allm = [D.stratified_masks(5, r, world) for r in range(world)]
        rows = np.arange(32 * 16, dtype=np.int64).astype(np.uint8).reshape(32, 16)
        pad = np.zeros((max(len(m) for m in allm), 16), np.uint8)
        pad[:len(allm[rank])] = rows[allm[rank]]
        gm = D.gather_rows(torch.from_numpy(pad.reshape(-1)), dist).numpy()
        q.put((rank, g.tobytes() == full.view(np.uint8).tobytes(),
               D.scatter_mask_rows(gm, allm, 32).tobytes() == rows.tobytes(),
               D.pooled_ratio(g) == D.pooled_ratio(full.view(np.uint8))))
    finally:
        dist.destroy_process_group()


def _table(n_scn, O=6):
    from paper_1910_07776_b200.speedrec import OPT_SCORE_DTYPE
    rng = np.random.default_rng(4)
    o = np.zeros(n_scn * O, dtype=OPT_SCORE_DTYPE)
    o["n_test"] = rng.integers(0, 40, size=o.size)
    o["sum_ratio"] = o["n_test"] * rng.uniform(0.5, 1.5, size=o.size)
    o["fp_train"] = rng.integers(0, 2**63, size=o.size)
    return o


def test_gloo_world2_score_table_gather_is_byte_identical():
    # one all_gather_into_tensor of fixed-size rows per table; the
    # gathered table (rank order = scenario order) equals the 1-process table
    # byte for byte, and the FP pooled statistic computed from it is the same.
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, same_masks, same_pool in res:
        assert same and same_masks and same_pool, (rank, same, same_masks, same_pool)

"""Multi-GPU plumbing of the scenario-sharded path.

One process per GPU (torchrun).  Scenarios are independent, so there is no
collective on the data path; the exchange steps come after it:
  (a) the per-scenario score tables (fixed-size sr_opt_score / sr_scn_score
      rows, or C5's sr_mask_score rows) gathered to rank 0 with ONE
      all_gather_into_tensor each (NCCL over NVLink on GPUs), in rank order =
      scenario order, so the N-GPU table is byte-identical to the 1-GPU one;
  (b) the pooled integer totals of A7 ("per config" sign accuracy,
      recommendation hits), an exact integer all-reduce;
  (c) for C5 the global top-K mask ranking, an exact integer-key merge.
FP statistics over scenarios are computed on rank 0 from the gathered table
(`pooled_ratio`), so they do not depend on the GPU count either.  Timing is
the max over ranks.  Works with "nccl" on GPUs and "gloo" on CPU
(tests/test_dist.py, tests/test_gpu_dist.py).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def weak_range(per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling: rank r evaluates scenarios [r*S, (r+1)*S) of the global batch."""
    return rank * per_rank, per_rank


def strong_range(total: int, rank: int, world: int, align: int = 1) -> Tuple[int, int]:
    """Strong scaling: split [0, total) into contiguous, `align`-aligned shards
    (align = n_splits for whole feature masks).  Shard sizes differ by <= align."""
    units = total // align
    lo = units * rank // world
    hi = units * (rank + 1) // world
    return lo * align, (hi - lo) * align


def stratified_masks(k: int, rank: int, world: int) -> np.ndarray:
    """C5 partition: sort the 2^k feature masks by (popcount,
    mask) and give the j-th to rank j mod W, so every rank gets the same
    number of masks of each size to within one (a fit's cost grows with the
    mask's popcount; contiguous or mod-W blocks leave the busiest rank ~36 %
    above the mean at W = 8).  Returns this rank's masks, ascending, so local
    index order is global mask order (ties in the top-K rule stay exact)."""
    m = np.arange(1 << k, dtype=np.int64)
    pc = np.zeros_like(m)
    for b in range(k):
        pc += (m >> b) & 1
    order = np.lexsort((m, pc))
    return np.sort(m[order[rank::world]])


def local_top_to_global(top_local: np.ndarray, masks: np.ndarray) -> np.ndarray:
    """Map the library's local top-K indices (into this rank's mask list) to
    global mask ids; -1 padding stays -1."""
    top_local = np.asarray(top_local, dtype=np.int64)
    out = np.full(len(top_local), -1, dtype=np.int64)
    ok = top_local >= 0
    out[ok] = masks[top_local[ok]]
    return out


def reduce_totals(totals, dist) -> "torch.Tensor":
    """Sum the 4 pooled int64 totals over ranks (exact)."""
    t = totals.clone()
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def max_over_ranks(value: float, dist, device="cpu") -> float:
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def topk_key(n_correct: int, mask_id: int) -> int:
    """The kernel's ranking key: more correct first, then smaller id."""
    return (int(n_correct) << 32) | (0xFFFFFFFF - int(mask_id))


def merge_top_masks(local_ids, local_correct, k: int, dist, device="cpu") -> np.ndarray:
    """Global top-k mask ids from each rank's local top-k (ids -1 padded):
    all-gather the (key) lists and select the k largest integer keys."""
    import torch
    keys = np.array([topk_key(c, m) if m >= 0 else 0 for m, c in zip(local_ids, local_correct)],
                    dtype=np.uint64).view(np.int64)
    t = torch.from_numpy(keys.copy()).to(device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(out, t)
        t = torch.cat(out)
    allk = t.cpu().numpy().view(np.uint64)
    allk = np.sort(allk[allk != 0])[::-1][:k]
    ids = (0xFFFFFFFF - (allk & np.uint64(0xFFFFFFFF))).astype(np.int64)
    return np.concatenate([ids, -np.ones(k - len(ids), dtype=np.int64)])


def gather_rows(rows, dist):
    """All-gather one rank's fixed-size score rows (a 1-D uint8 tensor of
    equal length on every rank: weak scaling gives each rank the same number
    of scenarios) into [world * len] in rank order, with ONE
    all_gather_into_tensor.  World 1: the rows themselves."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return rows
    out = torch.empty(rows.numel() * dist.get_world_size(), dtype=rows.dtype, device=rows.device)
    dist.all_gather_into_tensor(out, rows.contiguous())
    return out


def scatter_mask_rows(gathered, masks_of_rank, n_masks: int, row_bytes: int = 16):
    """C5: the gathered mask rows of every rank (rank r's rows for its
    stratified masks, padded to the longest list) -> one [n_masks] table in
    global mask order (numpy uint8 [n_masks * row_bytes])."""
    g = np.asarray(gathered).reshape(len(masks_of_rank), -1)
    out = np.zeros((n_masks, row_bytes), dtype=np.uint8)
    for r, m in enumerate(masks_of_rank):
        out[m] = g[r, :len(m) * row_bytes].reshape(len(m), row_bytes)
    return out.reshape(-1)


def pooled_ratio(opt_rows) -> dict:
    """Per-config FP statistics from a full (gathered) sr_opt_score table, in
    scenario order: sum of AC/EX over all test cases (math.fsum: correctly
    rounded, so the value is one function of the table) and its mean."""
    import math
    from .speedrec import OPT_SCORE_DTYPE
    o = np.asarray(opt_rows).view(OPT_SCORE_DTYPE).ravel()
    n = int(o["n_test"].astype(np.int64).sum())
    s = math.fsum(o["sum_ratio"][o["n_test"] > 0].tolist())
    return {"sum_ratio": s, "cases": n, "mean_ratio": s / n if n else None}

"""Multi-GPU plumbing of the scenario-sharded path.

One process per GPU (torchrun).  Scenarios are independent, so the only
exchange steps are (a) the pooled integer totals of A7 ("per config" sign
accuracy, recommendation hits) and (b) for C5 the global top-K mask ranking,
both exact because they are integer reductions / integer-key selections.
Timing is the max over ranks.  Works with the "nccl" backend on GPUs and the
"gloo" backend on CPU (tests/test_dist.py).
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

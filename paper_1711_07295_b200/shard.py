"""Multi-rank plumbing of the row-partitioned join (one process per GPU).

The self-join's pair space is split into contiguous row blocks balanced on
the length-window pair count (``ssjb_partition_rows``); every rank joins its
block independently against a full replica (``ssjb_join_rows``) -- no
collective on the data path.  The only exchange is the final gather of each
rank's sorted result run and counters to rank 0, which merges the runs into
the reference's global (id_r, id_s) order and sums the counters (counters of
disjoint row blocks add up exactly; reference tests/test_parallel.cpp:37-59).
"""
from __future__ import annotations

import heapq

import numpy as np

COUNTER_KEYS = ("candidates", "pruned_length", "pruned_positional", "pruned_suffix", "pruned_bitmap",
                "bitmap_tested", "filter_evaluations", "verified", "matched")


def merge_runs(runs):
    """k-way merge of (id_r, id_s)-sorted pair arrays (structured PAIR_DTYPE)."""
    runs = [r for r in runs if len(r)]
    if not runs:
        from .ssjoin import PAIR_DTYPE
        return np.zeros(0, dtype=PAIR_DTYPE)
    if len(runs) == 1:
        return runs[0]
    allp = np.concatenate(runs)
    key = (allp["id_r"].astype(np.uint64) << np.uint64(32)) | allp["id_s"].astype(np.uint64)
    # runs are individually sorted; a stable argsort of the concatenation is the merge
    return allp[np.argsort(key, kind="stable")]


def merge_counters(parts):
    out = {k: 0 for k in COUNTER_KEYS}
    sat = 0
    for counters, saturated in parts:
        for k in COUNTER_KEYS:
            out[k] += int(counters.get(k, 0))
        sat += int(saturated)
    return out, sat


def gather_to_root(pairs, counters, saturated, group=None):
    """Gather every rank's (pairs, counters, saturated) to rank 0 and merge.
    Returns (pairs, counters, saturated) on rank 0 and None elsewhere."""
    import torch.distributed as dist
    rank = dist.get_rank()
    world = dist.get_world_size()
    payload = (pairs.tobytes(), counters, int(saturated))
    bucket = [None] * world if rank == 0 else None
    dist.gather_object(payload, bucket, dst=0, group=group)
    if rank != 0:
        return None
    from .ssjoin import PAIR_DTYPE
    runs = [np.frombuffer(b, dtype=PAIR_DTYPE) for b, _, _ in bucket]
    merged_counters, sat = merge_counters([(c, s) for _, c, s in bucket])
    return merge_runs(runs), merged_counters, sat


def heap_merge(runs):
    """Reference-style k-way merge (used by tests to cross-check merge_runs)."""
    it = heapq.merge(*[[(int(p["id_r"]), int(p["id_s"]), int(p["overlap"])) for p in r] for r in runs])
    return list(it)

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


def merge_row_shards(lib, runs):
    """Canonical merge of ascending row-block results through the library's
    O(pairs) multi-threaded merge (ssjb_merge_row_shards)."""
    import ctypes as C
    from .ssjoin import PAIR_DTYPE
    runs = [np.ascontiguousarray(r) for r in runs]
    total = sum(len(r) for r in runs)
    out = np.empty(total, dtype=PAIR_DTYPE)
    if total == 0:
        return out
    ptrs = (C.c_void_p * len(runs))(*[r.ctypes.data if len(r) else None for r in runs])
    counts = (C.c_size_t * len(runs))(*[len(r) for r in runs])
    if lib.ssjb_merge_row_shards(ptrs, counts, len(runs), out.ctypes.data) != 0:
        raise RuntimeError("ssjb_merge_row_shards failed")
    return out


def gather_to_root_shm(pairs, counters, saturated, lib, group=None, tag="ssjb"):
    """Single-node gather through /dev/shm: every rank writes its sorted run to
    a shared-memory file, rank 0 maps all of them (no copy through a socket)
    and merges them with the library's row-shard merge.  Counters travel as
    one int64 all-gather.  Returns (pairs, counters, saturated) on rank 0."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    world = dist.get_world_size()
    head = torch.tensor([len(pairs), int(saturated)] + [int(counters.get(k, 0)) for k in COUNTER_KEYS],
                        dtype=torch.int64)
    heads = [torch.zeros_like(head) for _ in range(world)]
    dist.all_gather(heads, head, group=group)
    path = f"/dev/shm/{tag}_{rank}.bin"
    if len(pairs):
        np.ascontiguousarray(pairs).tofile(path)
    dist.barrier(group=group)
    out = None
    if rank == 0:
        from .ssjoin import PAIR_DTYPE
        runs = []
        for r in range(world):
            c = int(heads[r][0])
            if r == 0:
                runs.append(pairs)
            elif c:
                runs.append(np.memmap(f"/dev/shm/{tag}_{r}.bin", dtype=PAIR_DTYPE, mode="r", shape=(c,)))
        merged = merge_row_shards(lib, runs)
        merged_counters, sat = merge_counters(
            [({k: int(h[2 + i]) for i, k in enumerate(COUNTER_KEYS)}, int(h[1])) for h in heads])
        out = (merged, merged_counters, sat)
    dist.barrier(group=group)
    if len(pairs):
        import os
        os.unlink(path)
    return out


def gather_to_root(pairs, counters, saturated, group=None):
    """Gather every rank's (pairs, counters, saturated) to rank 0 and merge.
    Count-first: the pair counts and counters travel as one small int64
    all-gather, then each rank's pairs go to rank 0 as one raw byte tensor
    received in place into a preallocated buffer (no pickling).
    Returns (pairs, counters, saturated) on rank 0 and None elsewhere."""
    import torch
    import torch.distributed as dist
    from .ssjoin import PAIR_DTYPE
    rank = dist.get_rank()
    world = dist.get_world_size()
    head = torch.tensor([len(pairs), int(saturated)] + [int(counters.get(k, 0)) for k in COUNTER_KEYS],
                        dtype=torch.int64)
    heads = [torch.zeros_like(head) for _ in range(world)]
    dist.all_gather(heads, head, group=group)
    if rank != 0:
        if len(pairs):
            buf = np.ascontiguousarray(pairs).view(np.uint8)
            dist.send(torch.from_numpy(buf), dst=0, group=group)
        return None
    counts = [int(h[0]) for h in heads]
    allp = np.empty(sum(counts), dtype=PAIR_DTYPE)
    at = 0
    for r, c in enumerate(counts):
        if c == 0:
            continue
        dst = allp[at:at + c].view(np.uint8)
        if r == 0:
            dst[:] = np.ascontiguousarray(pairs).view(np.uint8)
        else:
            dist.recv(torch.from_numpy(dst), src=r, group=group)
        at += c
    merged_counters, sat = merge_counters(
        [({k: int(h[2 + i]) for i, k in enumerate(COUNTER_KEYS)}, int(h[1])) for h in heads])
    return merge_row_blocks(allp, counts), merged_counters, sat


def merge_row_blocks(allp, counts):
    """Canonical order of the concatenated results of ranks that own
    ascending, disjoint row blocks (rows are id_s): within one id_r, rank r's
    run precedes rank r+1's and each run is id_s-sorted, so a STABLE sort on
    id_r alone is the merge."""
    if sum(1 for c in counts if c) <= 1:
        return allp
    return allp[np.argsort(allp["id_r"], kind="stable")]


def heap_merge(runs):
    """Reference-style k-way merge (used by tests to cross-check merge_runs)."""
    it = heapq.merge(*[[(int(p["id_r"]), int(p["id_s"]), int(p["overlap"])) for p in r] for r in runs])
    return list(it)

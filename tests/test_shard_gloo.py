"""Multi-rank plumbing of the row-partitioned join on CPU (world_size 2, gloo).

Each rank takes its window-balanced row block from the library's own
partitioner (ssjb_partition_rows, host code), joins it -- here with the C
oracle standing in for the GPU engine, which has no device on this box -- and
rank 0 gathers and merges the runs with paper_1711_07295_b200.shard, exactly
as bench.py does under torchrun.  The merged pairs and summed counters must
equal the unsharded join (reference tests/test_parallel.cpp:37-59: the worker
count changes nothing observable)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

CASES = [  # (num_sets, mean, universe, seed, tau, capacity)
    (1200, 9, 100, 9, (3, 5), 2048),
    (800, 8, 60, 10, (1, 2), 3),
    (2000, 10, 60, 777, (3, 5), 1),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1711_07295_b200 import load_library, shard
    from paper_1711_07295_b200 import ssjoin as S
    lib = load_library()
    out = []
    for n, mean, universe, seed, tau, cap in CASES:
        coll = S.Collection.generate(lib, n, mean, universe, seed)
        opts = S.par_bitmap_options(lib, threshold=tau, buffer_capacity=cap)
        bounds = S.partition_rows(coll, opts, world)
        t, o = coll.csr()
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        if r1 > r0:
            pairs, cnt = O.par_bitmap_join(t, o, tau[0], tau[1], True, 1, 64, 0, O.INT64_MAX, cap, r0, r1)
        else:
            pairs, cnt = np.zeros(0, dtype=O.PAIR_DTYPE), {k: 0 for k in O.COUNTER_FIELDS}
        counters = {"candidates": cnt["candidates"], "pruned_bitmap": cnt["pruned_bitmap"],
                    "bitmap_tested": cnt["bitmap_tested"], "verified": cnt["verified"], "matched": cnt["matched"]}
        merged = shard.gather_to_root(pairs, counters, cnt["saturated_records"])
        via_shm = shard.gather_to_root_shm(pairs, counters, cnt["saturated_records"], lib,
                                           tag=f"ssjb_test_{port}")
        if rank == 0:
            assert (via_shm[0] == merged[0]).all() and via_shm[1] == merged[1] and via_shm[2] == merged[2]
            want, wcnt = O.par_bitmap_join(t, o, tau[0], tau[1], True, 1, 64, 0, O.INT64_MAX, cap)
            mp_pairs, mcnt, msat = merged
            ok = (len(mp_pairs) == len(want) and bool((mp_pairs == want).all())
                  and all(mcnt[k] == wcnt[k] for k in counters) and msat == wcnt["saturated_records"]
                  and bounds[0] == 0 and bounds[-1] == n)
            out.append((n, ok, len(want), list(map(int, bounds))))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_merge_to_the_full_join(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
    assert any(npairs > 0 for _, _, npairs, _ in res)


def test_merge_runs_is_a_kway_merge():
    from paper_1711_07295_b200 import shard
    from paper_1711_07295_b200.ssjoin import PAIR_DTYPE
    rng = np.random.default_rng(3)
    runs = []
    for _ in range(4):
        a = np.zeros(50, dtype=PAIR_DTYPE)
        a["id_r"] = rng.integers(0, 30, 50)
        a["id_s"] = rng.integers(30, 1000, 50)
        a["overlap"] = rng.integers(1, 9, 50)
        runs.append(np.sort(a, order=["id_r", "id_s"]))
    merged = shard.merge_runs(runs)
    assert [(int(p["id_r"]), int(p["id_s"]), int(p["overlap"])) for p in merged] == shard.heap_merge(runs)


def test_library_row_shard_merge_is_the_canonical_order(lib):
    """ssjb_merge_row_shards (the library's O(pairs) merge, capi.cpp merge_shards)
    on runs of ascending disjoint row blocks == the (id_r, id_s) sort of their
    union; large enough to split over several host threads."""
    from paper_1711_07295_b200 import shard
    from paper_1711_07295_b200.ssjoin import PAIR_DTYPE
    rng = np.random.default_rng(5)
    bounds = [0, 40000, 90000, 90000, 200000]  # one empty block
    runs = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        m = int(rng.integers(0, 300000)) if b > a else 0
        r = np.zeros(m, dtype=PAIR_DTYPE)
        r["id_s"] = rng.integers(a, b, m) if m else []
        r["id_r"] = (rng.random(m) * r["id_s"]).astype(np.uint32) if m else []
        r["overlap"] = rng.integers(1, 50, m)
        r = np.unique(r[r["id_r"] < r["id_s"]])
        runs.append(np.sort(r, order=["id_r", "id_s"]))
    got = shard.merge_row_shards(lib, runs)
    want = np.sort(np.concatenate(runs), order=["id_r", "id_s"])
    assert len(got) == len(want) > 500000 and (got == want).all()

#!/usr/bin/env python3
"""Headline benchmark: Bitmap-Filter self-join (paper Alg. 8) on B200.

Workload (default, BASELINE.json configs[3], "C4" -- the config the metric's
1/2/4/8-GPU numbers are quoted on; it fits one B200): ORKUT-shaped synthetic
collection, 2,732,271 sets, lognormal sizes (median 29, mean ~120, max
40,425), Zipf tokens over 8,730,857 (paper_1711_07295_b200/datasets.py c4),
Jaccard 0.7, Bitmap-Xor b = 64 (what the reference's auto width resolves to),
cutoff OFF, buffer 2048.  One STEP = one full join (4.31e11 window pairs,
42,380,999 matches).  ``--workload c2`` keeps round 1's DBLP-shaped 8-threshold
sweep (BASELINE configs[1]) as the step.

Metric: billion pair comparisons per second (one comparison = one (i, j) in
the length window, == ssj_counters.candidates), plus end-to-end join seconds.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c4|c2]

`value` = window pairs / device-timed step with the collection resident in
HBM (ssjb_collection_pin_device); `e2e` = the same metric through the
reference-facing C ABI (ssj_join on a host collection: H2D of tokens +
offsets and D2H of the sorted result pairs inside every step); `e2e_cold` =
the first ssj_join on a freshly created collection (host page registration
and every per-collection cache paid once).  Under torchrun each rank joins a
window-balanced row block (ssjb_join_rows); rank 0 gathers and merges.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "billion pair-comparisons/sec and end-to-end join seconds at 1/2/4/8 B200 vs CPU"
UNIT = "G pair-cmp/s"
WORKLOADS = {
    "c4": ("C4: ORKUT-shaped synthetic, 2,732,271 sets (lognormal sizes median 29 / mean ~120 / max 40,425, "
           "Zipf tokens over 8,730,857), Jaccard 0.7, Bitmap-Xor b=64, cutoff off, one join per step"),
    "c2": ("C2: DBLP-shaped synthetic, 100K sets (99K Zipf/4000 Poisson-86 + 1K planted near-dups), "
           "Jaccard sweep 0.50-0.95 (8 joins per step), Bitmap-Xor b=128, cutoff off"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("SSJB_BENCH_WORKLOAD", "c4"), choices=sorted(WORKLOADS))
    ap.add_argument("--bits", type=int, default=None, help="sketch width (default: 64 for c4, 128 for c2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary C2 / C3 measurements")
    ap.add_argument("--concurrency", type=int, default=int(os.environ.get("SSJB_BENCH_CONCURRENCY", "2")),
                    help="joins of a C2 step in flight at once (host threads; the C ABI is thread-safe)")
    a = ap.parse_args()
    if a.bits is None:
        a.bits = 64 if a.workload == "c4" else 128
    return a


def workload(lib, name, bits):
    """(collection, [options per join of one step])."""
    from paper_1711_07295_b200 import datasets as D
    if name == "c4":
        return D.c4(lib), [D.c4_options(lib, bits=bits)]
    return D.c2(lib), [D.c2_options(lib, tau, bits=bits) for tau in D.C2_TAUS]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("SSJB_BENCH_NO_CLOCKS"):  # (diagnostics only: a line without clocks is not a bench value)
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        ndev = max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local % ndev)
        if ndev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # plumbing check with more ranks than GPUs: NCCL needs one GPU per rank
            dist.init_process_group("gloo")
        return rank, world, local, dist.new_group(backend="gloo")
    return rank, world, local, None


def _reduce_device():
    import torch
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def barrier_sync(world):
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def flush_l2(buf):
    buf.add_(1)  # 256 MiB read+write: evicts the 126 MB L2 between timed steps


def pipe_peaks(device):
    exe = os.path.join(ROOT, "paper_1711_07295_b200", "lib", "pipe_peaks")
    try:
        out = subprocess.run([exe, str(device)], capture_output=True, text=True, timeout=120).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {}


# ------------------------------------------------------------------ our arm
def tc_ops_per_pair(rep, bits):
    """Algorithmic int8 tensor-core work of K2 per window pair: 2*(b+32) for
    the level-1 GEMM (b sketch bits + the 32-byte popcount extension), plus
    2*(256+32) when the join ran the level-2 GEMM (filter_kernel 2)."""
    return 2 * (bits + 32) + (2 * 288 if rep.extra["filter_kernel"] == 2 else 0)


def run_ours(args):
    import numpy as np  # noqa: F401
    import torch

    import paper_1711_07295_b200 as pkg
    from paper_1711_07295_b200 import shard
    from paper_1711_07295_b200 import ssjoin as S

    rank, world, local, gloo = dist_setup(args.gpus)
    device = local % max(torch.cuda.device_count(), 1)  # (identity on a full node)
    torch.cuda.set_device(device)
    lib = pkg.load_library()
    coll, opts = workload(lib, args.workload, args.bits)
    n = len(coll)
    bounds = [S.partition_rows(coll, o, world) for o in opts]
    rows = [(int(b[rank]), int(b[rank + 1])) for b in bounds]
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    debug = os.environ.get("SSJB_BENCH_DEBUG")
    concurrency = max(1, args.concurrency) if len(opts) > 1 else 1

    def one(o, r0, r1, pinned, c=coll):
        t0 = time.perf_counter()
        if world == 1 and not pinned:
            rep = S.join(c, o)  # the drop-in call
        else:
            rep = S.join_rows(c, o, r0, r1, device)
        if debug:
            x = rep.extra
            print(f"[bench] pinned={pinned} tau={o.threshold_num}/{o.threshold_den} "
                  f"wall_ms={(time.perf_counter() - t0) * 1e3:.3f} "
                  + " ".join(f"{k[3:]}={x[k]:.3f}" for k in x if k.startswith("ms_")), file=sys.stderr)
        return rep

    # the C2 sweep's joins are independent: with --concurrency > 1 several are
    # in flight from host threads (each on its own stream)
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=concurrency) if concurrency > 1 else None

    def step(pinned: bool):
        if pool is None:
            return [one(o, r0, r1, pinned) for o, (r0, r1) in zip(opts, rows)]
        futs = [pool.submit(one, o, r0, r1, pinned) for o, (r0, r1) in zip(opts, rows)]
        return [f.result() for f in futs]

    # ---- cold end-to-end: the first ssj_join on a freshly created collection ----
    # (host page registration, token-stream encoding and every per-collection
    # cache are paid inside this call; rank 0 / N=1 only, one sample)
    cold = None
    if world == 1:
        t, o = coll.csr()
        fresh = S.Collection.from_csr(lib, t, o)
        barrier_sync(world)
        t0 = time.perf_counter()
        reps = [one(op, 0, n, False, fresh) for op in opts]
        cold_s = time.perf_counter() - t0
        cold = {"value": round(sum(r.counters["candidates"] for r in reps) / cold_s / 1e9, 3), "unit": UNIT,
                "join_s": cold_s, "h2d_bytes": sum(r.extra["h2d_bytes"] for r in reps),
                "d2h_bytes": sum(r.extra["d2h_bytes"] for r in reps),
                "what": "first ssj_join(s) of one step on a collection created just before (from the same CSR): "
                        "includes host registration of the collection and every per-collection cache"}
        fresh.close()
        del fresh, reps

    # ---- device-resident timing (value) ----
    S.pin_device(coll, device)
    for _ in range(args.warmup):
        step(True)
    times, reps_last, launches, window, kstats = [], None, 0, 0, []
    with ClockSampler(device) as clocks:
        for _ in range(args.steps):
            flush_l2(l2)
            barrier_sync(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = step(True)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            if debug:
                print(f"[bench] resident step {len(times)}: {times[-1]:.2f} ms", file=sys.stderr)
            reps_last = reps
            launches += sum(r.extra["launches"] for r in reps)
            window += sum(r.counters["candidates"] for r in reps)
            for r in reps:  # (stats only from here on: the result block goes back to the library's cache,
                r.pairs = None  # as a client's does when it is done with a result)
            kstats.append(reps)
    if pool is not None:
        # per-kernel device times for the roofline come from serial steps (one
        # join at a time): with joins in flight a join's event intervals also
        # contain the other join's kernels.  (Not part of the timed value.)
        kstats = []
        for _ in range(min(args.steps, 5)):
            flush_l2(l2)
            reps = [one(o, r0, r1, True) for o, (r0, r1) in zip(opts, rows)]
            for r in reps:
                r.pairs = None
            kstats.append(reps)
    # K1 alone on the resident replica (its per-join cost is hidden by the
    # replica's sketch cache above): mean of 10 launches, L2 flushed before each
    k1_ms = None
    if rank == 0:
        import ctypes as C
        ms = C.c_double()
        if lib.ssjb_time_build(coll.handle, 1, args.bits, 0, device, 10, C.byref(ms)) == 0:
            k1_ms = ms.value
    S.unpin_device(coll, device)
    local_ms = sum(times)
    total_ms = max_over_ranks(local_ms, world)
    total_pairs = sum_over_ranks(window, world)
    ms_per_step = total_ms / args.steps
    value = total_pairs / (total_ms * 1e-3) / 1e9

    # ---- end-to-end through the C ABI with host buffers (e2e) ----
    for _ in range(min(args.warmup, 2)):
        step(False)
    e2e_times, h2d, d2h, e2e_pairs = [], 0, 0, 0
    for _ in range(args.steps):
        flush_l2(l2)
        barrier_sync(world)
        t0 = time.perf_counter()
        reps = step(False)
        if world > 1:  # one node: runs meet in /dev/shm, rank 0 merges them (ssjb_merge_row_shards)
            for r in reps:
                shard.gather_to_root_shm(r.pairs, r.counters, r.saturated_records, lib, group=gloo,
                                         tag=f"ssjb_{os.environ.get('MASTER_PORT', '0')}")
        t1 = time.perf_counter()
        e2e_times.append((t1 - t0) * 1e3)
        h2d += sum(r.extra["h2d_bytes"] for r in reps)
        d2h += sum(r.extra["d2h_bytes"] for r in reps)
        e2e_pairs += sum(r.counters["candidates"] for r in reps)
    e2e_ms = max_over_ranks(sum(e2e_times), world)
    e2e_value = sum_over_ranks(e2e_pairs, world) / (e2e_ms * 1e-3) / 1e9
    if pool is not None:
        pool.shutdown()

    # ---- roofline of the dominant kernel (library-internal CUDA events on its stream) ----
    peaks = pipe_peaks(device) if rank == 0 else {}
    mp = measured_peaks()
    nk = len(kstats)
    kms = {k: sum(r.extra[f"ms_{k}"] for reps in kstats for r in reps) / nk
           for k in ("filter", "head", "verify", "build", "rescan", "sort", "download", "upload")
           if f"ms_{k}" in reps_last[0].extra}
    flt_ms, ver_ms, head_ms = kms.get("filter", 0.0), kms.get("verify", 0.0), kms.get("head", 0.0)
    words32 = args.bits // 32
    pairs_step = sum(r.counters["candidates"] for r in reps_last)
    popc_per_step = pairs_step * words32
    tc_ops = sum(r.counters["candidates"] * tc_ops_per_pair(r, args.bits) for r in reps_last)
    uses_tc = all(r.extra["filter_kernel"] >= 1 for r in reps_last)
    hbm_peak = mp.get("hbm_gbs", 6650.0)
    popc_equiv = {"achieved": popc_per_step / (flt_ms * 1e-3) / 1e12,
                  "peak": peaks.get("popc_ops_per_s", float("nan")) / 1e12, "unit": "Tpopc/s",
                  "note": f"xor+popcount work the paper's filter needs ({words32} x 32-bit POPC per pair) per second "
                          "of filter time, against the measured POPC pipe peak"}
    popc_equiv["frac"] = popc_equiv["achieved"] / popc_equiv["peak"] if popc_equiv["peak"] == popc_equiv["peak"] else None
    vb_step = sum(r.extra["verify_bytes"] for reps in kstats for r in reps) / nk
    # K3a algorithmic work: a K-long head-indicator dot product (2K ops) per
    # region window pair (ssjb_stats.head_pairs)
    head_ops = sum(2.0 * r.extra.get("head_k", 0) * r.extra.get("head_pairs", 0) for r in reps_last)
    dominant = max((flt_ms, "filter"), (ver_ms, "verify"), (head_ms, "head"))[1]
    if dominant == "filter" and uses_tc:
        achieved = tc_ops / (flt_ms * 1e-3) / 1e12
        peak = peaks.get("tc_i8_ops_per_s", 4.5e15) / 1e12
        roofline = {"kernel": "filter_tc_kernel / filter_tcm_kernel (K2, tcgen05 kind::i8)", "bound": "tensor",
                    "achieved": achieved, "peak": peak, "unit": "TOPS(int8)", "frac": achieved / peak,
                    "traffic": None,
                    "peak_source": "tools/pipe_peaks.cu tc_i8_loop measured on this GPU (back-to-back "
                                   "M128xN256xK32 tcgen05.mma kind::i8); MEASURED_PEAKS.json has no int8 entry",
                    "work_per_pair": f"2*(b+32) = {2 * (args.bits + 32)} int8 ops (+576 with the level-2 GEMM)",
                    "popc_equivalent": popc_equiv}
    elif dominant == "filter":
        achieved = popc_per_step / (flt_ms * 1e-3) / 1e12
        peak = popc_equiv["peak"]
        roofline = {"kernel": "filter_kernel (K2, POPC)", "bound": "popc", "achieved": achieved, "peak": peak,
                    "unit": "Tpopc/s", "frac": achieved / peak if peak == peak else None, "traffic": None,
                    "peak_source": "tools/pipe_peaks.cu measured on this GPU (32-bit POPC, full chip)",
                    "work_per_pair": f"{words32} x 32-bit POPC (b={args.bits})"}
    elif dominant == "head":
        achieved = head_ops / (head_ms * 1e-3) / 1e12
        peak = peaks.get("tc_i8_ops_per_s", 4.5e15) / 1e12
        peak = peaks.get("tc_f4_ops_per_s", 9e15) / 1e12
        roofline = {"kernel": "head_overlap_kernel (K3a, tcgen05 kind::mxf4 exact head-token overlaps)",
                    "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS(fp4)",
                    "frac": achieved / peak, "traffic": None,
                    "peak_source": "tools/pipe_peaks.cu tc_f4_loop measured on this GPU"}
    else:
        achieved = vb_step / (ver_ms * 1e-3) / 1e9
        roofline = {"kernel": "verify_pairs (K3)", "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
                    "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if mp else "fallback 6650 GB/s"}
    roofline["kernel_ms_per_step"] = dict(kms, source="device events on the join stream (serial joins)")
    toks, offs = coll.csr()
    k1_bytes = 4 * len(toks) + 8 * (n + 1) + (args.bits // 8) * n
    roofline["secondary"] = {
        "K1_build_sketches": {
            "bound": "hbm", "unit": "GB/s", "peak": hbm_peak,
            "achieved": k1_bytes / (k1_ms * 1e-3) / 1e9 if k1_ms else None,
            "frac": k1_bytes / (k1_ms * 1e-3) / 1e9 / hbm_peak if k1_ms else None,
            "ms_per_launch": k1_ms, "bytes_per_launch": k1_bytes,
            "bytes_formula": "4*T tokens + 8*(n+1) offsets + (b/8)*n sketches (Bitmap-Xor, b as configured)",
            "timing": "ssjb_time_build: mean of 10 launches on the resident replica, L2 flushed before each",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if mp else "fallback"},
        "K3_verify": k3_roofline(vb_step, ver_ms, hbm_peak),
    }
    if head_ms and head_ops:
        f4_peak = peaks.get("tc_f4_ops_per_s")
        ach = head_ops / (head_ms * 1e-3) / 1e12
        roofline["secondary"]["K3a_head_overlap"] = {
            "bound": "tensor", "unit": "TOPS(fp4)", "achieved": ach,
            "peak": f4_peak / 1e12 if f4_peak else None,
            "frac": ach / (f4_peak / 1e12) if f4_peak else None,
            "ms_per_step": head_ms, "ops_per_step": head_ops,
            "ops_formula": "2*K per region window pair (K head tokens, ssjb_stats.head_k x head_pairs)",
            "peak_source": "tools/pipe_peaks.cu tc_f4_loop (back-to-back M128xN256xK64 tcgen05.mma "
                           "kind::mxf4.block_scale) measured on this GPU"}
    if dominant == "filter" and uses_tc:
        roofline.update(filter_traffic(args.workload))

    # ---- secondary workloads (rank 0, N=1): the C2 sweep and C3 ----
    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary:
        secondary = secondary_workloads(lib, args, device, l2)

    # ---- CPU baseline: the oracle port on a bounded row sample (rank 0, N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_port(coll, opts, args.bits)

    matched_all = int(sum_over_ranks(sum(r.counters["matched"] for r in reps_last), world))
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload], "sets": n,
                       "taus": [f"{o.threshold_num}/{o.threshold_den}" for o in opts],
                       "bits": args.bits, "method": "xor", "cutoff": "off", "buffer_capacity": 2048,
                       "window_pairs_per_step": int(total_pairs / args.steps), "matches_per_step": matched_all,
                       "l2": "flushed (256 MiB write) before every timed step; C4's inputs (1.3 GB of tokens) "
                             "exceed L2 as well",
                       "parallelism": f"row-block shards x{world}", "joins_in_flight": concurrency},
            "join_s": {"per_step_device_resident": ms_per_step / 1e3,
                       "per_join_mean": ms_per_step / 1e3 / len(opts),
                       "per_step_e2e": e2e_ms / args.steps / 1e3},
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                    "d2h_bytes_per_step": d2h // args.steps, "ms_per_step": e2e_ms / args.steps,
                    "api": "ssj_join (C ABI, host collection)" if world == 1 else "ssjb_join_rows + gather",
                    "state": "warm: the collection's host registration and encoded token stream are cached "
                             "by earlier calls (see e2e_cold for the first call)"},
            "e2e_cold": cold,
            "gpu_launches": launches // args.steps * args.steps,
            "roofline": roofline, "pipe_peaks": peaks, "clocks": clocks.summary(), "cpu_baseline": cpu,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def k3_roofline(vb_step, ver_ms, hbm_peak):
    """K3 against HBM with SURVEY 8d's algorithmic bytes -- an upper bound (the
    early exit reads less).  On C4 the merged records are L2-resident (ncu:
    ~0.1 GB of DRAM reads per verify launch), so the formula's rate can exceed
    the HBM peak; the fraction is reported only where it is a fraction."""
    if not ver_ms:
        return None
    ach = vb_step / (ver_ms * 1e-3) / 1e9
    out = {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "achieved": ach,
           "frac": ach / hbm_peak if ach <= hbm_peak else None,
           "ms_per_step": ver_ms, "bytes_per_step": vb_step,
           "bytes_formula": "4*(|r|+|s|) per merged survivor + 16 per match (SURVEY 8d upper bound)"}
    if ach > hbm_peak:
        out["note"] = ("algorithmic bytes above the HBM peak: the survivors' records are L2-resident and the "
                       "early exit stops most merges early; ncu of the launches: profiles/r02ao_c4_kernels_ncu.md")
    return out


def secondary_workloads(lib, args, device, l2):
    """The C2 sweep (round 1's headline: 8 joins per step, two in flight) and
    one C3 join (KOSARAK-shaped, 2e8 result pairs), device-resident and
    through ssj_join.  Reported beside the headline, not part of it."""
    import torch

    from paper_1711_07295_b200 import capi, datasets as D
    from paper_1711_07295_b200 import ssjoin as S
    from concurrent.futures import ThreadPoolExecutor
    out = {}
    c2 = D.c2(lib)
    opts = [D.c2_options(lib, tau, bits=128) for tau in D.C2_TAUS]
    with ThreadPoolExecutor(max_workers=2) as pool:
        def sweep(pinned):
            f = [pool.submit(S.join_rows if pinned else S.join, c2, o, *((0, len(c2), device) if pinned else ()))
                 for o in opts]
            return [x.result() for x in f]
        for mode in ("resident", "e2e"):
            pinned = mode == "resident"
            if pinned:
                S.pin_device(c2, device)
            for _ in range(3):
                sweep(pinned)
            ms, pairs = 0.0, 0
            for _ in range(10):
                flush_l2(l2)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                reps = sweep(pinned)
                ms += (time.perf_counter() - t0) * 1e3
                pairs += sum(r.counters["candidates"] for r in reps)
            if pinned:
                S.unpin_device(c2, device)
            out[f"C2_sweep_{mode}"] = {"value": round(pairs / (ms * 1e-3) / 1e9, 3), "unit": UNIT,
                                       "ms_per_sweep": ms / 10, "joins_in_flight": 2,
                                       "workload": WORKLOADS["c2"]}
    del c2
    c3 = D.c3(lib)
    for _ in range(2):
        r3 = S.join(c3, D.c3_options(lib))
    t0 = time.perf_counter()
    r3 = S.join(c3, D.c3_options(lib))
    dt = time.perf_counter() - t0
    out["C3_e2e"] = {"value": round(r3.counters["candidates"] / dt / 1e9, 3), "unit": UNIT, "join_s": dt,
                     "matches": r3.counters["matched"], "verify_ms": r3.extra["ms_verify"],
                     "verify_bytes": r3.extra["verify_bytes"],
                     "workload": "C3 KOSARAK-shaped (606,770 sets, tau 1/2, Bitmap-Next b=64), ssj_join, warm"}
    # the Bitmap Filter inside the prefix-filter algorithms (GPU
    # prefix-filter engine), PPJOIN with the bitmap as filter3 on C3; the
    # reference's own single-threaded run of the same join is in
    # tests/golden/prefix_large.jsonl (counters and pair sha checked here too)
    ref = None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "prefix_large.jsonl")) as f:
            ref = next(d for d in map(json.loads, f) if d["config"] == "c3" and d["algo"] == 2 and d["bitmap"] == "f3")
    except (OSError, StopIteration):
        pass
    po = S.default_options(lib, algorithm=capi.SSJ_ALGO_PPJOIN, threshold=(1, 2), bitmap_enabled=1)
    S.join(c3, po)
    t0 = time.perf_counter()
    rp = S.join(c3, po)
    dt = time.perf_counter() - t0
    out["C3_ppjoin_bitmap_e2e"] = {
        "join_s": dt, "encounters": rp.extra.get("window_pairs"), "matches": rp.counters["matched"],
        "workload": "C3, ssj_join(PPJOIN, tau 1/2, bitmap filter3): GPU prefix-filter engine",
        "reference_join_s": ref and ref["join_s"],
        "reference_note": "unmodified reference, 1 thread, build container (tests/golden/prefix_large.jsonl)",
        "same_counters_as_reference": bool(ref) and rp.counters == ref["counters"]}
    return out


def filter_traffic(workload_name):
    """DRAM bytes per filter launch from the committed `ncu --set full` capture
    of this workload (profiles/*_<workload>_filter_ncu.json, tools/ncu_summary.py)."""
    import glob
    pat = "*_filter_tc_ncu.json" if workload_name == "c2" else f"*_{workload_name}_filter_ncu.json"
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", pat)))
    if not files:
        return {"traffic": None, "traffic_source": f"no committed ncu capture of the {workload_name} filter"}
    d = json.load(open(files[-1]))
    return {"traffic": d["mean_dram_bytes_per_launch"],
            "traffic_source": f"{os.path.relpath(files[-1], ROOT)}: mean dram__bytes_read.sum + "
                              f"dram__bytes_write.sum over {len(d['launches'])} filter launches "
                              "(ncu flushes caches before each replay)"}


def cpu_baseline_port(coll, opts, bits, target_s=12.0):
    """Single-core oracle port (oracle/ssj_oracle.c) on a bounded, stratified
    row sample of every join of the step: the sketch store is built once per
    join (untimed setup, like the reference's index phase), then single rows
    drawn from 4096 equal strata in bit-reversed order are joined until
    target_s of CPU time is spent.  value = window pairs / seconds."""
    import numpy as np

    from oracle import oracle as O
    t, o = coll.csr()
    n = len(o) - 1
    strata = 4096
    order = [int(f"{k:012b}"[::-1], 2) for k in range(strata)]
    total_pairs, total_s, rows_done = 0, 0.0, 0
    per_join = target_s / len(opts)
    for op in opts:
        p, q = op.threshold_num, op.threshold_den
        store = O.build_bitmaps(t, o, 1, bits)
        spent = 0.0
        for k in order:
            r0 = min(n - 1, int((k + 0.5) * n / strata))
            t0 = time.perf_counter()
            _, cnt = O.par_bitmap_join_store(t, o, store, p, q, 1, bits, 0, O.INT64_MAX, 2048, r0, r0 + 1)
            dt = time.perf_counter() - t0
            spent += dt
            total_pairs += cnt["candidates"]
            rows_done += 1
            if spent >= per_join:
                break
        total_s += spent
        del store
    _ = np
    return {"value": round(total_pairs / total_s / 1e9, 5), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{rows_done} rows drawn from 4096 equal strata of each join's rows (bit-reversed order) "
                      f"until {target_s:.0f} s of CPU time: {total_pairs} window pairs in {total_s:.1f} s; "
                      "oracle/ssj_oracle.c single-threaded, sketch store built once per join (not timed)"}


# -------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's own CPU implementation (compiled from its sources into
    oracle/_ref) through its C ABI with all host threads, on a bounded sample
    of the step: a deterministic uniform record subsample of the workload's
    collection (every stride-th record: same size and token distributions),
    the same join options.  The value is the reference's pair-cmp/s on that
    sample; the full-size join time it implies is reported as a projection."""
    import ctypes as C
    import platform

    import numpy as np

    from paper_1711_07295_b200 import capi, datasets as D
    from paper_1711_07295_b200 import ssjoin as S

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    so = os.path.join(ROOT, "oracle", "_ref", "libssjoin_ref.so")
    if not os.path.exists(so):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libssjoin_ref.so not built"}))
        return
    ref = capi.bind(C.CDLL(so))
    cores = os.cpu_count() or 1
    cpu_model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu_model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    full, full_opts = workload(ref, args.workload, args.bits)
    t, o = full.csr()
    n = len(o) - 1
    full_window = sum(D.window_pairs(o, op.threshold_num, op.threshold_den) for op in full_opts)
    stride = int(os.environ.get("SSJB_REF_STRIDE", "100" if args.workload == "c4" else "10"))
    keep = np.arange(0, n, stride)
    o64 = o.astype(np.int64)
    lens = o64[keep + 1] - o64[keep]
    offs = np.zeros(len(keep) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum(lens)
    idx = np.concatenate([np.arange(o64[r], o64[r + 1]) for r in keep])
    sub = S.Collection.from_csr(ref, t[idx], offs)
    del full
    opts = [S.par_bitmap_options(ref, threshold=(op.threshold_num, op.threshold_den), method=capi.SSJ_BITMAP_XOR,
                                 bits=args.bits, cutoff_mode=capi.SSJ_CUTOFF_OFF, workers=cores) for op in full_opts]

    def step():
        pairs, secs = 0, 0.0
        for op in opts:
            t0 = time.perf_counter()
            rep = S.join(sub, op)
            secs += time.perf_counter() - t0
            pairs += rep.counters["candidates"]
        return pairs, secs

    for _ in range(args.warmup):
        step()
    tot_pairs, tot_s = 0, 0.0
    for _ in range(args.steps):
        p, s = step()
        tot_pairs += p
        tot_s += s
    value = tot_pairs / tot_s / 1e9
    sample = (f"every {stride}th record of the {args.workload.upper()} collection ({len(keep)} of {n} sets), "
              f"same join options, reference ssj_join(PAR_BITMAP, workers={cores}) on {cores} host threads "
              f"({cpu_model}); {tot_pairs // args.steps} window pairs per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": WORKLOADS[args.workload], "bits": args.bits, "sample": sample},
        "projection": {"full_window_pairs_per_step": full_window,
                       "projected_join_s": full_window / (value * 1e9),
                       "note": "PROJECTED full-size step time = the full step's window pairs / the sample's "
                               "pair-cmp/s (BASELINE.md section 4 step 4); not measured"},
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": cores, "cpu": cpu_model,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)

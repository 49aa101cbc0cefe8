/*
 * ssjoin_b200.h -- extensions of libssjoin.so beyond the reference ABI.
 *
 * Nothing here is needed by a drop-in client; these entry points expose the
 * multi-GPU row partition, resident device replicas, per-kernel statistics
 * and the sketch-build kernel for parity tests.  They never change the
 * behaviour of the ssj_* entry points in ssjoin.h.
 */
#ifndef SSJOIN_B200_H
#define SSJOIN_B200_H

#include "ssjoin.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Canonical collection from token-id records in CSR form: record r owns
 * tokens[offsets[r] .. offsets[r+1]).  Same canonicalisation as
 * ssj_collection_load(SSJ_INPUT_TOKEN_IDS) (reference src/collection.cpp:44-54,
 * 97-137): per-record sort + dedup, records by (size, tokens), ids as-is. */
ssj_status ssjb_collection_from_csr(const uint32_t* tokens, const uint64_t* offsets, size_t n,
                                    ssj_collection** out);

/* Borrowed view of the canonical CSR arrays (valid until the handle is freed). */
ssj_status ssjb_collection_csr(const ssj_collection* coll, const uint32_t** tokens,
                               const uint64_t** offsets, size_t* n);

/* Keep a replica of the collection resident in HBM of `device` so later joins
 * skip the host->device upload; unpin releases it. */
ssj_status ssjb_collection_pin_device(const ssj_collection* coll, int device);
ssj_status ssjb_collection_unpin_device(const ssj_collection* coll, int device);

/* The part of a PAR_BITMAP / NAIVE self-join whose later record (id_s) lies in
 * rows [row_begin, row_end), on one GPU (device < 0: the first configured).
 * Pairs, counters and saturated_records of disjoint row ranges add up exactly
 * to the full join's (the multi-GPU / multi-rank shard unit). */
ssj_status ssjb_join_rows(const ssj_collection* coll, const ssj_join_options* opts,
                          size_t row_begin, size_t row_end, int device, ssj_report** out);

/* parts+1 row boundaries balancing the length-window pair count of each part. */
ssj_status ssjb_partition_rows(const ssj_collection* coll, const ssj_join_options* opts,
                               int parts, uint64_t* bounds);

/* GPUs ssj_join spreads one join over (default: env SSJ_GPUS, else 1). */
int ssjb_device_count(void);
ssj_status ssjb_set_devices(int count);

/* Row shards per GPU of one self-join (default: env SSJB_SHARDS_PER_DEVICE,
 * else 1; 0 restores the default).  Values above 1 run the multi-GPU
 * partition and shard merge on fewer devices -- the worker-count invariance
 * check of reference tests/test_parallel.cpp:37-59 on a one-GPU host. */
ssj_status ssjb_set_shards_per_device(int count);

/* Canonical merge of row-shard results: runs[k] (counts[k] pairs, each run
 * sorted by (id_r, id_s)) are the results of ascending, disjoint row blocks of
 * one self-join (e.g. one per rank of a multi-process join); out receives the
 * sum of counts pairs in the reference's order.  O(pairs) on all host threads. */
ssj_status ssjb_merge_row_shards(const ssj_pair* const* runs, const size_t* counts, int nruns, ssj_pair* out);

/* Frees the idle join workspaces (survivor / result buffers a dense join grew
 * and the pool kept) of `device`, or of every device for -1.  Idle bytes kept
 * per device are bounded by env SSJB_WORKSPACE_KEEP_MB (default: 1/4 of HBM). */
ssj_status ssjb_trim(int device);

typedef struct ssjb_stats {
    uint64_t window_pairs;   /* pair comparisons = counters.candidates */
    uint64_t survivors;      /* filter survivors verified on the GPU */
    uint64_t batches;        /* survivor-buffer batches */
    uint64_t launches;       /* kernel launches issued */
    uint64_t h2d_bytes;      /* host->device bytes copied */
    uint64_t d2h_bytes;      /* device->host bytes copied */
    uint64_t verify_bytes;   /* algorithmic bytes of verification: 4*(|r|+|s|) per survivor + 16 per match */
    double ms_upload;        /* device event times per phase (max over GPUs) */
    double ms_build;
    double ms_filter;
    double ms_rescan;
    double ms_verify;
    double ms_sort;
    double ms_download;
    int devices;
    int filter_kernel;       /* 0 = POPC kernel */
    /* head-overlap phase of dense joins (K3a, exact head-token overlaps on the
     * tensor cores for the large-record region); zero when it did not run */
    uint64_t head_pairs;     /* region window pairs (the kernel's algorithmic work) */
    uint64_t head_survivors; /* region pairs passed to exact verification */
    double ms_head;          /* device ms of the head-overlap kernel (max over GPUs) */
    double ms_head_setup;    /* device ms of head selection + operand build */
    int head_k;              /* head tokens (GEMM depth) */
    double ms_merge;         /* host ms merging the row shards' sorted runs (multi-shard joins) */
} ssjb_stats;

ssj_status ssjb_report_stats(const ssj_report* report, ssjb_stats* out);

/* Runs the sketch-build kernel for the collection and copies the sketch store
 * (n * bits/64 words, row-major) into out_host.  method: SSJ_BITMAP_SET/XOR/NEXT. */
ssj_status ssjb_build_bitmaps(const ssj_collection* coll, int method, int bits, int hash,
                              int device, uint64_t* out_host);

/* ---- result delivery for outputs beyond host memory ----
 * The ssj_report these return holds the counters, timings and
 * saturated_records of the join (counters.matched = number of result pairs)
 * but NO pairs: ssj_report_pair_count() is 0.  RS-joins (s_or_null != NULL)
 * follow ssj_join's rules (NAIVE only). */

/* Receives consecutive chunks of the canonical (id_r, id_s)-sorted pair list;
 * a non-zero return stops the join (SSJ_ERROR_IO). */
typedef int (*ssjb_pair_sink)(const ssj_pair* pairs, size_t count, void* user);

/* Streams the join's pairs to `sink` in chunks of whole id_r ranges of about
 * chunk_pairs pairs (0: 16M), without ever holding the full list in host
 * memory: sorted result runs stay in HBM and are merged per chunk on the GPU.
 * `out` may be NULL. */
ssj_status ssjb_join_stream(const ssj_collection* r, const ssj_collection* s_or_null,
                            const ssj_join_options* opts, size_t chunk_pairs, ssjb_pair_sink sink,
                            void* user, ssj_report** out);

/* Count-first: counters (incl. matched) without sorting or downloading pairs. */
ssj_status ssjb_join_count(const ssj_collection* r, const ssj_collection* s_or_null,
                           const ssj_join_options* opts, ssj_report** out);

/* Streams the pairs into a text file in the reference CLI's pairs format,
 * one "id_r id_s overlap" line per pair (reference tools/ssjoin_cli.cpp:290-294).
 * `out` may be NULL. */
ssj_status ssjb_join_write_pairs(const ssj_collection* r, const ssj_collection* s_or_null,
                                 const ssj_join_options* opts, const char* path, ssj_report** out);

/* Writes a materialised report's pairs in the same text format. */
ssj_status ssjb_report_write_pairs(const ssj_report* report, const char* path);

/* Mean device time in ms of the sketch-build kernel (K1) over `reps` launches
 * on the device replica, L2 flushed before each (the K1 roofline probe). */
ssj_status ssjb_time_build(const ssj_collection* coll, int method, int bits, int hash, int device,
                           int reps, double* ms_per_launch);

const char* ssjb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SSJOIN_B200_H */

"""ctypes mirror of the reference C interface (``proj/include/ssjoin.h``).

The structs and constants below are byte-for-byte the reference layouts
(``ssj_join_options`` 80 B, ``ssj_pair`` 16 B, ``ssj_counters`` 72 B,
``ssj_timings`` 32 B, ``ssj_generator_config`` 48 B; reference
include/ssjoin.h:50-57,92-110,125-148).  :func:`bind` attaches prototypes to
any shared library exporting the ``ssj_*`` surface -- the B200 library
``libssjoin.so`` built from ``paper_1711_07295_b200/csrc`` or, in tests and
bench.py's reference arm only, the reference compiled under ``oracle/_ref``.
"""
from __future__ import annotations

import ctypes as C

# status codes -- reference include/ssjoin.h:15-21
SSJ_OK = 0
SSJ_ERROR_INVALID_ARGUMENT = 1
SSJ_ERROR_IO = 2
SSJ_ERROR_PARSE = 3
SSJ_ERROR_INTERNAL = 4

SSJ_INPUT_TOKEN_IDS, SSJ_INPUT_WORDS, SSJ_INPUT_QGRAMS = 0, 1, 2
SSJ_DIST_UNIFORM, SSJ_DIST_ZIPF = 0, 1

(SSJ_ALGO_NAIVE, SSJ_ALGO_ALLPAIRS, SSJ_ALGO_PPJOIN, SSJ_ALGO_PPJOIN_PLUS,
 SSJ_ALGO_GROUPJOIN, SSJ_ALGO_ADAPTJOIN, SSJ_ALGO_PAR_BITMAP) = range(7)
SSJ_SIM_OVERLAP, SSJ_SIM_JACCARD, SSJ_SIM_COSINE, SSJ_SIM_DICE = range(4)
SSJ_BITMAP_SET, SSJ_BITMAP_XOR, SSJ_BITMAP_NEXT, SSJ_BITMAP_COMBINED = range(4)
SSJ_HASH_MOD, SSJ_HASH_MULT = 0, 1
SSJ_CUTOFF_AUTO, SSJ_CUTOFF_OFF, SSJ_CUTOFF_EXPLICIT = 0, 1, 2
SSJ_PLACEMENT_DEFAULT, SSJ_PLACEMENT_FILTER2, SSJ_PLACEMENT_FILTER3 = 0, 1, 2
SSJ_SPACE_NORMALIZED, SSJ_SPACE_JACCARD = 0, 1

INT64_MAX = (1 << 63) - 1


class GeneratorConfig(C.Structure):
    _fields_ = [("distribution", C.c_int), ("num_sets", C.c_int64), ("mean_size", C.c_double),
                ("universe", C.c_int64), ("seed", C.c_uint64), ("zipf_exponent", C.c_double)]


class JoinOptions(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("similarity", C.c_int),
                ("threshold_num", C.c_int64), ("threshold_den", C.c_int64),
                ("bitmap_enabled", C.c_int), ("bitmap_method", C.c_int),
                ("bitmap_bits", C.c_int), ("bitmap_hash", C.c_int),
                ("cutoff_mode", C.c_int), ("cutoff_value", C.c_int64),
                ("placement", C.c_int), ("suffix_depth", C.c_int), ("ell_max", C.c_int),
                ("workers", C.c_int), ("buffer_capacity", C.c_int)]


class Pair(C.Structure):
    _fields_ = [("id_r", C.c_uint32), ("id_s", C.c_uint32), ("overlap", C.c_int64)]


class Counters(C.Structure):
    _fields_ = [(name, C.c_uint64) for name in (
        "candidates", "pruned_length", "pruned_positional", "pruned_suffix", "pruned_bitmap",
        "bitmap_tested", "filter_evaluations", "verified", "matched")]


class Timings(C.Structure):
    _fields_ = [("index_s", C.c_double), ("candidates_s", C.c_double),
                ("verify_s", C.c_double), ("total_s", C.c_double)]


assert C.sizeof(JoinOptions) == 80 and C.sizeof(Pair) == 16
assert C.sizeof(Counters) == 72 and C.sizeof(Timings) == 32 and C.sizeof(GeneratorConfig) == 48

P = C.c_void_p
_PROTOS = {
    # name: (restype, argtypes) -- reference include/ssjoin.h:24-173
    "ssj_last_error": (C.c_char_p, []),
    "ssj_collection_load": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(P)]),
    "ssj_collection_write": (C.c_int, [P, C.c_char_p]),
    "ssj_collection_free": (None, [P]),
    "ssj_collection_size": (C.c_size_t, [P]),
    "ssj_collection_median_size": (C.c_int64, [P]),
    "ssj_collection_mean_size": (C.c_double, [P]),
    "ssj_collection_max_size": (C.c_int64, [P]),
    "ssj_collection_universe": (C.c_int64, [P]),
    "ssj_collection_generate": (C.c_int, [C.POINTER(GeneratorConfig), C.POINTER(P)]),
    "ssj_join_options_init": (None, [C.POINTER(JoinOptions)]),
    "ssj_join": (C.c_int, [P, P, C.POINTER(JoinOptions), C.POINTER(P)]),
    "ssj_resolve_bitmap": (C.c_int, [P, C.POINTER(JoinOptions), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
    "ssj_report_pair_count": (C.c_size_t, [P]),
    "ssj_report_pairs": (C.POINTER(Pair), [P]),
    "ssj_report_counters": (None, [P, C.POINTER(Counters)]),
    "ssj_report_timings": (None, [P, C.POINTER(Timings)]),
    "ssj_report_saturated_records": (C.c_uint64, [P]),
    "ssj_report_free": (None, [P]),
    "ssj_expected_bound": (C.c_int, [C.c_int, C.c_int, C.c_int64, C.POINTER(C.c_double)]),
    "ssj_monte_carlo_bound": (C.c_int, [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_uint64,
                                        C.POINTER(C.c_double)]),
    "ssj_cutoff": (C.c_int, [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int,
                             C.POINTER(C.c_int64)]),
    "ssj_parse_threshold": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
}
SSJ_SYMBOLS = tuple(_PROTOS)

class Stats(C.Structure):
    """``ssjb_stats`` (include/ssjoin_b200.h)."""
    _fields_ = [(n, C.c_uint64) for n in ("window_pairs", "survivors", "batches", "launches",
                                          "h2d_bytes", "d2h_bytes", "verify_bytes")] + \
               [(n, C.c_double) for n in ("ms_upload", "ms_build", "ms_filter", "ms_rescan",
                                          "ms_verify", "ms_sort", "ms_download")] + \
               [("devices", C.c_int), ("filter_kernel", C.c_int),
                ("head_pairs", C.c_uint64), ("head_survivors", C.c_uint64),
                ("ms_head", C.c_double), ("ms_head_setup", C.c_double), ("head_k", C.c_int),
                ("ms_merge", C.c_double)]


# ssjb_pair_sink: int (*)(const ssj_pair*, size_t, void*)
PAIR_SINK = C.CFUNCTYPE(C.c_int, C.POINTER(Pair), C.c_size_t, C.c_void_p)

# Extension entry points of the B200 library (include/ssjoin_b200.h).
_EXT_PROTOS = {
    "ssjb_join_stream": (C.c_int, [P, P, C.POINTER(JoinOptions), C.c_size_t, PAIR_SINK, P,
                                   C.POINTER(P)]),
    "ssjb_join_count": (C.c_int, [P, P, C.POINTER(JoinOptions), C.POINTER(P)]),
    "ssjb_join_write_pairs": (C.c_int, [P, P, C.POINTER(JoinOptions), C.c_char_p, C.POINTER(P)]),
    "ssjb_report_write_pairs": (C.c_int, [P, C.c_char_p]),
    "ssjb_collection_from_csr": (C.c_int, [P, P, C.c_size_t, C.POINTER(P)]),
    "ssjb_collection_csr": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(C.c_size_t)]),
    "ssjb_collection_pin_device": (C.c_int, [P, C.c_int]),
    "ssjb_collection_unpin_device": (C.c_int, [P, C.c_int]),
    "ssjb_join_rows": (C.c_int, [P, C.POINTER(JoinOptions), C.c_size_t, C.c_size_t, C.c_int,
                                 C.POINTER(P)]),
    "ssjb_partition_rows": (C.c_int, [P, C.POINTER(JoinOptions), C.c_int, P]),
    "ssjb_device_count": (C.c_int, []),
    "ssjb_set_devices": (C.c_int, [C.c_int]),
    "ssjb_set_shards_per_device": (C.c_int, [C.c_int]),
    "ssjb_trim": (C.c_int, [C.c_int]),
    "ssjb_merge_row_shards": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int, C.c_void_p]),
    "ssjb_report_stats": (C.c_int, [P, C.POINTER(Stats)]),
    "ssjb_build_bitmaps": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, P]),
    "ssjb_time_build": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_double)]),
    "ssjb_version": (C.c_char_p, []),
}
SSJB_SYMBOLS = tuple(_EXT_PROTOS)


def bind(lib: C.CDLL, extensions: bool = False) -> C.CDLL:
    """Attach prototypes for the ``ssj_*`` surface (and ``ssjb_*`` when asked)."""
    protos = dict(_PROTOS)
    if extensions:
        protos.update(_EXT_PROTOS)
    for name, (res, args) in protos.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib

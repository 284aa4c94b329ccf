"""ctypes binding of the C ABI (include/quakescan_b200.h).

The CUDA library is built in-tree (`paper_1803_09835_b200/lib/
libquakescan_b200.so`, see csrc/Makefile / __graft_entry__.build()).  There
is no CPU fallback: if the library is missing every hot-path call raises.
"""

import ctypes
import os

from .errors import DataError, ParameterError

HERE = os.path.dirname(os.path.abspath(__file__))
# QS_LIB_PATH: an alternative build of the same library (kernel-configuration sweeps)
LIB_PATH = os.environ.get("QS_LIB_PATH") or os.path.join(HERE, "lib", "libquakescan_b200.so")

QS_OK, QS_ERR_ARG, QS_ERR_OOM, QS_ERR_CUDA, QS_ERR_DATA, QS_ERR_CAPACITY = 0, 1, 2, 3, 4, 5


class FpParamsC(ctypes.Structure):
    """struct qs_fp_params (include/quakescan_b200.h)."""
    _fields_ = [("window_len_s", ctypes.c_double), ("window_lag_s", ctypes.c_double),
                ("freq_bins", ctypes.c_uint32), ("time_bins", ctypes.c_uint32),
                ("top_k", ctypes.c_uint32), ("band_low_hz", ctypes.c_double),
                ("band_high_hz", ctypes.c_double), ("frame_len_s", ctypes.c_double),
                ("hop_s", ctypes.c_double)]


class SearchStatsC(ctypes.Structure):
    """struct qs_search_stats (include/quakescan_b200.h)."""
    _fields_ = [("n_fingerprints", ctypes.c_uint64), ("n_queries", ctypes.c_uint64),
                ("lookups_total", ctypes.c_uint64), ("distinct_pairs", ctypes.c_uint64),
                ("emitted_triplets", ctypes.c_uint64), ("filtered_fingerprints", ctypes.c_uint64),
                ("peak_table_entries", ctypes.c_uint64), ("n_buckets", ctypes.c_uint64),
                ("max_bucket", ctypes.c_uint64), ("top_bucket_mass", ctypes.c_double),
                ("n_partitions", ctypes.c_uint32)]

_u8p = ctypes.c_void_p
_p = ctypes.c_void_p
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_sz = ctypes.c_size_t
_int = ctypes.c_int
_dbl = ctypes.c_double

# name -> (restype, argtypes); must cover every function in include/quakescan_b200.h
SIGNATURES = {
    "qs_version": (ctypes.c_char_p, []),
    "qs_last_error": (ctypes.c_char_p, []),
    "qs_device_info": (_int, [ctypes.c_char_p, _sz]),
    "qs_host_ptr_pinned": (_int, [_p]),
    "qs_host_pack_u16": (_int, [_p, _p, _u64]),
    "qs_host_pack_u12": (_int, [_p, _p, _u64, ctypes.POINTER(ctypes.c_int)]),
    "qs_host_pack_f32": (_int, [_p, _p, _u64, ctypes.POINTER(ctypes.c_int)]),
    "qs_bits_widen_u16": (_int, [_p, _p, _u64, _p]),
    "qs_bits_widen_u12": (_int, [_p, _p, _u64, _p]),
    "qs_memcpy_h2d_async": (_int, [_p, _p, _sz, _p]),
    "qs_memcpy_d2h_async": (_int, [_p, _p, _sz, _p]),
    "qs_gen_hash_mapping": (_int, [_p, _u32, _u32, _u64, _p]),
    "qs_minmax_plan_bytes": (_sz, [_u32, _u32]),
    "qs_minmax_plan": (_int, [_p, _u32, _u32, _p, _p]),
    "qs_minmax_signatures": (_int, [_p, _u64, _u32, _p, _u32, _u32, _u32, _p, _p, _p]),
    "qs_minmax_signatures_search": (_int, [_p, _u64, _u32, _p, _u32, _u32, _u32, _p, _p, _p,
                                           _p, _p, _p]),
    "qs_minmax_signatures_search_rows": (_int, [_p, _u64, _u64, _u64, _u32, _p, _u32, _u32, _u32,
                                                _p, _p, _p, _p, _p, _p]),
    "qs_gen_signatures_range": (_int, [_p, _u64, _u32, _p, _u32, _u32, _i32, _i32, _p, _u64,
                                       _u64]),
    "qs_lsh_prep": (_int, [_p, _u64, _u32, _p, _p, _p, _p]),
    "qs_lsh_bucket_ws_bytes": (_sz, [_u64, _u32]),
    "qs_lsh_build_buckets": (_int, [_p, _u64, _u32, _p, _p, _p, _sz, _p]),
    "qs_lsh_list_ws_bytes": (_sz, [_u64, _u32]),
    "qs_lsh_list_buckets": (_int, [_p, _u64, _u32, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "qs_lsh_bucket_flags_ws_bytes": (_sz, [_u64, _u32]),
    "qs_lsh_build_bucket_flags": (_int, [_p, _u64, _u32, _p, _p, _p, _sz, _p]),
    "qs_lsh_list_flags_ws_bytes": (_sz, [_u64, _u32]),
    "qs_lsh_list_buckets_flags": (_int, [_p, _u64, _u32, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "qs_lsh_bucket_stats": (_int, [_p, _p, _p, _u64, _p, _p, _u32, _p, _u32, _p, _u64, _p, _p]),
    "qs_lsh_compact_ws_bytes": (_sz, [_u64]),
    "qs_lsh_compact_buckets": (_int, [_p, _p, _p, _p, _u64, _p, _p, _p, _p, _p, _p,
                                       _p, _u32, _p, _u64, _p, _p, _sz, _p]),
    "qs_lsh_pairs_ws_bytes": (_sz, [_u64]),
    "qs_lsh_pairs": (_int, [_p, _p, _p, _p, _u64, _p, _p, _u64, _u32, _u32, _u64, _p, _p, _u32,
                            _int, _p, _p, _p, _u64, _p, _p, _sz, _p]),
    "qs_lsh_pairs_ex": (_int, [_p, _p, _p, _p, _u64, _p, _p, _u64, _u32, _u32, _u64, _p, _p, _u32,
                               _int, _p, _p, _p, _u64, _p, _p, _sz, _u32, _u32, _p, _p]),
    "qs_lsh_core_first": (_int, [_p, _p, _p, _p, _u64, _u32, _p, _p, _p, _p]),
    "qs_lsh_core_skipped": (_int, [_p, _p, _p, _u64, _u32, _u32, _u32, _p, _p]),
    "qs_lsh_complete_sims": (_int, [_p, _p, _p, _u64, _p, _u32, _p]),
    "qs_lsh_occurrence_filter": (_int, [_p, _p, _u64, _u64, _dbl, _p, _u32, _p, _p, _p, _p]),
    "qs_lsh_occ_degree": (_int, [_p, _u64, _p, _u32, _p, _p]),
    "qs_lsh_occ_mark": (_int, [_p, _u64, _p, _u64, _dbl, _p, _u32, _p, _p]),
    "qs_lsh_occ_finish": (_int, [_p, _u64, _p, _p]),
    "qs_lsh_filter_pairs": (_int, [_p, _p, _p, _u32, _u64, _p, _p, _u32, _p, _p, _p, _p, _p]),
    "qs_sort_pairs_ws_bytes": (_sz, [_u64]),
    "qs_lsh_finalize": (_int, [_p, _p, _u64, _u32, _p, _p, _sz, _p]),
    "qs_fp_band_stft": (_int, [_p, _int, _u64, _u32, _u32, _u64, _u32, _p, _p, _p]),
    "qs_fp_windows": (_int, [_p, _u64, _u32, _p, _u64, _u64, _u64, _u64, _u32, _u32, _p, _p, _p,
                             _p, _p, _p, _u32, _u32, _u32, _u32, _p, _u32, _int, _p, _p, _u32, _p,
                             _p, _p]),
    "qs_fp_mad": (_int, [_p, _u32, _u64, _p, _p, _p, _p]),
    "qs_fp_transpose_f32": (_int, [_p, _u64, _u32, _p, _p]),
    "qs_fp_topk_bits": (_int, [_p, _int, _u64, _u32, _p, _p, _u32, _p, _p, _p]),
    "qs_fp_haar2d": (_int, [_p, _u64, _u32, _u32, _p, _u32, _int, _p]),
    "qs_fp_normalize": (_int, [_p, _int, _u64, _u32, _p, _p, _p, _p]),
    "qs_triplets_combine_ws_bytes": (_sz, [_u64]),
    "qs_sosfiltfilt_ws_bytes": (_sz, [_u64, _u64]),
    "qs_sosfiltfilt": (_int, [_p, _u64, _p, _u32, _p, _u64, _p, _p, _sz, _p]),
    "qs_triplets_combine": (_int, [_p, _u64, _u32, _u32, _p, _p, _p, _sz, _p]),
    "qs_fp_pack_records": (_int, [_p, _p, _p, _u64, _u32, _p, _p]),
    "qs_fp_unpack_records": (_int, [_p, _u64, _u32, _p, _p, _p, _p]),
    "qs_peak_launch": (_int, [_int, _u32, _u32, _p, ctypes.POINTER(ctypes.c_double), _p]),
    "qs_lsh_search_ws_bytes": (_sz, [_u64, _u32, _u64, _u32]),
    "qs_lsh_search": (_int, [_p, _u64, _u32, _u32, _u64, _dbl, _u32, _p, _u64,
                             ctypes.POINTER(_u64), ctypes.POINTER(SearchStatsC), _p, _sz, _p]),
    "qs_lsh_search_bits_ws_bytes": (_sz, [_u64, _u32, _u32, _u32, _u64, _u32]),
    "qs_lsh_search_bits": (_int, [_p, _u64, _u32, _u32, _u64, _u32, _u32, _u32, _u64, _dbl, _u32,
                                  _p, _u64, ctypes.POINTER(_u64), ctypes.POINTER(SearchStatsC), _p,
                                  _sz, _p]),
    "qs_fp_n_windows": (_int, [_u64, _dbl, ctypes.POINTER(FpParamsC), ctypes.POINTER(_u64)]),
    "qs_fingerprint_chain_ws_bytes": (_sz, [_u64, _dbl, ctypes.POINTER(FpParamsC), _u64]),
    "qs_fingerprint_chain": (_int, [_p, _int, _u64, _dbl, ctypes.POINTER(FpParamsC), _p, _u64, _p,
                                    _p, _p, ctypes.POINTER(_u64), _p, _sz, _p]),
    "qs_bench_pair_table": (_int, [_u64, _u64, _p, _u64, _p, _p]),
    "qs_radix_sort_ws_bytes": (_sz, [_u64, _u32]),
    "qs_radix_sort_pairs": (_int, [_p, _p, _u64, _u32, _u32, _p, _p, _p, _sz, _p, _p]),
}

_lib = None


class NativeMissing(RuntimeError):
    pass


def lib():
    """The loaded library; raises NativeMissing when it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeMissing(
                f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build() or "
                f"make -C paper_1803_09835_b200/csrc); there is no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def missing_symbols():
    handle = lib()
    return [n for n in SIGNATURES if not hasattr(handle, n)]


def last_error() -> str:
    return lib().qs_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == QS_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == QS_ERR_ARG:
        raise ParameterError(msg)
    if rc == QS_ERR_DATA:
        raise DataError(msg)
    if rc == QS_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


# ------------------------------------------------------------------ torch glue

def torch():
    import torch as _t
    if not _t.cuda.is_available():
        raise NativeMissing("no CUDA device: the quakescan-b200 hot path runs only on the GPU")
    return _t


def stream():
    """cudaStream_t of torch's current stream (kernels are ordered with torch work)."""
    t = torch()
    return ctypes.c_void_p(t.cuda.current_stream().cuda_stream)


def ptr(x):
    """Device pointer of a torch tensor (None -> NULL)."""
    if x is None:
        return None
    return ctypes.c_void_p(x.data_ptr())


def is_device_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)

"""ctypes binding of the C-ABI in include/txsite_b200.h (libtxsite_b200.so).

This is the reference-side binding a Python caller adds; the
engine itself is the sm_100a library.  There is no fallback: if the library is
missing, importing this module raises.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TXS_CHECKED=1 loads the bounds-checked build (tests only; traps on an
# out-of-range terrain load instead of reading it)
LIB_PATH = os.path.join(_HERE, "libtxsite_b200_checked.so" if os.environ.get("TXS_CHECKED") == "1"
                        else "libtxsite_b200.so")
# TXS_LIB=<path> loads an alternative build of the same C-ABI (kernel A/B runs)
LIB_PATH = os.environ.get("TXS_LIB", LIB_PATH)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libtxsite_b200.so not built ({LIB_PATH}); run `make` or __graft_entry__.build() — "
        "the engine has no CPU fallback")

lib = C.CDLL(LIB_PATH)

i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p

STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "OFF_GRID", 3: "STATE", 4: "CUDA",
          5: "OUT_OF_MEMORY", 6: "RANGE", 7: "SIZE_MISMATCH", 8: "NODATA"}
STOP = {0: "target-reached", 1: "zero-gain", 2: "exhausted", 3: "max-selected"}


class Params(C.Structure):
    _fields_ = [("roi", i32), ("tx_height", i32), ("rx_height", i32), ("samples_per_point", i32),
                ("per_block", i32), ("block_width", i32), ("site_mode", i32), ("los_arith", i32),
                ("target_coverage", dbl), ("max_selected", i64), ("seed", u64)]


class Candidate(C.Structure):
    _fields_ = [("row", i32), ("col", i32), ("score", i32), ("_pad", i32)]


class Window(C.Structure):
    _fields_ = [("row0", i32), ("col0", i32), ("h", i32), ("w", i32)]


class Step(C.Structure):
    _fields_ = [("index", i64), ("row", i32), ("col", i32), ("gain", i64), ("coverage", dbl)]


class Stats(C.Structure):
    _fields_ = [("ms_terrain", dbl), ("ms_vix", dbl), ("ms_findmax", dbl), ("ms_viewshed", dbl),
                ("ms_site", dbl), ("vix_los", i64), ("vix_crossings_full", i64),
                ("viewshed_crossings", i64), ("viewshed_cells", i64), ("site_iterations", i64),
                ("site_bytes", i64), ("site_launches", i64), ("candidates", i64),
                ("kernel_launches", i64), ("ms_site_rounds", dbl),
                ("vix_fp64_ties", i64), ("vix_fp64_flips", i64), ("vs_fp64_ties", i64), ("vs_fp64_flips", i64),
                ("ms_vix_kernel", dbl), ("ms_viewshed_kernel", dbl), ("device_bytes", i64), ("device_bytes_peak", i64),
                ("site_phase_ns", i64 * 5)]


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("txs_abi_version", C.c_int, [])
_sig("txs_device_ok", C.c_int, [])
_sig("txs_create", C.c_int, [C.c_int, C.POINTER(vp)])
_sig("txs_destroy", None, [vp])
_sig("txs_last_error", C.c_char_p, [vp])
_sig("txs_get_stats", C.c_int, [vp, C.POINTER(Stats)])
_sig("txs_reset_stats", C.c_int, [vp])
_sig("txs_synchronize", C.c_int, [vp])
_sig("txs_event_record", C.c_int, [vp, C.c_int])
_sig("txs_event_elapsed", C.c_int, [vp, C.c_int, C.c_int, C.POINTER(dbl)])
_sig("txs_set_terrain", C.c_int, [vp, vp, i64, i64])
_sig("txs_generate_fractal", C.c_int, [vp, i64, i64, dbl, u64, i32, i32])
_sig("txs_fill_rows", C.c_int, [vp, i64, i64, C.c_int16])
_sig("txs_get_terrain", C.c_int, [vp, vp])
_sig("txs_terrain_dims", C.c_int, [vp, C.POINTER(i64), C.POINTER(i64)])
_sig("txs_is_visible_batch", C.c_int, [vp, vp, i64, i32, i32, i32, vp])
_sig("txs_estimate_vix", C.c_int, [vp, C.POINTER(Params), vp])
_sig("txs_set_vix", C.c_int, [vp, vp])
_sig("txs_get_vix", C.c_int, [vp, i64, i64, vp])
_sig("txs_partition", C.c_int, [i64, i64, i32, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)])
_sig("txs_find_candidates", C.c_int, [vp, C.POINTER(Params), C.POINTER(i64), vp, i64])
_sig("txs_set_candidates", C.c_int, [vp, vp, i64])
_sig("txs_random_observers", C.c_int, [vp, i64, u64])
_sig("txs_get_candidates", C.c_int, [vp, vp, i64, C.POINTER(i64)])
_sig("txs_compute_viewsheds", C.c_int, [vp, C.POINTER(Params)])
_sig("txs_get_viewsheds", C.c_int, [vp, i64, i64, vp, vp, i64, vp])
_sig("txs_set_viewsheds", C.c_int, [vp, i32, i64, vp, vp, vp, vp, i64])
_sig("txs_site", C.c_int, [vp, C.POINTER(Params), vp, i64, C.POINTER(i64), C.POINTER(i32)])
_sig("txs_get_cumulative", C.c_int, [vp, vp])
_sig("txs_marginal_gains", C.c_int, [vp, vp, vp])
_sig("txs_run_pipeline", C.c_int, [vp, C.POINTER(Params), vp, i64, C.POINTER(i64), C.POINTER(i32), vp])
_sig("txs_set_shard", C.c_int, [vp, i64, i64, i64, i64, i32])
_sig("txs_shard_info", C.c_int, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)])
_sig("txs_set_candidate_base", C.c_int, [vp, i64])
_sig("txs_site_shard_begin", C.c_int, [vp, C.POINTER(Params)])
_sig("txs_site_shard_best", C.c_int, [vp, C.POINTER(u64)])
_sig("txs_site_shard_export", C.c_int, [vp, i64, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), vp, vp, i64])
_sig("txs_site_shard_apply", C.c_int, [vp, i32, i32, vp, vp])
_sig("txs_site_shard_best_dev", C.c_int, [vp, vp])
_sig("txs_site_shard_export_dev", C.c_int, [vp, vp, vp])
_sig("txs_site_shard_apply_dev", C.c_int, [vp, vp, vp, i64])
_sig("txs_site_shard_payload_words", i64, [vp])
_sig("txs_site_shard_export_keyed_dev", C.c_int, [vp, vp, vp])
_sig("txs_site_shard_select_dev", C.c_int, [vp, vp, i32, vp, vp])
_sig("txs_site_shard_result", C.c_int, [vp, vp, i64, C.POINTER(i64), C.POINTER(i32)])
_sig("txs_stream", vp, [vp])
_sig("txs_time_gain_pass", C.c_int, [vp, i32, C.POINTER(dbl), C.POINTER(i64)])
_sig("txs_measure_cache_read", C.c_int, [vp, i64, i32, C.POINTER(dbl)])
_sig("txs_ray_template", i64, [i32, vp, vp, vp, vp, vp, i64, i64, C.POINTER(i64)])
_sig("txs_selftest", C.c_int, [])
_sig("txs_event_template_info", C.c_int, [i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32)])

_sig("txs_get_cumulative_rows", C.c_int, [vp, i64, i64, vp])
_sig("txs_get_candidate_ids", C.c_int, [vp, vp, i64, C.POINTER(i64)])
_sig("txs_viewshed_record_words", i64, [i32])
_sig("txs_run_pipeline_host", C.c_int, [vp, vp, i64, i64, C.POINTER(Params), vp, i64, C.POINTER(i64), C.POINTER(i32), vp])
_sig("txs_viewsheds_pack", C.c_int, [vp, i64, vp, C.POINTER(i64)])
_sig("txs_site_gathered", C.c_int, [vp, C.POINTER(Params), i64, i64, vp, vp, i64, C.POINTER(i64), C.POINTER(i32)])
_sig("txs_default_ops", vp, [])
_sig("txs_plan_bands", C.c_int, [i64, i64, i32, vp])
_sig("txs_group_create", C.c_int, [C.c_int, vp, C.POINTER(vp)])
_sig("txs_group_create_with_ops", C.c_int, [C.c_int, vp, vp, C.POINTER(vp)])
_sig("txs_group_destroy", None, [vp])
_sig("txs_group_last_error", C.c_char_p, [vp])
_sig("txs_group_size", i32, [vp])
_sig("txs_group_context", vp, [vp, i32])
_sig("txs_group_set_exchange", C.c_int, [vp, i32])
_sig("txs_group_set_grid", C.c_int, [vp, i64, i64, C.POINTER(Params)])
_sig("txs_group_band", C.c_int, [vp, i32, C.POINTER(i64), C.POINTER(i64)])
_sig("txs_group_set_terrain", C.c_int, [vp, vp])
_sig("txs_group_generate_fractal", C.c_int, [vp, dbl, u64, i32, i32])
_sig("txs_group_fill_rows", C.c_int, [vp, i64, i64, C.c_int16])
_sig("txs_group_random_observers", C.c_int, [vp, i64, u64])
_sig("txs_group_run_pipeline", C.c_int, [vp, C.POINTER(Params), vp, i64, C.POINTER(i64), C.POINTER(i32), vp])
_sig("txs_group_get_cumulative", C.c_int, [vp, vp])

EXCHANGE = {"p2p": 0, "nccl": 1, "host": 2, "replicate": 3}

# every symbol the header declares (checked by the CPU test-suite)
EXPORTS = [
    "txs_abi_version", "txs_device_ok", "txs_create", "txs_destroy", "txs_last_error", "txs_get_stats",
    "txs_reset_stats", "txs_synchronize", "txs_event_record", "txs_event_elapsed", "txs_set_terrain", "txs_generate_fractal", "txs_fill_rows",
    "txs_get_terrain", "txs_terrain_dims", "txs_is_visible_batch", "txs_estimate_vix", "txs_set_vix", "txs_get_vix",
    "txs_partition", "txs_find_candidates", "txs_set_candidates", "txs_random_observers",
    "txs_get_candidates", "txs_compute_viewsheds", "txs_get_viewsheds", "txs_set_viewsheds", "txs_site",
    "txs_get_cumulative", "txs_marginal_gains", "txs_run_pipeline", "txs_ray_template", "txs_selftest",
    "txs_set_shard", "txs_shard_info", "txs_set_candidate_base", "txs_site_shard_begin", "txs_site_shard_best",
    "txs_site_shard_export", "txs_site_shard_apply", "txs_event_template_info",
    "txs_site_shard_best_dev", "txs_site_shard_export_dev", "txs_site_shard_apply_dev",
    "txs_site_shard_payload_words", "txs_site_shard_result", "txs_stream", "txs_time_gain_pass",
    "txs_site_shard_export_keyed_dev", "txs_site_shard_select_dev", "txs_measure_cache_read",
    "txs_get_cumulative_rows", "txs_get_candidate_ids", "txs_default_ops", "txs_viewshed_record_words",
    "txs_viewsheds_pack", "txs_site_gathered", "txs_run_pipeline_host", "txs_plan_bands", "txs_group_create", "txs_group_create_with_ops",
    "txs_group_destroy", "txs_group_last_error", "txs_group_size", "txs_group_context", "txs_group_set_exchange",
    "txs_group_set_grid", "txs_group_band", "txs_group_set_terrain", "txs_group_generate_fractal",
    "txs_group_fill_rows", "txs_group_random_observers", "txs_group_run_pipeline", "txs_group_get_cumulative",
]

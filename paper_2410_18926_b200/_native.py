"""ctypes binding of librrg.so (the C ABI declared in include/rrg.h).

There is no fallback: if the shared library is missing or fails to load,
importing this module raises, and every search entry point fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import BY_NAME, RrannError

LIB_PATH = Path(os.environ.get("RRG_LIB", Path(__file__).resolve().parent / "librrg.so"))

c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
c_size = ctypes.c_size_t
c_vp = ctypes.c_void_p
c_fp = ctypes.POINTER(ctypes.c_float)


class RrgIndexDesc(ctypes.Structure):
    _fields_ = [
        ("metric", c_i32), ("dim", c_i32), ("reduced_dim", c_i32), ("rank", c_i32),
        ("n_clusters", c_i32), ("n_points", c_i64), ("flags", c_u32),
        ("projection", c_vp), ("centroids", c_vp), ("cluster_sizes", c_vp), ("point_ids", c_vp),
        ("a_head", c_vp), ("a_scale", c_vp), ("a_values", c_vp),
        ("b_head", c_vp), ("b_scale", c_vp), ("b_values", c_vp),
        ("norms", c_vp), ("corpus", c_vp),
        ("a_values_f32", c_vp), ("b_values_f32", c_vp),
    ]


class RrgIndexInfo(ctypes.Structure):
    _fields_ = [
        ("metric", c_i32), ("dim", c_i32), ("reduced_dim", c_i32), ("rank", c_i32),
        ("n_clusters", c_i32), ("n_points", c_i64), ("flags", c_u32),
        ("n_exact_clusters", c_i32), ("max_cluster_size", c_i32), ("device", c_i32),
        ("device_bytes", c_u64),
    ]


class RrgFront(ctypes.Structure):
    _fields_ = [(n, c_vp) for n in ("xp", "qcodes", "qscale", "qhead", "pp", "xx", "sel", "prim")]


SIGNATURES = {
    "rrg_index_open": (c_int, [ctypes.c_char_p, c_int, ctypes.POINTER(c_vp)]),
    "rrg_index_open_shard": (c_int, [ctypes.c_char_p, c_int, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "rrg_index_create": (c_int, [ctypes.POINTER(RrgIndexDesc), c_int, ctypes.POINTER(c_vp)]),
    "rrg_index_create_shard": (c_int, [ctypes.POINTER(RrgIndexDesc), c_int, c_i32, c_i32,
                                       ctypes.POINTER(c_vp)]),
    "rrg_index_destroy": (None, [c_vp]),
    "rrg_index_info": (c_int, [c_vp, ctypes.POINTER(RrgIndexInfo)]),
    "rrg_index_cluster_sizes": (c_int, [c_vp, c_vp]),
    "rrg_search_workspace_bytes": (c_size, [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32]),
    "rrg_search": (c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32,
                           c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "rrg_search_host": (c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32,
                                c_vp, c_vp, c_vp]),
    "rrg_search_host_many": (c_int, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32,
                                     c_vp, c_vp, c_vp]),
    "rrg_stage_project": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rrg_stage_route": (c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_size, c_vp]),
    "rrg_stage_score_workspace_bytes": (c_size, [c_vp, c_i64, c_i32]),
    "rrg_stage_score": (c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                c_size, c_vp]),
    "rrg_index_reload_options": (c_int, [c_vp]),
    "rrg_shard_workspace_bytes": (c_size, [c_vp, c_i64, c_i32, c_i32, c_i32]),
    "rrg_shard_phase1": (c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp,
                                 c_vp, c_size, c_vp]),
    "rrg_front_workspace_bytes": (c_size, [c_vp, c_i64, c_i32]),
    "rrg_search_front": (c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_size, c_vp]),
    "rrg_search_from_front": (c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                                      c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "rrg_shard_phase1_from_front": (c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_vp,
                                            c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "rrg_merge_candidates": (c_int, [c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp,
                                     c_vp, c_vp]),
    "rrg_pack_candidates": (c_int, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rrg_unpack_candidates": (c_int, [c_i64, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      c_vp]),
    "rrg_shard_phase2": (c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp,
                                 c_vp, c_vp, c_size, c_vp]),
    "rrg_merge_results": (c_int, [c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_vp]),
    "rrg_ground_truth": (c_int, [c_vp, c_i64, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp]),
    "rrg_last_launch_count": (c_i64, []),
    "rrg_set_stage_timing": (None, [c_int]),
    "rrg_stage_times": (c_int, [c_vp, c_vp]),
    "rrg_path_times": (c_int, [c_vp, c_vp]),
    "rrg_search_counters": (c_int, [c_vp]),
    "rrg_last_error": (ctypes.c_char_p, []),
    "rrg_last_error_kind": (ctypes.c_char_p, []),
    "rrg_version": (ctypes.c_char_p, []),
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make`); the B200 query path has no CPU fallback")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc == 0:
        return
    kind = (lib.rrg_last_error_kind() or b"RrannError").decode()
    msg = (lib.rrg_last_error() or b"").decode()
    raise BY_NAME.get(kind, RrannError)(msg)

"""ctypes binding of the product C ABI (include/ebic_b200.h).

The library is the in-tree ``libebic_b200.so`` built for sm_100a.  There is no
fallback: if the library is missing or cannot be loaded, importing this module
raises, so nothing can silently run on a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

ABI_VERSION = 2  # EBIC_B200_ABI_VERSION of include/ebic_b200.h
LIB_PATH = Path(os.environ.get("EBIC_B200_LIB", Path(__file__).resolve().parent / "libebic_b200.so"))

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
szp = C.POINTER(C.c_size_t)
i64p = C.POINTER(C.c_int64)
vp = C.c_void_p


class CtxInfo(C.Structure):
    _fields_ = [
        ("n_rows", C.c_size_t),
        ("n_cols", C.c_size_t),
        ("row_begin", C.c_size_t),
        ("total_rows", C.c_size_t),
        ("n_shards", C.c_int),
        ("rows_per_tile", C.c_int),
        ("stages", C.c_int),
        ("grid", C.c_int),
        ("device_bytes", C.c_size_t),
        ("sm_count", C.c_int),
        ("layout", C.c_int),
        ("consumer_warps", C.c_int),
        ("kernel", C.c_int),
    ]


# (name, restype, argtypes) for every entry point declared in include/ebic_b200.h
SIGNATURES = [
    ("ebic_last_error", C.c_char_p, []),
    ("ebic_abi_version", C.c_int, []),
    ("ebic_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("ebic_ctx_create", C.c_int, [f64p, C.c_size_t, C.c_size_t, C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]),
    ("ebic_ctx_create_shard", C.c_int, [f64p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.POINTER(vp)]),
    ("ebic_ctx_create_shard_device", C.c_int, [vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.POINTER(vp)]),
    ("ebic_ctx_destroy", C.c_int, [vp]),
    ("ebic_ctx_get_info", C.c_int, [vp, C.POINTER(CtxInfo)]),
    ("ebic_count_matches", C.c_int, [vp, szp, u16p, C.c_size_t, C.c_double, u64p]),
    ("ebic_evaluate_population", C.c_int, [vp, szp, u16p, C.c_size_t, C.c_uint64, C.c_double, u64p, f64p]),
    ("ebic_fitness_score", C.c_double, [C.c_uint64, C.c_size_t, C.c_uint64]),
    ("ebic_default_sigma", C.c_uint64, [C.c_size_t]),
    ("ebic_fitness_scores_host", C.c_int, [u64p, szp, C.c_size_t, C.c_uint64, f64p]),
    ("ebic_count_matches_device", C.c_int, [vp, vp, vp, C.c_size_t, C.c_size_t, C.c_double, C.c_uint64, vp, vp, vp]),
    ("ebic_fitness_device", C.c_int, [vp, vp, vp, C.c_size_t, C.c_uint64, vp, vp]),
    ("ebic_ctx_phase_times", C.c_int, [vp, u64p, C.c_size_t, szp]),
    ("ebic_ctx_host_timers", C.c_int, [vp, f64p, u64p]),
    ("ebic_membership_bits", C.c_int, [vp, szp, u16p, C.c_size_t, C.c_double, C.c_size_t, u64p, u64p, u64p]),
    ("ebic_assign_rows", C.c_int, [vp, u16p, C.c_size_t, C.c_double, u64p, szp]),
    ("ebic_expand_bicluster", C.c_int, [vp, u16p, C.c_size_t, u64p, u8p, C.c_size_t, C.c_int, C.c_size_t, C.c_double, u64p, u8p, szp]),
    ("ebic_resolve_expand_batch", C.c_int, [vp, szp, u16p, C.c_size_t, C.c_int, C.c_size_t, C.c_double, u64p, u8p, szp]),
    ("ebic_synth_generate", C.c_int, [C.c_size_t, C.c_size_t, C.c_size_t, szp, szp, C.c_int, C.c_size_t, C.c_size_t, C.c_double, C.c_uint64, f64p]),
    ("ebic_xgroup_create", C.c_int, [vp, C.c_size_t, C.c_char_p, vp]),
    ("ebic_xgroup_join", C.c_int, [vp, vp, C.c_char_p, C.c_int, C.c_size_t, C.POINTER(vp)]),
    ("ebic_xgroup_evaluate", C.c_int, [vp, szp, u16p, C.c_size_t, C.c_uint64, C.c_double, C.c_uint64, u64p, f64p]),
    ("ebic_xgroup_count", C.c_int, [vp, vp, vp, C.c_size_t, C.c_size_t, C.c_double, C.c_uint64, C.c_int, C.c_uint64, vp]),
    ("ebic_xgroup_wait", C.c_int, [vp, C.c_uint64, C.c_size_t, u64p, f64p]),
    ("ebic_xgroup_destroy", C.c_int, [vp]),
    ("ebic_top_rank_update", C.c_int, [C.c_size_t, C.c_size_t, szp, u16p, f64p, u64p, C.c_size_t, szp, u16p, f64p, C.c_double, C.c_size_t, u64p, i64p, u64p, szp]),
]

EXPORTED = [s[0] for s in SIGNATURES]

EBIC_OK = 0
EBIC_ERR_INVALID_ARGUMENT = 1
EBIC_ERR_RUNTIME = 2
EBIC_ERR_CUDA = 3
EBIC_ERR_NO_DEVICE = 4


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ebic_abi_version() != ABI_VERSION:  # a stale build: struct layouts differ
        raise ImportError(f"{LIB_PATH} has ABI version {lib.ebic_abi_version()}, this binding "
                          f"expects {ABI_VERSION}: rebuild it")
    return lib


lib = _load()


def _fast(name, res, args):
    """A second handle on an entry point with raw-address (c_void_p) pointer
    arguments: the per-generation hot calls pass ndarray.ctypes.data ints
    instead of building ctypes pointer objects."""
    fn = getattr(C.CDLL(str(LIB_PATH)), name)
    fn.restype = res
    fn.argtypes = args
    return fn


fast_evaluate = _fast("ebic_evaluate_population", C.c_int,
                      [vp, vp, vp, C.c_size_t, C.c_uint64, C.c_double, vp, vp])
fast_count = _fast("ebic_count_matches", C.c_int, [vp, vp, vp, C.c_size_t, C.c_double, vp])


class EbicError(RuntimeError):
    """A failed C-ABI call (CUDA failure, no device)."""


def check(status: int) -> None:
    """Raise the exception the reference would raise for this status."""
    if status == EBIC_OK:
        return
    msg = (lib.ebic_last_error() or b"").decode()
    if status == EBIC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == EBIC_ERR_RUNTIME:
        raise RuntimeError(msg)
    raise EbicError(f"[status {status}] {msg}")


def ptr(a, typ):
    """ctypes pointer to a contiguous numpy array (None for None)."""
    if a is None:
        return None
    return a.ctypes.data_as(typ)

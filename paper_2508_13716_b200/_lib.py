"""ctypes binding of libcapgnn.so (the C ABI declared in include/capgnn.h).

There is no CPU fallback: if the library cannot be loaded, every entry point
raises.  ``lib()`` builds the library in-tree first when it is missing or
stale and nvcc is available (the build container); on a GPU box the prebuilt
``libcapgnn.so`` that travelled with the repo snapshot is used.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcapgnn.so")

P = C.c_void_p
I32, I64, U32, F32, F64 = C.c_int32, C.c_int64, C.c_uint32, C.c_float, C.c_double
INT = C.c_int
SZ = C.c_size_t


class PlanStatic(C.Structure):
    """Mirror of cg_plan_static (include/capgnn.h)."""

    _fields_ = [("n_union", I64), ("req_off", P), ("req_part", P), ("req_dev", P),
                ("req_pos", P), ("req_slot", P), ("req_needed", P), ("owner_dev", P),
                ("owner_row", P), ("gslot", P), ("lfree", P), ("score", P), ("lmin", P),
                ("gmin", F64), ("gfree", I32), ("policy", I32), ("n_parts", I32),
                ("req_snap", P), ("coalesce", I32)]


# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "cg_version": [],
    "cg_last_error": [],
    "cg_device_count": [P],
    "cg_device_sync": [INT],
    "cg_host_tier_alloc": [SZ, P],
    "cg_host_tier_free": [P],
    "cg_host_tier_register": [P, SZ],
    "cg_host_tier_unregister": [P],
    "cg_enable_peer_access": [INT, INT],
    "cg_ipc_get_handle": [P, P, P],
    "cg_ipc_open_handle": [P, INT, P],
    "cg_ipc_close_handle": [P],
    "cg_hash_features": [P, I64, P, I64, INT, U32, P, P],
    "cg_hash_labels": [P, P, I64, INT, U32, P],
    "cg_scale_rows": [P, I64, I64, INT, P, P],
    "cg_scale_rows_to": [P, I64, P, I64, I64, INT, P, P],
    "cg_copy_rows": [I64, INT, P, P, P, P, P, P, I64, P],
    "cg_copy_rows_bounded": [I64, INT, P, P, P, P, P, P, I64, INT, P],
    "cg_copy_rows_sel": [I64, INT, P, P, P, P, P, P, I64, INT, INT, INT, P],
    "cg_flag_signal": [P, C.c_uint32, P],
    "cg_flag_wait": [P, INT, INT, C.c_uint32, P],
    "cg_spmm": [I64, INT, P, P, I64, P, P, I64, P, P, I64, P, I64, P, I64, I64, P],
    "cg_spmm_mb": [I64, INT, P, P, I64, P, P, I64, P, P, I64, P, I64, P, I64, I64, P],
    "cg_relu_bits": [I64, INT, P, I64, P, I64, P],
    "cg_gemm_mb": [I64, INT, INT, P, I64, P, INT, P, I64, P, INT, P, INT, P, P, I64, P, I64, P,
                   I64, INT, P, P, P],
    "cg_gemm": [I64, INT, INT, P, I64, P, INT, P, I64, P, INT, P, INT, P, P, I64, P, I64, INT,
                P, P, P],
    "cg_split_tf32": [I64, P, P, P, P],
    "cg_split_tf32_t": [INT, P, P, P, P, P, P, I64, P],
    "cg_wgrad_workspace": [I64, INT, INT],
    "cg_wgrad": [I64, INT, INT, P, I64, P, I64, P, P, P, INT, P],
    "cg_colsum": [I64, INT, P, I64, P, P, P],
    "cg_softmax_ce": [I64, INT, P, I64, P, F32, P, I64, P, P, P, I64, P, P],
    "cg_adam": [I64, P, P, P, P, F32, F32, F32, F32, INT, P, P, P, P],
    "cg_set_epoch": [P, INT, P, F32, F32, INT, P],
    "cg_event_record": [P, P],
    "cg_plan_frozen": [P, INT, INT, INT, P, P, P, P, P, P, P, P, P, I32, I32, P, P, P],
    "cg_planner_create": [INT, INT, I64, P, I64, P, P],
    "cg_planner_destroy": [P],
    "cg_planner_set_halos": [P, P, P, P],
    "cg_planner_warm": [P],
    "cg_planner_epoch": [P, INT, INT, P, P, P, P, P, P, P, P, P],
    "cg_planner_state": [P, P, P, P, P, P, P, P, P, P],
    "cg_planner_lookup": [P, INT, I32, INT, INT, P],
    "cg_planner_admit": [P, INT, INT, I32, INT, P],
    "cg_planner_counters": [P, P, P, P, P],
    "cg_planner_occupancy": [P, P, P],
    "cg_csr_from_pairs": [I64, I64, P, P, P, P, P, P, P],
    "cg_undirected_csr": [I64, P, P, P, P, P, P],
    "cg_khop_halo": [I64, P, P, P, I32, INT, P, P],
    "cg_partition_stats": [I64, P, P, P, INT, P, P, P, P],
    "cg_influence_terms": [I64, P, P, P, P, P, P],
}
_RESTYPES = {"cg_last_error": C.c_char_p, "cg_wgrad_workspace": I64}

_lock = threading.Lock()
_lib = None


class CapgnnError(RuntimeError):
    """A libcapgnn entry point returned an error status."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        try:
            from . import build as _build
            if _build.stale():
                _build.build()
        except RuntimeError as exc:  # no nvcc here: must use the shipped .so
            if not os.path.exists(LIB_PATH):
                raise CapgnnError(f"libcapgnn.so missing and cannot be built: {exc}")
        if not os.path.exists(LIB_PATH):
            raise CapgnnError(f"libcapgnn.so not found at {LIB_PATH}")
        h = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, args in SIGNATURES.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, INT)
        _lib = h
    return _lib


# device entry points report how many kernels they launched; the running
# total is the bench's "gpu_launches" evidence
KERNEL_ENTRY = {"cg_hash_features", "cg_hash_labels", "cg_scale_rows", "cg_scale_rows_to",
                "cg_copy_rows", "cg_copy_rows_bounded", "cg_copy_rows_sel",
                "cg_spmm", "cg_spmm_mb", "cg_relu_bits", "cg_gemm", "cg_gemm_mb", "cg_wgrad",
                "cg_colsum", "cg_softmax_ce", "cg_adam",
                "cg_split_tf32", "cg_split_tf32_t",
                "cg_plan_frozen", "cg_set_epoch"}
launches = {"total": 0}


def call(name: str, *args) -> int:
    """Invoke an entry point; raise CapgnnError on a negative status."""
    rc = getattr(lib(), name)(*args)
    if name in _RESTYPES:
        return rc
    if rc < 0:
        msg = lib().cg_last_error()
        raise CapgnnError(f"{name}: {msg.decode() if msg else 'error'}")
    if name in KERNEL_ENTRY:
        launches["total"] += rc
        launches[name] = launches.get(name, 0) + rc
    return rc


def count_replay(per_entry: dict) -> None:
    """A CUDA-graph replay launches the kernels its capture recorded
    (per_entry maps entry point -> kernels; its "total" key, if present, is
    the same launches summed and is not counted twice)."""
    for name, n in per_entry.items():
        if name == "total":
            continue
        launches["total"] += n
        launches[name] = launches.get(name, 0) + n


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def ptr(x) -> int | None:
    """Raw address of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x).__name__}")

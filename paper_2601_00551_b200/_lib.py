"""ctypes binding of the in-tree sm_100a library ``libpaball_b200.so``.

The library is the product: if it is missing or cannot be loaded, every
compute entry point raises.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PAB_LIBRARY selects another build of the same library (tuning experiments)
LIB_PATH = os.environ.get("PAB_LIBRARY") or os.path.join(_HERE, "libpaball_b200.so")

_vp, _i, _i64, _d, _f = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_float
_SIGS = {
    "pab_version": ([], _i),
    "pab_device_info": ([_i, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)], _i),
    "pab_last_cuda_error": ([], C.c_char_p),
    "pab_record_sizes": ([C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)], _i),
    "pab_morton_keys": ([_vp, _vp, _i64, _d, _d, _d, _d, _d, _d, _i, _vp, _vp], _i),
    "pab_cloud_bounds_workspace_bytes": ([], C.c_size_t),
    "pab_cloud_bounds": ([_vp, _vp, _i64, _vp, _vp, _vp], _i),
    "pab_sort_keys": ([_vp, _vp, _i64, _vp, _i, _vp, _vp], _i),
    "pab_sort_perm_workspace_bytes": ([_i64], C.c_size_t),
    "pab_sort_perm": ([_vp, _i64, _vp, _vp, _vp], _i),
    "pab_pack": ([_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp], _i),
    "pab_forward_smem_bytes": ([_i, _i, _i], C.c_size_t),
    "pab_pair_table_bytes": ([_i64], C.c_size_t),
    "pab_pair_table": ([_vp, _vp, _i64, _vp, _vp], _i),
    "pab_forward": ([_vp, _vp, _vp, _vp, _i64, _vp, _vp, _i, _d, _d, _d, _i, _i, _d, _i, _d, _i, _i, _i, _i,
                     _vp, _vp, _i, _vp, _vp, _vp], _i),
    "pab_residual": ([_vp, _i, _i, _i, _vp, _vp, _vp, _vp], _i),
    "pab_adjoint": ([_vp, _vp, _vp, _i64, _vp, _vp, _i, _d, _d, _d, _i, _i, _d, _i, _d, _vp, _f, _i, _i, _i,
                     _vp, _vp, _vp, _vp], _i),
    "pab_grad_finalize": ([_vp, _i, _i64, _vp, _d, _i, _vp, _vp, _vp, _vp, _vp], _i),
    "pab_coincident": ([_vp, _vp, _i64, _vp, _vp, _i, _vp, _vp], _i),
    "pab_host_stage_copy": ([_vp, _vp, C.c_size_t, _i], _i),
    "pab_host_stage_narrow": ([_vp, _vp, C.c_size_t, _i], _i),
    "pab_pass_tail": ([_vp, _i, _vp, _vp, _vp, _vp], _i),
    "pab_decimate": ([_vp, _i, _i, _i, _vp, _vp], _i),
    "pab_adam": ([_vp, _vp, _vp, _vp, _i64, _d, _d, _d, _d, _i, _vp], _i),
    "pab_compact_workspace_bytes": ([_i64], C.c_size_t),
    "pab_compact": ([_vp, _i64, _i, _vp, _vp, _vp, _vp], _i),
    "pab_gather_f64": ([_vp, _i, _vp, _i64, _vp, _vp], _i),
    "pab_sumsq_workspace_bytes": ([_i64], C.c_size_t),
    "pab_sumsq_diff_f64": ([_vp, _vp, _i64, _vp, _vp, _vp], _i),
    "pab_select_workspace_bytes": ([], C.c_size_t),
    "pab_select_kth_f64": ([_vp, _i64, _i64, _vp, _vp, _vp], _i),
    "pab_density_keep_key": ([_vp, _vp, _i64, _vp, _vp, _d, _d, _d, _vp, _vp], _i),
    "pab_density_split_key": ([_vp, _i64, _d, _vp, _vp], _i),
    "pab_row_norms": ([_vp, _vp, _i64, _vp, _vp], _i),
    "pab_density_dup_key": ([_vp, _i64, _vp, _vp, _vp], _i),
    "pab_density_take_ties": ([_vp, _vp, _vp, _i, _i64, _vp, _vp], _i),
    "pab_split_children": ([_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp], _i),
    "pab_duplicate": ([_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp], _i),
    "pab_softplus_f64": ([_vp, _i64, _vp, _vp], _i),
    "pab_mul_sigmoid_f64": ([_vp, _vp, _i64, _vp, _vp], _i),
    "pab_vox_brick_count": ([_i, _i, _i], _i64),
    "pab_vox_count": ([_vp, _vp, _vp, _vp, _i64, _i, _i, _i, _d, _d, _d, _d, _d, _vp, _vp, _vp], _i),
    "pab_vox_emit": ([_vp, _vp, _i64, _i, _i, _i, _vp, _vp], _i),
    "pab_vox_gather": ([_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i, _i, _i, _d, _d, _d, _d, _d, _vp, _vp, _vp, _vp], _i),
    "pab_ubp": ([_vp, _i, _i, _d, _d, _vp, _d, _i, _i, _i, _d, _d, _d, _d, _vp, _vp, _vp, _vp], _i),
}
EXPORTED = tuple(_SIGS)

_lib = None


class LibraryError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library; raise if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


# Kernel launches issued through call() (bench.py reports the count inside
# its timed region as gpu_launches).  Every launching entry point issues one
# kernel, except these.
LAUNCHES = {"kernels": 0}
_KERNELS_PER_CALL = {"pab_host_stage_copy": 0, "pab_host_stage_narrow": 0, "pab_compact": 3, "pab_sumsq_diff_f64": 2,
                     "pab_cloud_bounds": 2, "pab_sort_perm": 15, "pab_forward": 2}


def call(name: str, *args) -> None:
    """Invoke an entry point and turn non-zero return codes into errors."""
    lib = load()
    rc = getattr(lib, name)(*args)
    LAUNCHES["kernels"] += _KERNELS_PER_CALL.get(name, 1)
    if rc != 0:
        if rc == 1:
            raise ValueError(f"{name}: invalid argument (rc=1)")
        err = lib.pab_last_cuda_error().decode()
        raise LibraryError(f"{name}: CUDA launch failed (rc={rc}): {err}")


def ptr(t) -> int | None:
    """Device/host address of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()

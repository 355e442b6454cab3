"""Python binding of libtci_b200.so (include/tci_b200.h) -- argument
marshalling only.

Every ``tci_*`` function below has the name and argument order of the C ABI
entry point it wraps and raises ``TciError`` (with ``.code`` = the
tci_status_t) on failure. All compute runs in the CUDA kernels of the shared
library; PyTorch is used only for device memory (tensors, the workspace),
streams and process groups. There is no CPU fallback: importing this package
raises if the compiled library is missing.

The ``Context`` class is a convenience layer over the same calls that takes
torch tensors (contiguous, on the context's device) and manages descriptors
and the workspace.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
from typing import Dict, Optional, Sequence, Tuple, Union

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtci_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2512_23917_b200/build.py` "
        "(or __graft_entry__.build()); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

# dtypes (tci_dtype_t)
TCI_R32, TCI_R64, TCI_C64, TCI_C128 = 1, 2, 3, 4
STATUS = {
    0: "OK", 1: "SHAPE_MISMATCH", 2: "ORDER_MISMATCH", 3: "OUT_OF_RANGE",
    4: "LABEL_CONFLICT", 5: "PARSE", 6: "DEAD_CONTEXT", 7: "UNSUPPORTED",
    8: "INVALID_ARGUMENT", 9: "WORKSPACE", 10: "CUDA", 11: "NCCL",
}
EXPORTED = [
    "tci_version", "tci_create_context", "tci_destroy_context", "tci_synchronize",
    "tci_last_error", "tci_workspace_attach", "tci_tensor_create", "tci_tensor_free",
    "tci_order", "tci_shape", "tci_size", "tci_size_bytes", "tci_copy", "tci_reshape",
    "tci_permute", "tci_contract_out_shape", "tci_contract", "tci_contract_str",
    "tci_contract_workspace_size", "tci_heff_workspace_size", "tci_heff_apply",
    "tci_tebd_theta", "tci_comm_init", "tci_comm_unique_id", "tci_allgather",
    "tci_launch_count", "tci_heff_plan_tree", "tci_profile_enable", "tci_profile_query",
    "tci_mps_overlap", "tci_norm", "tci_normalize", "tci_scale", "tci_linear_combine", "tci_inner",
    "tci_lanczos_workspace_size", "tci_heff_lanczos", "tci_set_gemm_algorithm", "tci_get_gemm_algorithm",
    "tci_ozaki_params", "tci_env_workspace_size", "tci_env_update", "tci_cplx_conj",
    "tci_svd_workspace_size", "tci_svd", "tci_trunc_svd", "tci_svd_info",
    "tci_mps_mpo_zipup_workspace_size", "tci_mps_mpo_zipup", "tci_heff_apply_staged",
    "tci_ipc_handle", "tci_ipc_open", "tci_ipc_close", "tci_gather_register", "tci_heff_apply_gather",
    "tci_gather_status", "tci_tebd_workspace_size", "tci_copy_async", "tci_lane_record", "tci_lane_wait",
    "tci_set_ozaki_guard", "tci_ozaki_guard_stats", "tci_ozaki_params_complex",
    "tci_set_ozaki_complex", "tci_set_f32_algorithm", "tci_ozaki_params_f32",
    "tci_graph_begin", "tci_graph_end", "tci_graph_launch", "tci_graph_destroy",
]


class TciError(RuntimeError):
    def __init__(self, code: int, fn: str):
        self.code = code
        msg = _lib.tci_last_error().decode(errors="replace")
        super().__init__(f"{fn}: {STATUS.get(code, code)} ({code}): {msg}")


_vp = ctypes.c_void_p
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_sig = {
    "tci_version": ([], ctypes.c_char_p),
    "tci_last_error": ([], ctypes.c_char_p),
    "tci_create_context": ([ctypes.POINTER(_vp), ctypes.c_int, _vp], ctypes.c_int),
    "tci_destroy_context": ([_vp], ctypes.c_int),
    "tci_synchronize": ([_vp], ctypes.c_int),
    "tci_workspace_attach": ([_vp, _vp, ctypes.c_size_t], ctypes.c_int),
    "tci_tensor_create": ([_vp, ctypes.c_int, ctypes.c_int, _i64p, _vp, ctypes.POINTER(_vp)], ctypes.c_int),
    "tci_tensor_free": ([_vp, _vp], ctypes.c_int),
    "tci_order": ([_vp, _vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tci_shape": ([_vp, _vp, _i64p], ctypes.c_int),
    "tci_size": ([_vp, _vp, _i64p], ctypes.c_int),
    "tci_size_bytes": ([_vp, _vp, _i64p], ctypes.c_int),
    "tci_copy": ([_vp, _vp, _vp], ctypes.c_int),
    "tci_copy_async": ([_vp, _vp, _vp, ctypes.c_int], ctypes.c_int),
    "tci_tebd_workspace_size": ([_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp,
                                 ctypes.c_char_p, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tci_lane_record": ([_vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "tci_lane_wait": ([_vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "tci_reshape": ([_vp, _vp, ctypes.c_int, _i64p], ctypes.c_int),
    "tci_permute": ([_vp, _vp, _i32p, _vp], ctypes.c_int),
    "tci_contract_out_shape": ([_vp, _vp, _i32p, _vp, _i32p, ctypes.c_int, _i32p, _i64p], ctypes.c_int),
    "tci_contract": ([_vp, _vp, _i32p, _vp, _i32p, _vp, _i32p], ctypes.c_int),
    "tci_contract_str": ([_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p], ctypes.c_int),
    "tci_contract_workspace_size": ([_vp, _vp, _i32p, _vp, _i32p, _vp, _i32p, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tci_heff_workspace_size": ([_vp, ctypes.c_int] + [ctypes.c_int64] * 8 + [ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tci_heff_apply": ([_vp] * 7, ctypes.c_int),
    "tci_heff_apply_staged": ([_vp] * 13, ctypes.c_int),
    "tci_env_workspace_size": ([_vp, ctypes.c_int] + [_vp] * 5 + [ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tci_env_update": ([_vp, ctypes.c_int] + [_vp] * 5, ctypes.c_int),
    "tci_cplx_conj": ([_vp] * 3, ctypes.c_int),
    "tci_svd_workspace_size": ([_vp, ctypes.c_int, ctypes.c_int, _i64p, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)],
                               ctypes.c_int),
    "tci_svd": ([_vp, _vp, ctypes.c_int, _vp, _vp, _vp], ctypes.c_int),
    "tci_trunc_svd": ([_vp, _vp, ctypes.c_int, _vp, _vp, _vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                       ctypes.c_int64, ctypes.c_double, ctypes.c_double, _i64p], ctypes.c_int),
    "tci_svd_info": ([_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tci_mps_mpo_zipup_workspace_size": ([_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.c_int64,
                                          ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tci_mps_mpo_zipup": ([_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                           ctypes.c_int64, ctypes.c_double, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tci_tebd_theta": ([_vp, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p, _vp, ctypes.c_char_p], ctypes.c_int),
    "tci_comm_init": ([_vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "tci_comm_unique_id": ([ctypes.c_char_p], ctypes.c_int),
    "tci_allgather": ([_vp, _vp, _vp], ctypes.c_int),
    "tci_ipc_handle": ([_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tci_ipc_open": ([ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(_vp)], ctypes.c_int),
    "tci_ipc_close": ([_vp], ctypes.c_int),
    "tci_gather_register": ([_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp)], ctypes.c_int),
    "tci_heff_apply_gather": ([_vp] * 7, ctypes.c_int),
    "tci_gather_status": ([_vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tci_launch_count": ([_vp, _i64p], ctypes.c_int),
    "tci_profile_enable": ([_vp, ctypes.c_int], ctypes.c_int),
    "tci_set_gemm_algorithm": ([_vp, ctypes.c_int], ctypes.c_int),
    "tci_ozaki_params": ([ctypes.c_int64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                          ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tci_ozaki_params_complex": ([ctypes.c_int64, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 5, ctypes.c_int),
    "tci_set_ozaki_complex": ([_vp, ctypes.c_int], ctypes.c_int),
    "tci_set_f32_algorithm": ([_vp, ctypes.c_int], ctypes.c_int),
    "tci_graph_begin": ([_vp], ctypes.c_int),
    "tci_graph_end": ([_vp, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "tci_graph_launch": ([_vp, _vp], ctypes.c_int),
    "tci_graph_destroy": ([_vp], ctypes.c_int),
    "tci_ozaki_params_f32": ([ctypes.c_int64, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 4, ctypes.c_int),
    "tci_get_gemm_algorithm": ([_vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tci_set_ozaki_guard": ([_vp, ctypes.c_double], ctypes.c_int),
    "tci_ozaki_guard_stats": ([_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tci_norm": ([_vp, _vp, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tci_normalize": ([_vp, _vp, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tci_scale": ([_vp, _vp, ctypes.c_double, ctypes.c_double, _vp], ctypes.c_int),
    "tci_linear_combine": ([_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_double), _vp], ctypes.c_int),
    "tci_inner": ([_vp, _vp, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "tci_lanczos_workspace_size": ([_vp] * 6 + [ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tci_heff_lanczos": ([_vp] * 6 + [ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "tci_mps_overlap": ([_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp], ctypes.c_int),
    "tci_profile_query": ([_vp, ctypes.c_int, _i64p] + [ctypes.POINTER(ctypes.c_double)] * 3, ctypes.c_int),
    "tci_heff_plan_tree": ([ctypes.c_int64] * 8 + [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
}
for _n, (_a, _r) in _sig.items():
    _f = getattr(_lib, _n)
    _f.argtypes = _a
    _f.restype = _r


def _ok(code: int, fn: str):
    if code != 0:
        raise TciError(code, fn)


def _i64arr(xs: Sequence[int]):
    xs = [int(x) for x in xs]
    return (ctypes.c_int64 * max(1, len(xs)))(*xs)


def _i32arr(xs: Sequence[int]):
    xs = [int(x) for x in xs]
    return (ctypes.c_int32 * max(1, len(xs)))(*xs)


def _labels(l) -> "ctypes.Array":
    if isinstance(l, (bytes, str)):
        b = l.encode("latin-1") if isinstance(l, str) else l
        return _i32arr(list(b))
    return _i32arr(list(l))


# ---------------------------------------------------------------------------
# 1:1 wrappers of the C ABI
# ---------------------------------------------------------------------------

def tci_version() -> str:
    return _lib.tci_version().decode()


def tci_last_error() -> str:
    return _lib.tci_last_error().decode(errors="replace")


def tci_create_context(device: int = 0, stream: int = 0) -> int:
    h = _vp()
    _ok(_lib.tci_create_context(ctypes.byref(h), int(device), _vp(int(stream) or None)), "tci_create_context")
    return h.value


def tci_destroy_context(ctx: int) -> None:
    _ok(_lib.tci_destroy_context(_vp(ctx)), "tci_destroy_context")


def tci_synchronize(ctx: int) -> None:
    _ok(_lib.tci_synchronize(_vp(ctx)), "tci_synchronize")


def tci_workspace_attach(ctx: int, ptr: int, nbytes: int) -> None:
    _ok(_lib.tci_workspace_attach(_vp(ctx), _vp(ptr or None), int(nbytes)), "tci_workspace_attach")


def tci_tensor_create(ctx: int, dtype: int, shape: Sequence[int], data_ptr: int) -> int:
    h = _vp()
    _ok(_lib.tci_tensor_create(_vp(ctx), int(dtype), len(shape), _i64arr(shape), _vp(data_ptr or None),
                               ctypes.byref(h)), "tci_tensor_create")
    return h.value


def tci_tensor_free(ctx: int, t: int) -> None:
    _ok(_lib.tci_tensor_free(_vp(ctx), _vp(t)), "tci_tensor_free")


def tci_order(ctx: int, t: int) -> int:
    o = ctypes.c_int()
    _ok(_lib.tci_order(_vp(ctx), _vp(t), ctypes.byref(o)), "tci_order")
    return o.value


def tci_shape(ctx: int, t: int) -> Tuple[int, ...]:
    n = tci_order(ctx, t)
    s = (ctypes.c_int64 * max(1, n))()
    _ok(_lib.tci_shape(_vp(ctx), _vp(t), s), "tci_shape")
    return tuple(s[i] for i in range(n))


def tci_size(ctx: int, t: int) -> int:
    n = ctypes.c_int64()
    _ok(_lib.tci_size(_vp(ctx), _vp(t), ctypes.byref(n)), "tci_size")
    return n.value


def tci_size_bytes(ctx: int, t: int) -> int:
    n = ctypes.c_int64()
    _ok(_lib.tci_size_bytes(_vp(ctx), _vp(t), ctypes.byref(n)), "tci_size_bytes")
    return n.value


def tci_copy(ctx: int, src: int, dst: int) -> None:
    _ok(_lib.tci_copy(_vp(ctx), _vp(src), _vp(dst)), "tci_copy")


def tci_tebd_workspace_size(ctx: int, A: int, la: str, B: int, lb: str, U: int, lu: str, T: int, lt: str) -> int:
    n = ctypes.c_size_t()
    _ok(_lib.tci_tebd_workspace_size(_vp(ctx), _vp(A), la.encode("latin-1"), _vp(B), lb.encode("latin-1"), _vp(U),
                                     lu.encode("latin-1"), _vp(T), lt.encode("latin-1"), ctypes.byref(n)),
        "tci_tebd_workspace_size")
    return n.value


def tci_copy_async(ctx: int, src: int, dst: int, lane: int) -> None:
    _ok(_lib.tci_copy_async(_vp(ctx), _vp(src), _vp(dst), int(lane)), "tci_copy_async")


def tci_lane_record(ctx: int, lane: int, slot: int) -> None:
    _ok(_lib.tci_lane_record(_vp(ctx), int(lane), int(slot)), "tci_lane_record")


def tci_lane_wait(ctx: int, lane: int, slot: int) -> None:
    _ok(_lib.tci_lane_wait(_vp(ctx), int(lane), int(slot)), "tci_lane_wait")


def tci_reshape(ctx: int, t: int, new_shape: Sequence[int]) -> None:
    _ok(_lib.tci_reshape(_vp(ctx), _vp(t), len(new_shape), _i64arr(new_shape)), "tci_reshape")


def tci_permute(ctx: int, src: int, new_order: Sequence[int], dst: int) -> None:
    _ok(_lib.tci_permute(_vp(ctx), _vp(src), _i32arr(new_order), _vp(dst)), "tci_permute")


def tci_contract_out_shape(ctx: int, a: int, la, b: int, lb, lc) -> Tuple[int, ...]:
    lcs = _labels(lc)
    nc = len(lc.encode("latin-1")) if isinstance(lc, str) else len(list(lc))
    out = (ctypes.c_int64 * max(1, nc))()
    _ok(_lib.tci_contract_out_shape(_vp(ctx), _vp(a), _labels(la), _vp(b), _labels(lb), nc, lcs, out),
        "tci_contract_out_shape")
    return tuple(out[i] for i in range(nc))


def tci_contract(ctx: int, a: int, la, b: int, lb, c: int, lc) -> None:
    _ok(_lib.tci_contract(_vp(ctx), _vp(a), _labels(la), _vp(b), _labels(lb), _vp(c), _labels(lc)),
        "tci_contract")


def tci_contract_str(ctx: int, a: int, la: str, b: int, lb: str, c: int, lc: str) -> None:
    _ok(_lib.tci_contract_str(_vp(ctx), _vp(a), la.encode("latin-1"), _vp(b), lb.encode("latin-1"),
                              _vp(c), lc.encode("latin-1")), "tci_contract_str")


def tci_contract_workspace_size(ctx: int, a: int, la, b: int, lb, c: int, lc) -> int:
    n = ctypes.c_size_t()
    _ok(_lib.tci_contract_workspace_size(_vp(ctx), _vp(a), _labels(la), _vp(b), _labels(lb), _vp(c),
                                         _labels(lc), ctypes.byref(n)), "tci_contract_workspace_size")
    return n.value


def tci_heff_workspace_size(ctx: int, dtype: int, chi_l, chi_lo, chi_r, chi_ro, d, D, D1, D2) -> int:
    n = ctypes.c_size_t()
    _ok(_lib.tci_heff_workspace_size(_vp(ctx), int(dtype), chi_l, chi_lo, chi_r, chi_ro, d, D, D1, D2,
                                     ctypes.byref(n)), "tci_heff_workspace_size")
    return n.value


def tci_heff_apply(ctx: int, L: int, W1: int, W2: int, R: int, psi: int, out: int) -> None:
    _ok(_lib.tci_heff_apply(*[_vp(x) for x in (ctx, L, W1, W2, R, psi, out)]), "tci_heff_apply")


def tci_heff_apply_staged(ctx: int, L_h: int, W1_h: int, W2_h: int, R_h: int, psi_h: int, out_h: int, L: int,
                          W1: int, W2: int, R: int, psi: int, out: int) -> None:
    _ok(_lib.tci_heff_apply_staged(*[_vp(x) for x in (ctx, L_h, W1_h, W2_h, R_h, psi_h, out_h, L, W1, W2, R, psi,
                                                        out)]), "tci_heff_apply_staged")


def tci_env_workspace_size(ctx: int, side: int, E: int, ket: int, W: int, bra: int, out: int) -> int:
    n = ctypes.c_size_t()
    _ok(_lib.tci_env_workspace_size(_vp(ctx), int(side), *[_vp(x) for x in (E, ket, W, bra, out)], ctypes.byref(n)),
        "tci_env_workspace_size")
    return n.value


def tci_env_update(ctx: int, side: int, E: int, ket: int, W: int, bra: int, out: int) -> None:
    _ok(_lib.tci_env_update(_vp(ctx), int(side), *[_vp(x) for x in (E, ket, W, bra, out)]), "tci_env_update")


def tci_cplx_conj(ctx: int, t_in: int, t_out: int) -> None:
    _ok(_lib.tci_cplx_conj(_vp(ctx), _vp(t_in), _vp(t_out)), "tci_cplx_conj")


def tci_svd_workspace_size(ctx: int, dtype: int, shape: Sequence[int], num_of_bds_as_row: int) -> int:
    n = ctypes.c_size_t()
    _ok(_lib.tci_svd_workspace_size(_vp(ctx), int(dtype), len(shape), _i64arr(shape), int(num_of_bds_as_row),
                                    ctypes.byref(n)), "tci_svd_workspace_size")
    return n.value


def tci_svd(ctx: int, a: int, num_of_bds_as_row: int, u: int, s_diag: int, v_dag: int) -> None:
    _ok(_lib.tci_svd(_vp(ctx), _vp(a), int(num_of_bds_as_row), _vp(u), _vp(s_diag), _vp(v_dag)), "tci_svd")


def tci_trunc_svd(ctx: int, a: int, num_of_bds_as_row: int, u: int, s_diag: int, v_dag: int, chi_min: int,
                  chi_max: int, target_trunc_err: float, s_min: float) -> Tuple[float, int]:
    """Returns (trunc_err, chi); the u / s_diag / v_dag descriptors are reshaped to chi."""
    err = ctypes.c_double()
    chi = ctypes.c_int64()
    _ok(_lib.tci_trunc_svd(_vp(ctx), _vp(a), int(num_of_bds_as_row), _vp(u), _vp(s_diag), _vp(v_dag),
                           ctypes.byref(err), int(chi_min), int(chi_max), float(target_trunc_err), float(s_min),
                           ctypes.byref(chi)), "tci_trunc_svd")
    return err.value, chi.value


def tci_mps_mpo_zipup_workspace_size(ctx: int, A: Sequence[int], W: Sequence[int], chi_max: int) -> int:
    n = ctypes.c_size_t()
    arr = lambda xs: (_vp * len(xs))(*[_vp(x) for x in xs])  # noqa: E731
    _ok(_lib.tci_mps_mpo_zipup_workspace_size(_vp(ctx), len(A), arr(A), arr(W), int(chi_max), ctypes.byref(n)),
        "tci_mps_mpo_zipup_workspace_size")
    return n.value


def tci_mps_mpo_zipup(ctx: int, A: Sequence[int], W: Sequence[int], B: Sequence[int], chi_max: int,
                      s_min: float) -> float:
    """Returns trunc_err; the B descriptors are reshaped to the kept bonds."""
    err = ctypes.c_double()
    arr = lambda xs: (_vp * len(xs))(*[_vp(x) for x in xs])  # noqa: E731
    _ok(_lib.tci_mps_mpo_zipup(_vp(ctx), len(A), arr(A), arr(W), arr(B), int(chi_max), float(s_min),
                               ctypes.byref(err)), "tci_mps_mpo_zipup")
    return err.value


def tci_svd_info(ctx: int) -> Tuple[int, float]:
    sw = ctypes.c_int()
    off = ctypes.c_double()
    _ok(_lib.tci_svd_info(_vp(ctx), ctypes.byref(sw), ctypes.byref(off)), "tci_svd_info")
    return sw.value, off.value


def tci_tebd_theta(ctx: int, A: int, la: str, B: int, lb: str, U: int, lu: str, T: int, lt: str) -> None:
    _ok(_lib.tci_tebd_theta(_vp(ctx), _vp(A), la.encode(), _vp(B), lb.encode(), _vp(U), lu.encode(),
                            _vp(T), lt.encode()), "tci_tebd_theta")


def tci_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _ok(_lib.tci_comm_unique_id(buf), "tci_comm_unique_id")
    return buf.raw


def tci_comm_init(ctx: int, uid: bytes, nranks: int, rank: int) -> None:
    _ok(_lib.tci_comm_init(_vp(ctx), uid, int(nranks), int(rank)), "tci_comm_init")


def tci_allgather(ctx: int, shard: int, full: int) -> None:
    _ok(_lib.tci_allgather(_vp(ctx), _vp(shard), _vp(full)), "tci_allgather")


def tci_ipc_handle(dev_ptr: int):
    """(64-byte cudaIpcMemHandle of the allocation, offset of dev_ptr in it)."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_size_t()
    _ok(_lib.tci_ipc_handle(_vp(dev_ptr), buf, ctypes.byref(off)), "tci_ipc_handle")
    return buf.raw, off.value


def tci_ipc_open(handle: bytes, offset: int) -> int:
    p = _vp()
    _ok(_lib.tci_ipc_open(handle, int(offset), ctypes.byref(p)), "tci_ipc_open")
    return p.value


def tci_ipc_close(dev_ptr: int) -> None:
    _ok(_lib.tci_ipc_close(_vp(dev_ptr)), "tci_ipc_close")


def tci_gather_register(ctx: int, nranks: int, rank: int, full_ptrs, flag_ptrs) -> None:
    fa = (_vp * len(full_ptrs))(*[_vp(int(x)) for x in full_ptrs])
    ga = (_vp * len(flag_ptrs))(*[_vp(int(x)) for x in flag_ptrs])
    _ok(_lib.tci_gather_register(_vp(ctx), int(nranks), int(rank), fa, ga), "tci_gather_register")


def tci_heff_apply_gather(ctx: int, L: int, W1: int, W2: int, R: int, psi: int, full: int) -> None:
    _ok(_lib.tci_heff_apply_gather(_vp(ctx), _vp(L), _vp(W1), _vp(W2), _vp(R), _vp(psi), _vp(full)),
        "tci_heff_apply_gather")


def tci_gather_status(ctx: int) -> int:
    """1 if a gather barrier timed out since registration (synchronizes the stream)."""
    v = ctypes.c_int()
    _ok(_lib.tci_gather_status(_vp(ctx), ctypes.byref(v)), "tci_gather_status")
    return v.value


def tci_launch_count(ctx: int) -> int:
    n = ctypes.c_int64()
    _ok(_lib.tci_launch_count(_vp(ctx), ctypes.byref(n)), "tci_launch_count")
    return n.value


def tci_mps_overlap(ctx: int, bra: Sequence[int], ket: Sequence[int], out: int) -> None:
    n = len(bra)
    b = (_vp * max(1, n))(*[_vp(x) for x in bra])
    k = (_vp * max(1, n))(*[_vp(x) for x in ket])
    _ok(_lib.tci_mps_overlap(_vp(ctx), n, b, k, _vp(out)), "tci_mps_overlap")


TCI_GEMM_DMMA_3M, TCI_GEMM_DMMA_4M, TCI_GEMM_OZAKI_INT8 = 0, 1, 2


def tci_set_gemm_algorithm(ctx: int, algo: int) -> None:
    _ok(_lib.tci_set_gemm_algorithm(_vp(ctx), int(algo)), "tci_set_gemm_algorithm")


def tci_ozaki_params(K: int):
    n, t = ctypes.c_int(), ctypes.c_int()
    mods = (ctypes.c_int * 16)()
    st = _lib.tci_ozaki_params(int(K), ctypes.byref(n), ctypes.byref(t), mods)
    return st, n.value, t.value, [mods[i] for i in range(n.value)]


def tci_graph_begin(ctx: int) -> None:
    _ok(_lib.tci_graph_begin(_vp(ctx)), "tci_graph_begin")


def tci_graph_end(ctx: int) -> int:
    g = ctypes.c_void_p()
    _ok(_lib.tci_graph_end(_vp(ctx), ctypes.byref(g)), "tci_graph_end")
    return g.value


def tci_graph_launch(ctx: int, graph: int) -> None:
    _ok(_lib.tci_graph_launch(_vp(ctx), _vp(graph)), "tci_graph_launch")


def tci_graph_destroy(graph: int) -> None:
    _ok(_lib.tci_graph_destroy(_vp(graph)), "tci_graph_destroy")


TCI_F32_OZAKI_INT8 = 0
TCI_F32_FP64_CORES = 1


def tci_ozaki_params_f32(K: int, cplx: bool):
    n, t, ppm = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    mods = (ctypes.c_int * 16)()
    st = _lib.tci_ozaki_params_f32(int(K), 1 if cplx else 0, ctypes.byref(n), ctypes.byref(t), mods,
                                   ctypes.byref(ppm))
    return st, n.value, t.value, [mods[i] for i in range(n.value)], ppm.value


def tci_set_f32_algorithm(ctx: int, algo: int) -> None:
    _ok(_lib.tci_set_f32_algorithm(_vp(ctx), int(algo)), "tci_set_f32_algorithm")


TCI_OZAKI_CPLX_GAUSS = 0
TCI_OZAKI_CPLX_3M = 1


def tci_set_ozaki_complex(ctx: int, variant: int) -> None:
    _ok(_lib.tci_set_ozaki_complex(_vp(ctx), int(variant)), "tci_set_ozaki_complex")


def tci_ozaki_params_complex(K: int, variant: int = TCI_OZAKI_CPLX_GAUSS):
    n, t, ppm = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    mods, roots = (ctypes.c_int * 16)(), (ctypes.c_int * 16)()
    st = _lib.tci_ozaki_params_complex(int(K), int(variant), ctypes.byref(n), ctypes.byref(t), mods, roots,
                                       ctypes.byref(ppm))
    return st, n.value, t.value, [mods[i] for i in range(n.value)], [roots[i] for i in range(n.value)], ppm.value


def tci_set_ozaki_guard(ctx: int, tol: float) -> None:
    _ok(_lib.tci_set_ozaki_guard(_vp(ctx), float(tol)), "tci_set_ozaki_guard")


def tci_ozaki_guard_stats(ctx: int, reset: bool = False) -> dict:
    g, f, b = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    le, me = ctypes.c_double(), ctypes.c_double()
    _ok(_lib.tci_ozaki_guard_stats(_vp(ctx), 1 if reset else 0, ctypes.byref(g), ctypes.byref(f), ctypes.byref(b),
                                   ctypes.byref(le), ctypes.byref(me)), "tci_ozaki_guard_stats")
    return {"gemms": g.value, "fallbacks": f.value, "balanced": b.value, "last_est": le.value,
            "max_est": me.value}


def tci_get_gemm_algorithm(ctx: int) -> int:
    x = ctypes.c_int()
    _ok(_lib.tci_get_gemm_algorithm(_vp(ctx), ctypes.byref(x)), "tci_get_gemm_algorithm")
    return x.value


def tci_norm(ctx: int, t: int) -> float:
    x = ctypes.c_double()
    _ok(_lib.tci_norm(_vp(ctx), _vp(t), ctypes.byref(x)), "tci_norm")
    return x.value


def tci_normalize(ctx: int, t: int) -> float:
    x = ctypes.c_double()
    _ok(_lib.tci_normalize(_vp(ctx), _vp(t), ctypes.byref(x)), "tci_normalize")
    return x.value


def tci_scale(ctx: int, src: int, s: complex, dst: int) -> None:
    s = complex(s)
    _ok(_lib.tci_scale(_vp(ctx), _vp(src), s.real, s.imag, _vp(dst)), "tci_scale")


def tci_linear_combine(ctx: int, ins: Sequence[int], coefs, out: int) -> None:
    m = len(ins)
    arr = (_vp * m)(*[_vp(x) for x in ins])
    if coefs is None:
        cp = None
    else:
        flat = []
        for c in coefs:
            c = complex(c)
            flat += [c.real, c.imag]
        cp = (ctypes.c_double * (2 * m))(*flat)
    _ok(_lib.tci_linear_combine(_vp(ctx), m, arr, cp, _vp(out)), "tci_linear_combine")


def tci_inner(ctx: int, a: int, b: int, conj_a: bool = True) -> complex:
    out = (ctypes.c_double * 2)()
    _ok(_lib.tci_inner(_vp(ctx), _vp(a), _vp(b), int(bool(conj_a)), out), "tci_inner")
    return complex(out[0], out[1])


def tci_lanczos_workspace_size(ctx: int, L: int, W1: int, W2: int, R: int, psi: int, max_iter: int) -> int:
    n = ctypes.c_size_t()
    _ok(_lib.tci_lanczos_workspace_size(_vp(ctx), _vp(L), _vp(W1), _vp(W2), _vp(R), _vp(psi), int(max_iter),
                                        ctypes.byref(n)), "tci_lanczos_workspace_size")
    return n.value


def tci_heff_lanczos(ctx: int, L: int, W1: int, W2: int, R: int, psi: int, max_iter: int, tol: float):
    e = ctypes.c_double()
    it = ctypes.c_int()
    _ok(_lib.tci_heff_lanczos(_vp(ctx), _vp(L), _vp(W1), _vp(W2), _vp(R), _vp(psi), int(max_iter), float(tol),
                              ctypes.byref(e), ctypes.byref(it)), "tci_heff_lanczos")
    return e.value, it.value


PROF_GEMM, PROF_SKINNY, PROF_PERMUTE, PROF_I8 = 0, 1, 2, 3


def tci_profile_enable(ctx: int, on: bool) -> None:
    _ok(_lib.tci_profile_enable(_vp(ctx), int(bool(on))), "tci_profile_enable")


def tci_profile_query(ctx: int, kind: int) -> dict:
    n = ctypes.c_int64()
    ms, fl, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _ok(_lib.tci_profile_query(_vp(ctx), int(kind), ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl),
                               ctypes.byref(by)), "tci_profile_query")
    return {"launches": n.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}


def tci_heff_plan_tree(chi_l, chi_lo, chi_r, chi_ro, d, D, D1, D2) -> Tuple[str, float, bool]:
    buf = ctypes.create_string_buffer(128)
    macs = ctypes.c_double()
    fast = _lib.tci_heff_plan_tree(chi_l, chi_lo, chi_r, chi_ro, d, D, D1, D2, buf, 128, ctypes.byref(macs))
    return buf.value.decode(), macs.value, bool(fast)


# ---------------------------------------------------------------------------
# torch convenience layer (marshalling only)
# ---------------------------------------------------------------------------

def _torch_dtype_code(t) -> int:
    import torch
    m = {torch.float32: TCI_R32, torch.float64: TCI_R64, torch.complex64: TCI_C64, torch.complex128: TCI_C128}
    if t.dtype not in m:
        raise TypeError(f"unsupported dtype {t.dtype}")
    return m[t.dtype]


class Context:
    """A TCI context on one CUDA device/stream with a torch-owned workspace."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        self.torch = torch
        self.device = int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        self.handle = tci_create_context(self.device, int(stream.cuda_stream))
        self._ws = None
        self._ws_bytes = 0
        self._desc: Dict[tuple, int] = {}
        self._ws_need: Dict[tuple, int] = {}

    # -- descriptors ---------------------------------------------------------
    def tensor(self, t) -> int:
        """Descriptor for a contiguous torch tensor (cached by pointer/shape/dtype)."""
        if not t.is_contiguous():
            raise ValueError("TCI tensors are dense row-major: pass a contiguous tensor")
        key = (t.data_ptr(), tuple(t.shape), t.dtype)
        h = self._desc.get(key)
        if h is None:
            if len(self._desc) >= 8192:   # bounded: descriptors are host-side only (no kernel holds one)
                for old in self._desc.values():
                    tci_tensor_free(self.handle, old)
                self._desc.clear()
            h = tci_tensor_create(self.handle, _torch_dtype_code(t), tuple(t.shape), t.data_ptr())
            self._desc[key] = h
        return h

    def host_tensor(self, t) -> int:
        return self.tensor(t)

    def free_descriptors(self):
        for h in self._desc.values():
            tci_tensor_free(self.handle, h)
        self._desc.clear()
        self._ws_need.clear()

    # -- workspace -----------------------------------------------------------
    def _on_stream(self):
        """Allocations for work on the context stream are made on that stream
        (the caching allocator then orders their reuse after it)."""
        return self.torch.cuda.stream(self.stream)

    def ensure_workspace(self, nbytes: int):
        if nbytes <= self._ws_bytes:
            return
        torch = self.torch
        nbytes = int(nbytes)
        if self._ws is not None:
            # kernels already queued on the context stream may still use the
            # old workspace: its memory is reused only after they complete
            self._ws.record_stream(self.stream)
        with self._on_stream():
            self._ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        ptr = (self._ws.data_ptr() + 255) // 256 * 256
        tci_workspace_attach(self.handle, ptr, nbytes)
        self._ws_bytes = nbytes

    def _on_current_stream(self) -> bool:
        return self.torch.cuda.current_stream(self.device).cuda_stream == self.stream.cuda_stream

    def _empty(self, shape, dtype, device=None):
        dev = device if device is not None else f"cuda:{self.device}"
        if self._on_current_stream():   # (the stream context manager costs several us per call)
            return self.torch.empty(shape, dtype=dtype, device=dev)
        with self._on_stream():
            return self.torch.empty(shape, dtype=dtype, device=dev)

    def _empty_like(self, x):
        with self._on_stream():
            return self.torch.empty_like(x)

    # -- operations ----------------------------------------------------------
    def permute(self, x, new_order, out=None):
        if out is None:
            out = self._empty([x.shape[p] for p in new_order], dtype=x.dtype, device=x.device)
        tci_permute(self.handle, self.tensor(x), list(new_order), self.tensor(out))
        return out

    def contract_out_shape(self, a, la, b, lb, lc):
        return tci_contract_out_shape(self.handle, self.tensor(a), la, self.tensor(b), lb, lc)

    def contract(self, a, la, b, lb, lc, out=None):
        if out is None:
            shape = self.contract_out_shape(a, la, b, lb, lc)
            out = self._empty(shape, dtype=a.dtype, device=a.device)
        ha, hb, hc = self.tensor(a), self.tensor(b), self.tensor(out)
        # the planner's workspace answer depends on dtype, shapes, labels and
        # whether the output aliases an input (R8) -- not on the addresses
        pc, nc = out.data_ptr(), out.numel() * out.element_size()
        alias = any(x.data_ptr() < pc + nc and pc < x.data_ptr() + x.numel() * x.element_size() for x in (a, b))
        key = (a.dtype, tuple(a.shape), tuple(b.shape), tuple(out.shape), alias,
               la if isinstance(la, str) else tuple(la), lb if isinstance(lb, str) else tuple(lb),
               lc if isinstance(lc, str) else tuple(lc))
        ws = self._ws_need.get(key)
        if ws is None:
            ws = tci_contract_workspace_size(self.handle, ha, _labels_list(la), hb, _labels_list(lb), hc,
                                             _labels_list(lc))
            self._ws_need[key] = ws
        self.ensure_workspace(ws)
        if isinstance(la, str) and isinstance(lb, str) and isinstance(lc, str):
            tci_contract_str(self.handle, ha, la, hb, lb, hc, lc)
        else:
            tci_contract(self.handle, ha, la, hb, lb, hc, lc)
        return out

    def heff_workspace_size(self, L, W1, W2, R, psi):
        return tci_heff_workspace_size(self.handle, _torch_dtype_code(L), L.shape[0], L.shape[2], psi.shape[3],
                                       R.shape[2], psi.shape[1], L.shape[1], W1.shape[1], W2.shape[1])

    def heff_apply(self, L, W1, W2, R, psi, out=None):
        if out is None:
            out = self._empty((L.shape[2], psi.shape[1], psi.shape[2], R.shape[2]), dtype=psi.dtype,
                                   device=psi.device)
        self.ensure_workspace(self.heff_workspace_size(L, W1, W2, R, psi))
        tci_heff_apply(self.handle, *[self.tensor(x) for x in (L, W1, W2, R, psi, out)])
        return out

    def heff_apply_staged(self, hosts, devs):
        """tci_heff_apply_staged: hosts / devs = (L, W1, W2, R, psi, out) host and
        device twins; the result lands in hosts[5] (copies overlap compute), or
        stays in devs[5] when hosts[5] is None (inputs staged only)."""
        self.ensure_workspace(self.heff_workspace_size(devs[0], devs[1], devs[2], devs[3], devs[4]))
        tci_heff_apply_staged(self.handle, *[None if x is None else self.tensor(x) for x in hosts],
                              *[self.tensor(x) for x in devs])
        return devs[5] if hosts[5] is None else hosts[5]

    def env_update(self, side, E, ket, W, bra=None, out=None):
        """Environment update (tci_env_update): side 0 = left, 1 = right; bra defaults to ket."""
        bra = ket if bra is None else bra
        if out is None:
            shape = ((ket.shape[2], W.shape[1], bra.shape[2]) if side == 0 else
                     (ket.shape[0], W.shape[0], bra.shape[0]))
            out = self._empty(shape, dtype=ket.dtype, device=ket.device)
        h = [self.tensor(x) for x in (E, ket, W, bra, out)]
        self.ensure_workspace(tci_env_workspace_size(self.handle, side, *h))
        tci_env_update(self.handle, side, *h)
        return out

    def cplx_conj(self, x, out=None):
        """Complex conjugate (tci_cplx_conj); out=x conjugates in place."""
        if out is None:
            out = self._empty_like(x)
        tci_cplx_conj(self.handle, self.tensor(x), self.tensor(out))
        return out

    def tebd_theta(self, A, la, B, lb, U, lu, lt, out=None):
        if out is None:
            dims = {}
            for t, l in ((A, la), (B, lb), (U, lu)):
                for ch, n in zip(l, t.shape):
                    dims[ch] = n
            out = self._empty([dims[ch] for ch in lt], dtype=A.dtype, device=A.device)
        self.ensure_workspace(tci_tebd_workspace_size(self.handle, self.tensor(A), la, self.tensor(B), lb,
                                                      self.tensor(U), lu, self.tensor(out), lt))
        tci_tebd_theta(self.handle, self.tensor(A), la, self.tensor(B), lb, self.tensor(U), lu,
                       self.tensor(out), lt)
        return out

    def _svd_outputs(self, a, k, cap):
        torch = self.torch
        u = self._empty(tuple(a.shape[:k]) + (cap,), dtype=a.dtype, device=a.device)
        s = self._empty((cap,), dtype=torch.float64, device=a.device)
        vd = self._empty((cap,) + tuple(a.shape[k:]), dtype=a.dtype, device=a.device)
        return u, s, vd

    def _fresh(self, t) -> int:
        # uncached descriptor (trunc_svd reshapes its outputs' descriptors)
        return tci_tensor_create(self.handle, _torch_dtype_code(t), tuple(t.shape), t.data_ptr())

    def svd(self, a, num_of_bds_as_row):
        """tci::svd: returns (u, s_diag, v_dag)."""
        k = int(num_of_bds_as_row)
        I = 1
        for x in a.shape[:k]:
            I *= int(x)
        kappa = min(I, a.numel() // max(I, 1))
        u, s, vd = self._svd_outputs(a, k, kappa)
        self.ensure_workspace(tci_svd_workspace_size(self.handle, _torch_dtype_code(a), tuple(a.shape), k))
        tci_svd(self.handle, self.tensor(a), k, self.tensor(u), self.tensor(s), self.tensor(vd))
        return u, s, vd

    def trunc_svd(self, a, num_of_bds_as_row, chi_min, chi_max, target_trunc_err, s_min):
        """tci::trunc_svd (2): returns (u, s_diag, v_dag, trunc_err),
        truncated to the chi the strategy keeps."""
        k = int(num_of_bds_as_row)
        I = 1
        for x in a.shape[:k]:
            I *= int(x)
        kappa = min(I, a.numel() // max(I, 1))
        cap = min(max(int(chi_min), int(chi_max)), kappa)
        u, s, vd = self._svd_outputs(a, k, max(cap, 1))
        self.ensure_workspace(tci_svd_workspace_size(self.handle, _torch_dtype_code(a), tuple(a.shape), k))
        hs = [self._fresh(x) for x in (u, s, vd)]
        try:
            err, chi = tci_trunc_svd(self.handle, self.tensor(a), k, *hs, chi_min, chi_max, target_trunc_err,
                                     s_min)
        finally:
            for h in hs:
                tci_tensor_free(self.handle, h)
        # the buffers hold the dense truncated tensors: view them with the chi shapes
        u = u.view(-1)[: u.numel() // cap * chi].view(tuple(a.shape[:k]) + (chi,))
        s = s[:chi]
        vd = vd.view(-1)[: vd.numel() // cap * chi].view((chi,) + tuple(a.shape[k:]))
        return u, s, vd, err

    def mps_mpo_zipup(self, A, W, chi_max, s_min=0.0):
        """Compressed W|psi> by zip-up (tci_mps_mpo_zipup): returns (B sites, trunc_err)."""
        torch = self.torch
        n = len(A)
        caps, left = [], 1
        for i in range(n):
            dout = W[i].shape[3]
            c = 1 if i == n - 1 else min(int(chi_max), left * dout, A[i].shape[2] * W[i].shape[1])
            caps.append((left, dout, c))
            left = c
        B = [self._empty(c, dtype=A[0].dtype, device=A[0].device) for c in caps]
        ha, hw = [self.tensor(x) for x in A], [self.tensor(x) for x in W]
        self.ensure_workspace(tci_mps_mpo_zipup_workspace_size(self.handle, ha, hw, chi_max))
        hb = [self._fresh(x) for x in B]
        try:
            err = tci_mps_mpo_zipup(self.handle, ha, hw, hb, chi_max, s_min)
            shapes = [tci_shape(self.handle, h) for h in hb]
        finally:
            for h in hb:
                tci_tensor_free(self.handle, h)
        out = [b.view(-1)[: int(np.prod(sh))].view(sh) for b, sh in zip(B, shapes)]
        return out, err

    def svd_info(self):
        return tci_svd_info(self.handle)

    def set_gemm_algorithm(self, algo: int):
        tci_set_gemm_algorithm(self.handle, algo)

    def set_ozaki_guard(self, tol: float):
        tci_set_ozaki_guard(self.handle, tol)

    def set_ozaki_complex(self, variant: int):
        tci_set_ozaki_complex(self.handle, variant)

    def set_f32_algorithm(self, algo: int):
        tci_set_f32_algorithm(self.handle, algo)

    def capture(self, fn):
        """Record the library calls fn() makes on this context into a CUDA
        graph (tci_graph_begin / tci_graph_end) without running them; returns
        (graph handle, fn's return value). Outputs must be preallocated
        (out=...) and the workspace already large enough: run fn once eagerly
        first. Replay with replay(graph); free with tci_graph_destroy."""
        tci_graph_begin(self.handle)
        try:
            r = fn()
        except BaseException:
            try:
                tci_graph_destroy(tci_graph_end(self.handle))
            except TciError:
                pass
            raise
        return tci_graph_end(self.handle), r

    def replay(self, graph: int):
        tci_graph_launch(self.handle, graph)

    def ozaki_guard_stats(self, reset: bool = False) -> dict:
        return tci_ozaki_guard_stats(self.handle, reset)

    def gemm_algorithm_name(self) -> str:
        return {TCI_GEMM_DMMA_3M: "dmma3m", TCI_GEMM_DMMA_4M: "dmma4m",
                TCI_GEMM_OZAKI_INT8: "ozaki"}.get(tci_get_gemm_algorithm(self.handle), "?")

    def norm(self, x) -> float:
        return tci_norm(self.handle, self.tensor(x))

    def inner(self, a, b, conj_a=True) -> complex:
        return tci_inner(self.handle, self.tensor(a), self.tensor(b), conj_a)

    def linear_combine(self, ins, coefs=None, out=None):
        if out is None:
            out = self._empty_like(ins[0])
        tci_linear_combine(self.handle, [self.tensor(x) for x in ins], coefs, self.tensor(out))
        return out

    def scale(self, x, s, out=None):
        if out is None:
            out = self._empty_like(x)
        tci_scale(self.handle, self.tensor(x), s, self.tensor(out))
        return out

    def heff_lanczos(self, L, W1, W2, R, psi, max_iter=60, tol=1e-12):
        """Lowest eigenpair of H_eff; psi (start vector) is overwritten by the Ritz vector."""
        hs = [self.tensor(x) for x in (L, W1, W2, R, psi)]
        self.ensure_workspace(tci_lanczos_workspace_size(self.handle, *hs, max_iter))
        return tci_heff_lanczos(self.handle, *hs, max_iter, tol)

    def mps_overlap(self, bra, ket, out=None):
        if out is None:
            out = self._empty((bra[-1].shape[2], ket[-1].shape[2]), dtype=bra[0].dtype, device=bra[0].device)
        tci_mps_overlap(self.handle, [self.tensor(x) for x in bra], [self.tensor(x) for x in ket], self.tensor(out))
        return out

    def copy(self, src, dst):
        tci_copy(self.handle, self.tensor(src), self.tensor(dst))
        return dst

    # asynchronous lanes: 0 = context stream, 1 = h2d copy lane, 2 = d2h copy lane
    def copy_async(self, src, dst, lane: int):
        tci_copy_async(self.handle, self.tensor(src), self.tensor(dst), lane)
        return dst

    def lane_record(self, lane: int, slot: int):
        tci_lane_record(self.handle, lane, slot)

    def lane_wait(self, lane: int, slot: int):
        tci_lane_wait(self.handle, lane, slot)

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        tci_comm_init(self.handle, uid, nranks, rank)

    def allgather(self, shard, full):
        tci_allgather(self.handle, self.tensor(shard), self.tensor(full))
        return full

    def gather_register(self, nranks: int, rank: int, full_ptrs, flag_ptrs):
        tci_gather_register(self.handle, nranks, rank, full_ptrs, flag_ptrs)

    def heff_apply_gather(self, L, W1, W2, R, psi, full):
        """tci_heff_apply_gather: this rank's slab, gathered into every rank's full."""
        self.ensure_workspace(self.heff_workspace_size(L, W1, W2, R, psi))
        tci_heff_apply_gather(self.handle, *[self.tensor(x) for x in (L, W1, W2, R, psi, full)])
        return full

    def gather_status(self) -> int:
        return tci_gather_status(self.handle)

    def launch_count(self) -> int:
        return tci_launch_count(self.handle)

    def synchronize(self):
        tci_synchronize(self.handle)

    def close(self):
        if self.handle:
            self.free_descriptors()
            tci_destroy_context(self.handle)
            self.handle = 0


def _labels_list(l):
    if isinstance(l, str):
        return list(l.encode("latin-1"))
    return list(l)

"""ctypes binding of ``librfxc.so`` (the C ABI declared in include/rfxc.h).

The library is built in-tree by ``paper_2511_19493_b200.build`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
shared object is missing or no CUDA device is present, every product call
raises.  Device buffers are torch tensors; their ``data_ptr()`` and the
current stream's handle are passed straight through.
"""

from __future__ import annotations

import ctypes
import os

from .errors import BudgetError, DataError, RfxError

_HERE = os.path.dirname(os.path.abspath(__file__))
BUILD_DIR = os.path.join(_HERE, "_build")
LIB_PATH = os.path.join(BUILD_DIR, "librfxc.so")

RFXC_OK, RFXC_EDATA, RFXC_EBUDGET, RFXC_ERUNTIME, RFXC_ECUDA = range(5)
NODES_F32, NODES_F64, NODES_F32_NUMERIC, NODES_F32_B2, NODES_F32_B2_NUMERIC = 0, 1, 2, 3, 4
UPPER_I32, UPPER_F64, BLOCK_I32 = 0, 1, 2
Q_MODES = {"f32": 0, "f16": 1, "i8": 2, "nf4": 3}

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double

# name -> (restype, argtypes); must match include/rfxc.h exactly
SIGNATURES = {
    "rfxc_last_error": (ctypes.c_char_p, []),
    "rfxc_version": (ctypes.c_int, []),
    "rfxc_device_info": (ctypes.c_int, [ctypes.c_int, P, P, P]),
    "rfxc_values_to_f32": (ctypes.c_int, [P, I64, P, P, P]),
    "rfxc_forest_pack": (ctypes.c_int, [P, P, P, P, P, P, P, I32, I64, P, I32, I32, P, P, P]),
    "rfxc_forest_pack_host": (ctypes.c_int, [P, P, P, P, P, P, P, I32, P, I32, I32, P, P, P,
                                             I32]),
    "rfxc_values_to_f32_host": (ctypes.c_int, [P, I64, P, P, I32]),
    "rfxc_leaf_codes": (ctypes.c_int, [P, P, I32, I32, I32, I32, P, I64, P, P]),
    "rfxc_transpose_i32": (ctypes.c_int, [P, I64, I64, P, P]),
    "rfxc_transpose_i32_ex": (ctypes.c_int, [P, I64, I64, I64, P, I64, P, P]),
    "rfxc_leaf_order": (ctypes.c_int, [P, I64, I32, P, P, P]),
    "rfxc_permute_rows_f32": (ctypes.c_int, [P, I64, I32, P, P, P]),
    "rfxc_bucket_scratch_bytes": (I64, [I64, I32]),
    "rfxc_outlier_work_bytes": (I64, [I64]),
    "rfxc_leaf_codes_rows": (ctypes.c_int, [P, P, I32, I32, I32, I32, P, I64, I64, I64, P, P]),
    "rfxc_h2d_rows": (ctypes.c_int, [P, P, I64, I64, I32, I64, I64, P]),
    "rfxc_oob_votes": (ctypes.c_int, [P, I64, I32, P, P, P, I32, P, P]),
    "rfxc_outlier_packed": (ctypes.c_int, [P, I64, F64, P, P, P]),
    "rfxc_outlier_lowrank": (ctypes.c_int, [P, I64, I32, F64, P, P]),
    "rfxc_bucket": (ctypes.c_int, [P, I64, I32, P, I32, P, P, P, P, P]),
    "rfxc_bucket_trees": (ctypes.c_int, [P, I64, I32, P, I32, I32, I32, P, P, P, P, P]),
    "rfxc_pair_counts": (ctypes.c_int, [P, I64, I32, I64, I64, I32, P, P, P]),
    "rfxc_pair_counts_leaf": (ctypes.c_int, [P, P, I32, P, P, P, I64, I32, I64, I64, I32, P, P, P]),
    "rfxc_pair_kernel_gate": (ctypes.c_int, [P, I64, I32, F64, P, P]),
    "rfxc_perm_positions": (ctypes.c_int, [P, I64, I32, P, P, P]),
    "rfxc_same_leaf_pairs": (ctypes.c_int, [P, I64, P, P]),
    "rfxc_triblock_count": (ctypes.c_int, [P, I64, I32, I64, I64, F64, P, P]),
    "rfxc_triblock_emit": (ctypes.c_int, [P, I64, I32, I64, I64, F64, P, P, P, P, P, P, P,
                                          P]),
    "rfxc_exclusive_scan_i64": (ctypes.c_int, [P, I64, P, P, P]),
    "rfxc_normals": (ctypes.c_int, [I64, I64, I64, P, P]),
    "rfxc_pack_f32": (ctypes.c_int, [P, I64, I32, I32, P, P]),
    "rfxc_leaf_sums": (ctypes.c_int, [P, P, I64, I64, P, I32, I32, P, P]),
    "rfxc_leaf_gather": (ctypes.c_int, [P, I64, I32, P, P, I32, I32, F64, I32, P, P]),
    "rfxc_sketch_plan": (ctypes.c_int, [P, I32, I64, I32, I64, P, P, P, P]),
    "rfxc_sketch_prepare": (ctypes.c_int, [P, P, I64, I32, I32, I32, I64, I32, P, P]),
    "rfxc_sketch_pass": (ctypes.c_int, [P, P, P, P, P, I64, I32, P, I32, I32, F64, I32, I64, I32,
                                        P, P, P]),
    "rfxc_gram_parts": (ctypes.c_int, [I64]),
    "rfxc_gram": (ctypes.c_int, [P, P, I64, I32, I32, P, P, P]),
    "rfxc_matmul_small": (ctypes.c_int, [P, I64, I32, P, I32, P, P, I32, P]),
    "rfxc_orth_map": (ctypes.c_int, [P, I32, P, P]),
    "rfxc_chol_inv": (ctypes.c_int, [P, I32, F64, P, P]),
    "rfxc_ritz_factor_map": (ctypes.c_int, [P, I32, I32, P, P]),
    "rfxc_sym_eig": (ctypes.c_int, [P, I32, P, P, P]),
    "rfxc_factor_quantize": (ctypes.c_int, [P, I64, I32, P, I32, I32, P, P, P, P, P]),
    "rfxc_dequantize": (ctypes.c_int, [P, P, I64, I32, I32, P, P]),
    "rfxc_pmax": (ctypes.c_int, [P, I64, I32, I64, P, P, P]),
    "rfxc_pmax_draws": (ctypes.c_int, [I64, I64, P, P]),
    "rfxc_mds_work_bytes": (I64, [I64, I32, I32]),
    "rfxc_mds_power": (ctypes.c_int, [P, P, P, I64, I32, F64, P, I32, I32, F64, I64, P, P, P, P,
                                      P]),
    "rfxc_gram_matvec": (ctypes.c_int, [P, I64, I32, F64, P, P, P, P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load librfxc.so and bind every symbol of include/rfxc.h (no CUDA
    context is created)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RfxError(
            f"{path} is missing: build it with paper_2511_19493_b200.build.build() "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Map a C ABI status onto the reference's exception types."""
    if rc == RFXC_OK:
        return
    msg = load().rfxc_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == RFXC_EDATA:
        raise DataError(text)
    if rc == RFXC_EBUDGET:
        raise BudgetError(text, {})
    raise RfxError(text)


# kernels launched per successful call (host-side count for bench.py's
# gpu_launches; rfxc_gram / rfxc_mds_power add their data-dependent extras)
LAUNCHES = {"rfxc_values_to_f32": 1, "rfxc_forest_pack": 1, "rfxc_leaf_codes": 1,
            "rfxc_transpose_i32": 1, "rfxc_transpose_i32_ex": 1, "rfxc_leaf_order": 3,
            "rfxc_permute_rows_f32": 1, "rfxc_bucket": 1, "rfxc_bucket_trees": 1, "rfxc_pair_counts": 1,
            "rfxc_triblock_count": 1, "rfxc_triblock_emit": 1, "rfxc_exclusive_scan_i64": 1,
            "rfxc_normals": 1, "rfxc_pack_f32": 1, "rfxc_leaf_sums": 1, "rfxc_leaf_gather": 1,
            "rfxc_sketch_prepare": 1, "rfxc_sketch_pass": 0, "rfxc_orth_map": 1,
            "rfxc_chol_inv": 1, "rfxc_ritz_factor_map": 1, "rfxc_sym_eig": 1,
            "rfxc_gram": 2, "rfxc_matmul_small": 1, "rfxc_factor_quantize": 3,
            "rfxc_dequantize": 1, "rfxc_pmax": 2, "rfxc_mds_power": 1, "rfxc_gram_matvec": 1,
            "rfxc_outlier_packed": 3, "rfxc_outlier_lowrank": 1,
            "rfxc_oob_votes": 1, "rfxc_leaf_codes_rows": 1, "rfxc_pair_counts_leaf": 1,
            "rfxc_perm_positions": 1, "rfxc_same_leaf_pairs": 1, "rfxc_pmax_draws": 1,
            "rfxc_pair_kernel_gate": 1}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(load(), name)(*args), name)
    launch_count += LAUNCHES.get(name, 0)
    if name == "rfxc_mds_power":
        launch_count += int(args[7])  # start-vector normals, one per component
    elif name == "rfxc_sketch_pass":  # a leaf-sum and a gather kernel per tree batch (the last adds up Y)
        Bl, T = int(args[6]), int(args[11])
        launch_count += 2 * ((Bl + T - 1) // T)
    elif name in ("rfxc_bucket", "rfxc_bucket_trees"):  # launches of <= 2 trees per SM
        trees = int(args[2]) if name == "rfxc_bucket" else int(args[6]) - int(args[5])
        launch_count += max(0, (trees + 2 * _sms() - 1) // (2 * _sms()) - 1)


def _sms() -> int:
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def ptr(t) -> ctypes.c_void_p:
    """Raw device pointer of a torch tensor (or None)."""
    return ctypes.c_void_p(None if t is None else t.data_ptr())


def stream_handle():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def require_cuda():
    """The product path runs on the GPU only; fail loudly otherwise."""
    import torch
    if not torch.cuda.is_available():
        raise RfxError("no CUDA device: the proximity path runs only on the GPU "
                       "(there is no CPU fallback)")
    load()
    return torch.device("cuda", torch.cuda.current_device())

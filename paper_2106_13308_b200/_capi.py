"""ctypes binding of the C ABI in include/vqmc_b200.h (libvqmc_b200.so, built in-tree).

There is no fallback: if the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libvqmc_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")

lib = C.CDLL(LIB_PATH)

VQMC_OK, VQMC_ERR_INVALID, VQMC_ERR_NUMERIC, VQMC_ERR_CUDA, VQMC_ERR_NCCL, VQMC_ERR_SR = 0, 1, 2, 3, 4, 5

_vp = C.c_void_p
_i32, _i64, _u64, _dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class StepStats(C.Structure):
    _fields_ = [("energy_mean", C.c_double), ("energy_var", C.c_double), ("grad_norm", C.c_double),
                ("cut_sum", C.c_int64), ("cut_sq_sum", C.c_int64), ("best_cut", C.c_int32),
                ("batch", C.c_int32)]


_SIGS = {
    "vqmc_gpu_device_count": [C.POINTER(C.c_int)],
    "vqmc_gpu_create": [C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _i64, C.c_int, C.POINTER(_vp)],
    "vqmc_gpu_destroy": [_vp],
    "vqmc_gpu_set_edges": [_vp, _vp, _i64],
    "vqmc_gpu_param_count": [_vp, C.POINTER(_i64)],
    "vqmc_gpu_set_params": [_vp, _vp],
    "vqmc_gpu_get_params": [_vp, _vp],
    "vqmc_gpu_sample": [_vp, C.c_int, _vp, _u64, _u64, _u64, _vp, _vp],
    "vqmc_gpu_log_psi": [_vp, _vp, C.c_int, _vp, _vp],
    "vqmc_gpu_maxcut_energy": [_vp, _vp, C.c_int, _vp, _vp],
    "vqmc_gpu_set_spec": [_vp, _vp, _vp, _vp, _vp, _vp, _i64],
    "vqmc_gpu_clear_spec": [_vp],
    "vqmc_gpu_local_energy": [_vp, _vp, C.c_int, _vp, _vp],
    "vqmc_gpu_weighted_grad": [_vp, _vp, _vp, C.c_int, _vp],
    "vqmc_gpu_gradient_from_locals": [_vp, _vp, _vp, C.c_int, _vp],
    "vqmc_gpu_adam_step": [_vp, _vp, _dbl, _dbl, _dbl, _dbl, _i64],
    "vqmc_gpu_adam_reset": [_vp],
    "vqmc_gpu_comm_unique_id": [_vp],
    "vqmc_gpu_comm_init": [_vp, _vp, C.c_int, C.c_int],
    "vqmc_gpu_train_step": [_vp, C.c_int, C.c_int, _vp, _u64, _u64, _u64, _dbl, _dbl, _dbl, _dbl, _i64,
                            C.POINTER(StepStats)],
    "vqmc_gpu_sr_direction": [_vp, _vp, C.c_int, _vp, _dbl, _dbl, C.c_int, C.c_int, _vp, C.POINTER(C.c_int),
                              C.POINTER(_dbl)],
    "vqmc_gpu_train_step_sr": [_vp, C.c_int, C.c_int, _vp, _u64, _u64, _u64, _dbl, _dbl, _dbl, C.c_int, C.c_int,
                               C.c_int, C.POINTER(StepStats), C.POINTER(C.c_int), C.POINTER(_dbl)],
    "vqmc_pooled_stats": [_i64, _i64, _i64, _i64, C.POINTER(_dbl), C.POINTER(_dbl)],
    "vqmc_gpu_last_cuts": [_vp, _vp, C.c_int],
    "vqmc_gpu_last_samples": [_vp, _vp, C.c_int],
    "vqmc_gpu_last_gradient": [_vp, _vp],
    "vqmc_gpu_evaluate": [_vp, C.c_int, _vp, _u64, _u64, _u64, _vp],
    "vqmc_gpu_synchronize": [_vp],
    "vqmc_gpu_set_phase_timing": [_vp, C.c_int],
    "vqmc_gpu_set_graph": [_vp, C.c_int],
    "vqmc_gpu_phase_times": [_vp, _vp],
    "vqmc_gpu_set_kernel_timing": [_vp, C.c_int],
    "vqmc_gpu_kernel_times": [_vp, _vp, _vp, C.c_int, C.POINTER(C.c_int)],
    "vqmc_gpu_kernel_timeline": [_vp, _vp, _vp, _vp, C.c_int, C.POINTER(C.c_int)],
    "vqmc_default_made_hidden": [C.c_int],
    "vqmc_made_init": [C.c_int, C.c_int, _u64, _vp, _vp],
    "vqmc_stream_uniforms": [_u64, _u64, _u64, _i64, _vp],
    "vqmc_random_maxcut_graph": [C.c_int, _u64, _vp, _i64, C.POINTER(_i64)],
    "vqmc_random_regular_graph": [C.c_int, C.c_int, _u64, _vp, _i64, C.POINTER(_i64)],
    "vqmc_erdos_renyi_graph": [C.c_int, C.c_double, _u64, _vp, _i64, C.POINTER(_i64)],
    "vqmc_random_tim": [C.c_int, _u64, _vp, _vp, _vp, _vp, _vp],
    "vqmc_load_spec": [C.c_char_p, C.POINTER(C.c_int), _vp, _vp, _vp, _vp, _vp, _i64, C.POINTER(_i64)],
    "vqmc_save_spec": [C.c_char_p, C.c_int, _vp, _vp, _vp, _vp, _vp, _i64],
    "vqmc_load_graph": [C.c_char_p, C.POINTER(C.c_int), _vp, _i64, C.POINTER(_i64)],
    "vqmc_save_graph": [C.c_char_p, C.c_int, _vp, _i64],
}
for _name, _args in _SIGS.items():
    fn = getattr(lib, _name)
    fn.argtypes = _args
    fn.restype = C.c_int
lib.vqmc_last_error.restype = C.c_char_p
lib.vqmc_last_error.argtypes = []
lib.vqmc_mix_seed.restype = C.c_uint64
lib.vqmc_mix_seed.argtypes = [_u64, _u64]
lib.vqmc_gpu_launch_count.restype = C.c_int64
lib.vqmc_gpu_launch_count.argtypes = [_vp]

# exported symbols declared in include/vqmc_b200.h (checked by tests/test_capi_symbols.py)
EXPORTS = sorted(list(_SIGS) + ["vqmc_last_error", "vqmc_mix_seed", "vqmc_gpu_launch_count"])


class VqmcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class SrSolveError(VqmcError):
    """SR conjugate gradient missed its residual contract (optimizer.hpp:46-55)."""


def check(rc: int) -> None:
    """Map a status code to the reference's exception types (ValueError ~ std::invalid_argument)."""
    if rc == VQMC_OK:
        return
    msg = lib.vqmc_last_error().decode()
    if rc == VQMC_ERR_INVALID:
        raise ValueError(msg)
    if rc == VQMC_ERR_SR:
        raise SrSolveError(rc, msg)
    raise VqmcError(rc, msg)


def ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C ABI must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def pack_bits(x: np.ndarray) -> np.ndarray:
    """B x n 0/1 -> B x ceil(n/32) uint32 words (bit i of sample b = bit i&31 of word i>>5)."""
    x = np.asarray(x)
    B, n = x.shape
    W = (n + 31) // 32
    pad = np.zeros((B, W * 32), np.uint8)
    pad[:, :n] = x != 0
    bits = np.packbits(pad.reshape(B, W, 4, 8)[:, :, :, ::-1], axis=-1).reshape(B, W, 4)
    return np.ascontiguousarray(bits.view("<u4").reshape(B, W))


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    words = np.ascontiguousarray(words, "<u4")
    B, W = words.shape
    by = words.view(np.uint8).reshape(B, W, 4, 1)
    bits = np.unpackbits(by, axis=-1)[:, :, :, ::-1].reshape(B, W * 32)
    return np.ascontiguousarray(bits[:, :n])

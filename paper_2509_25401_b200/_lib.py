"""ctypes binding of the C ABI in include/flashomni_b200.h.

The shared library `_fo_b200.so` is built in-tree by `build.py` (nvcc,
sm_100a). There is no CPU fallback: if the library or a CUDA device is
missing, every operator raises DeviceError.
"""

import ctypes
import pathlib

from .errors import (
    BoundsError,
    ConsistencyError,
    DeviceError,
    ParameterError,
    ShapeError,
    StateError,
)

LIB_PATH = pathlib.Path(__file__).with_name("_fo_b200.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "fo_abi_version": [],
    "fo_last_error": [],
    "fo_num_sms": [],
    "fo_kernel_launches": [],
    "fo_plan_workspace_bytes": [_I, _I],
    "fo_plan_offsets": [_I, _I, _P],
    "fo_plan_schedule_offset": [_I, _I],
    "fo_encode_symbols": [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P],
    "fo_decode_symbols": [_P, _P, _I, _I, _I, _I, _P, _P, _P],
    "fo_plan": [_P, _P, _I, _I, _I, _I, _I, _P, _I, _P, _P, _P],
    "fo_sparse_attention": [_P, _P, _P, _I, _I, _I, _P, _I, _I, _I, _P, _F, _I, _P, _P, _P, _I,
                            _P, _P, _P],
    "fo_sparse_attention_reuse": [_P, _P, _P, _I, _I, _I, _P, _I, _I, _I, _P, _F, _P, _P, _I, _P,
                                  _P, _P, _P, _P],
    "fo_forecast_materialize": [_P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "fo_check_finite": [_P, ctypes.c_longlong, _I, _P, _I, _P, _P],
    "fo_synthetic_x": [_P, _P, _P, _SZ, _I, _F, _F, _F, _P, _P],
    "fo_cache_push": [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P],
    "fo_cache_push_tile": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P],
    "fo_gemm_q": [_P, _I, _I, _P, _I, _I, _P, _P, _P, _F, _P, _I, _P, _P],
    "fo_gemm_qkv": [_P, _I, _I, _P, _I, _I, _P, _P, _P, _P, _F, _P, _I, _P, _P, _P, _P],
    "fo_gemm_o_update": [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "fo_gemm_o_dispatch": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P],
    "fo_gemm_o_dispatch_rows": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _I, _I, _I, _P, _P],
    "fo_check_active_match": [_P, _P, _I, _I, _I, _P, _P],
    "fo_policy_workspace_bytes": [_I, _I, _I],
    "fo_generate_masks": [_P, _P, _I, _I, _I, _I, _D, _D, _D, _I, _P, _P, _P, _SZ, _P],
    "fo_policy_map_workspace_bytes": [_I, _I, _I, _I, _I],
    "fo_policy_compressed_map": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _SZ, _P],
    "fo_policy_block_scores": [_P, _I, _I, _I, _I, _P, _P, _P],
    "fo_policy_select_cached": [_P, _P, _I, _I, _D, _P, _P],
    "fo_policy_select_skip": [_P, _P, _I, _I, _I, _I, _D, _I, _P, _P],
    "fo_online_softmax_update": [_P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P],
    "fo_online_softmax_finalize": [_P, _P, _I, _I, _P, _P, _P],
    "fo_update_entry": [_P, _I, _P, ctypes.c_longlong, _I, _P, _P],
    "fo_forecast_entry": [_P, ctypes.c_longlong, _I, _P, _P, _P],
    "fo_mean_pool_blocks": [_P, _I, _I, _I, _P, _P],
    "fo_rms_norm": [_P, _P, _I, _I, _D, _P, _P],
    "fo_rope": [_P, _P, _P, _I, _I, _P, _P],
    "fo_row_softmax": [_P, _I, _I, _P, _P],
    "fo_masked_block_attention_f32": [_P, _P, _P, _I, _I, _P, _P, _I, _I, _F, _P, _P, _P, _P],
    "fo_matmul_f32": [_P, _P, _P, _I, _I, _I, _I, _P],
}
_RESTYPES = {"fo_last_error": ctypes.c_char_p, "fo_plan_workspace_bytes": _SZ,
             "fo_plan_offsets": None, "fo_policy_workspace_bytes": _SZ,
             "fo_policy_map_workspace_bytes": _SZ,
             "fo_plan_schedule_offset": _SZ, "fo_kernel_launches": ctypes.c_longlong}

# return codes / status bits (flashomni_b200.h)
_CODE_ERRORS = {1: ShapeError, 2: ParameterError, 3: BoundsError, 4: ConsistencyError,
                5: StateError, 6: DeviceError}
ST_CONSISTENCY, ST_STATE, ST_BOUNDS, ST_PARAM, ST_TIMEOUT = 0x1, 0x2, 0x4, 0x8, 0x10

_lib = None

# kernel launches are counted inside the library (fo_kernel_launches): every
# launch site in csrc/ bumps one counter, so multi-kernel entry points count exactly
_launch_base = [0]


def reset_launch_count():
    _launch_base[0] = int(load().fo_kernel_launches())


def launch_count():
    return int(load().fo_kernel_launches()) - _launch_base[0]


def load():
    """Load the extension (once). Raises DeviceError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceError(
            f"CUDA extension {LIB_PATH.name} not built; run __graft_entry__.build() "
            "(the engine has no CPU fallback)"
        )
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:  # pragma: no cover - environment dependent
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from None
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, _I)
    _lib = lib
    return lib


def call(name, *args):
    """Invoke a C-ABI entry point and map a nonzero return code to the
    reference exception class."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc:
        msg = lib.fo_last_error().decode(errors="replace")
        raise _CODE_ERRORS.get(rc, DeviceError)(f"{name}: {msg}")
    return rc


def ptr(t):
    """Device pointer of a tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def raise_status(bits, what):
    """Map device status-word bits to the reference exception classes."""
    if not bits:
        return
    if bits & ST_TIMEOUT:
        raise DeviceError(f"{what}: pipeline watchdog fired")
    if bits & ST_CONSISTENCY:
        raise ConsistencyError(
            f"{what}: symbol contract violated (active query block with every key "
            "block skipped, or mask not uniform over pool groups)"
        )
    if bits & ST_STATE:
        raise StateError(f"{what}: cached tile with a cold cache, or stale symbols")
    if bits & ST_PARAM:
        raise ParameterError(f"{what}: invalid operand values")
    if bits & ST_BOUNDS:
        raise BoundsError(f"{what}: index out of range")

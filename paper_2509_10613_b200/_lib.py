"""ctypes binding of libsigkernel.so (include/sigkernel.h).

The library is built in-tree by paper_2509_10613_b200/build.py (sm_100a).  If
it is missing, or no CUDA device is visible, every entry point raises
NativeUnavailable -- there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes
import os

from .errors import InvalidArgument, InvalidState, NativeUnavailable

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("SK_LIBSIGKERNEL") or os.path.join(HERE, "_native", "libsigkernel.so")

SK_OK, SK_INVALID_ARGUMENT, SK_INVALID_STATE, SK_CUDA_ERROR = 0, 1, 2, 3
STATIC_LINEAR, STATIC_RBF = 0, 1
TRANSFORMS = {None: 0, "none": 0, "time_augment": 1, "lead_lag": 2}

# Every symbol include/sigkernel.h declares, with its ctypes signature.
_vp, _dp, _i64, _ci, _cd, _sz = (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                 ctypes.c_int, ctypes.c_double, ctypes.c_size_t)
SIGNATURES = {
    "sk_abi_version": ([], _ci),
    "sk_last_error": ([], ctypes.c_char_p),
    "sk_device_sms": ([], _ci),
    "sk_dfma_probe_scratch_bytes": ([], _sz),
    "sk_dfma_probe": ([_dp, _ci, ctypes.POINTER(ctypes.c_double), _vp], _ci),
    "sk_forward_batch_workspace_bytes": ([_i64, _i64, _i64, _i64, _ci, _ci, _ci], _sz),
    "sk_forward_batch": ([_dp, _dp, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _dp, _vp, _sz,
                          _vp], _ci),
    "sk_forward_gram_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci], _sz),
    "sk_forward_gram": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _i64, _i64,
                         _dp, _vp, _sz, _vp], _ci),
    "sk_solve_delta_workspace_bytes": ([_i64, _i64, _i64, _ci, _ci], _sz),
    "sk_solve_delta": ([_dp, _i64, _i64, _i64, _ci, _ci, _dp, _vp, _sz, _vp], _ci),
    "sk_solve_delta_grid": ([_dp, _i64, _i64, _ci, _ci, _dp, _vp], _ci),
    "sk_mirror_upper": ([_dp, _i64, _i64, _vp], _ci),
    "sk_backward_batch_workspace_bytes": ([_i64, _i64, _i64, _i64, _ci, _ci, _ci], _sz),
    "sk_backward_batch": ([_dp, _dp, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _dp, _dp, _dp,
                           _dp, _vp, _sz, _vp], _ci),
    "sk_backward_gram_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci],
                                         _sz),
    "sk_backward_gram": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _i64,
                          _i64, _dp, _dp, _dp, _vp, _sz, _vp], _ci),
    "sk_value_and_grad_gram": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd,
                                _i64, _i64, _dp, _dp, _dp, _dp, _vp, _sz, _vp], _ci),
    "sk_forward_batch_f32_workspace_bytes": ([_i64, _i64, _i64, _i64, _ci, _ci, _ci], _sz),
    "sk_forward_batch_f32": ([_vp, _vp, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _vp, _vp, _sz,
                              _vp], _ci),
    "sk_forward_gram_f32_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci],
                                            _sz),
    "sk_forward_gram_f32": ([_vp, _vp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _i64, _i64,
                             _vp, _vp, _sz, _vp], _ci),
    "sk_forward_batch_tf_workspace_bytes": ([_i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci], _sz),
    "sk_forward_batch_tf": ([_dp, _dp, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _ci, _dp, _vp,
                             _sz, _vp], _ci),
    "sk_forward_gram_tf_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci,
                                            _ci], _sz),
    "sk_forward_gram_tf": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _ci, _i64,
                            _i64, _dp, _vp, _sz, _vp], _ci),
    "sk_backward_batch_tf_workspace_bytes": ([_i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci], _sz),
    "sk_backward_batch_tf": ([_dp, _dp, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _ci, _dp, _dp,
                              _dp, _dp, _vp, _sz, _vp], _ci),
    "sk_backward_gram_tf_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci,
                                             _ci], _sz),
    "sk_backward_gram_tf": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _ci,
                             _i64, _i64, _dp, _dp, _dp, _dp, _vp, _sz, _vp], _ci),
    "sk_transform_adjoint": ([_dp, _i64, _i64, _i64, _ci, _dp, _ci, _vp], _ci),
    "sk_backward_gram_acc_tf_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci,
                                                 _ci, _ci], _sz),
    "sk_backward_gram_acc_tf": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _ci,
                                 _i64, _i64, _dp, _dp, _vp, _vp, _vp, _sz, _vp], _ci),
    "sk_signature_length": ([_i64, _ci], _i64),
    "sk_signature_workspace_bytes": ([_i64, _i64, _i64, _ci, _ci], _sz),
    "sk_signature": ([_dp, _dp, _i64, _i64, _i64, _ci, _ci, _dp, _vp, _sz, _vp], _ci),
    "sk_signature_backward_workspace_bytes": ([_i64, _i64, _i64, _ci, _ci], _sz),
    "sk_signature_backward": ([_dp, _dp, _i64, _i64, _i64, _ci, _ci, _dp, _dp, _vp, _sz, _vp],
                              _ci),
    "sk_grad_acc_bytes": ([_i64, _i64, _i64], _sz),
    "sk_grad_acc_init": ([_vp, _i64, _i64, _i64, _dp, _i64, _i64, _ci, _vp], _ci),
    "sk_grad_acc_finalize": ([_vp, _i64, _i64, _i64, _dp, _ci, _vp], _ci),
    "sk_backward_gram_acc_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _ci],
                                             _sz),
    "sk_backward_gram_acc": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _cd, _i64,
                              _i64, _dp, _dp, _vp, _vp, _vp, _sz, _vp], _ci),
    "sk_backward_gram_acc_cols": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci, _i64,
                                   _i64, _i64, _i64, _dp, _dp, _vp, _vp, _vp, _sz, _vp], _ci),
    "sk_backward_gram_acc_f32_workspace_bytes": ([_i64, _i64, _i64, _i64, _i64, _ci, _ci, _ci],
                                                 _sz),
    "sk_backward_gram_acc_f32": ([_dp, _dp, _i64, _i64, _i64, _i64, _i64, _ci, _ci, _i64, _i64,
                                  _dp, _dp, _vp, _vp, _vp, _sz, _vp], _ci),
}

_lib = None


def load(require_device: bool = True):
    """Load the library (once).  Raises NativeUnavailable when it cannot run."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise NativeUnavailable(
                f"{SO_PATH} is missing; run `python -m paper_2509_10613_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(SO_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.sk_abi_version() != 1:
            raise NativeUnavailable("libsigkernel ABI version mismatch")
        _lib = lib
    if require_device and not _device_ok:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 kernels cannot run here "
                                    "(there is no CPU fallback)")
        _set_device_ok()
    return _lib


_device_ok = False


def _set_device_ok():
    global _device_ok
    _device_ok = True


def check(rc: int) -> None:
    if rc == SK_OK:
        return
    msg = (_lib.sk_last_error() or b"").decode(errors="replace")
    if rc == SK_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == SK_INVALID_STATE:
        raise InvalidState(msg)
    raise RuntimeError(f"CUDA error in libsigkernel: {msg}")

"""B200-native (sm_100a) signature-kernel hot path of pySigLib (arXiv 2509.10613).

Public API (pySigLib style, torch autograd):
    sig_kernel, sig_kernel_gram, LinearKernel, RBFKernel
    sig_kernel_value_and_grad (k + gradients in one pass, the reference's
        kernel_batch_backward), sig_kernel_gram_value_and_grad (fused G + dF/dX)
    sig_mmd (autograd), sig_mmd_value_and_grad (fused)
    signature (truncated signatures, autograd; transforms inside the kernel)
Reference-compatible numpy facade (sigcore names): paper_2509_10613_b200.sigcore_compat
Multi-GPU Gram sharding: paper_2509_10613_b200.gram_dist
"""

from .api import (LinearKernel, RBFKernel, sig_kernel, sig_kernel_gram,
                  sig_kernel_gram_value_and_grad, sig_kernel_value_and_grad, sig_mmd,
                  sig_mmd_value_and_grad)
from .errors import InvalidArgument, InvalidState, NativeUnavailable
from .signatures import signature

__version__ = "0.1.0"

__all__ = ["signature", "sig_kernel", "sig_kernel_gram", "sig_kernel_gram_value_and_grad",
           "sig_kernel_value_and_grad", "sig_mmd",
           "sig_mmd_value_and_grad", "LinearKernel", "RBFKernel", "InvalidArgument",
           "InvalidState", "NativeUnavailable", "__version__"]

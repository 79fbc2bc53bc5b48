"""B200-native CSR sparse direct convolution (arXiv 2005.04091 hot path).

The compute lives in ``libspconv.so`` (include/spconv.h, sm_100a CUDA kernels);
``spconv`` is the thin ctypes binding with the C-ABI's names; ``parallel`` is
the batch-sharded multi-GPU driver over torch.distributed/NCCL.
"""
from .spconv import (KERNEL_AUTO, KERNEL_GENERIC, KERNEL_TILED, SparseConv2d,  # noqa: F401
                     SpconvError, load_library, spconv_create, spconv_debug_decoded,
                     spconv_destroy, spconv_forward, spconv_forward_host,
                     spconv_fused_relu_maxpool, spconv_output_dims, spconv_plan_info,
                     status_string)

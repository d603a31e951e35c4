"""B200-native facet-consensus deblurring (Mourya et al., arXiv 1705.06603).

The product is libdeblur.so (C ABI in include/deblur.h, CUDA kernels for
sm_100a in csrc/); `deblur` is its ctypes binding.  Importing this package
does not touch the GPU; creating a handle does, and fails loudly without one.
"""
from .deblur import (ABI_VERSION, CONV_AUTO, CONV_DIRECT, CONV_FFT, Deblur, DeblurError, Params,  # noqa: F401
                     lib, make_params, nccl_id, plan_facets, plan_messages, problem_params)

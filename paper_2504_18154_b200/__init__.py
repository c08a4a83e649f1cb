"""B200-native PaDG instance hot path of EcoServe (arXiv 2504.18154).

The product is the CUDA/C++ library ``libecoserve.so`` behind the C ABI in
``include/ecoserve.h``; this package is its thin Python binding:

* ``_lib``     -- ctypes prototypes of every exported symbol (loads the .so; no fallback)
* ``instance`` -- an instance handle (torch only allocates the borrowed buffers)
* ``macro``    -- the host macro-instance scheduler (Alg. 1/2) and its DES mode
* ``ops``      -- op-level entry points used by the kernel parity tests
* ``build``    -- in-tree nvcc build for sm_100a
"""
from ._lib import EcoError, load  # noqa: F401

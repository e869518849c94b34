"""B200-native hot path of Fast Ordering ICA (arXiv 2408.17118).

The product is liboica.so (CUDA kernels for sm_100a behind the C ABI in include/oica.h);
`oica` is its ctypes binding.  This package never imports the test oracle.
"""
from . import oica  # noqa: F401
from .oica import Context, Extraction, OicaError  # noqa: F401

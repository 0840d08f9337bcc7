"""B200-native QR-TEBD bond update (arXiv 2212.09782): sm_100a complex128
kernels behind a C-ABI (include/qrtebd_c.h); see DESIGN.md."""
from ._capi import LIB_PATH, load  # noqa: F401

__version__ = "0.1.0"

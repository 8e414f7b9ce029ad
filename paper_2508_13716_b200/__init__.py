"""B200-native CaPGNN hot path: halo exchange + neighbour aggregation.

Drop-in for halopart's train entry point (simulator.run) with real sm_100a
kernels behind a C ABI (include/capgnn.h, libcapgnn.so).
"""

from .errors import DomainError, HalopartError, ParseError

__version__ = "0.1.0"

__all__ = ["DomainError", "HalopartError", "ParseError", "__version__"]

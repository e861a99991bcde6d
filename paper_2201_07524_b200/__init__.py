"""B200-native NFFT fast-summation Sinkhorn (hot path of arXiv 2201.07524, Alg. 2).

The compute path is libsk_nfft.so (csrc/, C-ABI in include/sinkhorn_nfft.h); this package
is its ctypes binding. Importing ``capi`` fails loudly if the library is not built.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "libsk_nfft.so")


def load():
    """Import and return the binding module (raises ImportError if the library is missing)."""
    from . import capi
    return capi

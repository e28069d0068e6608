"""RIKI radial-pattern keyword search (arXiv 2001.06770): B200-native hot path.

The product is ``libriki.so`` (C-ABI, include/riki.h, CUDA for sm_100a); ``riki`` is its
thin ctypes binding.  Nothing here imports the CPU oracle (``oracle/``)."""
from .riki import Graph, RikiError, declared_symbols, load  # noqa: F401

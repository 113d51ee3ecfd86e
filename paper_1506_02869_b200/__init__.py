"""B200-native (sm_100a) SMC-in-MPC hot path of Eele & Maciejowski (arxiv 1506.02869).

``paper_1506_02869_b200.smcatm`` is the thin ctypes binding over the C-ABI
library ``libsmcatm.so`` (CUDA kernels for sm_100a).  ``scenarios`` holds the
seeded synthetic inputs.  Importing this package does not load the CUDA
library; ``smcatm.load()`` does, and raises if it is missing.
"""
__all__ = ["scenarios", "smcatm"]

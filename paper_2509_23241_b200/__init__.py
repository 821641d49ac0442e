"""B200-native (sm_100a) V-/I-TiMePReSt pipeline-parallel training step (arXiv 2509.23241).

`tps` is the ctypes binding of the C ABI in include/tps.h; the work runs in
lib/libtps.so (tcgen05/TMA GEMMs, fused update, NCCL p2p transport).
"""

"""B200-native (sm_100a) SonicMoE hot path: libsonic.so (CUDA, C ABI in include/sonic.h)
plus a thin ctypes binding (sonic.py).  See DESIGN.md."""

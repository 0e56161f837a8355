"""B200-native (sm_100a) SQNGD AF/CAF loss+gradient hot path (arXiv 2604.25728).

The compute path is the C-ABI library libsqngd.so (include/sqngd.h), hand-written
CUDA for sm_100a; `sqngd` is the thin ctypes binding (argument marshalling only).
"""

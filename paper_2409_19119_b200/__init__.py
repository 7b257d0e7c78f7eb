"""B200-native (sm_100a) FP64 SEM hot path of arXiv 2409.19119 (NekRS):
matrix-free Helmholtz operator, gather-scatter (local + NCCL halo) and
Jacobi-PCG, exported as the C ABI of include/nek.h (libnek.so) with a thin
ctypes binding in `nek`.  Import `paper_2409_19119_b200.nek` for the calls."""
__all__ = ["nek"]

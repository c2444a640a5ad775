"""B200-native tile-centric mixed-precision GEMM (arxiv 2508.14848).

C <- alpha*A*B + beta*C with a per-tile precision (FP64/FP32/FP16/BF16/E4M3)
chosen by a tile-norm criterion against a user tolerance; see DESIGN.md.
The compute path is libgemm_mp.so (CUDA, sm_100a) behind the C ABI of
include/gemm_mp.h; binding.py marshals arguments, api.py holds a small
torch-facing convenience wrapper (device memory and streams only)."""
from .binding import *  # noqa: F401,F403
from . import binding  # noqa: F401

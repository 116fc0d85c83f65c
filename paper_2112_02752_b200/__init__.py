"""B200-native sparse distributed embedding layer (arXiv 2112.02752's recommender hot path).

The product is libemb.so (include/emb.h, CUDA kernels for sm_100a under csrc/); `emb` is its thin
ctypes binding. Build: `python -m paper_2112_02752_b200.build`.
"""
from .emb import EmbeddingLayer, EmbError, get_unique_id, lib, LIB_PATH  # noqa: F401

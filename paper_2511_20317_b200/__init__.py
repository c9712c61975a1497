"""paper_2511_20317_b200 -- a B200-native (sm_100a) flip-graph walker for ternary
matrix-multiplication schemes (arXiv 2511.20317).  See DESIGN.md and include/fg.h.

The compute path is libfg.so (CUDA, built in-tree by __graft_entry__.build());
importing ``paper_2511_20317_b200.fg`` fails loudly if it is missing.
"""
__all__ = ["fg", "inputs", "pool_sync"]

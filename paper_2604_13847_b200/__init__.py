"""sparsebalance-b200: B200-native SparseBalance hot path (arxiv 2604.13847).

Host decision layer (cost model, sparsity tuner, sparsity-aware batcher) in C++ and the
dynamic block-sparse attention hot path (block scorer, top-k selector, varlen sparse
attention fwd/bwd) as hand-written sm_100a kernels, both behind plain C ABIs
(include/sb_host.h, include/sb_kernels.h). See DESIGN.md.
"""
__version__ = "0.1.0"

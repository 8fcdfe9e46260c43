"""paper_1203_0889_b200 — B200-native (sm_100a) FMM hot path.

The compute lives in ``lib/libfmm_b200.so`` (CUDA, built from ``csrc/``) behind the C-ABI of
``include/fmm_b200.h``; ``fmm`` mirrors the reference's tree / traversal / kernel-operator
API on top of it. Nothing here falls back to the CPU.
"""
from . import _capi
from .fmm import (FMMError, Context, Tree, KernelTables, KernelVisitor, TraversalConfig,
                  build_tree, upward_pass, dual_tree_traverse, downward_pass, potentials,
                  accelerations, evaluate, compute_bounds, morton_key, mac, split_pair, p2m,
                  m2m, m2l, m2l_mutual, l2l, l2p, p2p, evaluate_multipole, laplace_derivatives, m2p_flip,
                  generate_bodies, n_coef, index_of, exponents)

__all__ = ["FMMError", "Context", "Tree", "KernelTables", "KernelVisitor", "TraversalConfig",
           "build_tree", "upward_pass", "dual_tree_traverse", "downward_pass", "potentials",
           "accelerations", "evaluate", "compute_bounds", "morton_key", "mac", "split_pair",
           "p2m", "m2m", "m2l", "m2l_mutual", "l2l", "l2p", "p2p", "evaluate_multipole",
           "laplace_derivatives", "m2p_flip", "generate_bodies", "n_coef", "index_of",
           "exponents", "_capi"]

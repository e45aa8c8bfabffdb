"""B200-native HODLR-multifrontal preconditioner (arXiv 1410.2697 hot path).

Drop-in for the reference package's hot path (``mfhodlr``: ``mf_factorize``,
``mf_solve``, ``gmres``, ``full_pivot_lu``): same names, arguments, statistics
and error messages, with the numeric work in hand-written sm_100a CUDA kernels
behind the C-ABI of ``include/mfh.h`` (``libmfh.so``).
"""

from ._lib import PivotMonotonicityError
from .kernels import BACKEND as KERNEL_BACKEND, full_pivot_lu, full_pivot_lu_batched
from .krylov import (ConvergenceHistory, LinearOperator, Preconditioner, diagonal_preconditioner, gmres,
                     gmres_batched, identity_preconditioner, ilut, ilut_factors_as_csr, mf_preconditioner)
from .mmio import ScalingRecord, load_matrix_market, row_scale, write_matrix_market
from .multifrontal import (ACCELERATED, CONVENTIONAL, FactorStats, FrontRecord, MfFactorization,
                           MfParams, mf_factorize, mf_solve)
from .ordering import (EliminationTree, EtNode, SeparatorTree, SepNode, build_elimination_tree,
                       nested_dissection)
from .problems import gen_hex_q1, gen_p1_delaunay, gen_poisson7, gen_q1_2d, seeded_rhs
from .sparse import AdjGraph, SparseMatrix, adjacency_graph, spmv

__version__ = "0.1.0"

__all__ = [
    "ACCELERATED", "AdjGraph", "CONVENTIONAL", "ConvergenceHistory", "EliminationTree", "EtNode",
    "FactorStats", "FrontRecord", "KERNEL_BACKEND", "LinearOperator", "MfFactorization", "MfParams",
    "PivotMonotonicityError", "Preconditioner", "ScalingRecord", "SepNode", "SeparatorTree", "SparseMatrix",
    "adjacency_graph", "build_elimination_tree", "diagonal_preconditioner", "full_pivot_lu",
    "full_pivot_lu_batched", "gen_hex_q1", "gen_p1_delaunay", "gen_poisson7", "gen_q1_2d", "gmres",
    "gmres_batched", "identity_preconditioner", "ilut", "ilut_factors_as_csr", "load_matrix_market",
    "mf_factorize", "mf_preconditioner", "mf_solve", "nested_dissection", "row_scale", "seeded_rhs", "spmv",
    "write_matrix_market",
]

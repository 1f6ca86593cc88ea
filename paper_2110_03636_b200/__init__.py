"""B200-native HyKKT hybrid direct-iterative KKT solver (arXiv 2110.03636).

Host-side mirror of the reference C++ API (proj/core/include/hkkt/*.hpp)
over libhykkt.so, whose hand-written sm_100a kernels do all numeric work.
"""
from .kkt import BlockKkt4x4, CscMatrix, FullSolution, HGammaSystem, Reduced2x2
from .solver import (CgResult, CholeskyFactor, Device, FullSolveResult, LadderFailure,
                     NotSpdFailure, ReducedSolveResult,
                     RegularizationState, SequenceResult, SolveReport, SolverConfig,
                     SolveStatus, is_success, solve_full, solve_sequence)

__all__ = [
    "BlockKkt4x4", "CscMatrix", "FullSolution", "CholeskyFactor", "Device", "FullSolveResult",
    "NotSpdFailure", "RegularizationState", "SequenceResult", "SolveReport", "SolverConfig",
    "SolveStatus", "is_success", "solve_full", "solve_sequence", "Reduced2x2", "HGammaSystem",
    "CgResult", "LadderFailure", "ReducedSolveResult",
]

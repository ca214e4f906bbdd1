"""B200-native SSQA engine (drop-in for the reference's annealing loop).

The product is libssqa_b200.so (CUDA kernels for sm_100a behind the C ABI
of include/ssqa_cuda.h, plus the C++ facade of include/ssqa/*.hpp).  This
package is the Python view of the same ABI.
"""
from .api import (  # noqa: F401
    AnnealResult, Batch, IsingModel, K_TARGET_TOL, Problem, ReplicaLattice, RunOptions,
    SsaParams, SsqaParams, TracePoint, TrialOutcome, TtsValue, compute_tts, dense_ising,
    gi_compact, gi_ising, i0_schedule, init_lattice, ising_energy, jperp_schedule, pool_stats, pool_trim, replica_energies,
    run_trials, run_trials_fresh, ssa_run, ssa_run_batch, ssqa_run, ssqa_run_batch, ssqa_sweep,
    trial_instance_seeds, tune,
)
from ._lib import (  # noqa: F401
    ENGINE_AUTO, ENGINE_SIMT, ENGINE_TCGEN05, SsqaError, SsqaInvalidArgument, lib,
)

__version__ = "0.1.0"

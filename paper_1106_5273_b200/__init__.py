"""B200-native FMM evaluator for the vortex particle method of Yokota et al.
(arXiv 1106.5273): Biot-Savart velocity (Eq. 1) and vortex stretching (Eq. 3)
of Gaussian-regularised vortex particles in a periodic cube.

The compute path is libfmm_b200.so (hand-written sm_100a CUDA behind the C ABI
in include/fmm.h); ``fmm`` is its ctypes binding.  No CPU fallback exists.
"""
from .fmm import (FMM, FMMError, fmm_config_default, fmm_create, fmm_destroy, fmm_evaluate,  # noqa: F401
                  fmm_comm_unique_id, fmm_debug_mode, fmm_eval_cutoff, fmm_eval_pair_kernel, fmm_evaluate_parts, fmm_get_box, fmm_get_cells, fmm_get_expansions, fmm_get_keys,
                  fmm_get_lists, fmm_get_sizes, fmm_get_stats, fmm_last_error, fmm_set_particles, fmm_step,
                  fmm_evaluate_targets, fmm_rbf_reinit)

__all__ = ["FMM", "FMMError", "fmm_config_default", "fmm_create", "fmm_destroy", "fmm_evaluate",
           "fmm_comm_unique_id", "fmm_debug_mode", "fmm_eval_cutoff", "fmm_eval_pair_kernel", "fmm_evaluate_parts", "fmm_get_box", "fmm_get_cells", "fmm_get_expansions", "fmm_get_keys",
           "fmm_get_lists", "fmm_get_sizes", "fmm_get_stats", "fmm_last_error", "fmm_set_particles", "fmm_step",
           "fmm_evaluate_targets", "fmm_rbf_reinit"]

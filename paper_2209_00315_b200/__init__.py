"""paper_2209_00315_b200 -- B200-native (sm_100a, fp64) BB-preconditioned Newton
solver for the interior-point Benamou-Brenier optimal-transport method of
arXiv 2209.00315.

The product is libbbot.so (C-ABI: include/bbot.h); this package is its thin
ctypes binding.  Importing it without the built library raises ImportError --
there is deliberately no CPU fallback.
"""
from ._bbot import (BBOT_MEM_DEVICE, BBOT_MEM_HOST, EXPORTED, LIB_PATH, BbotError, Context, IpmOpts,
                    SolveStats, SolverOpts, default_ipm_opts, default_solver_opts, lib, nccl_unique_id,
                    slab_plan, time_blocks)

__all__ = ["Context", "SolverOpts", "IpmOpts", "SolveStats", "BbotError", "default_solver_opts",
           "default_ipm_opts", "lib", "LIB_PATH", "EXPORTED", "BBOT_MEM_HOST", "BBOT_MEM_DEVICE", "nccl_unique_id",
           "slab_plan", "time_blocks"]

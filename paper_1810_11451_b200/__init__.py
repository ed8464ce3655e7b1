"""B200-native beamforming (arXiv 1810.11451 "5Gperf", §III): R = W x S.

PAPER.md:84-86: W is a constant 64-antenna x f-flow precoder, S a changing
f x 60 block of symbols, 0 <= f <= 36.  The computation runs in libbf.so
(hand-written sm_100a CUDA, C ABI in include/bf.h); this package is its thin
Python binding.  Importing it loads libbf.so and fails loudly if it is absent.
"""
from ._lib import BfError, Layout, Status, Variant, lib
from .plan import MAX_F, N_ANT, N_RE, Plan, Server, apply_batch, plan_create_status
from .filter import FILTER_N, FilterPlan, filter_plan_create_status
from .ofdm import OFDM_N, OfdmPlan

lib()   # load now: no silent fallback path exists

__all__ = ["Plan", "Server", "apply_batch", "Layout", "Status", "Variant", "BfError", "plan_create_status", "N_ANT", "N_RE",
           "MAX_F", "FilterPlan", "FILTER_N", "filter_plan_create_status", "OfdmPlan", "OFDM_N"]

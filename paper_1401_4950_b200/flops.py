"""Algorithmic FP64 work of the k_rqi kernel, counted per executed element step.

FP64 instruction counts of the dd building blocks as written in csrc/dd.cuh (one FP64 pipe slot each;
an IEEE division costs w_div DFMA slots, measured by scripts/fp64_peak.cu):
  two_sum 6, fast_two_sum 3, two_prod 2, dd_add 20, dd_mul 9, dd_mul_d 6, dd_rcp 30 + w_div.
  qd_step (one dstqds or dqds element, csrc/kernels_vec.cuh) = dd_add + dd_rcp + 3 dd_mul + dd_sub
                                                            = 97 + w_div
  gamma_k (iteration-1 backward pass)                        = 2 dd_mul + dd_add = 38
  z-solve element (norm pass)                                = 2 dd_mul + dd_add = 38
  z-solve element that writes Z                              = 3 dd_mul + dd_add = 47
Flops are reported FMA-equivalent (2 per slot) so they compare with 2 x measured DFMA/s.
"""

SLOTS_QD = 97.0
SLOTS_GAMMA = 38.0
SLOTS_Z = 38.0
SLOTS_ZW = 47.0


def rqi_slots(stats: dict, w_div: float) -> float:
    return (stats["qd_steps"] * (SLOTS_QD + w_div) + stats["qdg_steps"] * SLOTS_GAMMA
            + stats["z_steps"] * SLOTS_Z + stats["zw_steps"] * SLOTS_ZW)


def rqi_flops(stats: dict, n: int, w_div: float) -> float:
    """FMA-equivalent FP64 flops executed by all k_rqi launches of the last solve."""
    return 2.0 * rqi_slots(stats, w_div)

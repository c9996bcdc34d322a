"""Algorithmic FP64 work of the singleton RQI kernel k_rqi2, per executed element step.

FP64 instruction counts of the dd building blocks as written in csrc/dd.cuh (one FP64 pipe slot each):
  two_sum 6, fast_two_sum 3, two_prod 2, dd_add 20, dd_add_d 10, dd_mul 9, dd_mul_d 6,
  dd_rcp 11 (MUFU seed, 5 FMA Newton, 2 FMA residual, 1 MUL, fast_two_sum; no IEEE division).
  qd_step (one dstqds or dqds element, csrc/kernels_vec.cuh) = dd_add + dd_rcp + 3 dd_mul + dd_sub = 78
  + the ||z||^2 recurrence S/T (dd_mul + dd_add_d + dd_mul)                                      = 28
  iteration-1 extras per element: t(i) = 2 dd_mul, gamma_k and S_k + T_k (2 dd_add)               = 58
  explicit z-solve element (zero-pivot fallback)                                                  = 38
  output element z * (1/||z||)                                                                     =  9
Flops are reported FMA-equivalent (2 per slot) so they compare with 2 x measured DFMA/s.
"""

SLOTS_QD = 78.0 + 28.0
SLOTS_ITER1 = 58.0
SLOTS_Z = 38.0
SLOTS_ZW = 9.0
# segmented RQI (kernels_rqi3.cuh): a row of the r-twisted pass on the pivot-recurrence form = reciprocal pair
# (5 FMA) + two dd quotients (2 x 5) + normalisation (3) + dd sum3 (22) + norm recurrence (28) = 68 slots;
# the RQC-only (light) pass drops one quotient, the normalisation and the dd norm (fp64 norm: 3) = 40;
# a row of the fp64 twist search (one lane) = reciprocal pair 5 + quotient 1 + 2 subtractions = 8.
SLOTS_QD_SEG = 68.0
SLOTS_QD_LIGHT = 40.0
SLOTS_TWIST = 8.0
# single/double realisation (seg_pass_sd): reciprocal pair 5 + two binary64 quotients (MUL + 2 FMA each) +
# 2 subtractions + norm recurrence 3 = 16 slots; light pass: one quotient and the fp64 norm = 14
SLOTS_QD_SD = 16.0
SLOTS_QD_LIGHT_SD = 14.0


def rqi_slots(stats: dict, w_div: float = 0.0, sd: bool = False, support: bool = True) -> float:
    """support: the numerical support (A-42) is on, so the z write multiplies only inside each
    column's support (a few hundred rows of C2's 8192): its element steps (stats['zw_steps'] counts whole
    columns) are not credited -- an under-count of ~1 % of the RQI work instead of an 8 % over-count."""
    seg = stats.get("twist_rows", 0) > 0 or stats.get("qd_light", 0) > 0
    qd = SLOTS_QD_SD if sd else (SLOTS_QD_SEG if seg else SLOTS_QD)
    light = SLOTS_QD_LIGHT_SD if sd else SLOTS_QD_LIGHT
    return (stats["qd_steps"] * qd + stats["qdg_steps"] * SLOTS_ITER1
            + stats["z_steps"] * SLOTS_Z + (0.0 if support else stats["zw_steps"] * SLOTS_ZW)
            + stats.get("qd_light", 0) * light + stats.get("twist_rows", 0) * SLOTS_TWIST)


def rqi_flops(stats: dict, n: int, w_div: float = 0.0, sd: bool = False, support: bool = True) -> float:
    """FMA-equivalent FP64 flops executed by the singleton-RQI kernels of the last solve."""
    return 2.0 * rqi_slots(stats, w_div, sd, support)


# x-NegCount (Alg. negcountLDL) per element: dp = d + s (DADD), q = s / dp (one IEEE division),
# s = q * dll - sigma (DMUL + DADD).  The division is counted at the cost the kernels ISSUE for it (north_star:
# "divisions weighted by their issue cost"): div_fast_nocheck (csrc/kernels.cuh) = 7 DFMA + 1 DMUL on the FP64
# pipe (+ one MUFU.RCP64H seed on the XU pipe, not an FP64 slot) -> 3 + 8 = 11 FP64 slots per element.  The
# survey's weighting by the measured cost of a compiler __ddiv_rn (w_div = 13.07 slots, profiles/fp64_peak_r01.json)
# is reported beside it but is not the roofline (it credits work the kernel does not issue).
W_DIV_ISSUE = 8.0


def negcount_slots_per_element(w_div: float = W_DIV_ISSUE) -> float:
    return 3.0 + w_div


def negcount_flops(stats: dict, nb: int, w_div: float = W_DIV_ISSUE) -> float:
    """Algorithmic flops (2 per FP64 slot) of the x-NegCount evaluations on the sequential bisection paths
    (shared-tree nodes, stats['negcount_x_alg']); k-section points off the path are speculative and not
    counted."""
    return 2.0 * stats["negcount_x_alg"] * nb * negcount_slots_per_element(w_div)

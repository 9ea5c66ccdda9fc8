"""FP64 flop accounting for the assembly roofline.

PAIR_FLOPS[kind] = FP64 flops executed per Green's-tensor point-pair
evaluation (2 per DFMA, 1 per DADD / DMUL), measured with ncu
(sm__sass_thread_inst_executed_op_d{fma,add,mul}_pred_on.sum) on the
eval_block kernel over a known number of pairs; see profiles/README.md for
the measurement log.  The factor arithmetic (ACA residual updates, Gram
columns, recompression, forming U' V') is counted exactly by libhmx
(hmx_stats.flops_assembly) from the actual ranks and step counts.
"""

# kind -> flops per pair, ncu round 1 (profiles/r01_pairflops.csv, 512 x 512
# pairs per launch): H 29 DFMA + 3 DADD + 10 DMUL; U 64 + 10 + 54; T 123 + 16 + 97
PAIR_FLOPS = {"H": 71.0, "U": 192.0, "T": 359.0}


def survey_flops(table, steps, rank_before, rank_after, d, kind, pairs):
    """FP64 flops of the REFERENCE algorithm on the actual steps / ranks, the
    work model SURVEY.md 8(d) fixes for the assembly roofline:

        F = F_pair * P + sum_adm [ 8 (d/2) (m+n) K^2        residual updates
                                 + 8 * 2 d (m+n) K^2        Householder QR of both panels
                                 + 8 d (m+n) K r            forming U', V'
                                 + 8 * 22 K^3 ]             K x K SVD

    (m, n in points, K = rank before, r = rank after recompression).  This
    implementation replaces the two QRs by the Gram matrices the ACA already
    accumulates (8 d^2 (m+n)(K+d) per step) and the SVD by a Hermitian
    eigen-solve, so it executes fewer flops than F; `hmx_stats.flops_assembly`
    counts those executed flops.  Returns (F, parts dict).
    """
    import numpy as np

    t = np.asarray(table)
    adm = t[:, 0] == 1
    mn = ((t[:, 2] - t[:, 1]) + (t[:, 4] - t[:, 3])).astype(np.float64)[adm]
    K = np.asarray(rank_before, dtype=np.float64)[adm]
    r = np.asarray(rank_after, dtype=np.float64)[adm]
    parts = {
        "pairs": PAIR_FLOPS[kind] * float(pairs),
        "residual": float(np.sum(8.0 * (d / 2.0) * mn * K * K)),
        "qr": float(np.sum(8.0 * 2.0 * d * mn * K * K)),
        "form": float(np.sum(8.0 * d * mn * K * r)),
        "svd": float(np.sum(8.0 * 22.0 * K ** 3)),
    }
    return sum(parts.values()), parts

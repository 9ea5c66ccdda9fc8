"""FP64 flop accounting for the assembly roofline.

PAIR_FLOPS[kind] = FP64 flops executed per Green's-tensor point-pair
evaluation (2 per DFMA, 1 per DADD / DMUL), measured with ncu
(sm__sass_thread_inst_executed_op_d{fma,add,mul}_pred_on.sum) on the
eval_block kernel over a known number of pairs; see profiles/README.md for
the measurement log.  The factor arithmetic (ACA residual updates, Gram
columns, recompression, forming U' V') is counted exactly by libhmx
(hmx_stats.flops_assembly) from the actual ranks and step counts.
"""

# kind -> flops per pair (initial hand estimates; replaced by the ncu
# calibration recorded in profiles/README.md)
PAIR_FLOPS = {"H": 60.0, "U": 200.0, "T": 330.0}

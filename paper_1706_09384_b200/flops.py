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

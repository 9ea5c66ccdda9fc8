# Refresh the round's profile evidence on one B200 (run under gpurun; the gpurun_out/ merge limit is
# 64 MiB, so the captures are split in two parts):
#   bash tools/profile_round.sh 1   bench line, ncu launch list, ncu --set full of the TC ACA / matvec / form
#   bash tools/profile_round.sh 2   ncu --set full of recompress_core (both modes) and the estimator
set -x
mkdir -p gpurun_out
if [ "${1:-1}" = "1" ]; then
python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
python tools/ncu_target.py U32k 3 > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_U32k.csv \
    python tools/ncu_target.py U32k 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"aca_(tc_)?kernel" -c 2 -o gpurun_out/prof_aca \
    python tools/ncu_target.py U32k 1 > gpurun_out/ncu_aca.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:mv_phase -c 2 -o gpurun_out/prof_mv \
    python tools/ncu_target.py U32k 1 > gpurun_out/ncu_mv.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:form_gemm -c 1 -o gpurun_out/prof_form \
    python tools/ncu_target.py U32k 1 > gpurun_out/ncu_form.log 2>&1
else
ncu --set full --clock-control none -k regex:recompress_core -c 3 -o gpurun_out/prof_rc \
    python tools/ncu_target.py U32k 1 > gpurun_out/ncu_rc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:err_tiles -c 1 -o gpurun_out/prof_est \
    python tools/est_target.py U32k > gpurun_out/ncu_est.log 2>&1
fi

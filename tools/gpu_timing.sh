# Per-role cycle counters of the Gram kernel (MHSK_GRAM_TIMING=1) on a config.
set -u
mkdir -p gpurun_out
for FP4 in ${FP4S:-1 0}; do
  MHSK_FP4=$FP4 MHSK_GRAM_TIMING=1 timeout 300 python tools/prof_run.py --config ${CFG:-c4} --reps 2 > gpurun_out/timing_fp4$FP4.log 2>&1
  echo "fp4=$FP4 rc=$?"; cat gpurun_out/timing_fp4$FP4.log | tail -6
done

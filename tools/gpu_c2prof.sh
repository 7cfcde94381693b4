# Per-kernel launch lists of one config under two sparse modes (PCFG, MODES).
set -u
mkdir -p gpurun_out
for M in ${MODES:-0 2}; do
  MHSK_SPARSE=$M python tools/prof_run.py --config ${PCFG:-c2} --reps 3 > gpurun_out/c2p_$M.log 2>&1; echo "mode $M rc=$? $(tail -1 gpurun_out/c2p_$M.log)"
  MHSK_SPARSE=$M timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2p_launches_$M.csv python tools/prof_run.py --config ${PCFG:-c2} --reps 2 > /dev/null 2>&1; echo "ncu rc=$?"
done

# One ncu --set full capture (with source) of the first Gram launch of a config.
set -u
mkdir -p gpurun_out
python tools/prof_run.py --config ${PCFG:-c4} > gpurun_out/prof_plain.log 2>&1; rc=$?; echo "prof plain rc=$rc"; cat gpurun_out/prof_plain.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tc2 -s ${SKIP:-0} -c 1 \
      -o gpurun_out/gram_full python tools/prof_run.py --config ${PCFG:-c4} > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  tail -2 gpurun_out/ncu_full.log
fi

# Profiling pass (one ncu session per gpurun call): int8 MMA peak, launch
# lists of the bench command, one full capture of the Gram kernel.
set -u
mkdir -p gpurun_out
./tools/mma_peak 3 > gpurun_out/mma_peak.json 2>&1; echo "mma_peak rc=$?"; cat gpurun_out/mma_peak.json
./tools/mxf4_probe peak 3 > gpurun_out/mxf4_peak.json 2>&1; echo "mxf4_peak rc=$?"; cat gpurun_out/mxf4_peak.json
B="python bench.py --config ${CFG:-c4} --steps 2 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/bench_plain.log 2>&1; rc=$?; echo "bench plain rc=$rc"; tail -1 gpurun_out/bench_plain.log | cut -c1-400
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
fi
python tools/prof_run.py --config ${PCFG:-c4} > gpurun_out/prof_plain.log 2>&1; rc=$?; echo "prof plain rc=$rc"; cat gpurun_out/prof_plain.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tc2 -c 1 \
      -o gpurun_out/gram_full python tools/prof_run.py --config ${PCFG:-c4} > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  tail -3 gpurun_out/ncu_full.log
fi

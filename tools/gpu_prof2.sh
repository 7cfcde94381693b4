set -u
mkdir -p gpurun_out
python tools/prof_run.py --config c2 --reps 3 > gpurun_out/p2_c2.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_run.py --config c2 --reps 3 > /dev/null 2>&1; echo "c2 launches rc=$?"
python tools/prof_run.py --config c3 > gpurun_out/p2_c3.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/prof_run.py --config c3 > /dev/null 2>&1; echo "c3 launches rc=$?"
python tools/prof_run.py --config c5 > gpurun_out/p2_c5.log 2>&1; echo "c5 plain rc=$?"; cat gpurun_out/p2_c5.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gram_tc2 -c 1 -o gpurun_out/gram_c5 python tools/prof_run.py --config c5 > gpurun_out/ncu_c5.log 2>&1; echo "c5 ncu rc=$?"; tail -2 gpurun_out/ncu_c5.log

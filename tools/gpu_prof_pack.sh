set -u
mkdir -p gpurun_out
python tools/prof_run.py --config ${PCFG:-c4} > gpurun_out/pp_plain.log 2>&1; echo "plain rc=$?"; cat gpurun_out/pp_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pp_launches.csv python tools/prof_run.py --config ${PCFG:-c4} > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack|transpose|need" -c 3 -o gpurun_out/pack_full python tools/prof_run.py --config ${PCFG:-c4} > gpurun_out/pp_ncu.log 2>&1; echo "full rc=$?"

# One ncu --set full capture (with source) of the round-1 edge pack of c4.
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pack_rows -c 1 -o gpurun_out/pack1_full python tools/prof_run.py --config c4 --reps 1 > gpurun_out/pack1_ncu.log 2>&1; echo "full rc=$?"

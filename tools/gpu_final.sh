# Round evidence: smoke, default bench, every config + reference arm, launch
# list and one ncu --set full capture of the headline Gram kernel.
set -u
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-300
CFGS="c1 c2 c3 c3a3 c4 c4-twins c5" STEPS=3 bash tools/gpu_configs.sh
B="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
bash tools/gpu_ncu_gram.sh

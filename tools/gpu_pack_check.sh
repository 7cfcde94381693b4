# Row-scatter repack check: full GPU suite, then c4 / c4-twins / c5 timings and the c4 launch list.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for C in c4 c4-twins c5; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pk_$C.log 2>&1
  echo "cfg=$C rc=$? $(tail -1 gpurun_out/pk_$C.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['rounds'], d['deleted'])")"
done
B="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"

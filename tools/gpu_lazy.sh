# Lazy vertex operand: new tests, full suite, dense configs + launch list.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "candidate or probe or lazy" > gpurun_out/pytest_new.log 2>&1; echo "new tests rc=$?"; tail -5 gpurun_out/pytest_new.log
if [ "${FULL:-1}" = "1" ]; then
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
CFGS="${CFGS:-c4 c4-twins c5}" STEPS=3 bash tools/gpu_configs.sh 2>&1 | grep -v "^ref\|^{"
B="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_table.py gpurun_out/launches.csv | head -20

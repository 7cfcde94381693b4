set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "candidate or probe or lazy or golden or incremental" > gpurun_out/pytest_new.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pytest_new.log
CFGS="c4 c5 c4-twins" STEPS=3 bash tools/gpu_configs.sh 2>&1 | grep -v "^ref\|^{"
B="python bench.py --config c4-twins --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tw.csv $B > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_table.py gpurun_out/launches_tw.csv | head -30

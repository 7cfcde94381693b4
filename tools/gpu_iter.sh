# Quick iteration: probe-related parity tests, c4/c5 bench, role timing on c4.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "candidate or probe or lazy or golden" > gpurun_out/pytest_new.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_new.log
CFGS="${CFGS:-c4 c5}" STEPS=3 bash tools/gpu_configs.sh 2>&1 | grep -v "^ref\|^{"
FP4S=1 bash tools/gpu_timing.sh 2>&1 | grep -E "gram timing|rounds" | head -3

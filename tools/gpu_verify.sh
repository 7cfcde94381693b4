# New parity tests first, then the full GPU suite, then the dense configs.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "candidate or probe" > gpurun_out/pytest_new.log 2>&1; echo "new tests rc=$?"; tail -5 gpurun_out/pytest_new.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CFGS="${CFGS:-c4 c4-twins c5}" STEPS=3 bash tools/gpu_configs.sh 2>&1 | grep -v "^ref"

# Round-end check: full GPU suite, then the evidence run.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
bash tools/gpu_final.sh

# Chunked-upload check: its parity test, the validation tests, c4 bench (e2e).
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "large_instance_validation or invalid or device_pointer" > gpurun_out/pytest_chunk.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_chunk.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_chunk.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_c4_chunk.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"

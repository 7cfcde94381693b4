nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --maxfail 30 -x -k "simt" > gpurun_out/pytest_simt.log 2>&1; echo "pytest simt rc=$?"
tail -5 gpurun_out/pytest_simt.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --maxfail 30 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --cpu-budget 6 > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
tail -3 gpurun_out/bench_c2.log
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --cpu-budget 8 > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"
tail -3 gpurun_out/bench_c4.log

set -u
mkdir -p gpurun_out
for R in ${RASTERS}; do
  MHSK_RASTER=$R timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x --timeout 600 -k "oracle or config or backends or sharded" > gpurun_out/pytest_r$R.log 2>&1; echo "raster $R pytest rc=$? $(tail -1 gpurun_out/pytest_r$R.log)"
  MHSK_RASTER=$R timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r$R.log 2>&1
  echo "raster=$R rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_r$R.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), 'ms', round(d['roofline']['achieved']), 'TOPS e2e', round(d['e2e']['ms_per_step'],1), d['clocks'], d['rounds'], d['deleted'])")"
done

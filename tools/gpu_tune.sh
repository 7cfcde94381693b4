# Raster sweep for the Gram schedule on one config (bench values only).
set -u
mkdir -p gpurun_out
for R in ${RASTERS:-"8,9"}; do
  MHSK_RASTER=$R timeout 600 python bench.py --config ${CFG:-c4} --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/tune_$R.log 2>&1
  echo "raster=$R rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/tune_$R.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), 'ms', round(d['roofline']['achieved']), 'TOPS', d['clocks'])")"
done

set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x --timeout 600 -k "oracle or config or backends or sharded or pipeline" > gpurun_out/pytest_thr.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_thr.log)"
for C in ${CFGS:-c5 c4}; do
for T in ${THR:-"4,0" "4,8" "4,4" "3,8" "5,4"}; do
  MHSK_THROTTLE=$T timeout 900 python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/thr_${C}_$T.log 2>&1
  echo "cfg=$C thr=$T rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/thr_${C}_$T.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), 'ms', round(d['roofline']['achieved']), 'TOPS', d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done; done

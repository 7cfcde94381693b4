set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pt_all.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pt_all.log)"
for C in ${CFGS:-c1 c2 c3 c3a3}; do for G in 1 0; do
  MHSK_GRAPHS=$G timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gr_${C}_$G.log 2>&1
  echo "cfg=$C graphs=$G $(python -c "import json; d=json.loads(open('gpurun_out/gr_${C}_$G.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms share', round(d['roofline']['gram_share_of_step'],3), 'launches/step', d['gpu_launches']//d['steps'])" 2>&1 | tail -1)"
done; done

set -u
mkdir -p gpurun_out
for C in ${CFGS:-c1 c2 c3}; do for F in 1 0; do
  MHSK_FAST_LOOP=$F timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${C}_$F.log 2>&1
  echo "cfg=$C fast=$F $(python -c "import json; d=json.loads(open('gpurun_out/ab_${C}_$F.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms gram share', round(d['roofline']['gram_share_of_step'],3), 'launches/step', d['gpu_launches']//d['steps'])" 2>&1 | tail -1)"
done; done

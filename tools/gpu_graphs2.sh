set -u
for C in c2 c3 c3a3; do for G in 0 1; do
  MHSK_GRAPHS=$G timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gr_${C}_$G.log 2>&1
  echo "cfg=$C graphs=$G $(python -c "import json; d=json.loads(open('gpurun_out/gr_${C}_$G.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms', d['rounds'], d['deleted'])" 2>&1 | tail -1)"
done; done

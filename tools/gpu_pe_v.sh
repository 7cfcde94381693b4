set -u
for C in c4 c5 c4-twins; do for PE in 12 14 16; do
  MHSK_PROBE_ENTRIES=$PE timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pev_${C}_$PE.log 2>&1
  echo "cfg=$C pe_v=$PE $(python -c "import json; d=json.loads(open('gpurun_out/pev_${C}_$PE.log').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],3), 'ms gram', round(r['gram_share_of_step']*d['ms_per_step'],3))" 2>&1 | tail -1)"
done; done

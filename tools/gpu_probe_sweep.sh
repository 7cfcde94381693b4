# Probe-length sweep (MHSK_PROBE_ENTRIES) on the dense configs.
set -u
mkdir -p gpurun_out
for C in ${CFGS:-c4 c4-twins c5}; do
  for PE in ${PES:-12 14 16 18 20}; do
    MHSK_PROBE_ENTRIES=$PE timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pe_${C}_$PE.log 2>&1
    echo "cfg=$C pe=$PE rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/pe_${C}_$PE.log').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],3), 'ms', 'gram', round(r['gram_share_of_step']*d['ms_per_step'],3), 'ms', round(r['achieved']), 'TF', 'pruned', r['pruned_tiles'], 'del', d['deleted'])" 2>&1 | tail -1)"
  done
done

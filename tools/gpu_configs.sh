# Bench every BASELINE config (+ planted-twin variants) and the reference arm.
set -u
mkdir -p gpurun_out
for C in ${CFGS:-c1 c2 c3 c3a3 c4 c4-twins c5}; do
  timeout 1200 python bench.py --config $C --steps ${STEPS:-3} --warmup 3 --cpu-budget 8 > gpurun_out/cfg_$C.log 2>&1
  echo "cfg=$C rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/cfg_$C.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms', '%.3g'%d['value'], 'e/s', round(d['roofline']['achieved']), 'TOPS share', round(d['roofline']['gram_share_of_step'],3), 'rounds', d['rounds'], d['deleted'], 'pruned', d['roofline'].get('pruned_tiles'), 'cpu', '%.3g'%(d['cpu_baseline'] or {}).get('value',0), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/ref_c4.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/ref_c4.log | cut -c1-300

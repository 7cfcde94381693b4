set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "incremental or oracle or config or backends or sharded or idempotent or reference" > gpurun_out/pt_inc.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pt_inc.log)"
for C in ${CFGS:-c2 c3 c3a3 c4-twins}; do for I in 1 0; do
  MHSK_INCREMENTAL=$I timeout 900 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/inc_${C}_$I.log 2>&1
  echo "cfg=$C inc=$I $(python -c "import json; d=json.loads(open('gpurun_out/inc_${C}_$I.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms gram share', round(d['roofline']['gram_share_of_step'],3), 'rounds', d['rounds'], d['deleted'])" 2>&1 | tail -1)"
done; done

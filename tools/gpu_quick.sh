# Quick GPU loop: smoke, a parity subset over all backends, bench on configs.
set -u
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "${PYK:-oracle or config or known or backends}" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
for C in ${CFGS:-c4}; do
 for BK in ${BACKS:-tc}; do
  timeout 600 python bench.py --config $C --backend $BK --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/bench_${C}_${BK}.log 2>&1
  echo "bench $C $BK rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/bench_${C}_${BK}.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'ms', round(d['roofline']['achieved']), 'TOPS frac', round(d['roofline']['frac'],3), 'share', round(d['roofline']['gram_share_of_step'],3), d['clocks'])" 2>&1 | tail -1)"
 done
done

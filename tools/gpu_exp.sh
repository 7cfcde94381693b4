# Gram kernel experiments (MHSK_GRAM_TUNE bits), c4 role timing + bench.
set -u
for T in 0 1 2 3; do
  echo "== tune=$T"; MHSK_GRAM_TUNE=$T MHSK_GRAM_TIMING=1 timeout 300 python tools/prof_run.py --config c4 2>&1 | grep -E "gram timing|rounds" | grep -v " kernel [0-9]\{5\} cyc" | cut -c1-250
  MHSK_GRAM_TUNE=$T timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step'],3), 'ms')"
done

# Bounds-checked run of the default path with every stage engaged
# (tools/sanitize_run.py on the MHSK_CHECKED build: device assertions at every
# data-derived index, __trap on a violation).  compute-sanitizer is closed on
# this pool (round 2: every tool refused, rc 86, profiles/r02_sanitize.txt).
#   bash tools/gpu_sanitize.sh TAG
set -u
T=${1:-chk}
O=gpurun_out
mkdir -p $O
timeout 900 python tools/sanitize_run.py 20000 > $O/${T}_plain.log 2>&1; echo "plain rc=$?"
for n in 20000 40000; do
    MHSK_LIB=checked timeout 1200 python tools/sanitize_run.py $n > $O/${T}_checked_$n.log 2>&1
    echo "checked $n rc=$? $(grep -c 'MHSK_CHECK failed' $O/${T}_checked_$n.log) violations"
done

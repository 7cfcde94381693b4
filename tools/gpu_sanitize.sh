# compute-sanitizer on the default path with every stage engaged
# (tools/sanitize_run.py; one tool per run):  bash tools/gpu_sanitize.sh TAG
set -u
T=${1:-san}
O=gpurun_out
mkdir -p $O
timeout 600 python tools/sanitize_run.py 20000 > $O/${T}_plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
    n=20000; [ "$tool" = racecheck ] && n=8000
    timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py $n \
        > $O/${T}_${tool}.log 2>&1
    echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${T}_${tool}.log | tail -1)"
done

set -u
for T in 0 16; do
echo "== tune=$T"; MHSK_GRAM_TUNE=$T MHSK_GRAM_TIMING=1 timeout 300 python tools/prof_run.py --config c4 2>&1 | grep -E "gram timing" | grep -v " kernel [0-9]\{5\} cyc" | cut -c1-200
done
for T in 0 4; do

done

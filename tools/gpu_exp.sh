set -u
for L in libmhsk_st4.so libmhsk_st5.so libmhsk.so; do
echo "== $L"; MHSK_LIB=$PWD/paper_2109_06042_b200/$L MHSK_GRAM_TIMING=1 timeout 300 python tools/prof_run.py --config c4 2>&1 | grep -E "gram timing" | grep -v " kernel [0-9]\{5\} cyc" | cut -c1-200
done

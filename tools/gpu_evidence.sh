# Round evidence on one B200 (run through gpurun from the repo root):
#   bash tools/gpu_evidence.sh TAG
# smoke, the default bench line, the reference arm, every config through
# tools/ab.py, the launch list of the headline bench command, and one
# `ncu --set full` capture of each probe Gram phase, the member scan and the
# round-1 edge pack (each command runs once without ncu before it is
# profiled).  Outputs: gpurun_out/TAG_*; summaries go to profiles/ by hand
# (tools/ncu_summary.py, tools/one_kernelization.py).
set -u
T=${1:-ev}
O=gpurun_out
mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/${T}_reference.json 2> $O/${T}_reference.err
echo "reference rc=$?"
timeout 1200 python tools/ab.py c1,c2,c3,c3a3,c4,c4-twins,c4-planted,c5,c5-planted > $O/${T}_configs.jsonl 2>&1
echo "configs rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --secondary none"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv $B \
    > $O/${T}_launches.log 2>&1; echo "launch list rc=$?"
# third kernelization of `ab.py c4 --steps 2` (warm).  Per kernelization:
# gram_tc2_kernel x4 (edge probe, edge full-K pass, vertex probe, vertex
# full-K pass), scan_members x2, pack_rows_csr x3 (round-1 edge pack first)
P="python tools/ab.py c4 --steps 2"
for spec in "gram_tc2_kernel:8:gram_edge_probe" "gram_tc2_kernel:10:gram_vertex_probe" \
            "scan_members:2:scan_members" "pack_rows_csr:6:pack_rows_csr"; do
    IFS=: read -r k skip f <<< "$spec"
    timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${k}" -s $skip -c 1 \
        -o $O/${T}_${f} $P > $O/${T}_${f}.log 2>&1; echo "ncu $f rc=$?"
done

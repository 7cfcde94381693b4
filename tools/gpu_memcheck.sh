# compute-sanitizer memcheck (ONE tool per call) on small kernelizations and a pipeline.
set -u
mkdir -p gpurun_out
cat > /tmp/mc_run.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2109_06042_b200 import _native, interval_trains, nested_chains, plant_twins, random_csr
ctx = _native.context()
for b in ("tc", "tc1", "simt"):
    ctx.set_backend(b)
    for csr in (interval_trains(3000, 1200, 1, 1), plant_twins(random_csr(700, 900, 0.03, 2, 2), 0.03, 0.03, 3),
                nested_chains(12, 30, 3, 4)):
        ctx.kernelize(csr); ctx.reduce_edges(csr, "se"); ctx.reduce_vertices(csr)
        ctx.run_pipeline(csr, ("fe", "dp", "md"), True)
ctx.set_backend("tc")
ctx.generate_random(3000, 2500, 0.01, 3, 5)
print("done")
PY
python /tmp/mc_run.py > gpurun_out/mc_plain.log 2>&1; echo "plain rc=$?"
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python /tmp/mc_run.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.log

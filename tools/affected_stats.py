"""Per-round sizes of the 'affected' sets that incremental rounds would
process (edges containing a vertex deleted in the previous vertex phase;
vertices in an edge deleted in this round's edge phase)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_06042_b200 import _native, config_instance

ctx = _native.context()
for name in sys.argv[1:] or ["c2", "c3", "c3a3", "c4-twins"]:
    if name.startswith("c4"):
        from paper_2109_06042_b200.generate import COUNTER_CONFIGS
        csr, _ = ctx.generate_random(*COUNTER_CONFIGS["c4"], 0)
        if name.endswith("twins"):
            from paper_2109_06042_b200 import plant_twins
            csr = plant_twins(csr, 0.01, 0.01, 1)
    else:
        csr = config_instance(name, 0)
    owner = np.repeat(np.arange(csr.m), np.diff(csr.edge_ptr))
    vtx = csr.edge_vtx
    prev_va = np.ones(csr.n, bool); prev_ea = np.ones(csr.m, bool)
    rows = []
    r = 1
    while True:
        va, ea, st = ctx.kernelize(csr, "dp", r)
        va = va.astype(bool); ea = ea.astype(bool)
        # edge phase of round r: deleted edges = prev_ea & ~ea ; vertex phase deleted = prev_va & ~va
        edel = prev_ea & ~ea
        vdel = prev_va & ~va
        aff_v = np.zeros(csr.n, bool); np.logical_or.at(aff_v, vtx, edel[owner]); aff_v &= prev_va
        aff_e_next = np.zeros(csr.m, bool); np.logical_or.at(aff_e_next, owner, vdel[vtx]); aff_e_next &= ea
        rows.append(dict(round=r, n_alive_start=int(prev_va.sum()), m_alive_start=int(prev_ea.sum()),
                         edel=int(edel.sum()), aff_v_this_round=int(aff_v.sum()), vdel=int(vdel.sum()),
                         aff_e_next_round=int(aff_e_next.sum())))
        if st["rounds"] < r or (edel.sum() == 0 and vdel.sum() == 0):
            break
        prev_va, prev_ea = va, ea
        r += 1
    print(name, csr.n, csr.m)
    for x in rows:
        print("  ", x)

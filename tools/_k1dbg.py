import sys, numpy as np
sys.path.insert(0, '.')
from paper_2502_00778_b200 import Engine, meshgen
from oracle.oracle import Oracle
O = Oracle()
eng = Engine(0)
ms = [meshgen.tet_cube(4, amp=0.1), meshgen.tet_cube(12, amp=0.1), meshgen.tri_square(9, diag_seed=3, amp=0.2),
      meshgen.permute(meshgen.tet_cube(10, amp=0.1)), meshgen.fan_in(meshgen.tet_cube(8, amp=0.1)),
      meshgen.flip23(meshgen.tet_cube(10, amp=0.1)), meshgen.permute(meshgen.tri_square(20, diag_seed=3, amp=0.2))]
for m in ms:
    eng.set_mesh(m)
    eng.build_edges()
    el = eng.edges()
    e, o = O.build_edges(m)
    ok = np.array_equal(el.edges, e) and np.array_equal(el.origin_start, o)
    e2l, ip, inc = O.edge_maps(m, e, o)
    gip, ginc = eng.incidence()
    print("edges", ok, np.array_equal(eng.e2l(), e2l), np.array_equal(gip, ip), np.array_equal(ginc, inc), flush=True)

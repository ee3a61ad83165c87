import sys, os, threading
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2502_00778_b200 import Engine, Mesh, _lib, meshgen
from oracle.oracle import Oracle
O = Oracle()
# (1) more side edges than the side list holds -> whole-mesh fallback, still right
rng = np.random.default_rng(11)
nv, ne = 6000, 1500000
el = rng.integers(0, nv, size=(ne, 4), dtype=np.int32)
ok = (np.sort(el, 1)[:, 1:] != np.sort(el, 1)[:, :-1]).all(1)
el = el[ok]
m = Mesh(3, rng.random(3 * nv), el.reshape(-1), np.zeros(0, np.int32))
eng = Engine(0)
eng.set_mesh(m); n = eng.build_edges()
e, o = O.build_edges(m)
assert np.array_equal(eng.edges().edges, e)
want = O.navs_dualfree(m, e, o)
eng.navs(); g = eng.get_navs()
print("big soup: edges", n, "plan", eng.plan_info(), "side", eng.side_edges(), "err", np.abs(g - want).max() / np.abs(want).max(), flush=True)
eng.volumes(); v = eng.get_volumes(); wv = O.volumes_edge(m, e, want)
print("  vols err", np.abs(v - wv).max() / np.abs(wv).max(), flush=True)
eng.close()
# (2) two contexts interleaved on two host threads
res = {}
def work(tag, mesh):
    en = Engine(0)
    en.set_mesh(mesh); en.build_edges()
    out = []
    for _ in range(5):
        en.navs(); en.volumes(); out.append((en.get_navs().copy(), en.get_volumes().copy()))
    res[tag] = out
    en.close()
ma, mb = meshgen.tet_cube(20, amp=0.15), meshgen.permute(meshgen.tet_cube(18, amp=0.1))
ta = threading.Thread(target=work, args=("a", ma)); tb = threading.Thread(target=work, args=("b", mb))
ta.start(); tb.start(); ta.join(); tb.join()
for tag, mesh in (("a", ma), ("b", mb)):
    e, o = O.build_edges(mesh); w = O.navs_dualfree(mesh, e, o)
    errs = [np.abs(nv_ - w).max() / np.abs(w).max() for nv_, _ in res[tag]]
    same = all(np.array_equal(res[tag][0][0], r[0]) and np.array_equal(res[tag][0][1], r[1]) for r in res[tag])
    print("threads", tag, "max err", max(errs), "repeatable", same, flush=True)

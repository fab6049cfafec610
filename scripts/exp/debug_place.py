"""Compare GPU placement with the oracle on a test case; print the first mismatching call."""
import sys
import numpy as np
sys.path.insert(0, '.')
from gen import make, place_cfg_for
from oracle import oracle as O
from paper_2605_00528_b200 import saga
O.build()
d = make("C4", n_sessions=150, n_nodes=4)
pc = place_cfg_for(d); pc.update(kappa=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
o = O.Oracle(d, pc)
on, om, os_, orr = o.placement()
for rep in range(3):
    t = saga.Trace(d, pc)
    gn, gm, gs, gr = t.placement()
    diff = np.nonzero(on != gn)[0]
    e = d.call_t_us // 100000 + 1
    print("rep", rep, "steals", os_, gs, "reroutes", orr, gr, "n_mig", len(om), len(gm), "ndiff", diff.size)
    if diff.size:
        c = diff[0]
        print("first diff call", c, "epoch", e[c], "session", d.call_session[c], "oracle", on[c], "gpu", gn[c])
        mo = [tuple(x) for x in om]; mg = [tuple(x) for x in gm]
        print("migs oracle", mo[:8]); print("migs gpu", mg[:8])
    t.free()

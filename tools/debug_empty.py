import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2003_03572_b200.sacd import Sacd
dims = (5, 4, 3)
c, v = np.zeros((0, 3), np.uint32), np.zeros(0, np.float32)
for ug in (False, True):
    g = Sacd(c, v, dims, 3, 1, use_graph=ug)
    print("init U", g.factors(0)[0], "M0", g.mttkrp(0)[0])
    for n in range(3):
        out = g.mode_update(n, branch=0, decisions=True)
        print("mode", n, out["E"], out["ti"], "F", g.factors(n)[0], "z", g.get_zprev(n)[0])
    g.close()
ora = O.sacd_run(c, v, dims, 3, 1, 2)
print("oracle U", ora["F"][0][0], ora["f"])

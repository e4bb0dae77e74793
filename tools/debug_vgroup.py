import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_04081_b200 import AdaptiveConfig, problems
from paper_1908_04081_b200.dist import VirtualGroup
from paper_1908_04081_b200.partition import CsrRows
prob = problems.make_problem("c1")
for P in (3,):
    grp = VirtualGroup(CsrRows.of(prob.a), P, depth=8)
    for p in grp.parts:
        print(p.rank, p.n_own, p.n_rows, p.n_local, len(p.values), p.peers, p.send_off, p.recv_off)
    x, t, c, logs = grp.solve(prob, AdaptiveConfig(sigma=8, eps_star=1e-10))
    print(t.total_outer, t.converged)

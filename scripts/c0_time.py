import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1305_5120_b200 as G
from paper_1305_5120_b200.workloads import baseline_matrix
h, lt, _ = baseline_matrix(0, 1000)
cfg = G.SolverConfig(nev=100, buffer=20, degree=15, max_outer_iters=20000)
G.chfsi_solve(h, None, G.SolverConfig(nev=100, buffer=20, degree=15, max_outer_iters=20000, interval="block_top"), seed=1)
t = time.perf_counter(); lam, v, rep = G.chfsi_solve(h, None, cfg, seed=1); dt = time.perf_counter() - t
print("c0 s/solve %.3f iters %d tf %.3f tq %.3f trr %.3f err %.2e" % (dt, rep.outer_iterations, rep.t_filter, rep.t_qr, rep.t_rr, np.max(np.abs(lam - lt[:100]) / np.abs(lt[:100]))))

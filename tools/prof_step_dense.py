"""One c2 MPC update on a dense wind grid (for ncu): python tools/prof_step_dense.py Nx Ny Nz [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02869_b200 import scenarios as sc, smcatm  # noqa: E402

g = tuple(int(v) for v in sys.argv[1:4])
K = int(sys.argv[4]) if len(sys.argv) > 4 else 2
scn, cfg = sc.config(2)
scn["wind_n"] = g
sol = smcatm.Solver(scn, L=cfg.L, S=cfg.S, K=K, sigma=cfg.sigma, seed=cfg.seed)
sol.solve()
torch.cuda.synchronize()
print("ok", sol.launches)

"""One c<N> MPC update through smc_solve (for ncu captures): python tools/prof_step.py [config] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02869_b200 import scenarios as sc, smcatm  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
scn, cfg = sc.config(cfgn)
sol = smcatm.Solver(scn, L=cfg.L, S=cfg.S, K=K, sigma=cfg.sigma, seed=cfg.seed)
sol.solve()
torch.cuda.synchronize()
print("ok", sol.launches)

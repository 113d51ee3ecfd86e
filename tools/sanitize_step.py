"""A small MPC update for compute-sanitizer (racecheck / synccheck / memcheck):
python tools/sanitize_step.py CONFIG L K [S]  -- the config's scenario and solver with L particles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02869_b200 import scenarios as sc, smcatm  # noqa: E402

num, L, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
scn, cfg = sc.config(num)
S = int(sys.argv[4]) if len(sys.argv) > 4 else min(cfg.S, 4)
sol = smcatm.Solver(scn, L=L, S=S, K=K, sigma=cfg.sigma, seed=cfg.seed)
sol.iterate(K - 1)
sol.best_controls(allow_infeasible=True)
sol.mpc_step(scn["x0"])
torch.cuda.synchronize()
print("ok", sol.launches)

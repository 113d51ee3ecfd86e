"""One rank of a world-size-2 libsmcatm context on a shared GPU (used by
test_multirank_gpu.py): collectives through the host shim over a gloo process
group (include/smcatm.h smc_host_collectives), parent rows read in place from
the other process's workspace through CUDA IPC (peer mode) or all-gathered
(SMC_P2P=0).  No kernel of one rank waits on the other: every exchange is a
host-synchronised collective.

    python tests/multirank_worker.py RANK WORLD PORT CONFIG L S K OUT.npz
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, port, num, L, S, K, out = sys.argv[1:9]
    rank, world, L, S, K, num = int(rank), int(world), int(L), int(S), int(K), int(num)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1506_02869_b200 import scenarios as sc, smcatm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    scn, cfg = sc.config(num)
    sol = smcatm.Solver(scn, L=L, S=S, K=K, sigma=cfg.sigma, seed=cfg.seed, rank=rank, world_size=world,
                        host_collectives=True, use_graph=False)
    res = {}
    for k in range(K - 1):
        sol.iterate(1)
        pop = sol.population()
        for key in ("cur", "prop", "surv_mask", "ell", "lam"):
            res[f"{key}_{k}"] = pop[key]
    best, lam, idx = sol.best_controls(allow_infeasible=True)
    res["best"], res["lam_best"], res["idx_best"] = best, np.array([lam]), np.array([idx])
    res["launches"] = np.array([sol.launches])
    np.savez(out, **res)
    sol.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""The library's own world_size > 1 code path on one GPU:
two processes, each a rank of one libsmcatm context (collectives through the
host shim over gloo, so neither rank's kernels wait on the other), against a
single-rank run of the same problem.  Populations (both MH candidates, survivor
masks, log-weights, lambdas) must be bit-identical slice by slice for every
round, and so must the selected controls: the Philox streams are keyed by the
global particle index and the integer CDF makes the ancestors G-invariant.
Both exchange modes: peer (parent rows and CDFs read in place through CUDA IPC
mappings of the other process's workspace) and all-gather (SMC_P2P=0)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("num,L", [(2, 4099), (5, 20000)])
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_world2_bitexact_vs_single(tmp_path, num, L, p2p):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1506_02869_b200 import scenarios as sc, smcatm
    S, K = 3, 4
    port = _port()
    env = dict(os.environ, SMC_P2P=p2p)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "multirank_worker.py"), str(r), "2", str(port),
                               str(num), str(L), str(S), str(K), str(tmp_path / f"r{r}.npz")], env=env)
             for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    scn, cfg = sc.config(num)
    sol = smcatm.Solver(scn, L=L, S=S, K=K, sigma=cfg.sigma, seed=cfg.seed)
    ranks = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    b1 = smcatm.shard_range(L, 2, 1)[0]
    for k in range(K - 1):
        sol.iterate(1)
        pop = sol.population()
        for key in ("cur", "prop", "surv_mask", "lam"):
            both = np.concatenate([ranks[0][f"{key}_{k}"], ranks[1][f"{key}_{k}"]])
            assert np.array_equal(both, pop[key]), (k, key)
        ell = np.concatenate([ranks[0][f"ell_{k}"], ranks[1][f"ell_{k}"]], axis=1)
        assert np.array_equal(ell, pop["ell"]), k
        assert ranks[1][f"cur_{k}"].shape[0] == L - b1
    best, lam, idx = sol.best_controls(allow_infeasible=True)
    for r in range(2):
        assert np.array_equal(ranks[r]["best"], best) and ranks[r]["lam_best"][0] == lam
        assert ranks[r]["idx_best"][0] == idx
    sol.close()

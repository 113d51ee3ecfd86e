"""K2 time per round vs particle count (wave quantisation probe): python tools/wave_probe.py L1 L2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02869_b200 import scenarios as sc, smcatm  # noqa: E402

scn, cfg = sc.config(2)
stream = torch.cuda.Stream()
for L in [int(a) for a in sys.argv[1:]]:
    sol = smcatm.Solver(scn, L=L, S=cfg.S, K=21, sigma=cfg.sigma, seed=cfg.seed, anneal=cfg.anneal,
                        mh=cfg.mh, profile=True, use_graph=True, stream=stream)
    with torch.cuda.stream(stream):
        sol.solve()
        torch.cuda.synchronize()
        sol.phase_times()
        for _ in range(3):
            sol.solve()
        torch.cuda.synchronize()
    ph = sol.phase_times()
    ms, n = ph["rollout"]
    print(f"L={L}: K2 {1000 * ms / n:.1f} us/launch avg over {n} launches, {1e3 * ms / n / L * 1e3:.3f} ns/particle", flush=True)

"""Step time of one c<N> MPC update with and without the per-kernel timing events:
python tools/prof_overhead.py [config] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02869_b200 import scenarios as sc, smcatm  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
scn, cfg = sc.config(cfgn)
stream = torch.cuda.Stream()
for prof in (False, True, False, True):
    sol = smcatm.Solver(scn, L=cfg.L, S=cfg.S, K=cfg.K, sigma=cfg.sigma, seed=cfg.seed, anneal=cfg.anneal,
                        mh=cfg.mh, profile=prof, use_graph=True, stream=stream)
    with torch.cuda.stream(stream):
        for _ in range(3):
            sol.solve()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            sol.solve()
        b.record(stream)
        torch.cuda.synchronize()
    ph = sol.phase_times() if prof else None
    print(f"profile={prof}: {a.elapsed_time(b) / steps:.3f} ms/step", {k: round(v[0] / steps, 3) for k, v in ph.items()} if ph else "")

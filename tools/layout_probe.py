"""K2 layout re-calibration: MPC-step time of the segment vs transposed layout per aircraft count.
python tools/layout_probe.py [K rounds]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1506_02869_b200 import scenarios as sc, smcatm  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 21
_, cfg = sc.config(2)
for n in (5, 6, 7, 9, 10, 11, 12, 13, 17, 18, 20, 22, 24, 26):
    scn = sc.snapshot((n + 1) // 2, n // 2, seed=1002)
    scn["nominal"] = [8.0, 0.0]
    scn["turb_sigma"] = 1.0
    out = {"n": n}
    for lay in ("segment", "transposed"):
        os.environ["SMC_K2_LAYOUT"] = lay
        st = torch.cuda.Stream()
        sol = smcatm.Solver(scn, L=cfg.L, S=cfg.S, K=K, sigma=cfg.sigma, seed=cfg.seed, use_graph=True, stream=st)
        with torch.cuda.stream(st):
            sol.solve()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(3):
                sol.solve()
            e1.record(st)
        torch.cuda.synchronize()
        out[lay] = round(e0.elapsed_time(e1) / 3, 3)
        sol.close()
    print(json.dumps(out), flush=True)

"""Copy one tools/gpu_round2.sh run (gpurun_out/*_TAG.*) into profiles/r02_*: bench lines, reference
arm, GPU test log, closed loops, launch list + summary, ncu --set full metrics, K2 DRAM traffic.
usage: python tools/refresh_profiles.py TAG"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
G = lambda name: os.path.join(ROOT, "gpurun_out", name)      # noqa: E731
P = lambda name: os.path.join(ROOT, "profiles", name)        # noqa: E731


def line(path):
    return next(l for l in open(path) if l.startswith("{"))


open(P("r02_bench_c5.json"), "w").write(line(G(f"bench_c5_{tag}.log")))
open(P("r02_bench_configs.jsonl"), "w").writelines(line(G(f"bench_c{c}_{tag}.log")) for c in (2, 3, 4, 6, 7))
open(P("r02_bench_reference_c5.json"), "w").write(line(G(f"bench_ref_{tag}.log")))
open(P("r02_pytest_gpu.log"), "w").write(open(G(f"pytest_{tag}.log")).read() + open(G(f"smoke_{tag}.log")).read())
# closed loops: the three traffic streams of this run; the mh = 2 / warm-start variants kept from before
old = [json.loads(l) for l in open(P("r02_mpc_loop_audit.jsonl"))]
keep = [json.dumps(d) + "\n" for d in old if "mh=2" in d["config"] or "warm" in d["config"]]
new = [line(G(f"loop_{tr}_{tag}.log")) for tr in ("c3", "mixed", "congested")]
open(P("r02_mpc_loop_audit.jsonl"), "w").writelines(new + keep)
subprocess.run(["cp", G(f"launches_c5_{tag}.csv"), P("r02_launches_bench_c5.csv")], check=True)
with open(P("r02_launches_bench_c5_summary.txt"), "w") as f:
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), G(f"launches_c5_{tag}.csv")],
                   stdout=f, check=True)
for src, dst in ((f"prof_k2c5_{tag}", "r02_ncu_full_c5_k2.json"), (f"prof_k2c2_{tag}", "r02_ncu_full_c2_k2.json"),
                 (f"prof_rsc5_{tag}", "r02_ncu_full_c5_resample.json")):
    if os.path.exists(G(src + ".json")):                    # converted on the box (gpu_round2.sh)
        subprocess.run(["cp", G(src + ".json"), P(dst)], check=True)
        continue
    with open(P(dst), "w") as f:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_full_json.py"), G(src + ".ncu-rep")], stdout=f,
                       check=True)


def gb(v):
    x, u = v.split()
    return float(x) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


tr = json.load(open(P("k2_traffic.json")))
for c in ("c5", "c2"):
    r = json.load(open(P(f"r02_ncu_full_{c}_k2.json")))[0]
    tr[c] = int(gb(r["dram__bytes_read.sum"]) + gb(r["dram__bytes_write.sum"]))
json.dump(tr, open(P("k2_traffic.json"), "w"))
print("profiles refreshed from", tag)

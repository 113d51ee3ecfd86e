"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and its pure-host partition helpers are exact."""
import os
import re
import subprocess
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1506_02869_b200 import build, smcatm
    build.build()
    return smcatm.load()


def _declared():
    txt = open(os.path.join(ROOT, "include", "smcatm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(smc_[a-z0-9_]+|mpc_step)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    from paper_1506_02869_b200 import smcatm
    names = _declared()
    assert "smc_init" in names and "mpc_step" in names and len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", smcatm.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert sorted(smcatm.EXPORTED) == names


def test_library_is_sm100a(lib):
    from paper_1506_02869_b200 import smcatm
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", smcatm.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_workspace_bytes_validation(lib):
    from paper_1506_02869_b200 import smcatm
    cfg = smcatm.Config()
    assert lib.smc_workspace_bytes(cfg) == 0               # L = 0 is invalid
    cfg.n_particles, cfg.max_aircraft, cfg.max_horizon = 1000, 8, 6
    nb = lib.smc_workspace_bytes(cfg)
    assert nb >= 4 * 1000 * 8 * 6 * 3 * 4
    cfg.max_aircraft = 33
    assert lib.smc_workspace_bytes(cfg) == 0


def test_shard_range_partitions(lib):
    from paper_1506_02869_b200 import smcatm
    for L in (1, 7, 1000, 1 << 20):
        for G in (1, 2, 3, 8):
            spans = [smcatm.shard_range(L, G, r) for r in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_shard_offsets(lib):
    from paper_1506_02869_b200 import smcatm
    rng = np.random.default_rng(0)
    Q = rng.integers(0, 2**40, (4, 6)).astype(np.uint64)
    for r in range(4):
        off, tot = smcatm.shard_offsets(Q, r)
        assert np.array_equal(off, Q[:r].sum(0) if r else np.zeros(6, np.uint64))
        assert np.array_equal(tot, Q.sum(0))


def test_slot_count_exact(lib):
    """#{j : floor((jQ+R)/L) < C} against exact rational enumeration."""
    from paper_1506_02869_b200 import smcatm
    rng = np.random.default_rng(1)
    for _ in range(300):
        L = int(rng.integers(1, 60))
        Q = int(rng.integers(1, 2**45))
        R = int(rng.integers(0, Q))
        C = int(rng.integers(0, Q + 1))
        ref = sum(1 for j in range(L) if (j * Q + R) // L < C)
        assert smcatm.slot_count(C, Q, R, L) == ref
    # large L, Q near the 2^62 design bound
    L, Q = 1 << 20, (1 << 20) * (1 << 32)
    R = Q // 3
    for C in (0, 1, Q // 2, Q - 1, Q):
        j = smcatm.slot_count(C, Q, R, L)
        assert (j == 0 or ((j - 1) * Q + R) // L < C) and (j == L or (j * Q + R) // L >= C)


def test_bench_particle_schedule_matches_oracle():
    """bench.py counts work with roofline.particles_of; it must be the schedule
    the oracle (and smc_config.n_particles_final) defines (R44)."""
    import oracle as O
    from paper_1506_02869_b200 import roofline
    for L, Lf, K in ((1000, 400, 4), (16384, 4096, 101), (256, 40, 6), (100, 0, 5), (100, 200, 5), (7, 3, 1)):
        for k in range(K + 2):
            assert roofline.particles_of(L, Lf, K, k) == O.particles_of(L, Lf, K, min(k, max(K - 1, 0))), (L, Lf, K, k)


def test_bench_sample_schedule_matches_oracle():
    import oracle as O
    from paper_1506_02869_b200 import roofline, scenarios as sc
    assert [roofline.sample_schedule(k) for k in range(101)] == [O.sample_schedule(k) for k in range(101)]
    _, cfg = sc.config(6)
    assert sum(roofline.samples_list(cfg)) == 15370


def test_closed_loop_audit_counts():
    """mpc_loop.audit: Eq. avoidance on realised states, completion counts."""
    import numpy as np
    from paper_1506_02869_b200 import mpc_loop, scenarios as sc
    base, _ = sc.config(3)
    tr = sc.traffic(2, 1, seed=3)
    Pr, Ph = float(base["P_r"]), float(base["P_h"])
    st = lambda x, y, z: np.array([x, y, z, 100.0, 0.0, 6e4])
    log = [
        {0: st(0, 0, 1000), 1: st(2 * Pr - 1, 0, 1000), 2: st(0, 0, 1000 + 2 * Ph + 1)},   # 0-1 conflict only
        {0: st(0, 0, 1000), 1: st(2 * Pr + 1, 0, 1000)},                                   # clear (boundary +1)
        {0: st(0, 0, 1000), 2: st(10, 0, 1000 + 2 * Ph - 1)},                              # conflict
    ]
    a = mpc_loop.audit(base, tr, log, {0: (3, "landed"), 2: (5, "exited")}, {0: 10.0, 1: 5.5})
    assert a.sep_violations == 2
    assert a.min_sep_m == 10.0                    # step 2, pair 0-2 (step 0: 0-2 is 2 Ph + 1 apart vertically)
    assert (a.landed, a.exited, a.unfinished, a.n_aircraft) == (1, 1, 1, 3)
    assert a.fuel_total_kg == 15.5


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the oracle on the host cores) prints one JSON line with
    the driver's keys; N > 1 ranks other than 0 print nothing."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                          "--config", "1"], cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--config", "1"], cwd=root, capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0 and not out.stdout.strip()

"""Multi-rank (world_size 2, gloo on CPU) test of the particle-sharded
resampling protocol of DESIGN.md section 9, driven by libsmcatm's host
partition helpers (smc_shard_range, smc_shard_offsets, smc_slot_count):

  1. all-reduce MAX of the per-column log-weight maxima,
  2. all-gather of per-rank integer weight totals -> exclusive offsets,
  3. per rank: marks at the first global offspring slot of each local
     particle, all-reduce MAX of the marks, prefix-max -> ancestors.

The ancestors of every rank's own slots must equal the single-process
oracle's systematic resampling of the whole column bit for bit (G-invariance).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ell, k, seed, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_1506_02869_b200 import smcatm
    N, L = ell.shape
    b, e = smcatm.shard_range(L, world, rank)
    loc = ell[:, b:e]
    # 1. column max (all-reduce MAX)
    m = torch.tensor(loc.max(axis=1) if e > b else np.full(N, -np.inf), dtype=torch.float64)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    m = m.numpy()
    # 2. local integer weights and totals; all-gather totals
    infeasible = ~np.isfinite(m)
    q = np.array([[1 if infeasible[i] else O.det_quant(float(loc[i, l]) - float(m[i])) for l in range(e - b)]
                  for i in range(N)], dtype=np.uint64).reshape(N, e - b)
    Qr = torch.tensor(q.sum(axis=1).astype(np.int64))
    gathered = [torch.zeros_like(Qr) for _ in range(world)]
    dist.all_gather(gathered, Qr)
    Q_all = np.stack([g.numpy() for g in gathered]).astype(np.uint64)
    off, Qtot = smcatm.shard_offsets(Q_all, rank)
    # 3. marks at global slots, all-reduce MAX, prefix max
    marks = np.full((N, L), -1, dtype=np.int64)
    for i in range(N):
        R = (O.r64(6, i, k, seed) * int(Qtot[i])) >> 64
        C = int(off[i])
        for l in range(e - b):
            qq = int(q[i, l])
            if not qq:
                continue
            s0 = smcatm.slot_count(C, int(Qtot[i]), R, L)
            C += qq
            s1 = smcatm.slot_count(C, int(Qtot[i]), R, L)
            if s1 > s0:
                marks[i, s0] = b + l
    mt = torch.tensor(marks)
    dist.all_reduce(mt, op=dist.ReduceOp.MAX)
    anc = np.maximum.accumulate(mt.numpy(), axis=1)
    ret[rank] = anc[:, b:e].tolist()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_resampling_matches_single_process(world):
    import oracle as O
    rng = np.random.default_rng(3)
    N, L = 4, 301
    ell = rng.normal(-20, 6, (N, L))
    ell[rng.uniform(size=(N, L)) < 0.25] = -np.inf
    ell[2] = -np.inf                                   # infeasible column: uniform
    ell[3, :200] = -np.inf                             # all mass on rank 1's particles
    k, seed = 5, 0x5EED0002
    mgr = mp.Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, ell, k, seed, ret), nprocs=world, join=True)
    anc = np.concatenate([np.array(ret[r]) for r in range(world)], axis=1)
    for i in range(N):
        ref = O.resample_column(ell[i], i, k, seed)["anc"]
        assert np.array_equal(anc[i], ref), i

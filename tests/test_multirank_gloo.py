"""Multi-rank (world_size 2, gloo on CPU) test of the particle-sharded
resampling protocol of DESIGN.md section 9, driven by libsmcatm's host
partition helpers (smc_shard_range, smc_shard_offsets, smc_slot_count):

  1. all-reduce MAX of the per-column log-weight maxima,
  2. all-gather of per-rank integer weight totals -> exclusive offsets,
  3. per rank: marks at the first global offspring slot of each local
     particle, all-reduce MAX of the marks, prefix-max -> ancestors.

The ancestors of every rank's own slots must equal the single-process
oracle's systematic resampling of the whole column bit for bit (G-invariance).
The second test follows the exchange the library implements for world > 1
(per-rank integer CDFs all-gathered, owner search, bisection, parent rows read
in place from their owner by survivor mask -- the NVLink peer mode) and checks
ancestors and gathered rows the same way.
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


def _worker_cdf(rank, world, port, ell, rows, surv, k, seed, ret):
    """The implemented exchange (capi.cu run_round, world > 1):
    all-reduce MAX of the column maxima; local inclusive integer CDFs all-gathered;
    each rank's new slot j -> owner rank rho by the prefix of the per-rank totals ->
    bisection in rho's CDF -> parent row read where rho keeps it (x' or x* by
    rho's published survivor mask; the gloo all-gather of the row arrays stands in
    for the NVLink peer mapping)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_1506_02869_b200 import smcatm
    N, L = ell.shape
    b, e = smcatm.shard_range(L, world, rank)
    Lmax = max(smcatm.shard_range(L, world, r)[1] - smcatm.shard_range(L, world, r)[0] for r in range(world))
    loc = ell[:, b:e]
    m = torch.tensor(loc.max(axis=1) if e > b else np.full(N, -np.inf), dtype=torch.float64)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    m = m.numpy()
    infeasible = ~np.isfinite(m)
    C = np.zeros((N, Lmax), dtype=np.int64)                     # local inclusive CDFs, stride Lmax
    for i in range(N):
        run = 0
        for l in range(e - b):
            run += 1 if infeasible[i] else O.det_quant(float(loc[i, l]) - float(m[i]))
            C[i, l] = run
    Call = [torch.zeros_like(torch.tensor(C)) for _ in range(world)]
    dist.all_gather(Call, torch.tensor(C))
    Call = [c.numpy().astype(object) for c in Call]
    lens = [smcatm.shard_range(L, world, r)[1] - smcatm.shard_range(L, world, r)[0] for r in range(world)]
    # peer stand-in: every rank's (x', x*) pair and published masks
    mine = torch.tensor(np.stack([rows[0][b:e], rows[1][b:e]]))
    pad = torch.zeros((2, Lmax) + rows[0].shape[1:], dtype=mine.dtype)
    pad[:, :e - b] = mine
    peers = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(peers, pad)
    ms = torch.zeros(Lmax, dtype=torch.int64)
    ms[:e - b] = torch.tensor(surv[b:e].astype(np.int64))
    pmask = [torch.zeros_like(ms) for _ in range(world)]
    dist.all_gather(pmask, ms)
    anc = np.zeros((N, e - b), dtype=np.int64)
    xnew = np.zeros((e - b,) + rows[0].shape[1:], dtype=rows[0].dtype)
    for i in range(N):
        Qr = [int(Call[r][i, lens[r] - 1]) if lens[r] else 0 for r in range(world)]
        Q = sum(Qr)
        R = (O.r64(6, i, k, seed) * Q) >> 64
        for jl in range(e - b):
            j = b + jl
            t = (j * Q + R) // L
            rho, off = 0, 0
            while rho < world - 1 and t >= off + Qr[rho]:
                off += Qr[rho]
                rho += 1
            c = Call[rho][i, :lens[rho]]
            a = int(np.searchsorted(np.array(c, dtype=object), t - off, side="right"))   # min{a: C_a > t - off}
            anc[i, jl] = smcatm.shard_range(L, world, rho)[0] + a
            bit = (int(pmask[rho][a]) >> i) & 1
            xnew[jl, i] = peers[rho][bit, a, i].numpy()
    ret[rank] = (anc.tolist(), xnew.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_matches_single_process(world):
    """The implemented multi-GPU round (CDF all-gather, owner search, bisection,
    in-place parent read by survivor mask) gives every rank the single-process
    oracle's ancestors and parent rows bit for bit."""
    import oracle as O
    rng = np.random.default_rng(11)
    N, L, H = 3, 257, 4
    ell = rng.normal(-18, 5, (N, L))
    ell[rng.uniform(size=(N, L)) < 0.3] = -np.inf
    ell[1, 100:] = -np.inf                              # mass on the first rank(s) only
    rows = [rng.normal(size=(L, N, H, 3)).astype(np.float32) for _ in range(2)]
    surv = rng.integers(0, 1 << N, size=L).astype(np.uint32)      # per-aircraft survivor masks
    k, seed = 3, 0x5EED0004
    mgr = mp.Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.spawn(_worker_cdf, args=(world, port, ell, rows, surv, k, seed, ret), nprocs=world, join=True)
    anc = np.concatenate([np.array(ret[r][0], dtype=np.int64).reshape(N, -1) for r in range(world)], axis=1)
    xnew = np.concatenate([np.array(ret[r][1], dtype=np.float32).reshape(-1, N, H, 3) for r in range(world)])
    for i in range(N):
        ref = O.resample_column(ell[i], i, k, seed)["anc"]
        assert np.array_equal(anc[i], ref), i
        bits = (surv[ref] >> i) & 1
        want = np.where(bits[:, None, None] == 1, rows[1][ref, i], rows[0][ref, i])
        assert np.array_equal(xnew[:, i], want), i

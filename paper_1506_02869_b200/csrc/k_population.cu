// k_population.cu -- population kernels of libsmcatm (sm_100a):
//   K1  k_init_population   uniform initial controls       (Alg.1 l.3-5)
//   K4a k_qsum              integer resampling weights per column, totals Q_i, ESS sums
//   K4b k_scan / k_scan_cluster  inclusive scan of the integer weights: decoupled
//                           look-back, or one 8-CTA cluster per column (DSMEM); (Q, R)
//                           per column     (R25)
//   K5  k_mp_splits +       merge-path systematic ancestors (large populations)
//       k_ancestors_mp
//   K6  k_gather_propose    per-aircraft recombination + Gaussian proposal
//                           (Alg.1 l.22-23)
//   K7  k_select            argmax of the joint weight (Alg.1 l.27)
//   K8  k_plant             apply the first control, realised wind
// plus the population-density grid, the multi-GPU exchange kernels and the
// MH debug hooks.
#include <cfloat>

#include <cooperative_groups.h>

#include "smc_device.cuh"
#include "smc_kernels.h"

namespace smc {

// ============================================================== K1
__global__ void k_init_population(const DevScen sc, const PopArgs p, float *ctrl) {
    const size_t total = (size_t)p.L * p.n * p.H;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int t = idx % p.H;
        const int i = (idx / p.H) % p.n;
        const uint32_t l = p.l0 + (uint32_t)(idx / ((size_t)p.H * p.n));
        float *c = ctrl + idx * 3;
        const int wi = l < p.Lw ? p.warm_map[i] : -1;
        if (wi >= 0 && *p.warm_ok >= 0) {
            // warm start (R45): previous winner shifted one step, + N(0, sigma^2) for l > 0
            const float *b = p.warm_row + ((size_t)wi * p.H + (t + 1 < p.H ? t + 1 : p.H - 1)) * 3;
            float o0 = b[0], o1 = b[1], o2 = b[2];
            if (l != 0) {
                const uint4 w = draw(TAG_INIT, l, 1u << 16, (uint32_t)t | ((uint32_t)i << 8), *p.mpcp, p.key0, p.key1);
                const float2 z01 = box_muller(w.x, w.y), z23 = box_muller(w.z, w.w);
                o0 = fmaf(p.sig[0], z01.x, o0); o1 = fmaf(p.sig[1], z01.y, o1); o2 = fmaf(p.sig[2], z23.x, o2);
                if (p.clamp) {
                    const float *lo = p.lo3 + 3 * i, *hi = p.hi3 + 3 * i;
                    o0 = fminf(fmaxf(o0, lo[0]), hi[0]);
                    o1 = fminf(fmaxf(o1, lo[1]), hi[1]);
                    o2 = fminf(fmaxf(o2, lo[2]), hi[2]);
                }
            }
            c[0] = o0; c[1] = o1; c[2] = o2;
            continue;
        }
        const uint4 w = draw(TAG_INIT, l, 0u, (uint32_t)t | ((uint32_t)i << 8), *p.mpcp, p.key0, p.key1);
        const DevAircraft &A = sc.ac[i];
        c[0] = A.T_min + (A.T_max - A.T_min) * unif(w.x);
        c[1] = -A.phi_max + 2.0f * A.phi_max * unif(w.y);
        c[2] = -A.gamma_max + 2.0f * A.gamma_max * unif(w.z);
    }
}

cudaError_t launch_init_population(const DevScen &sc, const PopArgs &p, float *ctrl, cudaStream_t st) {
    const size_t total = (size_t)p.L * p.n * p.H;
    if (!total) return cudaSuccess;
    const unsigned grid = (unsigned)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    k_init_population<<<grid, 256, 0, st>>>(sc, p, ctrl);
    return cudaGetLastError();
}

// ============================================================== slot arithmetic (R25)
// t_j = floor((j Q + R) / L) = j floor(Q/L) + floor((j (Q mod L) + R) / L), all in 64 bits.
__host__ __device__ static inline uint64_t slot_t(uint64_t j, uint64_t qd, uint64_t qm, uint64_t R, uint64_t L) {
    return j * qd + (j * qm + R) / L;
}

// #{ j in [0, L) : t_j < C }  (t_j is non-decreasing in j).
__host__ __device__ uint64_t slot_count(uint64_t C, uint64_t Q, uint64_t R, uint32_t L) {
    if (Q == 0 || L == 0) return 0;
    const uint64_t qd = Q / L, qm = Q % L;
    double approx = ((double)C * (double)L - (double)R) / (double)Q;
    int64_t j;
    if (!(approx > 0.0)) j = 0;
    else if (approx >= (double)L) j = L;
    else j = (int64_t)ceil(approx);
    while (j > 0 && slot_t((uint64_t)(j - 1), qd, qm, R, L) >= C) --j;
    while (j < (int64_t)L && slot_t((uint64_t)j, qd, qm, R, L) < C) ++j;
    return (uint64_t)j;
}

// ============================================================== K4a
constexpr int kScanThreads = 256;
// Items per thread of the look-back scan: 2 (512-element tiles, more blocks in
// flight) for small populations, 8 (2048-element tiles) for large ones.
int scan_items(uint32_t L) { return L < (1u << 17) ? 2 : 8; }
int scan_tiles(uint32_t L) {
    const uint32_t tile = (uint32_t)kScanThreads * scan_items(L);
    return (int)((L + tile - 1) / tile);
}
int scan_tiles_max(uint32_t L) { return (int)((L + 511) / 512); }

__device__ __forceinline__ bool column_infeasible(uint32_t cm) {
    return cm == 0u || cm == f2ord(-INFINITY);
}

__device__ __forceinline__ uint64_t qweight(const float *ell, uint32_t l, float m, bool infeasible) {
    if (infeasible) return 1ull;
    return det_quant((double)ell[l] - (double)m);
}

__global__ void __launch_bounds__(kScanThreads) k_qsum(const ResampleArgs r) {
    const int i = blockIdx.y;
    const uint32_t cm = r.colmax[i];
    const bool inf = column_infeasible(cm);
    const float m = ord2f(cm);
    const float *ell = r.ell + (size_t)i * (r.ell_stride ? r.ell_stride : r.L);
    unsigned long long sum = 0;
    double s1 = 0.0, s2 = 0.0;
    for (uint32_t l = blockIdx.x * kScanThreads + threadIdx.x; l < r.L; l += gridDim.x * kScanThreads) {
        const uint64_t q = qweight(ell, l, m, inf);
        sum += q;
        const double w = (double)q * 0x1.0p-32;
        s1 += w;
        s2 += w * w;
    }
    __shared__ unsigned long long s_sum[kScanThreads / 32];
    __shared__ double s_d1[kScanThreads / 32], s_d2[kScanThreads / 32];
    for (int o = 16; o; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    const int wid = threadIdx.x / 32;
    if ((threadIdx.x & 31) == 0) { s_sum[wid] = sum; s_d1[wid] = s1; s_d2[wid] = s2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        double a = 0.0, b = 0.0;
        for (int w = 0; w < kScanThreads / 32; ++w) { t += s_sum[w]; a += s_d1[w]; b += s_d2[w]; }
        atomicAdd(&r.Q[i], t);
        atomicAdd(&r.ess[2 * i], a);
        atomicAdd(&r.ess[2 * i + 1], b);
    }
}

cudaError_t launch_qsum(const ResampleArgs &r, cudaStream_t st) {
    unsigned gx = (r.L + kScanThreads * 16 - 1) / (kScanThreads * 16);
    if (gx < 1) gx = 1;
    if (gx > 1024) gx = 1024;
    k_qsum<<<dim3(gx, r.n), kScanThreads, 0, st>>>(r);
    return cudaGetLastError();
}

// ============================================================== decoupled look-back
// Status word per (column, tile): bits 63..62 = flag (1 aggregate, 2 inclusive
// prefix), bits 61..0 = value.  One 64-bit store publishes flag and value together.
constexpr unsigned long long kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_status(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

struct OpSum {
    __device__ static unsigned long long id() { return 0ull; }
    __device__ static unsigned long long op(unsigned long long a, unsigned long long b) { return a + b; }
};
struct OpMax {  // values are (int32 + 1) >= 0
    __device__ static unsigned long long id() { return 0ull; }
    __device__ static unsigned long long op(unsigned long long a, unsigned long long b) { return a > b ? a : b; }
};

// Exclusive prefix of `tile` within its column: publish the aggregate, walk
// back over predecessors until an inclusive prefix is found.  Thread 0 only.
template <class Op>
__device__ unsigned long long lookback(unsigned long long *status, int tile, unsigned long long agg) {
    if (tile == 0) {
        st_status(&status[0], kFlagP | agg);
        return Op::id();
    }
    st_status(&status[tile], kFlagA | agg);
    unsigned long long pre = Op::id();
    int j = tile - 1;
    while (true) {
        const unsigned long long s = ld_status(&status[j]);
        const unsigned long long f = s & ~kValMask;
        if (f == 0ull) continue;           // predecessor not published yet
        pre = Op::op(pre, s & kValMask);
        if (f == kFlagP) break;
        --j;
    }
    st_status(&status[tile], kFlagP | Op::op(pre, agg));
    return pre;
}

// The same look-back run by one warp: lane k probes predecessor tile - 1 - k, so a
// window of 32 predecessors costs one round of loads (the serial walk above costs
// one load latency per predecessor).  All 32 lanes of warp 0 call it.
template <class Op>
__device__ unsigned long long lookback_warp(unsigned long long *status, int tile, unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_status(&status[0], kFlagP | agg);
        return Op::id();
    }
    if (lane == 0) st_status(&status[tile], kFlagA | agg);
    unsigned long long pre = Op::id();
    int j = tile - 1;
    while (true) {
        const int jj = j - lane;
        unsigned long long s = jj >= 0 ? ld_status(&status[jj]) : kFlagP;   // before tile 0: prefix 0
        while (__any_sync(0xffffffffu, (s & ~kValMask) == 0ull))
            if ((s & ~kValMask) == 0ull) s = ld_status(&status[jj]);        // predecessor not published yet
        const unsigned pm = __ballot_sync(0xffffffffu, (s & ~kValMask) == kFlagP);
        const int stop = pm ? __ffs(pm) - 1 : 31;                           // nearest inclusive prefix
        unsigned long long v = lane <= stop ? (s & kValMask) : Op::id();
        for (int o = 16; o; o >>= 1) v = Op::op(v, __shfl_xor_sync(0xffffffffu, v, o));
        pre = Op::op(pre, v);
        if (pm) break;
        j -= 32;
    }
    if (lane == 0) st_status(&status[tile], kFlagP | Op::op(pre, agg));
    return pre;
}

// Block-wide exclusive scan of per-thread values; returns the thread's
// exclusive prefix, *agg = block total.
template <class Op>
__device__ unsigned long long block_exclusive(unsigned long long v, unsigned long long *agg) {
    __shared__ unsigned long long s_w[kScanThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = Op::op(x, y);
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    unsigned long long wpre = Op::id(), tot = Op::id();
    for (int w = 0; w < kScanThreads / 32; ++w) {
        if (w < wid) wpre = Op::op(wpre, s_w[w]);
        tot = Op::op(tot, s_w[w]);
    }
    const unsigned long long excl_in_warp = __shfl_up_sync(0xffffffffu, x, 1);
    *agg = tot;
    return Op::op(wpre, lane ? excl_in_warp : Op::id());
}

// ============================================================== K4b
// Inclusive scan C_l = sum_{l' <= l} q_l' per column (uint64, exact), single pass
// with decoupled look-back.  The block that owns the last tile of a column also
// publishes (Q, R): Q = C_{L-1}, R = floor(r64 * Q / 2^64) (RESAMPLE stream).
// Grid (n, ntiles): x = column, so the blocks resident at any moment are spread over all
// columns (a few tiles of each) rather than hundreds of tiles of one column, whose look-backs
// would each walk back over many predecessors that only hold aggregates (c5: 170 -> 135 us).
template <int kScanItems>
__global__ void __launch_bounds__(kScanThreads) k_scan(const ResampleArgs r, int ntiles) {
    constexpr int kTile = kScanThreads * kScanItems;
    const int i = blockIdx.x;
    __shared__ int s_tile;
    __shared__ unsigned long long s_pre;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(&r.tile_ctr[i], 1u);
    __syncthreads();
    const int tile = s_tile;
    const uint32_t cm = r.colmax[i];
    const bool inf = column_infeasible(cm);
    const float m = ord2f(cm);
    const float *ell = r.ell + (size_t)i * (r.ell_stride ? r.ell_stride : r.L);
    const uint32_t base = (uint32_t)tile * kTile + threadIdx.x * kScanItems;
    uint64_t inc[kScanItems];
    uint64_t run = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        const uint32_t l = base + it;
        run += l < r.L ? qweight(ell, l, m, inf) : 0ull;
        inc[it] = run;
    }
    unsigned long long agg;
    const unsigned long long texcl = block_exclusive<OpSum>(run, &agg);
    if (threadIdx.x < 32) {
        const unsigned long long pw = lookback_warp<OpSum>(r.status + (size_t)i * ntiles, tile, agg);
        if (threadIdx.x == 0) s_pre = pw;
    }
    __syncthreads();
    const uint64_t pre = s_pre + texcl;
    unsigned long long *C = r.C + (size_t)i * (r.Cstride ? r.Cstride : r.L);
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        const uint32_t l = base + it;
        if (l < r.L) {
            C[l] = pre + inc[it];
            if (r.Cs && ((l % kCdfSample) == kCdfSample - 1 || l == r.L - 1))
                r.Cs[(size_t)i * r.Cs_stride + l / kCdfSample] = pre + inc[it];
        }
    }
    if (inf && tile == 0 && threadIdx.x == 0 && r.inf_round) atomicCAS(&r.inf_round[i], -1, (int)r.k);
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        const uint64_t Q = s_pre + agg;
        const uint64_t rw = r64(TAG_RESAMPLE, (uint32_t)i, r.k, *r.mpcp, r.key0, r.key1);
        r.QR[2 * i] = Q;
        r.QR[2 * i + 1] = __umul64hi(rw, Q);                  // R = floor(r64 Q / 2^64)
        if (r.Q) r.Q[i] = Q;
    }
}

cudaError_t launch_scan(const ResampleArgs &r, cudaStream_t st) {
    const int nt = scan_tiles(r.L);
    if (scan_items(r.L) == 2) k_scan<2><<<dim3(r.n, nt), kScanThreads, 0, st>>>(r, nt);
    else k_scan<8><<<dim3(r.n, nt), kScanThreads, 0, st>>>(r, nt);
    return cudaGetLastError();
}

// ============================================================== K4b' (cluster scan)
// Populations up to kClusterScanMax: one 8-CTA thread-block cluster per column, no global
// atomics and no look-back.  CTA r scans its contiguous eighth of the column into shared
// memory (sub-tiles of 2048 with a running carry), publishes its total, and after a
// cluster barrier reads the totals of CTAs 0..r-1 through distributed shared memory
// (DSMEM) for its exclusive offset; every CTA also forms Q.  One pass over ell, one over C.
constexpr int kClusterCtas = 8, kClusterSeg = 8192;
constexpr uint32_t kClusterScanMax = (uint32_t)kClusterCtas * kClusterSeg;

__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kScanThreads)
k_scan_cluster(const ResampleArgs r) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ unsigned long long s_loc[];                // [seg] local inclusive sums
    __shared__ unsigned long long s_agg;
    const int i = blockIdx.y;
    const int rank = (int)cluster.block_rank();
    const uint32_t L = r.L;
    const uint32_t seg = (((L + kClusterCtas - 1) / kClusterCtas) + 7u) & ~7u;
    const uint32_t b = min(L, (uint32_t)rank * seg), e = min(L, b + seg);
    const uint32_t cm = r.colmax[i];
    const bool inf = column_infeasible(cm);
    const float m = ord2f(cm);
    const float *ell = r.ell + (size_t)i * (r.ell_stride ? r.ell_stride : L);
    constexpr int kIt = 8, kSub = kScanThreads * kIt;
    unsigned long long carry = 0;
    for (uint32_t s0 = b; s0 < e; s0 += kSub) {
        const uint32_t base = s0 + threadIdx.x * kIt;
        uint64_t inc[kIt];
        uint64_t run = 0;
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const uint32_t l = base + it;
            run += l < e ? qweight(ell, l, m, inf) : 0ull;
            inc[it] = run;
        }
        unsigned long long agg;
        const unsigned long long texcl = block_exclusive<OpSum>(run, &agg);
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const uint32_t l = base + it;
            if (l < e) s_loc[l - b] = carry + texcl + inc[it];
        }
        carry += agg;
        __syncthreads();                                         // s_w of block_exclusive reused
    }
    if (threadIdx.x == 0) s_agg = carry;
    cluster.sync();
    unsigned long long pre = 0, Q = 0;
    for (int q = 0; q < kClusterCtas; ++q) {
        const unsigned long long aq = *cluster.map_shared_rank(&s_agg, q);
        if (q < rank) pre += aq;
        Q += aq;
    }
    cluster.sync();                                              // no CTA leaves while its s_agg is read
    unsigned long long *C = r.C + (size_t)i * (r.Cstride ? r.Cstride : L);
    for (uint32_t l = b + threadIdx.x; l < e; l += kScanThreads) {
        const unsigned long long v = pre + s_loc[l - b];
        C[l] = v;
        if (r.Cs && ((l % kCdfSample) == kCdfSample - 1 || l == L - 1))
            r.Cs[(size_t)i * r.Cs_stride + l / kCdfSample] = v;
    }
    if (rank == 0 && threadIdx.x == 0) {
        if (inf && r.inf_round) atomicCAS(&r.inf_round[i], -1, (int)r.k);
        const uint64_t rw = r64(TAG_RESAMPLE, (uint32_t)i, r.k, *r.mpcp, r.key0, r.key1);
        r.QR[2 * i] = Q;
        r.QR[2 * i + 1] = __umul64hi(rw, Q);                  // R = floor(r64 Q / 2^64)
        if (r.Q) r.Q[i] = Q;
    }
}

bool cluster_scan_fits(uint32_t L) { return L >= 1 && L <= kClusterScanMax; }

cudaError_t launch_scan_cluster(const ResampleArgs &r, cudaStream_t st) {
    const uint32_t seg = (((r.L + kClusterCtas - 1) / kClusterCtas) + 7u) & ~7u;
    const size_t smem = (size_t)seg * sizeof(unsigned long long);
    if (smem > 48 * 1024) {   // per device and cheap: set on every launch that needs it, checked
        const cudaError_t e = cudaFuncSetAttribute(k_scan_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)(kClusterSeg * sizeof(unsigned long long)));
        if (e != cudaSuccess) return e;
    }
    k_scan_cluster<<<dim3(kClusterCtas, r.n), kScanThreads, smem, st>>>(r);
    return cudaGetLastError();
}

// Systematic slot j takes min{ l : C_l > t_j }, t_j = floor((j Q + R) / L) (R25).
// M new particles drawn from L (M = L unless the population shrinks).
__device__ __forceinline__ int32_t find_ancestor(const unsigned long long *C, uint32_t L, uint32_t M, uint64_t Q,
                                                 uint64_t R, uint32_t j) {
    const uint64_t tj = slot_t(j, Q / M, Q % M, R, M);
    uint32_t lo = 0, hi = L - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(&C[mid]) > tj) hi = mid; else lo = mid + 1;
    }
    return (int32_t)lo;
}

// Two-level search: the group g of kCdfSample entries whose sample Cs[g] first exceeds t_j
// (bisection over L / 16 samples: a small, cache-resident array), then the slot's ancestor
// inside that group (four steps within one 128-byte line).  Same result as find_ancestor.
#ifndef SMC_K6_ARY
#define SMC_K6_ARY 3   // c2 A/B (MPC step, 3 repeats): 2 -> 29.233 ms, 3 -> 29.209, 4 -> 29.257, 8 -> 29.527
#endif
// First index in [lo, hi] whose entry exceeds tj (hi if none), for a non-decreasing array.
// K-ary rounds: the K - 1 probes of a round are independent loads, so a search over n
// entries waits on ~log_K(n) load latencies instead of log_2(n); same result as bisection.
template <int K>
__device__ __forceinline__ uint32_t first_above(const unsigned long long *A, uint32_t lo, uint32_t hi, uint64_t tj) {
    if constexpr (K > 2) {
        while (hi - lo >= (uint32_t)K) {
            const uint32_t span = hi - lo;
            uint32_t p[K - 1];
            unsigned long long c[K - 1];
#pragma unroll
            for (int q = 0; q < K - 1; ++q) {
                p[q] = lo + (uint32_t)(((uint64_t)span * (uint32_t)(q + 1)) / (uint32_t)K);
                c[q] = __ldg(&A[p[q]]);
            }
            uint32_t nlo = p[K - 2] + 1, nhi = hi;
#pragma unroll
            for (int q = K - 2; q >= 0; --q) {
                if (c[q] > tj) { nhi = p[q]; nlo = q ? p[q - 1] + 1 : lo; }
            }
            lo = nlo; hi = nhi;
        }
    }
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(&A[mid]) > tj) hi = mid; else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ int32_t find_ancestor2(const unsigned long long *C, const unsigned long long *Cs,
                                                  uint32_t L, uint32_t M, uint64_t Q, uint64_t R, uint32_t j) {
    const uint64_t tj = slot_t(j, Q / M, Q % M, R, M);
    const uint32_t g = first_above<SMC_K6_ARY>(Cs, 0, cdf_samples(L) - 1, tj);
    const uint32_t a = g * kCdfSample, b = min(a + kCdfSample, L) - 1;
    return (int32_t)first_above<SMC_K6_ARY>(C, a, b, tj);
}

__global__ void k_ancestors(const ResampleArgs r) {
    const int i = blockIdx.y;
    const uint64_t Q = r.QR[2 * i], R = r.QR[2 * i + 1];
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < r.M; j += gridDim.x * blockDim.x)
        r.anc[(size_t)i * r.M + j] = find_ancestor(r.C + (size_t)i * r.L, r.L, r.M, Q, R, j);
}

// The production K6 search (find_ancestor2: K-ary rounds over the every-16th samples Cs, then
// inside one 128-byte line of C) as a stand-alone pass, for the bit-exact debug sweep.
__global__ void k_ancestors2(const ResampleArgs r) {
    const int i = blockIdx.y;
    const uint64_t Q = r.QR[2 * i], R = r.QR[2 * i + 1];
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < r.M; j += gridDim.x * blockDim.x)
        r.anc[(size_t)i * r.M + j] = find_ancestor2(r.C + (size_t)i * r.L, r.Cs + (size_t)i * r.Cs_stride, r.L, r.M,
                                                    Q, R, j);
}

cudaError_t launch_ancestors_two_level(const ResampleArgs &r, cudaStream_t st) {
    unsigned gx = (r.M + 255) / 256;
    if (gx > 1024) gx = 1024;
    k_ancestors2<<<dim3(gx, r.n), 256, 0, st>>>(r);
    return cudaGetLastError();
}

cudaError_t launch_ancestors_bisect(const ResampleArgs &r, cudaStream_t st) {
    unsigned gx = (r.M + 255) / 256;
    if (gx > 1024) gx = 1024;
    k_ancestors<<<dim3(gx, r.n), 256, 0, st>>>(r);
    return cudaGetLastError();
}

// ============================================================== K5 (merge path)
// The same ancestors as find_ancestor, without a bisection over the whole CDF per
// slot.  Both C (sources) and t_j (slots) are non-decreasing, so a(j) =
// #{l : C_l <= t_j} is the position of slot j in the merge of the two sequences
// (a source goes first on ties).  Block b owns diagonals [bT, (b+1)T) of that
// merge: it finds its two split points (a0, j0), (a1, j1) by a 32-ary warp search,
// loads the window C[a0, a1) (<= T entries, coalesced) into shared memory and
// gives every slot j in [j0, j1) the ancestor a0 + #{a in window : C_a <= t_j}
// (bisection in shared memory).  Traffic: C read once, anc written once.
constexpr int kMpThreads = 256, kMpTile = 2048;

struct SlotGen {
    uint64_t qd, qm, R, M;
    __device__ uint64_t t(uint64_t j) const { return slot_t(j, qd, qm, R, M); }
};

// First a in [lo, hi) with C[a] > t(d - 1 - a) (hi if none): the merge-path split
// at diagonal d.  All 32 lanes of a warp call it; each round probes 32 points.
__device__ uint32_t mp_split(const unsigned long long *C, const SlotGen &g, uint64_t d, uint32_t lo, uint32_t hi) {
    const int lane = threadIdx.x & 31;
    while (lo < hi) {
        const uint32_t span = hi - lo, step = (span + 31) / 32;
        const uint32_t a = lo + (uint32_t)lane * step;
        const bool ok = a < hi && __ldg(&C[a]) <= g.t(d - 1 - a);      // source a precedes slot d-1-a
        const unsigned b = __ballot_sync(0xffffffffu, ok);
        const int c = __popc(b);                                         // predicate true on a lane prefix
        if (c == 0) break;                                               // answer = lo
        const uint32_t last = lo + (uint32_t)(c - 1) * step;
        lo = last + 1;
        if (c < 32) hi = min(hi, lo - 1 + step);
    }
    return lo;
}

// One warp per split point: splits[i][b] = a(b T) for b = 0..nblocks (all in parallel, so the
// 32-ary searches of all blocks overlap instead of heading every block's critical path).
__global__ void k_mp_splits(const ResampleArgs r, uint32_t *splits, uint32_t nsplit) {
    const int i = blockIdx.y;
    const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= nsplit) return;
    const uint32_t L = r.L, M = r.M;
    const unsigned long long *C = r.C + (size_t)i * (r.Cstride ? r.Cstride : L);
    const uint64_t Q = r.QR[2 * i];
    const SlotGen g{Q / M, Q % M, r.QR[2 * i + 1], M};
    const uint64_t d = min((uint64_t)L + M, (uint64_t)b * kMpTile);
    const uint32_t lo = d > M ? (uint32_t)(d - M) : 0u, hi = (uint32_t)min(d, (uint64_t)L);
    const uint32_t a = mp_split(C, g, d, lo, hi);
    if ((threadIdx.x & 31) == 0) splits[(size_t)i * nsplit + b] = a;
}

__global__ void __launch_bounds__(kMpThreads) k_ancestors_mp(const ResampleArgs r, const uint32_t *splits,
                                                              uint32_t nsplit) {
    __shared__ unsigned long long s_c[kMpTile];
    const int i = blockIdx.y;
    const uint32_t L = r.L, M = r.M;
    const unsigned long long *C = r.C + (size_t)i * (r.Cstride ? r.Cstride : L);
    const uint64_t Q = r.QR[2 * i];
    const SlotGen g{Q / M, Q % M, r.QR[2 * i + 1], M};
    const uint64_t total = (uint64_t)L + M;
    const uint32_t a0 = splits[(size_t)i * nsplit + blockIdx.x], a1 = splits[(size_t)i * nsplit + blockIdx.x + 1];
    const uint64_t d0 = (uint64_t)blockIdx.x * kMpTile, d1 = min(total, d0 + kMpTile);
    const uint32_t j0 = (uint32_t)(d0 - a0), j1 = (uint32_t)(d1 - a1);
    const int nw = (int)(a1 - a0);
    for (int e = threadIdx.x; e < nw; e += kMpThreads) s_c[e] = __ldg(&C[a0 + e]);
    // t_j = j qd + floor((j qm + R) / M) without a 64-bit division per slot: with
    // j0 qm + R = u0 M + v0 (one division per block), slot j0 + dj has
    // floor(...) = u0 + floor(x / M), x = v0 + dj qm < 2^44 -- a double-precision
    // quotient (error < 1 / M) and an integer fix-up
    __shared__ uint64_t s_u0, s_v0;
    if (threadIdx.x == 0) {
        const uint64_t num = (uint64_t)j0 * g.qm + g.R;
        s_u0 = num / M;
        s_v0 = num - s_u0 * M;
    }
    __syncthreads();
    const uint64_t u0 = s_u0, v0 = s_v0;
    const double invM = 1.0 / (double)M;
    int32_t *anc = r.anc + (size_t)i * M;
    for (uint32_t j = j0 + threadIdx.x; j < j1; j += kMpThreads) {
        const uint64_t x = v0 + (uint64_t)(j - j0) * g.qm;
        uint64_t u = (uint64_t)((double)x * invM);
        const int64_t rem = (int64_t)(x - u * M);
        if (rem < 0) --u;
        else if (rem >= (int64_t)M) ++u;
        const uint64_t tj = (uint64_t)j * g.qd + u0 + u;
        int lo = 0, hi = nw;                                             // first window entry with C > t_j
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_c[mid] > tj) hi = mid; else lo = mid + 1;
        }
        anc[j] = (int32_t)(a0 + (uint32_t)lo);
    }
}

size_t mp_split_words(uint32_t L, uint32_t M) { return ((uint64_t)L + M + kMpTile - 1) / kMpTile + 1; }

cudaError_t launch_ancestors(const ResampleArgs &r, cudaStream_t st) {
    if (!r.M || !r.L) return cudaSuccess;
    const uint32_t blocks = (uint32_t)(((uint64_t)r.L + r.M + kMpTile - 1) / kMpTile), nsplit = blocks + 1;
    k_mp_splits<<<dim3((nsplit + 3) / 4, r.n), 128, 0, st>>>(r, r.splits, nsplit);
    k_ancestors_mp<<<dim3(blocks, r.n), kMpThreads, 0, st>>>(r, r.splits, nsplit);
    return cudaGetLastError();
}

// Zero the next round's accumulators (column maxima, accept count, look-back
// status words and tile counters): saves four memset nodes per round.
__device__ __forceinline__ void reset_round_state(const ProposeArgs &p) {
    if (!p.reset_n) return;
    const size_t gtid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    for (size_t e = gtid; e < p.reset_status_n; e += stride) p.reset_status[e] = 0ull;
    if (gtid < (size_t)p.reset_n) { p.reset_colmax[gtid] = 0u; p.reset_tiles[gtid] = 0u; }
    if (gtid == 0) *p.reset_accept = 0ull;
}

// ============================================================== K6
// A block owns kRowsPerBlock rows (new particle j, aircraft i).  Phase 1: one
// thread per row finds the ancestor by bisection of the integer CDF and the
// buffer (x' or x*) that holds the ancestor's survivor row (no survivor copy
// is made).  Phase 2: one thread per (row, step) copies the parent's control
// triple and writes the Gaussian proposal -- consecutive threads write
// consecutive 12-byte triples, so both output streams are coalesced.
#ifndef SMC_K6_ROWS
#define SMC_K6_ROWS 128   // c2 A/B (MPC step, 3 repeats): 256 rows 29.24 ms, 128 rows 29.17, 128 rows + batch 6 29.15
#endif
#ifndef SMC_K6_BATCH
#define SMC_K6_BATCH 6    // 256 rows + batch 6: 29.72 ms; 512 rows + batch 6: 29.83 ms
#endif
constexpr int kRowsPerBlock = SMC_K6_ROWS;   // = blockDim: every thread runs one bisection in phase 1

// Phase 2 of K6 for the block's rows q0 .. q0 + kRowsPerBlock - 1: copy each parent's control
// triples (s_src[r] + 3 t) to x' and write the Gaussian proposal x* (P:221).  Batches of
// kBatch elements per thread: all parent loads (read-only path) are issued before any store, so
// their latencies overlap.
__device__ __forceinline__ void propose_rows(const ProposeArgs &p, const float *const *s_src, const uint32_t *s_j,
                                             const uint32_t *s_perturb_x2, uint32_t q0, uint32_t rows, uint32_t mpc,
                                             uint32_t invH) {
    const int H = p.H;
    const int tot = (int)(min((uint32_t)kRowsPerBlock, rows - q0) * (uint32_t)H);
    float *const xp = p.xp + (size_t)q0 * H * 3, *const xs = p.xs + (size_t)q0 * H * 3;
    constexpr int kBatch = SMC_K6_BATCH;
    for (int e0 = 0; e0 < tot; e0 += kBatch * (int)blockDim.x) {
        float cv[kBatch][3];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int e = e0 + u * (int)blockDim.x + (int)threadIdx.x;
            if (e < tot) {
                const int r = (int)__umulhi((uint32_t)e, invH), t = e - r * H;
                const float *src = s_src[r] + 3 * t;
                cv[u][0] = __ldg(src); cv[u][1] = __ldg(src + 1); cv[u][2] = __ldg(src + 2);
            }
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int e = e0 + u * (int)blockDim.x + (int)threadIdx.x;
            if (e >= tot) break;
            const int r = (int)__umulhi((uint32_t)e, invH), t = e - r * H;
            const uint32_t x2 = s_perturb_x2[r];
            const float c0 = cv[u][0], c1 = cv[u][1], c2 = cv[u][2];
            xp[3 * e] = c0; xp[3 * e + 1] = c1; xp[3 * e + 2] = c2;
            const uint4 w = draw_ks(TAG_PERTURB, p.l0 + s_j[r], p.k << 16, (uint32_t)t | x2, mpc, p.ks);
            const float4 z = box_muller4(w);
            float o0 = fmaf(p.sig[0], z.x, c0), o1 = fmaf(p.sig[1], z.y, c1), o2 = fmaf(p.sig[2], z.z, c2);
            if (p.clamp) {
                const int i = (int)(x2 >> 8);
                const float *lo = p.lo3 + 3 * i, *hi = p.hi3 + 3 * i;
                o0 = fminf(fmaxf(o0, lo[0]), hi[0]);
                o1 = fminf(fmaxf(o1, lo[1]), hi[1]);
                o2 = fminf(fmaxf(o2, lo[2]), hi[2]);
            }
            xs[3 * e] = o0; xs[3 * e + 1] = o1; xs[3 * e + 2] = o2;
        }
    }
}

__global__ void __launch_bounds__(kRowsPerBlock) k_gather_propose(const ProposeArgs p) {
    __shared__ const float *s_src[kRowsPerBlock];
    __shared__ uint32_t s_j[kRowsPerBlock];
    __shared__ uint32_t s_perturb_x2[kRowsPerBlock];     // (i << 8): the aircraft part of the PERTURB counter
    const uint32_t rows = p.L * (uint32_t)p.n;            // < 2^31 (smc_init bounds L n)
    const uint32_t mpc = *p.mpcp;
    const uint32_t invH = 0xFFFFFFFFu / (uint32_t)p.H + 1u;  // e / H = umulhi(e, invH) for e < 2^32 / H^2
    for (uint32_t q0 = blockIdx.x * kRowsPerBlock; q0 < rows; q0 += gridDim.x * kRowsPerBlock) {
        {
            const uint32_t q = q0 + threadIdx.x;
            const float *src = nullptr;
            if (q < rows) {
                const uint32_t j = q / (uint32_t)p.n;
                const int i = (int)(q - j * (uint32_t)p.n);
                int32_t a;
                if (p.anc) {
                    a = __ldg(&p.anc[(size_t)i * p.L + j]);
                } else {
                    const uint64_t Q = p.QR[2 * i], R = p.QR[2 * i + 1];
                    a = p.Cs ? find_ancestor2(p.C + (size_t)i * p.Lsrc, p.Cs + (size_t)i * p.Cs_stride, p.Lsrc, p.L,
                                              Q, R, j)
                             : find_ancestor(p.C + (size_t)i * p.Lsrc, p.Lsrc, p.L, Q, R, j);
                }
                src = p.src[(__ldg(&p.surv[a]) >> i) & 1u] + ((size_t)a * p.n + i) * p.H * 3;
                s_j[threadIdx.x] = j;
                s_perturb_x2[threadIdx.x] = (uint32_t)i << 8;
            }
            s_src[threadIdx.x] = src;
        }
        __syncthreads();
        propose_rows(p, s_src, s_j, s_perturb_x2, q0, rows, mpc, invH);
        __syncthreads();
    }
    reset_round_state(p);
}

cudaError_t launch_gather_propose(const ProposeArgs &p0, cudaStream_t st) {
    const size_t rows = (size_t)p0.L * p0.n;
    if (!rows) return cudaSuccess;
    ProposeArgs p = p0;                     // Philox round keys as kernel parameters (as in K2)
    for (int r = 0; r < 10; ++r) {
        p.ks[2 * r] = p.key0 + (uint32_t)r * 0x9E3779B9u;
        p.ks[2 * r + 1] = p.key1 + (uint32_t)r * 0xBB67AE85u;
    }
    size_t g = (rows + kRowsPerBlock - 1) / kRowsPerBlock;
    if (g > 148 * 16 * 256 / kRowsPerBlock) g = 148 * 16 * 256 / kRowsPerBlock;   // same thread count for any block size
    k_gather_propose<<<(unsigned)g, kRowsPerBlock, 0, st>>>(p);
    return cudaGetLastError();
}

// ============================================================== K7
__device__ __forceinline__ bool better(double la, long long ia, double lb, long long ib) {
    if (ia < 0) return false;
    if (ib < 0) return true;
    return la > lb || (la == lb && ia < ib);
}

int select_blocks(uint32_t L) {
    int b = (int)((L + 255) / 256);
    return b < 1 ? 1 : (b > 512 ? 512 : b);
}

// Keys: survivors l -> l0 + l; per-aircraft MH (lam2 != NULL) candidates (l, c) -> 2 (l0 + l) + c,
// so ties go to the lowest particle, then x' before x* (R27, R46).
__global__ void k_select(const SelectArgs s) {
    double bl = -INFINITY;
    long long bi = -1;
    const uint32_t ne = s.lam2 ? 2 * s.L : s.L;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
        const double v = s.lam2 ? s.lam2[(e & 1u) * s.lam2_stride + (e >> 1)] : s.lam[e];
        const long long key = s.lam2 ? 2 * (long long)(s.l0 + (e >> 1)) + (e & 1u) : (long long)(s.l0 + e);
        if (v != -INFINITY && better(v, key, bl, bi)) { bl = v; bi = key; }
    }
    for (int o = 16; o; o >>= 1) {
        const double ol = __shfl_xor_sync(0xffffffffu, bl, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (better(ol, oi, bl, bi)) { bl = ol; bi = oi; }
    }
    __shared__ double s_l[8];
    __shared__ long long s_i[8];
    __shared__ bool s_last;
    if ((threadIdx.x & 31) == 0) { s_l[threadIdx.x / 32] = bl; s_i[threadIdx.x / 32] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x / 32); ++w)
            if (better(s_l[w], s_i[w], bl, bi)) { bl = s_l[w]; bi = s_i[w]; }
        s.part_lam[blockIdx.x] = bl;
        s.part_idx[blockIdx.x] = bi;
        __threadfence();
        const unsigned done = atomicAdd(s.done_ctr, 1u);
        s_last = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __shared__ long long s_win;
    if (threadIdx.x == 0) {
        __threadfence();
        double gl = -INFINITY;
        long long gi = -1;
        for (unsigned b = 0; b < gridDim.x; ++b) {
            const double pl = ((volatile double *)s.part_lam)[b];
            const long long pi = ((volatile long long *)s.part_idx)[b];
            if (better(pl, pi, gl, gi)) { gl = pl; gi = pi; }
        }
        s.best_lam[0] = gl;
        s.best_idx[0] = (s.lam2 && gi >= 0) ? gi >> 1 : gi;   // reported: particle index
        s_win = gi;
        *s.done_ctr = 0u;
    }
    __syncthreads();
    const long long gi = s_win;
    if (gi < 0) return;
    const uint32_t ll = (uint32_t)((s.lam2 ? gi >> 1 : gi) - s.l0);
    const int cbuf = s.lam2 ? (int)(gi & 1) : (int)(s.surv[ll] & 1u);
    const float *src = s.src[cbuf] + (size_t)ll * s.n * s.H * 3;
    for (int e = threadIdx.x; e < s.n * s.H * 3; e += blockDim.x) s.best_row[e] = src[e];
}

cudaError_t launch_select(const SelectArgs &s, cudaStream_t st) {
    k_select<<<select_blocks(s.L), 256, 0, st>>>(s);
    return cudaGetLastError();
}

// ============================================================== K8 (FP64)
__device__ double d_angdist(double d) {
    double r = fmod(fabs(d), 2.0 * 3.141592653589793);
    return r > 3.141592653589793 ? 2.0 * 3.141592653589793 - r : r;
}

__global__ void k_plant(const PlantScen ps, const PlantArgs p) {
    constexpr int G2M = 2 * kMaxWindNodes;
    __shared__ double sV[G2M + 4], sZ[G2M], sW[G2M];
    const int tid = threadIdx.x;
    const int G = ps.ng, G2 = 2 * ps.ng, nblk = (G2 + 3) / 4;
    if (*p.best_idx < 0) {                       // infeasible solve: nothing is applied
        if (tid < p.n) {
            for (int a = 0; a < 6; ++a) p.next[6 * tid + a] = p.states[6 * tid + a];
            p.flags[tid] = 4;
            p.applied[3 * tid] = p.applied[3 * tid + 1] = p.applied[3 * tid + 2] = 0.0f;
        }
        return;
    }
    // realised field: normal e = 4 blk + j -> component e / G, grid point e % G
    for (int blk = tid; blk < nblk; blk += blockDim.x) {
        const uint4 w = draw(TAG_PLANT_WIND, 0u, 0u, (uint32_t)blk << 16, *p.mpcp, p.key0, p.key1);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        for (int pr = 0; pr < 2; ++pr) {
            const double u1 = ((double)(ws[2 * pr] >> 9) + 0.5) * 0x1.0p-23;
            const double u2 = ((double)(ws[2 * pr + 1] >> 9) + 0.5) * 0x1.0p-23;
            const double r = sqrt(-2.0 * log(u1));
            sV[4 * blk + 2 * pr] = r * cos(2.0 * 3.141592653589793 * u2);
            sV[4 * blk + 2 * pr + 1] = r * sin(2.0 * 3.141592653589793 * u2);
        }
    }
    __syncthreads();
    const int zi = *p.zinit;
    for (int e = tid; e < G2; e += blockDim.x) {
        const double z = zi ? ps.a * p.Z[e] + ps.b * sV[e] : sV[e];
        sZ[e] = z;
        p.Z[e] = z;
    }
    __syncthreads();
    for (int e = tid; e < G2; e += blockDim.x) {
        const int comp = e / G, node = e % G;
        double acc = 0.0;
        for (int m = 0; m < G; ++m) acc += ps.Qd[node * G + m] * sZ[comp * G + m];
        sW[e] = acc;
    }
    __syncthreads();
    if (tid == 0) *p.zinit = 1;
    if (tid >= p.n) return;
    const int i = tid;
    const double *st = p.states + 6 * i;
    double *nx = p.next + 6 * i;
    const float *u0 = p.best_row + (size_t)i * p.H * 3;
    p.applied[3 * i] = u0[0]; p.applied[3 * i + 1] = u0[1]; p.applied[3 * i + 2] = u0[2];
    p.flags[i] = 0;
    if (ps.first_step[i] != 0) {
        for (int a = 0; a < 6; ++a) nx[a] = st[a];
        return;
    }
    // trilinear interpolation in the grid cell holding the aircraft, clamped
    double f[3];
    int c0[3];
    for (int a = 0; a < 3; ++a) {
        double t = (st[a] - ps.wind_lo[a]) / (ps.wind_hi[a] - ps.wind_lo[a]);
        t = t > 0.0 ? (t < 1.0 ? t : 1.0) : 0.0;
        const double gcoord = t * (double)(ps.wn[a] - 1);
        int i0 = (int)floor(gcoord);
        if (i0 > ps.wn[a] - 2) i0 = ps.wn[a] - 2;
        c0[a] = i0;
        f[a] = gcoord - (double)i0;
    }
    double wxy[2];
    for (int c = 0; c < 2; ++c) {
        double acc = 0.0;
        for (int nd = 0; nd < 8; ++nd) {
            const int node = (c0[0] + (nd & 1)) + ps.wn[0] * ((c0[1] + ((nd >> 1) & 1)) + ps.wn[1] * (c0[2] + (nd >> 2)));
            acc += ((nd & 1) ? f[0] : 1 - f[0]) * ((nd & 2) ? f[1] : 1 - f[1]) * ((nd & 4) ? f[2] : 1 - f[2]) * sW[c * G + node];
        }
        wxy[c] = acc + ps.nominal[c];
    }
    if (ps.turb_sigma > 0.0) {
        const uint4 w = draw(TAG_PLANT_TURB, 0u, 0u, (uint32_t)i << 8, *p.mpcp, p.key0, p.key1);
        const double u1 = ((double)(w.x >> 9) + 0.5) * 0x1.0p-23, u2 = ((double)(w.y >> 9) + 0.5) * 0x1.0p-23;
        const double r = sqrt(-2.0 * log(u1));
        wxy[0] += ps.turb_sigma * r * cos(2.0 * 3.141592653589793 * u2);
        wxy[1] += ps.turb_sigma * r * sin(2.0 * 3.141592653589793 * u2);
    }
    const double T = u0[0], ph = u0[1], ga = u0[2];
    const double x = st[0], y = st[1], z = st[2], v = st[3], chi = st[4], m = st[5];
    double rho = ps.rho_const;
    if (ps.density_mode == 0) {
        double base = 1.0 - 2.2558e-5 * z;
        rho = 1.225 * pow(base > 0.0 ? base : 0.0, 4.2559);
    }
    const double qd = rho * v * v * ps.halfS[i];
    const double Lf = m * ps.g / cos(ph);
    const double CL = Lf / qd;
    const double D = qd * (ps.cd0[i] + ps.cd2[i] * CL * CL);
    nx[0] = x + ps.dt * (v * cos(chi) * cos(ga)) + wxy[0] * ps.dt;
    nx[1] = y + ps.dt * (v * sin(chi) * cos(ga)) + wxy[1] * ps.dt;
    nx[2] = z + ps.dt * (v * sin(ga));
    nx[3] = v + ps.dt * ((T - D) / m - ps.g * sin(ga));
    nx[4] = chi + ps.dt * (Lf * sin(ph) / (m * v));
    nx[5] = m - ps.dt * (ps.eta[i] * T);
    int fl = 0;
    const double rh = sqrt(nx[0] * nx[0] + nx[1] * nx[1]);
    const double th = atan2(nx[1], nx[0]);
    if (ps.kind[i] == 0) {
        const double at = fabs(th);
        const double s = at == 0.0 ? rh : rh * at / sin(at);
        const double beta = atan2(nx[2], s);
        if (rh <= ps.P_runway && beta <= ps.P_beta && at <= ps.P_chi && d_angdist(nx[4] - 3.141592653589793) <= ps.P_chi &&
            nx[3] <= ps.P_vs)
            fl |= 1;
    } else if (rh >= ps.tma_radius) {
        fl |= 2;
    }
    bool bad = fabs(ga) > ps.gamma_max[i] || !(fabs(ph) < ps.phi_max[i]) || T < ps.T_min[i] || T > ps.T_max[i];
    bad = bad || nx[2] < ps.z_min[i] || nx[2] > ps.z_max[i] || nx[3] < ps.v_min[i] || nx[3] > ps.v_max[i] ||
          nx[5] < ps.m_empty[i];
    for (int a = 0; a < 6; ++a) bad = bad || !isfinite(nx[a]);
    if (bad) fl |= 4;
    p.flags[i] = fl;
}

cudaError_t launch_plant(const PlantScen &ps, const PlantArgs &p, cudaStream_t st) {
    k_plant<<<1, 128, 0, st>>>(ps, p);
    return cudaGetLastError();
}

// ============================================================== popdense grid
__global__ void k_popgrid(const double *centres, int nc, int nx, int ny, double x0, double y0, double dx, float *out,
                          int pad) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int sx = nx + pad;                                  // row stride
    if (idx >= sx * (ny + pad)) return;
    const int ix = min(idx % sx, nx - 1), iy = min(idx / sx, ny - 1);   // padding repeats the edge
    const double x = x0 + ix * dx, y = y0 + iy * dx;
    double sum = 0.0;
    for (int c = 0; c < nc; ++c) {
        const double bx = (x - centres[3 * c]) * 1e-3, by = (y - centres[3 * c + 1]) * 1e-3;
        const double ci = centres[3 * c + 2] * 1e-3;
        sum += exp(-(bx * bx + by * by) / (2.0 * ci * ci)) / (ci * 2.5066282746310002);
    }
    out[idx] = (float)(sum < 1.0 ? sum : 1.0);
}

cudaError_t launch_popgrid(const double *centres, int n_centres, int nx, int ny, double x0, double y0,
                           double dx, float *out, float *outp, cudaStream_t st) {
    if (nx * ny == 0) return cudaSuccess;
    k_popgrid<<<(nx * ny + 255) / 256, 256, 0, st>>>(centres, n_centres, nx, ny, x0, y0, dx, out, 0);
    const int np = (nx + 1) * (ny + 1);
    k_popgrid<<<(np + 255) / 256, 256, 0, st>>>(centres, n_centres, nx, ny, x0, y0, dx, outp, 1);
    return cudaGetLastError();
}

// ============================================================== MH debug hook
__global__ void k_mh_debug(const double *lc, const double *lp, uint32_t L, uint32_t k, const uint32_t *mpcp,
                           uint32_t key0, uint32_t key1, uint8_t *acc) {
    const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < L) acc[l] = mh_decide(lc[l], lp[l], l, k, *mpcp, key0, key1) ? 1 : 0;
}

__global__ void k_mh_aircraft_debug(const float *ec, const float *ep, uint32_t L, int n, uint32_t k,
                                    const uint32_t *mpcp, uint32_t key0, uint32_t key1, uint32_t *mask) {
    const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    uint32_t m = 0u;
    for (int i = 0; i < n; ++i)
        if (mh_decide_aircraft((double)ec[(size_t)l * n + i], (double)ep[(size_t)l * n + i], l, (uint32_t)i, k, *mpcp,
                               key0, key1))
            m |= 1u << i;
    mask[l] = m;
}

cudaError_t launch_mh_aircraft_debug(const float *ec, const float *ep, uint32_t L, int n, uint32_t k,
                                     const uint32_t *mpcp, uint32_t key0, uint32_t key1, uint32_t *mask,
                                     cudaStream_t st) {
    if (!L) return cudaSuccess;
    k_mh_aircraft_debug<<<(L + 255) / 256, 256, 0, st>>>(ec, ep, L, n, k, mpcp, key0, key1, mask);
    return cudaGetLastError();
}

cudaError_t launch_mh_debug(const double *lc, const double *lp, uint32_t L, uint32_t k, const uint32_t *mpcp,
                            uint32_t key0, uint32_t key1, uint8_t *acc, cudaStream_t st) {
    if (!L) return cudaSuccess;
    k_mh_debug<<<(L + 255) / 256, 256, 0, st>>>(lc, lp, L, k, mpcp, key0, key1, acc);
    return cudaGetLastError();
}

}  // namespace smc

namespace smc {
// ============================================================== column max (debug path; K2 fuses it)
__global__ void k_colmax(const float *ell, int n, uint32_t L, uint32_t *colmax) {
    const int i = blockIdx.y;
    uint32_t mx = 0u;
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < L; l += gridDim.x * blockDim.x)
        mx = max(mx, f2ord(ell[(size_t)i * L + l]));
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(&colmax[i], mx);
}

cudaError_t launch_colmax(const float *ell, int n, uint32_t L, uint32_t *colmax, cudaStream_t st) {
    unsigned gx = (L + 255) / 256;
    if (gx < 1) gx = 1;
    if (gx > 256) gx = 256;
    k_colmax<<<dim3(gx, n), 256, 0, st>>>(ell, n, L, colmax);
    return cudaGetLastError();
}
}  // namespace smc

namespace smc {
// ============================================================== multi-GPU (R43)
// Particle sharding: rank r owns global particles [L r / G, L (r+1) / G) (smc_shard_range).

// Compact this rank's survivor rows (x' or x* per survivor flag) for the all-gather.
__global__ void k_compact_survivors(const float *xp, const float *xs, const uint32_t *surv, uint32_t Lloc, int n,
                                    int rowlen, float *out) {
    const size_t total = (size_t)Lloc * rowlen;
    const int arow = rowlen / n;                         // H * 3 floats per aircraft
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const uint32_t l = (uint32_t)(e / rowlen);
        const int i = (int)((e % rowlen) / arow);
        out[e] = (((surv[l] >> i) & 1u) ? xs : xp)[e];
    }
}

cudaError_t launch_compact_survivors(const float *xp, const float *xs, const uint32_t *surv, uint32_t Lloc, int n,
                                     int rowlen, float *out, cudaStream_t st) {
    const size_t total = (size_t)Lloc * rowlen;
    if (!total) return cudaSuccess;
    size_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_compact_survivors<<<(unsigned)g, 256, 0, st>>>(xp, xs, surv, Lloc, n, rowlen, out);
    return cudaGetLastError();
}

// Gather + propose for this rank's new particles, on K6's two-phase
// structure.  Every rank holds only its own inclusive CDF; the ranks' column totals Q_r were
// all-gathered (Qall), so slot j's target t_j = floor((j Q + R) / L) on the global total
// Q = sum_r Q_r names its owner rho (the rank whose cumulative offset range holds t_j) and
// the owner-local target t_j - off_rho.  Phase 1 searches the owner's CDF in place -- two-
// level through its every-16th samples, over NVLink through CUDA IPC mappings (peer mode), in
// the all-gathered CDFs (all-gather mode) or in slices of one buffer (virtual ranks) -- and
// points at the parent's survivor row where its owner keeps it (x' or x* by the published
// mask bit) or in the all-gathered compacted rows.  Phase 2 is K6's (copy + proposal).  The
// ancestors equal the single-GPU ones bit for bit: the global CDF is the concatenation of the
// per-rank CDFs shifted by the rank offsets (G-invariance).
__device__ __forceinline__ uint32_t first_above_t(const unsigned long long *C, const unsigned long long *Cs,
                                                 uint32_t L, uint64_t tj) {
    if (Cs) {
        const uint32_t g = first_above<SMC_K6_ARY>(Cs, 0, cdf_samples(L) - 1, tj);
        const uint32_t a = g * kCdfSample, b = min(a + kCdfSample, L) - 1;
        return first_above<SMC_K6_ARY>(C, a, b, tj);
    }
    return first_above<2>(C, 0, L - 1, tj);
}

__global__ void __launch_bounds__(kRowsPerBlock) k_gather_propose_multi(const MultiArgs m) {
    const ProposeArgs &p = m.p;
    __shared__ const float *s_src[kRowsPerBlock];
    __shared__ uint32_t s_j[kRowsPerBlock];
    __shared__ uint32_t s_perturb_x2[kRowsPerBlock];
    __shared__ uint64_t s_qd[kMaxAc], s_qm[kMaxAc], s_R[kMaxAc], s_off[kMaxAc][9];
    const uint32_t mpc = *p.mpcp;
    const int n = p.n;
    if (threadIdx.x < (unsigned)n) {                       // per column: global total, offset R, rank offsets
        const int i = threadIdx.x;
        uint64_t Q = 0;
        for (int r = 0; r < m.G; ++r) {
            s_off[i][r] = Q;
            Q += m.Qall[(size_t)r * m.Qstride + i];
        }
        s_off[i][m.G] = Q;
        const uint64_t rw = r64(TAG_RESAMPLE, (uint32_t)i, p.k, mpc, p.key0, p.key1);
        s_R[i] = __umul64hi(rw, Q);
        s_qd[i] = Q / m.Lg;
        s_qm[i] = Q % m.Lg;
    }
    __syncthreads();
    const uint32_t rows = p.L * (uint32_t)n;
    const uint32_t invH = 0xFFFFFFFFu / (uint32_t)p.H + 1u;
    for (uint32_t q0 = blockIdx.x * kRowsPerBlock; q0 < rows; q0 += gridDim.x * kRowsPerBlock) {
        {
            const uint32_t q = q0 + threadIdx.x;
            const float *src = nullptr;
            if (q < rows) {
                const uint32_t jl = q / (uint32_t)n;
                const int i = (int)(q - jl * (uint32_t)n);
                const uint64_t t = slot_t(p.l0 + jl, s_qd[i], s_qm[i], s_R[i], m.Lg);
                int rho = 0;
                while (rho < m.G - 1 && t >= s_off[i][rho + 1]) ++rho;
                const uint64_t tl = t - s_off[i][rho];
                const unsigned long long *Cs = m.peer_Cs[rho] ? m.peer_Cs[rho] + (size_t)i * m.Cs_stride : nullptr;
                const uint32_t a = first_above_t(m.peer_C[rho] + (size_t)i * m.Cstride, Cs, m.len[rho], tl);
                if (m.Sall) {
                    src = m.Sall + (((size_t)rho * m.Lmax + a) * n + i) * p.H * 3;
                } else {
                    const uint32_t bit = (__ldg(&m.peer_surv[rho][a]) >> i) & 1u;
                    src = m.peer_ctrl[rho] + bit * m.prow + ((size_t)a * n + i) * p.H * 3;
                }
                s_j[threadIdx.x] = jl;
                s_perturb_x2[threadIdx.x] = (uint32_t)i << 8;
            }
            s_src[threadIdx.x] = src;
        }
        __syncthreads();
        propose_rows(p, s_src, s_j, s_perturb_x2, q0, rows, mpc, invH);
        __syncthreads();
    }
    reset_round_state(p);
}

cudaError_t launch_gather_propose_multi(const MultiArgs &m0, cudaStream_t st) {
    const size_t rows = (size_t)m0.p.L * m0.p.n;
    if (!rows) return cudaSuccess;
    MultiArgs m = m0;
    for (int r = 0; r < 10; ++r) {
        m.p.ks[2 * r] = m.p.key0 + (uint32_t)r * 0x9E3779B9u;
        m.p.ks[2 * r + 1] = m.p.key1 + (uint32_t)r * 0xBB67AE85u;
    }
    size_t g = (rows + kRowsPerBlock - 1) / kRowsPerBlock;
    if (g > 148 * 16 * 256 / kRowsPerBlock) g = 148 * 16 * 256 / kRowsPerBlock;
    k_gather_propose_multi<<<(unsigned)g, kRowsPerBlock, 0, st>>>(m);
    return cudaGetLastError();
}

// Global winner from the all-gathered per-rank selection records
// {double lambda, int64 index, float row[n][H][3]}: greatest lambda, ties ->
// lowest global index, -1 index = rank had no feasible particle.
__global__ void k_select_merge(const unsigned char *recs, int G, size_t rec_bytes, int rowlen, unsigned char *out) {
    __shared__ int s_best;
    if (threadIdx.x == 0) {
        int best = -1;
        double bl = 0.0;
        long long bi = -1;
        for (int r = 0; r < G; ++r) {
            const double lr = *reinterpret_cast<const double *>(recs + r * rec_bytes);
            const long long ir = *reinterpret_cast<const long long *>(recs + r * rec_bytes + 8);
            if (ir < 0) continue;
            if (bi < 0 || lr > bl || (lr == bl && ir < bi)) { best = r; bl = lr; bi = ir; }
        }
        s_best = best;
        *reinterpret_cast<double *>(out) = best >= 0 ? bl : -INFINITY;
        *reinterpret_cast<long long *>(out + 8) = bi;
    }
    __syncthreads();
    if (s_best < 0) return;
    const float *src = reinterpret_cast<const float *>(recs + s_best * rec_bytes + 16);
    float *dst = reinterpret_cast<float *>(out + 16);
    for (int e = threadIdx.x; e < rowlen; e += blockDim.x) dst[e] = src[e];
}

cudaError_t launch_select_merge(const unsigned char *recs, int G, size_t rec_bytes, int rowlen, unsigned char *out,
                                cudaStream_t st) {
    k_select_merge<<<1, 128, 0, st>>>(recs, G, rec_bytes, rowlen, out);
    return cudaGetLastError();
}
}  // namespace smc

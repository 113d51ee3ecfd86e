// k_rollout.cu -- K2: batched Monte Carlo evaluation (Alg.1 l.9-18)
// fused with the Metropolis-Hastings accept step (R1).
//
// Mapping: one warp segment of W = next_pow2(N) lanes per
// particle l, lane = aircraft i.  Each lane keeps its aircraft's state for
// both MH candidates (c = 0: resampled x', c = 1: proposal x*) in registers;
// both candidates see the same wind realisation (common random numbers).
// Per step t the segment
//   1. draws the 16 normals of the 2x2x2 wind field (Philox, Box-Muller),
//      advances the AR(1) state Z and forms W = Qhat Z, directly in
//      trilinear-coefficient form (Cq = M Qhat, tripoly) -- the 16 entries are
//      distributed over the lanes and exchanged via shared memory;
//   2. every lane interpolates W at its aircraft, adds the nominal wind
//      and gust, and applies Eq. hor to both candidates;
//   3. checks the envelope / mass and the landing sector
//      (Eq. TO_init);
//   4. checks separation against every other lane of the segment through a
//      shared-memory broadcast of positions (Eq. avoidance);
//   5. accumulates the per-step cost terms.
// After S samples: ell += sum_s log2 J_T (R24); lambda = sum_i ell in
// double; MH decision (R1); survivor ell / lambda / flag written; per-column
// max of ell folded into an atomicMax (first step of the resampling reduce).
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "smc_device.cuh"
#include "smc_kernels.h"
#include "smc_vec.cuh"

#ifndef SMC_K2_TUNROLL
#define SMC_K2_TUNROLL 2   // unroll factor of the horizon loop (A/B on c2: 1 -> 29.2, 2 -> 28.2, 3 -> 29.0 ms of K2)
#endif
#ifndef SMC_K2_MINB
#define SMC_K2_MINB 4   // resident 128-thread blocks per SM the register budget targets, two candidates
#endif
#ifndef SMC_K2_MINB1
#define SMC_K2_MINB1 5  // the same for single-candidate launches (round 0, paper mode; sweep: 5 > 6 > 4)
#endif
#ifndef SMC_K2_FASTTRIG
#define SMC_K2_FASTTRIG 1   // control staging: MUFU sin/cos (A/B on c2: 27.80 vs 28.11 ms of K2)
#endif
#ifndef SMC_K2_MINBSP
#define SMC_K2_MINBSP 3   // sample-pair launches (Table-1 workload: 3 -> 181.4, 5 -> 184.1, 4 -> 188.5 ms)
#endif
#ifndef SMC_K2_MINB32
#define SMC_K2_MINB32 SMC_K2_MINB  // two candidates in 32-lane segments (N > 16)
#endif

namespace smc {

constexpr int kTUnroll = SMC_K2_TUNROLL;

__device__ __forceinline__ float clamp01(float v) { return fminf(fmaxf(v, 0.0f), 1.0f); }

// a - 2 pi rint(a / 2 pi): the integer by the magic-number form (one packed FMA adding
// 1.5 * 2^23, one packed subtract: FMA pipe) instead of FRND per candidate on the XU pipe, which
// the MUFU work keeps busy (c5 K2 2166 -> 2154 ms over 21 rounds; round 1, before the XU load
// grew, it measured slower: 28.62 vs 28.13 ms of c2 K2).  A tie at an odd multiple of pi may
// round either way: +pi and -pi are the same heading for every later use (sin, cos, |chi|).
#ifndef SMC_K2_WRAPMAGIC
#define SMC_K2_WRAPMAGIC 1
#endif
template <class V>
__device__ __forceinline__ V wrap_pi(V a) {
#if SMC_K2_WRAPMAGIC
    // rint(a / 2 pi) on the FMA pipe: adding 1.5 * 2^23 rounds to an integer (|a| < 2^22 pi)
    const V k = vfma(a, 1.0f / kTwoPi, 12582912.0f) - 12582912.0f;
    return vfma(k, -kTwoPi, a);
#else
    return vfma(vmap(a * (1.0f / kTwoPi), [](float u) { return rintf(u); }), -kTwoPi, a);
#endif
}

// popdense bilinear lookup on the 1 km grid, clamped at its edge.
// pop: the grid in global memory (read-only path) or staged in shared memory by the caller
__device__ __forceinline__ float popdense(const DevScen &sc, const float *pop, float x, float y) {
    float gx = (x - sc.pop_x0) * sc.pop_inv_dx, gy = (y - sc.pop_y0) * sc.pop_inv_dx;
    const float mx = (float)(sc.pop_nx - 1), my = (float)(sc.pop_ny - 1);
    gx = fminf(fmaxf(gx, 0.0f), mx);
    gy = fminf(fmaxf(gy, 0.0f), my);
    int ix = min((int)gx, max(sc.pop_nx - 2, 0));
    int iy = min((int)gy, max(sc.pop_ny - 2, 0));
    const float fx = sc.pop_nx > 1 ? gx - (float)ix : 0.0f;
    const float fy = sc.pop_ny > 1 ? gy - (float)iy : 0.0f;
    const int ix1 = sc.pop_nx > 1 ? ix + 1 : ix, iy1 = sc.pop_ny > 1 ? iy + 1 : iy;
    const float v00 = pop[iy * sc.pop_nx + ix], v10 = pop[iy * sc.pop_nx + ix1];
    const float v01 = pop[iy1 * sc.pop_nx + ix], v11 = pop[iy1 * sc.pop_nx + ix1];
    const float a = fmaf(fx, v10 - v00, v00), b = fmaf(fx, v11 - v01, v01);
    return fmaf(fy, b - a, a);
}

// popdense on the edge-padded grid pp = [pop_ny + 1][pop_nx + 1], both candidates of a
// chain.  u = clamp((x - x0) / dx, 0, nx - 1) / (nx - 1) is one saturated FMA; the cell comes from
// adding 1.5 * 2^23 to u (nx - 1) - 1/2 (round to nearest: floor, or one cell lower at an integer
// coordinate, whose weight is then 1), read off the float's low bits -- no F2I, no index clamp (the
// padding makes column nx and row ny valid).  pp: shared memory or global (inlined per space).
template <class V, bool LDG = false>
__device__ __forceinline__ V popdense_pad(const DevScen &sc, const float *pp, V x, V y) {
    constexpr int NCV = (int)(sizeof(V) / sizeof(float));
    constexpr float kMagic = 12582912.0f;                       // 1.5 * 2^23
    V ux, uy;
#pragma unroll
    for (int c = 0; c < NCV; ++c) {
        cset(ux, c, __saturatef(fmaf(cget(x, c), sc.pop_ax, sc.pop_bx)));
        cset(uy, c, __saturatef(fmaf(cget(y, c), sc.pop_ay, sc.pop_by)));
    }
    const V kx = vfma(ux, sc.pop_mx, -0.5f) + kMagic, ky = vfma(uy, sc.pop_my, -0.5f) + kMagic;
    const V fx = vfma(ux, sc.pop_mx, kMagic - kx), fy = vfma(uy, sc.pop_my, kMagic - ky);
    const int P = sc.pop_nx + 1;
    V v00, v10, v01, v11;
#pragma unroll
    for (int c = 0; c < NCV; ++c) {
        const uint32_t e = __float_as_uint(cget(ky, c)) * (uint32_t)P + __float_as_uint(cget(kx, c)) -
                           0x4B400000u * (uint32_t)(P + 1);
        const float *r0 = pp + e, *r1 = r0 + P;
        if constexpr (LDG) {
            cset(v00, c, __ldg(r0)); cset(v10, c, __ldg(r0 + 1));
            cset(v01, c, __ldg(r1)); cset(v11, c, __ldg(r1 + 1));
        } else {
            cset(v00, c, r0[0]); cset(v10, c, r0[1]);
            cset(v01, c, r1[0]); cset(v11, c, r1[1]);
        }
    }
    const V a = vfma(fx, v10 - v00, v00), b = vfma(fx, v11 - v01, v01);
    return vfma(fy, b - a, a);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// atan2 on the MUFU reciprocal and a degree-15 odd polynomial (least-squares
// fit of atan(a)/a on [0,1] in a^2; |error| < 1.5e-7 rad in binary32), both
// candidates at once (packed polynomial, per-candidate octant selects).
template <class V>
__device__ __forceinline__ V fast_atan2(V y, V x) {
    const V ax = vabs(x), ay = vabs(y);
    V mx, mn;
#pragma unroll
    for (int c = 0; c < (int)(sizeof(V) / sizeof(float)); ++c) {
        cset(mx, c, fmaxf(cget(ax, c), cget(ay, c)));
        cset(mn, c, fminf(cget(ax, c), cget(ay, c)));
    }
    const V a = mn * vmap(mx, [](float u) { return rcp_approx(fmaxf(u, 1e-30f)); });   // mx = 0 -> mn = 0 -> a = 0
    const V s = a * a;
    V p = vfma(s, -0.0040731243789196014f, 0.021945973858237267f);
    p = vfma(p, s, -0.056062303483486176f);
    p = vfma(p, s, 0.0965619683265686f);
    p = vfma(p, s, -0.13915780186653137f);
    p = vfma(p, s, 0.19948504865169525f);
    p = vfma(p, s, -0.3333010673522949f);
    p = vfma(p, s, 0.999999463558197f);
    const V r = p * a;
    const V r1 = 1.57079632679489662f - r;
    V q;
#pragma unroll
    for (int c = 0; c < (int)(sizeof(V) / sizeof(float)); ++c)
        cset(q, c, cget(ay, c) > cget(ax, c) ? cget(r1, c) : cget(r, c));
    const V q1 = kPi - q;
    V out;
#pragma unroll
    for (int c = 0; c < (int)(sizeof(V) / sizeof(float)); ++c)
        cset(out, c, copysignf(cget(x, c) < 0.0f ? cget(q1, c) : cget(q, c), cget(y, c)));
    return out;
}

// atan2(y, x) for x >= 0 (right half-plane), without octant selects: for a, b >= 0,
// atan2(a, b) = pi/4 + atan(t), t = (a - b) / (a + b) in [-1, 1], where the same odd polynomial
// holds; the sign of y is restored by copysign.  Absolute error ~2e-7 rad, but not relative
// accuracy near 0 (pi/4 - pi/4 cancels) -- used for beta, which enters only absolute terms.
template <class V>
__device__ __forceinline__ V fast_atan2_xpos(V y, V x) {
    const V ay = vabs(y);
    const V t = (ay - x) * vmap(ay + (x + 1e-37f), [](float u) { return rcp_approx(u); });   // x = y = 0 -> t = 0
    const V s = t * t;
    V p = vfma(s, -0.0040731243789196014f, 0.021945973858237267f);
    p = vfma(p, s, -0.056062303483486176f);
    p = vfma(p, s, 0.0965619683265686f);
    p = vfma(p, s, -0.13915780186653137f);
    p = vfma(p, s, 0.19948504865169525f);
    p = vfma(p, s, -0.3333010673522949f);
    p = vfma(p, s, 0.999999463558197f);
    const V r = vfma(p, t, 0.78539816339744831f);
    V out;
#pragma unroll
    for (int c = 0; c < (int)(sizeof(V) / sizeof(float)); ++c) cset(out, c, copysignf(cget(r, c), cget(y, c)));
    return out;
}

// Shared-memory strides of the wind field per segment: normals (VST) and
// AR(1) state / node values (ZST: even, so the node-major (x, y) state loads as float2;
// the + 2 shifts neighbouring segments by two banks).
__host__ __device__ constexpr int dense_vst(int G) { return 4 * ((2 * G + 3) / 4); }
__host__ __device__ constexpr int dense_zst(int G) { return 2 * G + 2; }
// row stride of the transposed factor Qhat^T [G][QTS] (multiple of 4 for 16-byte rows, zero padded)
__host__ __device__ constexpr int dense_qts(int G) { return 4 * ((G + 3) / 4) + 4; }

// R: separation ring size, n <= R <= W: lanes < R publish their position (NaN when they carry no
// flying aircraft) and scan partners d = 1..R/2 (mod R) at compile time; lanes >= R publish
// nothing.  R = W is the plain segment ring.
// SP (sample pairs, single-candidate launches): the two float2 slots carry samples s and s+1 of
// the same particle instead of two MH candidates -- each slot its own wind / gust draws, the
// two log-weights summed at the end; launched as NC = 2 with both control pointers equal.
template <int W, int NC, bool DEBUG, bool DENSE, int R = W, bool SP = false>
__global__ void __launch_bounds__(kBlock, SP ? SMC_K2_MINBSP : (NC == 1 ? SMC_K2_MINB1 : (W >= 32 ? SMC_K2_MINB32 : SMC_K2_MINB)))
k_rollout(const DevScen sc, const RolloutArgs args) {
    static_assert(!SP || (NC == 2 && !DENSE && !DEBUG && W >= 8), "sample pairs: two slots, 2x2x2 grid, W >= 8");
    constexpr int NSL = SP ? 2 : 1;                 // wind realisations per segment and step
    constexpr int SEGS = kBlock / W;
    constexpr int TU = W >= 32 ? 1 : kTUnroll;      // W = 32 spills when unrolled
    constexpr int EN = W >= 8 ? 1 : 8 / W;          // wind-grid nodes owned per lane (lanes >= 8 idle)
    extern __shared__ __align__(16) float smem[];
    const int H = sc.H, n = sc.n;
    float4 *s_ctrl = reinterpret_cast<float4 *>(smem);               // [H][NC][kBlock] (T, tan phi, sin g, cos g)
    constexpr int GB = (W >= 8 && !DENSE) ? W / 4 : 1;             // steps whose normals one batch draws
    // 2x2x2 grid: [SEGS][GB][16] normals, [SEGS][16] state, [SEGS][16] coefficients, Cq [8][9];
    // dense grid (G = N_x N_y N_z > 8): [SEGS][VST] normals, [SEGS][ZST] state and node values,
    // Qhat [G][G+1]
    const int G = DENSE ? sc.wng : 8;
    const int VST = DENSE ? dense_vst(G) : GB * 16 * NSL, ZST = DENSE ? dense_zst(G) : 16 * NSL;
    float *s_V = reinterpret_cast<float *>(s_ctrl + H * NC * kBlock);
    float *s_Z = s_V + SEGS * VST;
    float *s_W = s_Z + SEGS * ZST;
    // positions for the separation scan, each segment's entries stored twice so partner
    // lane + d is a constant offset: [2 kBlock] float4 (NC = 2: (x0, x1, y0, y1)) + [2 kBlock] float2 (z0, z1)
    float4 *s_pos = reinterpret_cast<float4 *>(s_W + ((SEGS * ZST + 3) & ~3));
    float *s_Q = reinterpret_cast<float *>(s_pos + 3 * kBlock);

    const int tid = threadIdx.x, lane = tid % W, seg = tid / W;
    const uint32_t lloc = blockIdx.x * SEGS + seg;
    const bool valid = lloc < args.L;
    const uint32_t l = args.l0 + lloc;                         // global particle index
    const bool isac = lane < n;
    const uint32_t k = args.k, mpc = *args.mpcp;

    if constexpr (DENSE) {
        const int qts = dense_qts(G);
        for (int q = tid; q < G * qts; q += kBlock) {
            const int m = q / qts, r = q % qts;                 // s_Q[m][r] = Qhat[r][m]
            s_Q[q] = r < G ? sc.Qf[r * G + m] : 0.0f;
        }
    } else {
        if (tid < 64) s_Q[(tid >> 3) * 9 + (tid & 7)] = sc.Cq[tid];   // W = Cq Z: trilinear coefficients
    }

    // ---- per-lane aircraft constants needed every step (the rest is read when needed)
    const DevAircraft *Ap = sc.ac + (isac ? lane : 0);
    const int kind = Ap->kind;
    const int first = isac ? Ap->first_step : (1 << 20);
    const float halfS = Ap->halfS, cd0 = Ap->cd0, cd2 = Ap->cd2, dt_eta = Ap->dt_eta;
    const float zmin = Ap->z_min, zmax = Ap->z_max, vmin = Ap->v_min, vmax = Ap->v_max, mempty = Ap->m_empty;
    const float gA = kind ? Ap->theta_F : Ap->beta_f;          // goal of the A/D term or the E term
    const float z_tf = Ap->z_tf, v_D = Ap->v_D;

    // ---- controls: (T, tan phi, sin gamma, cos gamma) to shared memory; envelope bits to registers.
    // NC = 1: one float4 (T, tan phi, sin g, cos g) per (t, lane).  NC = 2: the candidates
    // interleaved so each quantity loads as a float2 pair -- (T0, T1, tphi0, tphi1) and
    // (sg0, sg1, cg0, cg1) at s_ctrl[(2t + h) kBlock + tid], h = 0, 1.
    uint32_t cbad[NC];
    // SP (one candidate, sample pairs): the airframe -- z, v, chi, m; wind-independent (Eq. hor,
    // P:246-251) -- is integrated once per particle here, as in k_rollout_2s: per step the
    // air-relative ground velocity, z and chi after the step (s_rec) and the fuel increment
    // (s_rfi); envelope / landing speed-heading flags as bit t of vbadm / lokm
    float4 *const s_rec = reinterpret_cast<float4 *>(s_ctrl);              // SP: [H][kBlock]
    float *const s_rfi = reinterpret_cast<float *>(s_rec + H * kBlock);      // SP: [H][kBlock]
    uint32_t vbadm = 0u, lokm = 0u;
    float sCc = 0.0f;
    if constexpr (SP) {
#pragma unroll
        for (int c = 0; c < NC; ++c) cbad[c] = 0;
        const float gmax = Ap->gamma_max, pmax = Ap->phi_max, Tmin = Ap->T_min, Tmax = Ap->T_max;
        const float cq1 = (sc.density_mode == 0 ? 1.225f : sc.rho_const) * halfS;
        const float *src = args.ctrl[0] + ((size_t)lloc * n + lane) * H * 3;
        float v = Ap->x0[3], z = Ap->x0[2], chi = Ap->x0[4], m = Ap->x0[5];
        const float dt1 = sc.dt, g1 = sc.g;
        bool broken = false;
        for (int t = 0; t < H; ++t) {
            float T = 0.f, ph = 0.f, ga = 0.f;
            if (isac && valid) { T = src[3 * t]; ph = src[3 * t + 1]; ga = src[3 * t + 2]; }
            float sph, cph, sga, cga;
            __sincosf(ph, &sph, &cph);
            __sincosf(ga, &sga, &cga);
            const float tph = sph * rcp_approx(cph);
            const bool cbd = (fabsf(ga) > gmax) || !(fabsf(ph) < pmax) || (T < Tmin) || (T > Tmax);
            const bool act = first <= t;
            const float dta = act ? dt1 : 0.0f, dtea = act ? dt_eta : 0.0f;
            float qd = cq1 * v * v;
            if (sc.density_mode == 0) qd = qd * ex2_approx(lg2_approx(fmaxf(fmaf(z, -2.2558e-5f, 1.0f), 0.0f)) * 4.2559f);
            const float mgq = (m * g1) * rcp_approx(qd);
            const float D = qd * fmaf(fmaf(tph, tph, 1.0f) * cd2, mgq * mgq, cd0);
            float sch, cch;
            __sincosf(chi, &sch, &cch);
            const float vcg = v * cga;
            float ax = vcg * cch, ay = vcg * sch;
            float nz = fmaf(dta * v, sga, z);
            const float nv = fmaf(dta, fmaf(T - D, rcp_approx(m), sga * (-g1)), v);
            float nchi = wrap_pi(fmaf((dta * g1) * tph, rcp_approx(v), chi));
            const float nm = fmaf(-dtea, T, m);
            float fi = T * dtea;
            const bool fin = (fabsf(ax) < INFINITY) & (fabsf(ay) < INFINITY) & (fabsf(nz) < INFINITY) &
                             (fabsf(nv) < INFINITY) & (fabsf(nchi) < INFINITY) & (fabsf(nm) < INFINITY);
            broken |= !fin;
            bool bad, lok;
            if (broken) {                       // non-finite: far-away sentinel (see k_rollout_2s)
                ax = ay = nz = 1e30f; nchi = 0.0f; fi = 0.0f;
                bad = true; lok = false;
            } else {
                bad = cbd | !(nz >= zmin) | !(nz <= zmax) | !(nv >= vmin) | !(nv <= vmax) | !(nm >= mempty);
                lok = (nv <= sc.P_vs) & (fabsf(nchi) >= sc.P_chi_west);
                if (act) sCc += fabsf(nv - v_D);
            }
            vbadm |= (bad ? 1u : 0u) << t;
            lokm |= (lok ? 1u : 0u) << t;
            s_rec[t * kBlock + tid] = make_float4(ax, ay, nz, nchi);
            s_rfi[t * kBlock + tid] = fi;
            v = nv; z = nz; chi = nchi; m = nm;
        }
    } else {
        const float gmax = Ap->gamma_max, pmax = Ap->phi_max, Tmin = Ap->T_min, Tmax = Ap->T_max;
        const float *src[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            cbad[c] = 0;
            src[c] = args.ctrl[c] + ((size_t)lloc * n + lane) * H * 3;
        }
        for (int t = 0; t < H; ++t) {
            float q[NC][4];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                float T = 0.f, ph = 0.f, ga = 0.f;
                if (isac && valid) { T = src[c][3 * t]; ph = src[c][3 * t + 1]; ga = src[c][3 * t + 2]; }
                float sph, cph, sga, cga;
#if SMC_K2_FASTTRIG
                __sincosf(ph, &sph, &cph);                    // |phi| < 30 deg, |gamma| < 6 deg: MUFU
                __sincosf(ga, &sga, &cga);
#else
                sincosf(ph, &sph, &cph);
                sincosf(ga, &sga, &cga);
#endif
                q[c][0] = T; q[c][1] = SMC_K2_FASTTRIG ? sph * rcp_approx(cph) : sph / cph; q[c][2] = sga; q[c][3] = cga;
                const bool bad = (fabsf(ga) > gmax) || !(fabsf(ph) < pmax) || (T < Tmin) || (T > Tmax);
                cbad[c] |= (bad ? 1u : 0u) << t;
            }
            if constexpr (NC == 2) {
                s_ctrl[(2 * t) * kBlock + tid] = make_float4(q[0][0], q[1][0], q[0][1], q[1][1]);
                s_ctrl[(2 * t + 1) * kBlock + tid] = make_float4(q[0][2], q[1][2], q[0][3], q[1][3]);
            } else {
                s_ctrl[t * kBlock + tid] = make_float4(q[0][0], q[0][1], q[0][2], q[0][3]);
            }
        }
    }
    __syncthreads();

    // W >= 8: every wind entry a lane owns belongs to node lane & 7 -> keep that Qhat row in registers
    float qrow[8];
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) qrow[mm] = (W >= 8 && !DENSE) ? s_Q[(lane & 7) * 9 + mm] : 0.0f;

    float ell[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) ell[c] = (SP && c == 1) ? 0.0f : args.ell0;

    using V = vec_t<NC>;
    const float dt = sc.dt, g = sc.g;
    // wind-box coordinates f = sat(p inv + nlo) (clamped to the box, R14)
    const float inv0 = sc.wind_inv_ext[0], inv1 = sc.wind_inv_ext[1], inv2 = sc.wind_inv_ext[2];
    const float nlo0 = -sc.wind_lo[0] * inv0, nlo1 = -sc.wind_lo[1] * inv1, nlo2 = -sc.wind_lo[2] * inv2;
    // dynamic pressure factor: q = rho v^2 S / 2 = cq e(z) v^2, e(z) the ISA ratio or 1
    const float cq = (sc.density_mode == 0 ? 1.225f : sc.rho_const) * halfS;
    // The deviation arguments as FMA chains with per-lane coefficients (kind is per aircraft):
    //   departure A = theta - theta_F, B = z_tf - z;  arrival A = chi - pi - 2 theta (R8), B = beta - beta_f
    const float cA_th = kind ? 1.0f : -2.0f, cA_chi = kind ? 0.0f : 1.0f, cA_0 = kind ? -gA : -kPi;
    const float cB_z = kind ? -1.0f : 0.0f, cB_b = kind ? 0.0f : 1.0f, cB_0 = kind ? z_tf : -gA;
    const uint32_t s_lo = 0, s_hi = args.S;
    for (uint32_t s = s_lo; s < s_hi; s += NSL) {
        V x = vsplat<V>(Ap->x0[0]), y = vsplat<V>(Ap->x0[1]), z = vsplat<V>(Ap->x0[2]);
        V v = vsplat<V>(Ap->x0[3]), chi = vsplat<V>(Ap->x0[4]), m = vsplat<V>(Ap->x0[5]);
        V fuel = vsplat<V>(0.0f), sA = fuel, sB = fuel, sC = fuel, sN = fuel;
        // per-candidate flags as bit masks (bit c = candidate c)
        constexpr int ALLC = (1 << NC) - 1;
        int landedm = 0, violm = 0;
        constexpr int ENS = SP ? (W >= 16 ? 1 : 2) : EN;   // (node, slot) pairs a lane owns
        float2 Zr[ENS];                                  // AR(1) state of the lane's nodes, (x, y)
        float2 gust_odd = make_float2(0.f, 0.f), gust_odd_b = gust_odd;
        const uint32_t x1 = (s & 0xFFFFu) | (k << 16);
        const uint32_t x1b = ((s + 1) & 0xFFFFu) | (k << 16);   // SP: the second slot's sample

#pragma unroll TU
        for (int t = 0; t < H; ++t) {
            // ---------------- 1. wind realisation for step t (Alg.1 l.10).
            float Wn[16];
            float *const sWs = s_W + seg * ZST;
            if constexpr (DENSE) {
                // dense grid: 2G normals from ceil(2G/4) Philox blocks, AR(1) in shared
                // memory, node values W = Qhat Z (lower-triangular rows) -- spread over the lanes
                float *const sVs = s_V + seg * VST, *const sZs = s_Z + seg * ZST;
                const int G2 = 2 * G, nblk = (G2 + 3) >> 2;
                for (int b = lane; b < nblk; b += W) {
                    const uint4 w = draw_ks(TAG_WIND, l, x1, (uint32_t)t | ((uint32_t)b << 16), mpc, sc.ks);
                    *reinterpret_cast<float4 *>(&sVs[4 * b]) = box_muller4(w);
                }
                __syncwarp();
                // AR(1) state node-major, both components of a node in one float2 (normal e of
                // the step is component e / G, node e mod G, R48)
                float2 *const sZ2 = reinterpret_cast<float2 *>(sZs);
                for (int nd = lane; nd < G; nd += W) {
                    const float2 ve = make_float2(sVs[nd], sVs[G + nd]);
                    sZ2[nd] = (t == 0) ? ve : vfma(sZ2[nd], sc.a, ve * sc.b);
                }
                __syncwarp();
                // W = Qhat Z from the transposed factor, four consecutive rows per task: one
                // 16-byte load of Qhat^T[m][r0..r0+3] per 4 FMAs of each component the task
                // covers.  The lower triangle makes row block q cost 4q + 4 iterations, so a lane
                // takes the blocks q and nq - 1 - q together (every pair costs the same).  With
                // more pairs than lanes a task covers both components (one Z (x, y) float2 load
                // per 8 FMAs: half the shared-memory traffic); otherwise one component, so that
                // more lanes work (4x4x4 in 8 lanes: 207 -> 143 ms per c2 MPC step)
                const int nq = (G + 3) >> 2, half = (nq + 1) >> 1;
                const bool both = 2 * half > W;
                const int ntask = both ? half : 2 * half;
                for (int pt = lane; pt < ntask; pt += W) {
                    const int comp = (!both && pt >= half) ? 1 : 0, qa = pt - comp * half;
                    for (int side = 0; side < 2; ++side) {
                        const int q = side ? nq - 1 - qa : qa;
                        if (side && q == qa) break;
                        const int r0 = 4 * q;
                        const int mend = min(r0 + 4, G);         // Qhat lower triangular: m <= r
                        float4 ax = make_float4(0.f, 0.f, 0.f, 0.f), ay = ax;
                        if (both) {
                            for (int m = 0; m < mend; ++m) {
                                const float4 q4 = *reinterpret_cast<const float4 *>(&s_Q[m * dense_qts(G) + r0]);
                                const float2 zm = sZ2[m];
                                ax.x = fmaf(q4.x, zm.x, ax.x); ax.y = fmaf(q4.y, zm.x, ax.y);
                                ax.z = fmaf(q4.z, zm.x, ax.z); ax.w = fmaf(q4.w, zm.x, ax.w);
                                ay.x = fmaf(q4.x, zm.y, ay.x); ay.y = fmaf(q4.y, zm.y, ay.y);
                                ay.z = fmaf(q4.z, zm.y, ay.z); ay.w = fmaf(q4.w, zm.y, ay.w);
                            }
                        } else {
                            const float *zc = sZs + comp;                // node-major: Z[m].comp
                            for (int m = 0; m < mend; ++m) {
                                const float4 q4 = *reinterpret_cast<const float4 *>(&s_Q[m * dense_qts(G) + r0]);
                                const float zm = zc[2 * m];
                                ax.x = fmaf(q4.x, zm, ax.x); ax.y = fmaf(q4.y, zm, ax.y);
                                ax.z = fmaf(q4.z, zm, ax.z); ax.w = fmaf(q4.w, zm, ax.w);
                            }
                        }
                        float *wx = sWs + comp * G + r0, *wy = sWs + G + r0;
                        wx[0] = ax.x;
                        if (r0 + 1 < G) wx[1] = ax.y;
                        if (r0 + 2 < G) wx[2] = ax.z;
                        if (r0 + 3 < G) wx[3] = ax.w;
                        if (both) {
                            wy[0] = ay.x;
                            if (r0 + 1 < G) wy[1] = ay.y;
                            if (r0 + 2 < G) wy[2] = ay.z;
                            if (r0 + 3 < G) wy[3] = ay.w;
                        }
                    }
                }
                __syncwarp();
            } else {
            // Every GB steps the segment's lanes draw the 4 Philox blocks of GB
            // consecutive steps at once (lane -> block lane&3 of step t + lane/4); SP: the
            // blocks of both slots' samples (slot = task / (4 GB)).
            const int tb = t % GB;
            if (tb == 0) {
                for (int task = lane; task < 4 * GB * NSL; task += W) {
                    const int sl = SP ? task / (4 * GB) : 0, tk = task - sl * 4 * GB;
                    const int b = tk & 3, ts = t + (tk >> 2);
                    if (ts < H) {
                        const uint4 w = draw_ks(TAG_WIND, l, sl ? x1b : x1, (uint32_t)ts | ((uint32_t)b << 16), mpc, sc.ks);
                        *reinterpret_cast<float4 *>(&s_V[((seg * NSL + sl) * GB + (tk >> 2)) * 16 + 4 * b]) = box_muller4(w);
                    }
                }
            }
            __syncwarp();
            // AR(1) and W = Cq Z with both components of a node packed in one float2:
            // lane owns (node, slot) pair lane + q W (q < ENS; node = pair & 7, slot = pair >> 3);
            // Z is kept node-major [slot][node](x, y) in shared memory
            // (segments wider than the 8 NSL pairs: every lane computes pair lane mod 8 NSL -- the
            // duplicates store identical values -- so no lane branches around the work)
            float2 *const sZ2 = reinterpret_cast<float2 *>(s_Z + seg * 16 * NSL);
            constexpr bool FULL = W >= 8 * NSL;
#pragma unroll
            for (int q = 0; q < ENS; ++q) {
                const int pq = FULL ? (lane & (8 * NSL - 1)) : lane + q * W;
                const int node = SP ? (pq & 7) : pq, sl = SP ? (pq >> 3) : 0;
                if (FULL || pq < 8 * NSL) {
                    const float *vv = &s_V[((seg * NSL + sl) * GB + tb) * 16];
                    const float2 ve = make_float2(vv[node], vv[8 + node]);
                    Zr[q] = (t == 0) ? ve : vfma(Zr[q], sc.a, ve * sc.b);
                    sZ2[sl * 8 + node] = Zr[q];
                }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < ENS; ++q) {
                const int pq = FULL ? (lane & (8 * NSL - 1)) : lane + q * W;
                const int node = SP ? (pq & 7) : pq, sl = SP ? (pq >> 3) : 0;
                if (FULL || pq < 8 * NSL) {
                    const float4 *z4 = reinterpret_cast<const float4 *>(sZ2 + sl * 8);
                    const float *qr = (W >= 8) ? qrow : &s_Q[node * 9];
                    float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float4 zz = z4[mm];
                        acc = vfma(make_float2(zz.x, zz.y), qr[2 * mm], acc);
                        acc = vfma(make_float2(zz.z, zz.w), qr[2 * mm + 1], acc);
                    }
                    if constexpr (SP) {                          // interleaved [coefficient][slot]
                        s_W[(seg * 16 + node) * 2 + sl] = acc.x;
                        s_W[(seg * 16 + 8 + node) * 2 + sl] = acc.y;
                    } else {
                        s_W[seg * 16 + node] = acc.x;
                        s_W[seg * 16 + 8 + node] = acc.y;
                    }
                }
            }
            __syncwarp();
            if constexpr (!SP) {
                const float4 *w4 = reinterpret_cast<const float4 *>(&s_W[seg * 16]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 a4 = w4[q];
                    Wn[4 * q] = a4.x; Wn[4 * q + 1] = a4.y; Wn[4 * q + 2] = a4.z; Wn[4 * q + 3] = a4.w;
                }
            }
            }
            // gusts (R15): one Philox call covers steps 2u and 2u+1 (SP: one per slot)
            float gx = sc.nominal[0], gy = sc.nominal[1], gxb = gx, gyb = gy;
            if (sc.turb_sigma > 0.0f) {
                float2 gg, ggb = make_float2(0.f, 0.f);
                if ((t & 1) == 0) {
                    const uint4 w = draw_ks(TAG_TURB, l, x1, ((uint32_t)t >> 1) | ((uint32_t)lane << 8), mpc, sc.ks);
                    const float4 g4 = box_muller4(w);
                    gg = make_float2(g4.x, g4.y);
                    gust_odd = make_float2(g4.z, g4.w);
                    if constexpr (SP) {
                        const uint4 wb = draw_ks(TAG_TURB, l, x1b, ((uint32_t)t >> 1) | ((uint32_t)lane << 8), mpc, sc.ks);
                        const float4 g4b = box_muller4(wb);
                        ggb = make_float2(g4b.x, g4b.y);
                        gust_odd_b = make_float2(g4b.z, g4b.w);
                    }
                } else {
                    gg = gust_odd;
                    ggb = gust_odd_b;
                }
                gx = fmaf(sc.turb_sigma, gg.x, gx);
                gy = fmaf(sc.turb_sigma, gg.y, gy);
                gxb = fmaf(sc.turb_sigma, ggb.x, gxb);
                gyb = fmaf(sc.turb_sigma, ggb.y, gyb);
            }
            float c0x = gx, c0y = gy;                                   // nominal + gust (+ c0)
            if constexpr (!DENSE && !SP) { c0x += Wn[0]; c0y += Wn[8]; }
            const float2 *const sW2 = reinterpret_cast<const float2 *>(&s_W[seg * 32]);   // SP: [k](slot a, slot b)

            // ---------------- 2-3. dynamics, unary checks and geometry, both candidates at once
            const bool act = first <= t;
            // Alg.1 l.11-13: every active aircraft flies its own controls to H and stays in
            // every pair test, violated or not (a failure only zeroes its weight); only a
            // landed arrival stops (R18)
            const int flym = act ? (~landedm & ALLC) : 0;
            V flyf;                                   // 1 while the candidate's aircraft flies, else 0
#pragma unroll
            for (int c = 0; c < NC; ++c) cset(flyf, c, ((flym >> c) & 1) ? 1.0f : 0.0f);
            V T, tph, sga, cga;
            if constexpr (SP) {
                T = tph = sga = cga = vsplat<V>(0.0f);           // (airframe from the records)
            } else if constexpr (NC == 2) {
                const float4 a = s_ctrl[(2 * t) * kBlock + tid], b = s_ctrl[(2 * t + 1) * kBlock + tid];
                T = make_float2(a.x, a.y); tph = make_float2(a.z, a.w);
                sga = make_float2(b.x, b.y); cga = make_float2(b.z, b.w);
            } else {
                const float4 a = s_ctrl[t * kBlock + tid];
                T = a.x; tph = a.y; sga = a.z; cga = a.w;
            }
            // wind at the pre-step position (trilinear, clamped to the box)
            V wx, wy;
            if constexpr (DENSE) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    // grid cell holding the aircraft (clamped), trilinear over its 8 corners
                    float f3[3];
                    int base = 0, mul = 1;
                    const float p3[3] = {cget(x, c), cget(y, c), cget(z, c)};
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const float gc = clamp01((p3[a] - sc.wind_lo[a]) * sc.wind_inv_ext[a]) * (float)(sc.wn[a] - 1);
                        const int i0 = min((int)gc, sc.wn[a] - 2);
                        f3[a] = gc - (float)i0;
                        base += i0 * mul;
                        mul *= sc.wn[a];
                    }
                    const int sy = sc.wn[0], sz = sc.wn[0] * sc.wn[1];
                    const float *sWs = s_W + seg * ZST;
#pragma unroll
                    for (int comp = 0; comp < 2; ++comp) {
                        const float *w0 = sWs + comp * G + base;
                        const float a0 = fmaf(f3[0], w0[1] - w0[0], w0[0]);
                        const float a1 = fmaf(f3[0], w0[sy + 1] - w0[sy], w0[sy]);
                        const float a2 = fmaf(f3[0], w0[sz + 1] - w0[sz], w0[sz]);
                        const float a3 = fmaf(f3[0], w0[sz + sy + 1] - w0[sz + sy], w0[sz + sy]);
                        const float b0 = fmaf(f3[1], a1 - a0, a0), b1 = fmaf(f3[1], a3 - a2, a2);
                        const float wv = fmaf(f3[2], b1 - b0, b0) + (comp ? c0y : c0x);
                        if (comp) cset(wy, c, wv); else cset(wx, c, wv);
                    }
                }
            } else {
                const V fx = vmap(x, [&](float p) { return __saturatef(fmaf(p, inv0, nlo0)); });
                const V fy = vmap(y, [&](float p) { return __saturatef(fmaf(p, inv1, nlo1)); });
                const V fz = vmap(z, [&](float p) { return __saturatef(fmaf(p, inv2, nlo2)); });
                if constexpr (SP) {
                    const float2 cx0 = sW2[0], cy0 = sW2[8];
                    wx = tripoly2(sW2, make_float2(cx0.x + c0x, cx0.y + gxb), fx, fy, fz);
                    wy = tripoly2(sW2 + 8, make_float2(cy0.x + c0y, cy0.y + gyb), fx, fy, fz);
                } else {
                    wx = tripoly(Wn, c0x, fx, fy, fz);
                    wy = tripoly(Wn + 8, c0y, fx, fy, fz);
                }
            }
            V nx, ny, nz, nv, nchi, nm;
            int vnowm = 0, lokt = ALLC;
            const V dtf = flyf * dt, dtef = flyf * dt_eta;
            if constexpr (SP) {
                // the candidate's airframe after the step (both samples): per-particle records
                const float4 rec = s_rec[t * kBlock + tid];
                nx = vfma(dtf, wx + rec.x, x);
                ny = vfma(dtf, wy + rec.y, y);
                nz = vsplat<V>(rec.z); nchi = vsplat<V>(rec.w);
                nv = nm = vsplat<V>(0.0f);                       // (flags precomputed)
                vnowm = ((vbadm >> t) & 1u) ? ALLC : 0;
                lokt = ((lokm >> t) & 1u) ? ALLC : 0;
            } else {
                // Eq. hor, coordinated-turn lift and parabolic drag (R12):
                // C_L^2 = (m g / q)^2 (1 + tan^2 phi); a landed / inactive aircraft advances with
                // dt_f = 0 (its state stays frozen, R18/R20)
                V qd = cq * v * v;
                if (sc.density_mode == 0) {
                    const V base = vmap(vfma(z, -2.2558e-5f, 1.0f), [](float a) { return fmaxf(a, 0.0f); });
                    qd = qd * vmap(vmap(base, lg2_approx) * 4.2559f, ex2_approx);
                }
                const V mgq = (m * g) * vmap(qd, rcp_approx);
                const V D = qd * vfma(vfma(tph, tph, 1.0f) * cd2, mgq * mgq, cd0);
                const V chr = chi;                                    // kept in [-pi, pi] (wrapped once per step)
                V sch, cch;
    #pragma unroll
                for (int c = 0; c < NC; ++c) {
                    float s_, c_;
                    __sincosf(cget(chr, c), &s_, &c_);
                    cset(sch, c, s_); cset(cch, c, c_);
                }
                const V vcg = v * cga;
                nx = vfma(dtf, vfma(vcg, cch, wx), x);
                ny = vfma(dtf, vfma(vcg, sch, wy), y);
                nz = vfma(dtf * v, sga, z);
                nv = vfma(dtf, vfma(T - D, vmap(m, rcp_approx), sga * (-g)), v);
                nchi = wrap_pi(vfma((dtf * g) * tph, vmap(v, rcp_approx), chi));   // heading, wrapped (R32)
                nm = vfma(-dtef, T, m);
                // envelope and mass at j = t+1 (R17)
    #pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const float zc = cget(nz, c), vc = cget(nv, c);
                    // unordered compares (a NaN fails every bound), OR-ed without short-circuit branches
                    const bool bad = (((cbad[c] >> t) & 1u) != 0u) | !(zc >= zmin) | !(zc <= zmax) | !(vc >= vmin) |
                                     !(vc <= vmax) | !(cget(nm, c) >= mempty);
                    // (x, y, chi stay finite whenever v, z, m and the controls pass: no extra test needed)
                    vnowm |= (bad ? 1 : 0) << c;
                }
            }
            const V th = fast_atan2(ny, nx);
            // descent angle on the flow-field arc (Eq. flow, R9) and landing test (R10):
            // s = rho_h |theta| / sin|theta| with sin|theta| = |y| / rho_h, i.e. s = rho_h^2 |theta| / |y|
            const V r2 = vfma(nx, nx, ny * ny);
            const V rh = r2 * vmap(r2, [](float a) { return rsqrt_approx(fmaxf(a, 1e-30f)); });
            const V at = vabs(th);
            const V sfull = (r2 * at) * vmap(ny, [](float a) { return rcp_approx(fabsf(a)); });   // unconditional:
            V sarc;                                                                             // no branch
#pragma unroll
            for (int c = 0; c < NC; ++c) cset(sarc, c, cget(at, c) > 1e-4f ? cget(sfull, c) : cget(rh, c));
            const V beta = fast_atan2_xpos(nz, sarc);              // s >= 0: right half-plane
            int lnowm = 0;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const bool ln = (cget(rh, c) <= sc.P_runway) & (cget(beta, c) <= sc.P_beta) & (cget(at, c) <= sc.P_chi) &
                                (SP || ((fabsf(cget(nchi, c)) >= sc.P_chi_west) & (cget(nv, c) <= sc.P_vs)));
                lnowm |= (ln ? 1 : 0) << c;
            }
            if constexpr (SP) lnowm &= lokt;                     // speed / heading: precomputed
            if (kind != 0) lnowm = 0;                            // only arrivals land (Eq. TO_init)
            // a landed / inactive aircraft is a NaN position: every comparison fails (as it does for a
            // violator whose state has become non-finite)
            V px;
#pragma unroll
            for (int c = 0; c < NC; ++c) cset(px, c, ((flym >> c) & 1) ? cget(nx, c) : __int_as_float(0x7fffffff));
            // own entry at seg*2W + lane and + R: partner lane + d (mod R) sits at offset d
            const int pb = seg * 2 * W + lane;
            float4 *s_pxy = s_pos;                                           // [2 kBlock]
            float2 *s_pz = reinterpret_cast<float2 *>(s_pos + 2 * kBlock);   // [2 kBlock] (NC = 2)
            if (R == W || lane < R) {
                if constexpr (NC == 2) {
                    const float4 e = make_float4(px.x, px.y, ny.x, ny.y);
                    s_pxy[pb] = e; s_pxy[pb + R] = e;
                    s_pz[pb] = nz; s_pz[pb + R] = nz;
                } else {
                    const float4 e = make_float4(px, ny, nz, 0.0f);
                    s_pxy[pb] = e; s_pxy[pb + R] = e;
                }
            }
            __syncwarp();
            // ---------------- 4. separation (Eq. avoidance), each unordered pair once:
            // lane checks partner lane+d (d = 1..R/2) and hands the verdict to that
            // partner with a segment-wide shuffle (for d = R/2, R even, both lanes check).
            // A pair conflicts iff d^2 < (2P_r)^2 and |dz| < 2P_h, i.e. iff u = d^2 - (2P_r)^2 and
            // w = |dz| - 2P_h are both negative: the verdict is the sign bit of bits(u) & bits(w)
            // (equality gives +0: separated; a NaN or infinite coordinate gives a
            // non-negative u or w: no conflict).  Candidate c's verdict sits in bit 31 - 8c of the
            // word that is OR-ed over the partners and shuffled to them.
            uint32_t confw = 0u;
#pragma unroll
            for (int d = 1; d <= R / 2; ++d) {
                V dx, dy, dz;
                if constexpr (NC == 2) {
                    const float4 q = s_pxy[pb + d];
                    dx = px - make_float2(q.x, q.y);
                    dy = ny - make_float2(q.z, q.w);
                    dz = nz - s_pz[pb + d];
                } else {
                    const float4 q = s_pxy[pb + d];
                    dx = px - q.x; dy = ny - q.y; dz = nz - q.z;
                }
                const V u = vfma(dx, dx, vfma(dy, dy, -sc.twoPr2));
                const V w = vabs(dz) - sc.twoPh;
                uint32_t hv;
                if constexpr (NC == 2)       // byte 3 of each candidate's word: bits 31 (c = 0) and 23 (c = 1)
                    hv = __byte_perm(__float_as_uint(u.x) & __float_as_uint(w.x),
                                     __float_as_uint(u.y) & __float_as_uint(w.y), 0x3700);
                else
                    hv = __float_as_uint(u) & __float_as_uint(w);
                // one shuffle hands both candidates' verdicts to the partner, from lane - d (mod R);
                // lanes >= R (R < W) compute ignored verdicts
                if (2 * d < R)
                    confw |= hv | __shfl_sync(0xffffffffu, hv, R == W ? lane + W - d : (lane >= d ? lane - d : lane - d + R), W);
                else
                    confw |= hv;
            }
            const int confm = NC == 2 ? (int)((confw >> 31) | ((confw >> 22) & 2u)) : (int)(confw >> 31);
            // ---------------- 5. per-step cost terms at j = t+1 (frozen aircraft add 0), state update
            // departure: A = |wrap(theta - theta_F)|, B = |z_tf - z|, C = |v - v_D|
            // arrival:   D = |wrap(chi - chi_hat)|, chi_hat = pi + 2 theta (R8); E = |beta - beta_f|
            const V argA = vfma(th, cA_th, vfma(nchi, cA_chi, cA_0));
            const V wA = wrap_pi(argA);
            sA = vfma(vabs(wA), flyf, sA);
            sB = vfma(vabs(vfma(nz, cB_z, vfma(beta, cB_b, cB_0))), flyf, sB);
            if constexpr (SP) {
                fuel = vfma(flyf, vsplat<V>(s_rfi[t * kBlock + tid]), fuel);
            } else {
                sC = vfma(vabs(nv - v_D), flyf, sC);
                fuel = vfma(dtef, T, fuel);
            }
            if (sc.has_noise) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const float zz = cget(nz, c) * sc.inv_Ac;
                    const float nzs = 1.0f - fmaxf(1.0f - zz * zz, 0.0f) * popdense(sc, sc.pop, cget(nx, c), cget(ny, c));
                    // "best possible cost, 1, for all remaining steps" after landing
                    cset(sN, c, cget(sN, c) + (((flym >> c) & 1) ? nzs : ((act && ((landedm >> c) & 1)) ? 1.0f : 0.0f)));
                }
            }
            violm |= flym & (vnowm | confm);
            landedm |= flym & lnowm;
            x = nx; y = ny; z = nz;
            if constexpr (!SP) { v = nv; chi = nchi; m = nm; }
            if (DEBUG && valid && isac && args.dbg_traj) {
                float *tr = args.dbg_traj + ((((size_t)lloc * args.S + s) * n + lane) * (H + 1) + t + 1) * 6;
                tr[0] = cget(x, 0); tr[1] = cget(y, 0); tr[2] = cget(z, 0);
                tr[3] = cget(v, 0); tr[4] = cget(chi, 0); tr[5] = cget(m, 0);
                if (t == 0) {
                    float *t0 = tr - 6;
                    for (int a = 0; a < 6; ++a) t0[a] = Ap->x0[a];
                }
            }
            if (DEBUG && valid && isac && args.dbg_landed && (lnowm & flym & 1))
                args.dbg_landed[((size_t)lloc * args.S + s) * n + lane] = t + 1;
        }  // t

        // ---------------- utility J_T and weight
        {
            const int Ha = Ap->Ha;
            const float invHa = Ap->invHa, invFmax = Ap->invFmax;
            const float supB = Ap->supB, invDenB = Ap->invDenB, invSupC = Ap->invSupC, invSupE = Ap->invSupE;
            const int flagB = Ap->flagB;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (SP && c == 1 && s + 1 >= s_hi) continue;         // odd sample count: no second sample
                float J = 1.0f, c0 = 1.f, c1 = 1.f, c2 = 1.f, c3 = 1.f;
                if (Ha > 0 && isac) {
                    const float Jfuel = clamp01(1.0f - cget(fuel, c) * invFmax);
                    const float J1 = clamp01(1.0f - cget(sA, c) * invHa * (1.0f / kPi));
                    if (kind == 1) {
                        c0 = J1;
                        c1 = Jfuel;
                        c2 = flagB ? 1.0f : clamp01((supB - cget(sB, c) * invHa) * invDenB);
                        c3 = clamp01(1.0f - (SP ? sCc : cget(sC, c)) * invHa * invSupC);
                        J = sc.alpha_dep[0] * c0 + sc.alpha_dep[1] * c1 + sc.alpha_dep[2] * c2 + sc.alpha_dep[3] * c3;
                    } else {
                        c0 = J1;
                        c1 = clamp01(1.0f - cget(sB, c) * invHa * invSupE);
                        c2 = Jfuel;
                        c3 = 0.0f;
                        J = sc.alpha_arr[0] * c0 + sc.alpha_arr[1] * c1 + sc.alpha_arr[2] * c2;
                    }
                    if (sc.has_noise) J = (1.0f - sc.noise_w) * J + sc.noise_w * cget(sN, c) * invHa;
                }
                ell[c] = (((violm >> c) & 1) || !(J > 0.0f)) ? -INFINITY : ell[c] + __log2f(J);
                if (DEBUG && c == 0 && valid && isac) {
                    const size_t o = ((size_t)lloc * args.S + s) * n + lane;
                    if (args.dbg_J) args.dbg_J[o] = J;
                    if (args.dbg_viol) args.dbg_viol[o] = (violm >> c) & 1;
                    if (args.dbg_fuel) args.dbg_fuel[o] = cget(fuel, c);
                    if (args.dbg_comp) { float *cp = args.dbg_comp + 4 * o; cp[0] = c0; cp[1] = c1; cp[2] = c2; cp[3] = c3; }
                }
            }
        }
    }  // s

    constexpr int ENC = SP ? 1 : NC;               // candidates in the epilogue
    if constexpr (SP) ell[0] = ell[0] + ell[1];    // both slots' samples of the single candidate
    // ---------------- epilogue: lambda (double, ascending i), MH (R1), survivor
    __syncthreads();
    float *s_ell = reinterpret_cast<float *>(s_pos);          // reuse [NC][kBlock]
    int *s_dec = reinterpret_cast<int *>(s_V);                 // [SEGS]
#pragma unroll
    for (int c = 0; c < ENC; ++c) s_ell[c * kBlock + tid] = ell[c];
    __syncwarp();
    double lam[ENC];
#pragma unroll
    for (int c = 0; c < ENC; ++c) {
        lam[c] = 0.0;
        for (int i = 0; i < n; ++i) lam[c] += (double)s_ell[c * kBlock + seg * W + i];
    }
    // survivor mask: bit i set = aircraft i keeps the proposal x* (joint MH: all bits alike)
    uint32_t mask = args.surv_single;
    int nacc = 0;
    float ell_s = ell[0];
    double lam_s = lam[0];
    if constexpr (ENC == 2) {
        if (args.mh_mode == 2) {
            // per-aircraft MH (R46): every lane decides for its own aircraft
            const bool ai = isac && mh_decide_aircraft((double)ell[0], (double)ell[ENC - 1], l, (uint32_t)lane, k, mpc,
                                                       sc.key0, sc.key1);
            const unsigned b = __ballot_sync(0xffffffffu, ai);
            mask = (W == 32) ? b : ((b >> ((tid & 31) & ~(W - 1))) & ((1u << (W & 31)) - 1u));
            ell_s = ai ? ell[ENC - 1] : ell[0];
            lam_s = 0.0;
            for (int i = 0; i < n; ++i) lam_s += (double)s_ell[(((mask >> i) & 1u) ? ENC - 1 : 0) * kBlock + seg * W + i];
            nacc = __popc(mask);
        } else {
            const bool acc = mh_decide(lam[0], lam[1], l, k, mpc, sc.key0, sc.key1);
            mask = acc ? 0xFFFFFFFFu : 0u;
            ell_s = acc ? ell[ENC - 1] : ell[0];
            lam_s = acc ? lam[ENC - 1] : lam[0];
            nacc = acc ? 1 : 0;
        }
    }
    if (valid && isac) args.ell_out[(size_t)lane * args.L + lloc] = ell_s;
    if (valid && lane == 0) {
        args.lam_out[lloc] = lam_s;
        args.surv_out[lloc] = mask;
        if (args.lam_cand) {
            args.lam_cand[lloc] = lam[0];
            args.lam_cand[args.L + lloc] = lam[ENC - 1];
        }
        if (DEBUG && args.dbg_ell_c) {
            for (int c = 0; c < ENC; ++c)
                for (int i = 0; i < n; ++i)
                    args.dbg_ell_c[((size_t)c * args.L + lloc) * n + i] = s_ell[c * kBlock + seg * W + i];
        }
    }
    if (lane == 0) s_dec[seg] = (valid && ENC == 2) ? nacc : 0;
    // per-column max of the survivor log-weights (K3, first half)
    __syncthreads();
    uint32_t *s_cm = reinterpret_cast<uint32_t *>(s_ctrl);
    s_cm[tid] = (valid && isac) ? f2ord(ell_s) : 0u;
    __syncthreads();
    if (tid < n) {
        uint32_t mx = 0u;
        for (int sg = 0; sg < SEGS; ++sg) mx = max(mx, s_cm[sg * W + tid]);
        if (mx) atomicMax(&args.colmax[tid], mx);
    }
    if (ENC == 2 && tid == 0) {
        unsigned long long cnt = 0;
        for (int sg = 0; sg < SEGS; ++sg) cnt += s_dec[sg];
        if (cnt) atomicAdd(args.n_accept, cnt);
    }
}

// ============================================================== K2, two sample chains per lane
// NC = 2 launches (both MH candidates) on the 2x2x2 grid with W >= 8: every lane carries samples s
// and s + 1 of its aircraft as two independent chains, each a float2 over the candidates, so a
// warp has two independent dependency chains in flight (the scheduler can issue from one while
// the other waits on a fixed-latency result) at the same arithmetic per aircraft-step.  Shared by
// both chains: the staged controls (one pair of LDS.128 per step), the per-lane constants, one
// separation exchange (three LDS.128 per partner for four (sample, candidate) positions instead
// of two per two) and one verdict shuffle per partner (four verdict bytes).  The two samples'
// wind fields are drawn like the sample-pair instances' (two slots per segment).  Results are
// identical to k_rollout<W, 2>: the same operations in the same order per (sample, candidate).
#ifndef SMC_K2_MINB2S
#define SMC_K2_MINB2S 4     // 128 registers: no spill once the airframe left the sample loop (c2 -5.6 %, c4 -4.3 %)
#endif
#ifndef SMC_K2_SP4
#define SMC_K2_SP4 1
#endif
#ifndef SMC_K2_MINB2SP4
#define SMC_K2_MINB2SP4 3   // single-candidate four-sample instances (four wind slots)
#endif
#ifndef SMC_K2_MINB2S32
#define SMC_K2_MINB2S32 3   // 32-lane segments (25-32 aircraft): more live state per lane
#endif

#ifndef SMC_K2_2S_MINW
#define SMC_K2_2S_MINW 8    // narrowest segment launched with two sample chains (W = 8: c2 K2 24.95 -> 21.06 ms)
#endif
#ifndef SMC_K2_TUNROLL2S
#define SMC_K2_TUNROLL2S 1
#endif
#ifndef SMC_K2_POP_SMEM
#define SMC_K2_POP_SMEM 0   // 1: stage the noise grid in shared memory (c4: 27 KB per block -> 2 blocks/SM)
#endif
// the 1 km population grid is staged in shared memory when it fits (c4: 81 x 81, 26 KB)
constexpr int kPopSmem = 8192;
__host__ __device__ inline int pop_smem_floats(int nx, int ny) { return nx * ny <= kPopSmem ? nx * ny : 0; }

// Segments of W lanes that do not divide a warp (W = 12, 20, 24, ...) are packed contiguously over
// the block and cross warp boundaries: their exchanges synchronise the block and the verdict
// hand-back goes through shared memory.  The block's last kBlock mod W threads form a phantom
// segment (own scratch, no particle).
__host__ __device__ constexpr bool k2_cross_warp(int W) { return (32 % W) != 0; }
__host__ __device__ constexpr int k2_segs_alloc(int W) { return kBlock / W + (k2_cross_warp(W) && kBlock % W ? 1 : 0); }

size_t rollout2s_smem_bytes(int W, int H, int npop, int nsl) {
    const int SEGA = k2_segs_alloc(W), GB = W / 4;
    const size_t pos = (size_t)2 * SEGA * W;                      // entries per position array
    return sizeof(float) * (size_t)npop + sizeof(float) * ((size_t)H * 10 * kBlock)   // airframe records
           + sizeof(float) * (SEGA * nsl * GB * 16                // normals [SEGA][slot][GB][16]
                              + SEGA * nsl * 16                   // AR(1) state [SEGA][slot][8] (x, y)
                              + SEGA * nsl * 16)                  // coefficients [SEGA][slot][16]
           + sizeof(float4) * 2 * pos + sizeof(float2) * pos      // positions x4, y4, z2, each twice
           + (k2_cross_warp(W) ? sizeof(uint32_t) * (size_t)(W / 2) * SEGA * W : 0)   // verdicts
           + sizeof(float) * 72 + 16;
}

// SP4: a single-candidate round (round 0, the paper-literal Alg. 1): the two float2 components of a
// chain are two more samples of the one candidate (4 samples per lane and pass, 4 wind slots).
template <int W, int R, bool SP4 = false>
__global__ void __launch_bounds__(kBlock, W >= 32 ? SMC_K2_MINB2S32 : (SP4 ? SMC_K2_MINB2SP4 : SMC_K2_MINB2S)) k_rollout_2s(const DevScen sc, const RolloutArgs args) {
    static_assert(W >= 8 && W % 4 == 0, "two-chain instances need W >= 8 (eight AR(1) nodes per slot), W = 4 GB");
    constexpr bool XW = k2_cross_warp(W);
    static_assert(!XW || R == W, "packed segments use the whole segment as the separation ring");
    constexpr int NSL = SP4 ? 4 : 2, SEGS = kBlock / W, SEGA = k2_segs_alloc(W), GB = W / 4;
    constexpr int NP = 8 * NSL;                                   // (node, slot) pairs of a segment
    constexpr int ENS = W >= NP ? 1 : (NP + W - 1) / W;           // pairs a lane owns
    constexpr int TU2 = SMC_K2_TUNROLL2S;
    // exchange barrier of a segment: its warp, or the block when segments cross warps
    auto seg_sync = [] { if constexpr (XW) __syncthreads(); else __syncwarp(); };
    extern __shared__ __align__(16) float smem_all[];
    const int H = sc.H, n = sc.n;
    const int npop = (SMC_K2_POP_SMEM && sc.has_noise) ? pop_smem_floats(sc.pop_nx + 1, sc.pop_ny + 1) : 0;
    float *smem = smem_all + ((npop + 3) & ~3);
    for (int e = threadIdx.x; e < npop; e += kBlock) smem_all[e] = __ldg(&sc.popp[e]);   // staged when it fits
    constexpr int NPOS = 2 * SEGA * W;                           // entries per position array
    float *s_V = smem + (size_t)H * 10 * kBlock;                 // after the airframe records (below)
    float *s_Z = s_V + SEGA * NSL * GB * 16;
    float *s_W = s_Z + SEGA * NSL * 16;
    float4 *s_p4 = reinterpret_cast<float4 *>(s_W + SEGA * NSL * 16);   // [2][NPOS] x4, y4; [NPOS] z2
    uint32_t *s_hv = reinterpret_cast<uint32_t *>(s_p4 + 2 * NPOS + NPOS / 2);   // [W/2][SEGA W] verdicts (XW)
    float *s_Q = reinterpret_cast<float *>(s_hv + (XW ? (W / 2) * SEGA * W : 0));

    const int tid = threadIdx.x, lane = tid % W, seg = tid / W;
    const uint32_t lloc = blockIdx.x * SEGS + seg;
    const bool valid = seg < SEGS && lloc < args.L;
    const uint32_t l = args.l0 + lloc;
    const bool isac = lane < n;
    const uint32_t k = args.k, mpc = *args.mpcp;
    if (tid < 64) s_Q[(tid >> 3) * 9 + (tid & 7)] = sc.Cq[tid];

    const DevAircraft *Ap = sc.ac + (isac ? lane : 0);
    const int kind = Ap->kind;
    const int first = isac ? Ap->first_step : (1 << 20);
    const float halfS = Ap->halfS, cd0 = Ap->cd0, cd2 = Ap->cd2, dt_eta = Ap->dt_eta;
    const float zmin = Ap->z_min, zmax = Ap->z_max, vmin = Ap->v_min, vmax = Ap->v_max, mempty = Ap->m_empty;
    const float gA = kind ? Ap->theta_F : Ap->beta_f;
    const float z_tf = Ap->z_tf, v_D = Ap->v_D;

    // ---------------- airframe trajectory (Eq. hor), once per particle.  z, v, chi and m
    // do not depend on the wind -- it enters only dx/dt and dy/dt -- so for both candidates they are
    // integrated here and every sample reads them; samples differ only in the ground track and what
    // depends on it.  Per step t: the air-relative ground velocity (v cos g cos chi, v cos g sin chi)
    // at t, z and chi at t+1, the fuel increment; the envelope (with the control bounds) and the
    // landing sector's speed / heading conditions at t+1 as bit masks (bit 2t + c).  A trajectory
    // that becomes non-finite (v reached 0: already outside the envelope, so every sample flying it
    // is violated) is replaced by a far-away finite sentinel: it fails the envelope and can no longer
    // conflict (the oracle's non-finite rule), and a sample in which the aircraft has landed before
    // keeps finite cost terms.
    float4 *const s_r0 = reinterpret_cast<float4 *>(smem);                // [H][kBlock] (ax0, ax1, ay0, ay1)
    float4 *const s_r1 = s_r0 + H * kBlock;                                 // [H][kBlock] (z'0, z'1, chi'0, chi'1)
    float2 *const s_rf = reinterpret_cast<float2 *>(s_r1 + H * kBlock);     // [H][kBlock] fuel increments
    using V = float2;
    const float dt = sc.dt, g = sc.g;
    uint32_t vbadm = 0u, lokm = 0u;
    V sCc = make_float2(0.0f, 0.0f);           // departures (never land): sum of |v - v_D| over active steps
    {
        const float gmax = Ap->gamma_max, pmax = Ap->phi_max, Tmin = Ap->T_min, Tmax = Ap->T_max;
        const float cq = (sc.density_mode == 0 ? 1.225f : sc.rho_const) * halfS;
        const float *src[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) src[c] = args.ctrl[SP4 ? 0 : c] + ((size_t)lloc * n + lane) * H * 3;
        V v = vsplat<V>(Ap->x0[3]), z = vsplat<V>(Ap->x0[2]), chi = vsplat<V>(Ap->x0[4]), m = vsplat<V>(Ap->x0[5]);
        int broken = 0;
        for (int t = 0; t < H; ++t) {
            V T, tph, sga, cga;
            int cb = 0;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                float Tc = 0.f, ph = 0.f, ga = 0.f;
                if (isac && valid) { Tc = src[c][3 * t]; ph = src[c][3 * t + 1]; ga = src[c][3 * t + 2]; }
                float sph, cph, sg, cg;
                __sincosf(ph, &sph, &cph);
                __sincosf(ga, &sg, &cg);
                cset(T, c, Tc); cset(tph, c, sph * rcp_approx(cph)); cset(sga, c, sg); cset(cga, c, cg);
                const bool bad = (fabsf(ga) > gmax) || !(fabsf(ph) < pmax) || (Tc < Tmin) || (Tc > Tmax);
                cb |= (bad ? 1 : 0) << c;
            }
            const bool act = first <= t;
            const float dta = act ? dt : 0.0f, dtea = act ? dt_eta : 0.0f;
            V qd = cq * v * v;
            if (sc.density_mode == 0) {
                const V base = vmap(vfma(z, -2.2558e-5f, 1.0f), [](float a) { return fmaxf(a, 0.0f); });
                qd = qd * vmap(vmap(base, lg2_approx) * 4.2559f, ex2_approx);
            }
            const V mgq = (m * g) * vmap(qd, rcp_approx);
            const V D = qd * vfma(vfma(tph, tph, 1.0f) * cd2, mgq * mgq, cd0);
            V sch, cch;
            __sincosf(chi.x, &sch.x, &cch.x);
            __sincosf(chi.y, &sch.y, &cch.y);
            const V vcg = v * cga;
            V ax = vcg * cch, ay = vcg * sch;
            V nz = vfma(dta * v, sga, z);
            const V nv = vfma(vsplat<V>(dta), vfma(T - D, vmap(m, rcp_approx), sga * (-g)), v);
            V nchi = wrap_pi(vfma((dta * g) * tph, vmap(v, rcp_approx), chi));
            const V nm = vfma(vsplat<V>(-dtea), T, m);
            V fi = T * dtea;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const bool fin = (fabsf(cget(ax, c)) < INFINITY) & (fabsf(cget(ay, c)) < INFINITY) &
                                 (fabsf(cget(nz, c)) < INFINITY) & (fabsf(cget(nv, c)) < INFINITY) &
                                 (fabsf(cget(nchi, c)) < INFINITY) & (fabsf(cget(nm, c)) < INFINITY);
                if (!fin) broken |= 1 << c;
                int bad, lok;
                if ((broken >> c) & 1) {
                    cset(ax, c, 1e30f); cset(ay, c, 1e30f); cset(nz, c, 1e30f); cset(nchi, c, 0.0f); cset(fi, c, 0.0f);
                    bad = 1; lok = 0;
                } else {
                    const float zc = cget(nz, c), vc = cget(nv, c);
                    bad = (((cb >> c) & 1) | !(zc >= zmin) | !(zc <= zmax) | !(vc >= vmin) | !(vc <= vmax) |
                           !(cget(nm, c) >= mempty)) ? 1 : 0;
                    lok = ((vc <= sc.P_vs) & (fabsf(cget(nchi, c)) >= sc.P_chi_west)) ? 1 : 0;
                    if (act) cset(sCc, c, cget(sCc, c) + fabsf(vc - v_D));
                }
                vbadm |= (uint32_t)bad << (2 * t + c);
                lokm |= (uint32_t)lok << (2 * t + c);
            }
            s_r0[t * kBlock + tid] = make_float4(ax.x, ax.y, ay.x, ay.y);
            s_r1[t * kBlock + tid] = make_float4(nz.x, nz.y, nchi.x, nchi.y);
            s_rf[t * kBlock + tid] = fi;
            v = nv; z = nz; chi = nchi; m = nm;
        }
    }
    __syncthreads();
    float qrow[8];
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) qrow[mm] = s_Q[(lane & 7) * 9 + mm];

    float ell[2] = {args.ell0, args.ell0};
    const float inv0 = sc.wind_inv_ext[0], inv1 = sc.wind_inv_ext[1], inv2 = sc.wind_inv_ext[2];
    const float nlo0 = -sc.wind_lo[0] * inv0, nlo1 = -sc.wind_lo[1] * inv1, nlo2 = -sc.wind_lo[2] * inv2;
    const float cA_th = kind ? 1.0f : -2.0f, cA_chi = kind ? 0.0f : 1.0f, cA_0 = kind ? -gA : -kPi;
    const float cB_z = kind ? -1.0f : 0.0f, cB_b = kind ? 0.0f : 1.0f, cB_0 = kind ? z_tf : -gA;
    const int pb = seg * 2 * W + lane;                             // own entry; + R: duplicate
    float4 *const s_px = s_p4, *const s_py = s_p4 + NPOS;
    float2 *const s_pz = reinterpret_cast<float2 *>(s_p4 + 2 * NPOS);   // z: shared by the two samples
    const uint32_t S = args.S;

    for (uint32_t s = 0; s < S; s += NSL) {
        const bool two = s + 1 < S;                                // odd S: the second chain is not counted
        V x[2], y[2], fuel[2], sA[2], sB[2], sN[2];
        V z = vsplat<V>(Ap->x0[2]);                                // the airframe altitude (both samples)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            x[q] = vsplat<V>(Ap->x0[0]); y[q] = vsplat<V>(Ap->x0[1]);
            fuel[q] = sA[q] = sB[q] = sN[q] = vsplat<V>(0.0f);
        }
        int landedm[2] = {0, 0}, violm[2] = {0, 0};
        float2 Zr[ENS];
        float2 gust_odd[NSL];
        uint32_t x1[NSL];                                          // slot sl: sample s + sl (SP4: chain sl / 2, component sl % 2)
        if constexpr (SP4) {
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl) {
                gust_odd[sl] = make_float2(0.f, 0.f);
                x1[sl] = ((s + sl) & 0xFFFFu) | (k << 16);
            }
        } else {
            gust_odd[0] = gust_odd[1] = make_float2(0.f, 0.f);
            x1[0] = (s & 0xFFFFu) | (k << 16);
            x1[1] = ((s + 1) & 0xFFFFu) | (k << 16);
        }

#pragma unroll TU2
        for (int t = 0; t < H; ++t) {
            // ---------------- 1. both samples' wind fields for step t (Alg.1 l.10)
            const int tb = t % GB;
            if (tb == 0) {
#pragma unroll
                for (int task0 = 0; task0 < 4 * GB * NSL; task0 += W) {
                    const int task = task0 + lane, sl = task / (4 * GB), tk = task - sl * 4 * GB;
                    const int b = tk & 3, ts = t + (tk >> 2);
                    if (ts < H) {
                        const uint4 w = draw_ks(TAG_WIND, l, x1[sl], (uint32_t)ts | ((uint32_t)b << 16), mpc, sc.ks);
                        *reinterpret_cast<float4 *>(&s_V[((seg * NSL + sl) * GB + (tk >> 2)) * 16 + 4 * b]) = box_muller4(w);
                    }
                }
            }
            seg_sync();
            float2 *const sZ2 = reinterpret_cast<float2 *>(s_Z + seg * 16 * NSL);
            // (node, slot) pair pq of the NP a segment advances: W >= NP: pair lane mod NP (duplicates
            // store identical values); else pairs lane + e W < NP
            constexpr bool QREG = (W % 8) == 0;                 // node = lane mod 8 for every pair
#pragma unroll
            for (int e = 0; e < ENS; ++e) {
                const int pq = W >= NP ? (lane & (NP - 1)) : lane + e * W, node = pq & 7, sl = pq >> 3;
                if (W >= NP || pq < NP) {
                    const float *vv = &s_V[((seg * NSL + sl) * GB + tb) * 16];
                    const float2 ve = make_float2(vv[node], vv[8 + node]);
                    Zr[e] = (t == 0) ? ve : vfma(Zr[e], sc.a, ve * sc.b);
                    sZ2[sl * 8 + node] = Zr[e];
                }
            }
            seg_sync();
#pragma unroll
            for (int e = 0; e < ENS; ++e) {
                const int pq = W >= NP ? (lane & (NP - 1)) : lane + e * W, node = pq & 7, sl = pq >> 3;
                if (W >= NP || pq < NP) {
                    const float4 *z4 = reinterpret_cast<const float4 *>(sZ2 + sl * 8);
                    const float *qr = QREG ? qrow : &s_Q[node * 9];
                    float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float4 zz = z4[mm];
                        acc = vfma(make_float2(zz.x, zz.y), qr[2 * mm], acc);
                        acc = vfma(make_float2(zz.z, zz.w), qr[2 * mm + 1], acc);
                    }
                    if constexpr (SP4) {                         // [seg][chain][k](component): float2 pairs
                        s_W[((seg * 2 + (sl >> 1)) * 16 + node) * 2 + (sl & 1)] = acc.x;
                        s_W[((seg * 2 + (sl >> 1)) * 16 + 8 + node) * 2 + (sl & 1)] = acc.y;
                    } else {
                        s_W[(seg * NSL + sl) * 16 + node] = acc.x;
                        s_W[(seg * NSL + sl) * 16 + 8 + node] = acc.y;
                    }
                }
            }
            seg_sync();
            // gusts (R15): one Philox call per sample covers steps 2u and 2u+1; slot sl's gust goes to
            // chain sl (both candidates) or, SP4, to chain sl / 2, component sl % 2
            using GT = std::conditional_t<SP4, V, float>;
            GT gxq[2], gyq[2];
            if constexpr (SP4) {
#pragma unroll
                for (int q = 0; q < 2; ++q) { gxq[q] = vsplat<GT>(sc.nominal[0]); gyq[q] = vsplat<GT>(sc.nominal[1]); }
                if (sc.turb_sigma > 0.0f) {
#pragma unroll
                    for (int sl = 0; sl < NSL; ++sl) {
                        float2 gg;
                        if ((t & 1) == 0) {
                            const uint4 w = draw_ks(TAG_TURB, l, x1[sl], ((uint32_t)t >> 1) | ((uint32_t)lane << 8), mpc, sc.ks);
                            const float4 g4 = box_muller4(w);
                            gg = make_float2(g4.x, g4.y);
                            gust_odd[sl] = make_float2(g4.z, g4.w);
                        } else {
                            gg = gust_odd[sl];
                        }
                        cset(gxq[sl >> 1], sl & 1, fmaf(sc.turb_sigma, gg.x, sc.nominal[0]));
                        cset(gyq[sl >> 1], sl & 1, fmaf(sc.turb_sigma, gg.y, sc.nominal[1]));
                    }
                }
            } else {
                gxq[0] = gxq[1] = sc.nominal[0];
                gyq[0] = gyq[1] = sc.nominal[1];
                if (sc.turb_sigma > 0.0f) {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        float2 gg;
                        if ((t & 1) == 0) {
                            const uint4 w = draw_ks(TAG_TURB, l, x1[q], ((uint32_t)t >> 1) | ((uint32_t)lane << 8), mpc, sc.ks);
                            const float4 g4 = box_muller4(w);
                            gg = make_float2(g4.x, g4.y);
                            gust_odd[q] = make_float2(g4.z, g4.w);
                        } else {
                            gg = gust_odd[q];
                        }
                        gxq[q] = fmaf(sc.turb_sigma, gg.x, gxq[q]);
                        gyq[q] = fmaf(sc.turb_sigma, gg.y, gyq[q]);
                    }
                }
            }
            // airframe state of step t (shared by both chains: wind-independent)
            const float4 r0 = s_r0[t * kBlock + tid], r1 = s_r1[t * kBlock + tid];
            const V fi = s_rf[t * kBlock + tid];
            const V ax = make_float2(r0.x, r0.y), ay = make_float2(r0.z, r0.w);
            const V nz = make_float2(r1.x, r1.y), nchi = make_float2(r1.z, r1.w);
            const bool act = first <= t;
            const int vbt = (int)((vbadm >> (2 * t)) & 3u), lkt = (int)((lokm >> (2 * t)) & 3u);
            const V fz = vmap(z, [&](float p) { return __saturatef(fmaf(p, inv2, nlo2)); });

            // ---------------- 2-3. per chain: ground track, geometry, landing test
            V nx[2], ny[2], th[2], beta[2], px[2], flyf[2];
            int flym[2], lnowm[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                flym[q] = act ? (~landedm[q] & 3) : 0;
                flyf[q] = make_float2((flym[q] & 1) ? 1.0f : 0.0f, (flym[q] & 2) ? 1.0f : 0.0f);
                const V fx = vmap(x[q], [&](float p) { return __saturatef(fmaf(p, inv0, nlo0)); });
                const V fy = vmap(y[q], [&](float p) { return __saturatef(fmaf(p, inv1, nlo1)); });
                V wx, wy;
                if constexpr (SP4) {                               // per-component coefficients
                    const float2 *c2 = reinterpret_cast<const float2 *>(&s_W[(seg * 2 + q) * 32]);
                    wx = tripoly2(c2, c2[0] + gxq[q], fx, fy, fz);
                    wy = tripoly2(c2 + 8, c2[8] + gyq[q], fx, fy, fz);
                } else {
                    const float4 *w4 = reinterpret_cast<const float4 *>(&s_W[(seg * NSL + q) * 16]);
                    float Wn[16];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float4 a4 = w4[e];
                        Wn[4 * e] = a4.x; Wn[4 * e + 1] = a4.y; Wn[4 * e + 2] = a4.z; Wn[4 * e + 3] = a4.w;
                    }
                    wx = tripoly(Wn, Wn[0] + gxq[q], fx, fy, fz);
                    wy = tripoly(Wn + 8, Wn[8] + gyq[q], fx, fy, fz);
                }
                const V dtf = flyf[q] * dt;
                nx[q] = vfma(dtf, ax + wx, x[q]);
                ny[q] = vfma(dtf, ay + wy, y[q]);
                th[q] = fast_atan2(ny[q], nx[q]);
                const V r2 = vfma(nx[q], nx[q], ny[q] * ny[q]);
                const V rh = r2 * vmap(r2, [](float a) { return rsqrt_approx(fmaxf(a, 1e-30f)); });
                const V at = vabs(th[q]);
                const V sfull = (r2 * at) * vmap(ny[q], [](float a) { return rcp_approx(fabsf(a)); });
                V sarc;
#pragma unroll
                for (int c = 0; c < 2; ++c) cset(sarc, c, cget(at, c) > 1e-4f ? cget(sfull, c) : cget(rh, c));
                beta[q] = fast_atan2_xpos(nz, sarc);
                lnowm[q] = 0;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const bool ln = (cget(rh, c) <= sc.P_runway) & (cget(beta[q], c) <= sc.P_beta) &
                                    (cget(at, c) <= sc.P_chi);
                    lnowm[q] |= (ln ? 1 : 0) << c;
                }
                lnowm[q] &= kind == 0 ? lkt : 0;                  // speed / heading conditions: precomputed
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    cset(px[q], c, ((flym[q] >> c) & 1) ? cget(nx[q], c) : __int_as_float(0x7fffffff));
            }
            // ---------------- 4. separation (Eq. avoidance): one exchange for both chains
            if (R == W || lane < R) {
                const float4 ex = make_float4(px[0].x, px[0].y, px[1].x, px[1].y);
                const float4 ey = make_float4(ny[0].x, ny[0].y, ny[1].x, ny[1].y);
                s_px[pb] = ex; s_px[pb + R] = ex;
                s_py[pb] = ey; s_py[pb + R] = ey;
                s_pz[pb] = nz; s_pz[pb + R] = nz;
            }
            seg_sync();
            // verdict bytes: bit 31 (sample s, candidate 0), 23 (s, 1), 15 (s + 1, 0), 7 (s + 1, 1)
            uint32_t confw = 0u;
#pragma unroll
            for (int d = 1; d <= R / 2; ++d) {
                const float4 qx = s_px[pb + d], qy = s_py[pb + d];
                const float2 qz = s_pz[pb + d];
                const V dx0 = px[0] - make_float2(qx.x, qx.y), dx1 = px[1] - make_float2(qx.z, qx.w);
                const V dy0 = ny[0] - make_float2(qy.x, qy.y), dy1 = ny[1] - make_float2(qy.z, qy.w);
                const V w = vabs(nz - qz) - sc.twoPh;
                const V u0 = vfma(dx0, dx0, vfma(dy0, dy0, -sc.twoPr2)), u1 = vfma(dx1, dx1, vfma(dy1, dy1, -sc.twoPr2));
                // sign bytes first, then one AND: w (per candidate) is shared by the two chains
                const uint32_t pu = __byte_perm(__byte_perm(__float_as_uint(u0.x), __float_as_uint(u0.y), 0x3737),
                                                __byte_perm(__float_as_uint(u1.x), __float_as_uint(u1.y), 0x3737), 0x3254);
                const uint32_t hv = pu & __byte_perm(__float_as_uint(w.x), __float_as_uint(w.y), 0x3737);
                if constexpr (XW) {
                    // partner lane + d learns this verdict from shared memory after the scan
                    if (2 * d < R) s_hv[(d - 1) * (SEGA * W) + seg * W + lane] = hv;
                    confw |= hv;
                } else if (2 * d < R) {
                    confw |= hv | __shfl_sync(0xffffffffu, hv, R == W ? lane + W - d : (lane >= d ? lane - d : lane - d + R), W);
                } else {
                    confw |= hv;
                }
            }
            if constexpr (XW) {
                seg_sync();
#pragma unroll
                for (int d = 1; 2 * d < R; ++d)
                    confw |= s_hv[(d - 1) * (SEGA * W) + seg * W + (lane >= d ? lane - d : lane - d + R)];
            }
            const int confm[2] = {(int)((confw >> 31) | ((confw >> 22) & 2u)), (int)(((confw >> 15) & 1u) | ((confw >> 6) & 2u))};
            // ---------------- 5. per chain: cost terms, flags, state update
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const V argA = vfma(th[q], cA_th, vfma(nchi, cA_chi, cA_0));
                const V wA = wrap_pi(argA);
                sA[q] = vfma(vabs(wA), flyf[q], sA[q]);
                sB[q] = vfma(vabs(vfma(nz, cB_z, vfma(beta[q], cB_b, cB_0))), flyf[q], sB[q]);
                fuel[q] = vfma(flyf[q], fi, fuel[q]);
                if (sc.has_noise) {
#if SMC_K2_POP_SMEM
                    const V pd = popdense_pad(sc, smem_all, nx[q], ny[q]);   // staged (launch_rollout checks it fits)
#else
                    const V pd = popdense_pad<V, true>(sc, sc.popp, nx[q], ny[q]);   // L1-resident, read-only path
#endif
                    const V zz = nz * sc.inv_Ac;
                    V f;
#pragma unroll
                    for (int c = 0; c < 2; ++c) cset(f, c, __saturatef(fmaf(-cget(zz, c), cget(zz, c), 1.0f)));   // max(1 - zz^2, 0)
                    const V nzs = vfma(f, -pd, 1.0f);
#pragma unroll
                    for (int c = 0; c < 2; ++c)
                        cset(sN[q], c, cget(sN[q], c) + (((flym[q] >> c) & 1) ? cget(nzs, c)
                                                                               : ((act && ((landedm[q] >> c) & 1)) ? 1.0f : 0.0f)));
                }
                violm[q] |= flym[q] & (vbt | confm[q]);
                landedm[q] |= flym[q] & lnowm[q];
                x[q] = nx[q]; y[q] = ny[q];
            }
            z = nz;
        }  // t

        // ---------------- utility J_T and weight, both chains
        {
            const int Ha = Ap->Ha;
            const float invHa = Ap->invHa, invFmax = Ap->invFmax;
            const float supB = Ap->supB, invDenB = Ap->invDenB, invSupC = Ap->invSupC, invSupE = Ap->invSupE;
            const int flagB = Ap->flagB;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (!SP4 && q == 1 && !two) continue;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (SP4 && s + 2 * q + c >= S) continue;          // sample count not a multiple of 4
                    float J = 1.0f;
                    if (Ha > 0 && isac) {
                        const float Jfuel = clamp01(1.0f - cget(fuel[q], c) * invFmax);
                        const float J1 = clamp01(1.0f - cget(sA[q], c) * invHa * (1.0f / kPi));
                        if (kind == 1) {
                            const float c2 = flagB ? 1.0f : clamp01((supB - cget(sB[q], c) * invHa) * invDenB);
                            const float c3 = clamp01(1.0f - cget(sCc, c) * invHa * invSupC);
                            J = sc.alpha_dep[0] * J1 + sc.alpha_dep[1] * Jfuel + sc.alpha_dep[2] * c2 + sc.alpha_dep[3] * c3;
                        } else {
                            const float c1 = clamp01(1.0f - cget(sB[q], c) * invHa * invSupE);
                            J = sc.alpha_arr[0] * J1 + sc.alpha_arr[1] * c1 + sc.alpha_arr[2] * Jfuel;
                        }
                        if (sc.has_noise) J = (1.0f - sc.noise_w) * J + sc.noise_w * cget(sN[q], c) * invHa;
                    }
                    float &e = ell[SP4 ? 0 : c];                      // SP4: every sample adds to the one candidate
                    e = (((violm[q] >> c) & 1) || !(J > 0.0f)) ? -INFINITY : e + __log2f(J);
                }
            }
        }
    }  // s

    // ---------------- epilogue: lambda (double, ascending i), MH (R1, R46), survivor
    __syncthreads();
    float *s_ell = reinterpret_cast<float *>(s_p4);
    int *s_dec = reinterpret_cast<int *>(s_V);
    if constexpr (SP4) ell[1] = ell[0];                         // one candidate
    s_ell[tid] = ell[0];
    s_ell[kBlock + tid] = ell[1];
    seg_sync();
    double lam[2] = {0.0, 0.0};
    for (int i = 0; i < n; ++i) {
        lam[0] += (double)s_ell[seg * W + i];
        lam[1] += (double)s_ell[kBlock + seg * W + i];
    }
    uint32_t mask;
    int nacc;
    float ell_s;
    double lam_s;
    if (SP4) {                                                  // no MH: the caller's survivor mask
        mask = args.surv_single;
        ell_s = ell[0];
        lam_s = lam[0];
        nacc = 0;
    } else if (args.mh_mode == 2) {
        const bool ai = isac && mh_decide_aircraft((double)ell[0], (double)ell[1], l, (uint32_t)lane, k, mpc, sc.key0,
                                                   sc.key1);
        if constexpr (XW) {                                       // segments cross warps: via shared memory
            uint32_t *s_ai = reinterpret_cast<uint32_t *>(s_ell + 2 * kBlock);
            s_ai[tid] = ai ? 1u : 0u;
            __syncthreads();
            mask = 0u;
            for (int i = 0; i < n; ++i) mask |= s_ai[seg * W + i] << i;
        } else {
            const unsigned b = __ballot_sync(0xffffffffu, ai);
            mask = (W == 32) ? b : ((b >> ((tid & 31) & ~(W - 1))) & ((1u << (W & 31)) - 1u));
        }
        ell_s = ai ? ell[1] : ell[0];
        lam_s = 0.0;
        for (int i = 0; i < n; ++i) lam_s += (double)s_ell[(((mask >> i) & 1u) ? kBlock : 0) + seg * W + i];
        nacc = __popc(mask);
    } else {
        const bool acc = mh_decide(lam[0], lam[1], l, k, mpc, sc.key0, sc.key1);
        mask = acc ? 0xFFFFFFFFu : 0u;
        ell_s = acc ? ell[1] : ell[0];
        lam_s = acc ? lam[1] : lam[0];
        nacc = acc ? 1 : 0;
    }
    if (valid && isac) args.ell_out[(size_t)lane * args.L + lloc] = ell_s;
    if (valid && lane == 0) {
        args.lam_out[lloc] = lam_s;
        args.surv_out[lloc] = mask;
        if (args.lam_cand) {
            args.lam_cand[lloc] = lam[0];
            args.lam_cand[args.L + lloc] = lam[1];
        }
    }
    if (lane == 0) s_dec[seg] = valid ? nacc : 0;
    __syncthreads();
    uint32_t *s_cm = reinterpret_cast<uint32_t *>(s_r0);
    s_cm[tid] = (valid && isac) ? f2ord(ell_s) : 0u;
    __syncthreads();
    if (tid < n) {
        uint32_t mx = 0u;
        for (int sg = 0; sg < SEGS; ++sg) mx = max(mx, s_cm[sg * W + tid]);
        if (mx) atomicMax(&args.colmax[tid], mx);
    }
    if (tid == 0) {
        unsigned long long cnt = 0;
        for (int sg = 0; sg < SEGS; ++sg) cnt += s_dec[sg];
        if (cnt) atomicAdd(args.n_accept, cnt);
    }
}

template <int W, int R, bool SP4 = false>
static cudaError_t launch_2s_r(const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    const int npop = (SMC_K2_POP_SMEM && sc.has_noise) ? pop_smem_floats(sc.pop_nx + 1, sc.pop_ny + 1) : 0;
    const size_t smem = rollout2s_smem_bytes(W, sc.H, (npop + 3) & ~3, SP4 ? 4 : 2);
    auto kern = k_rollout_2s<W, R, SP4>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (a.L + kBlock / W - 1) / (kBlock / W);
    if (grid == 0) return cudaSuccess;
    kern<<<grid, kBlock, smem, st>>>(sc, a);
    return cudaGetLastError();
}

size_t rollout_smem_bytes(int W, int NC, int H, int ng, bool sp) {
    const int SEGS = kBlock / W, NSL = sp ? 2 : 1;
    if (ng > 8) {
        const size_t zs = ((size_t)SEGS * dense_zst(ng) + 3) & ~(size_t)3;
        return sizeof(float4) * ((size_t)H * NC * kBlock) +
               sizeof(float) * ((size_t)SEGS * dense_vst(ng) + SEGS * dense_zst(ng) + zs) +
               sizeof(float4) * 3 * kBlock + sizeof(float) * (size_t)ng * dense_qts(ng) + 16;
    }
    const int GB = (W >= 8) ? W / 4 : 1;
    return sizeof(float4) * ((size_t)H * NC * kBlock) + sizeof(float) * NSL * (SEGS * GB * 16 + 2 * SEGS * 16) +
           sizeof(float4) * 3 * kBlock + sizeof(float) * 72 + 16;
}

template <int W, int NC, bool DEBUG, bool DENSE, int R = W, bool SP = false>
static cudaError_t launch_w(const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    const size_t smem = rollout_smem_bytes(W, NC, sc.H, DENSE ? sc.wng : 8, SP);
    auto kern = k_rollout<W, NC, DEBUG, DENSE, R, SP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int segs = kBlock / W;
    const unsigned grid = (a.L + segs - 1) / segs;
    if (grid == 0) return cudaSuccess;
    kern<<<grid, kBlock, smem, st>>>(sc, a);
    return cudaGetLastError();
}

static bool ring_enabled() {
    static const bool on = [] { const char *e = getenv("SMC_K2_RING"); return !(e && strcmp(e, "0") == 0); }();
    return on;
}

static bool ns2_enabled() {
    static const bool on = [] { const char *e = getenv("SMC_K2_2S"); return !(e && strcmp(e, "0") == 0); }();
    return on;
}

// Two-candidate launches on the 2x2x2 grid with W >= 16: two sample chains per lane (k_rollout_2s);
// SMC_K2_2S=0 runs one sample per lane (k_rollout<W, 2>).
static bool pack_enabled() {
    static const bool on = [] { const char *e = getenv("SMC_K2_PACK"); return !(e && strcmp(e, "0") == 0); }();
    return on;
}

template <bool SP4>
static cudaError_t launch_2s(int W, int R, const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    // packed segments (W not dividing a warp, ring = segment): 9-12 aircraft in 12 lanes (10 per block),
    // 17-20 in 20 (6 per block), 21-24 in 24 (5 per block) -- instead of 16- / 32-lane segments
    if (!SP4 && pack_enabled()) {   // (SP4 instances: segments within warps only)
        if (sc.n >= 9 && sc.n <= 12) return launch_2s_r<12, 12, SP4>(sc, a, st);
        if (sc.n >= 17 && sc.n <= 20) return launch_2s_r<20, 20, SP4>(sc, a, st);
        if (sc.n >= 21 && sc.n <= 24) return launch_2s_r<24, 24, SP4>(sc, a, st);
    }
    switch (W) {
#if SMC_K2_2S_MINW <= 8
        case 8:
            if (R == 6) return launch_2s_r<8, 6, SP4>(sc, a, st);
            return launch_2s_r<8, 8, SP4>(sc, a, st);
#endif
        case 16:
            if (R == 10) return launch_2s_r<16, 10, SP4>(sc, a, st);
            if (R == 12) return launch_2s_r<16, 12, SP4>(sc, a, st);
            if (R == 14) return launch_2s_r<16, 14, SP4>(sc, a, st);
            return launch_2s_r<16, 16, SP4>(sc, a, st);
        case 32:
            if (R == 20) return launch_2s_r<32, 20, SP4>(sc, a, st);
            if (R == 24) return launch_2s_r<32, 24, SP4>(sc, a, st);
            if (R == 28) return launch_2s_r<32, 28, SP4>(sc, a, st);
            return launch_2s_r<32, 32, SP4>(sc, a, st);
    }
    return cudaErrorInvalidValue;
}

static bool sp_enabled() {
    static const bool on = [] { const char *e = getenv("SMC_K2_SP"); return !(e && strcmp(e, "0") == 0); }();
    return on;
}

// Single-candidate launches on the 2x2x2 grid with W >= 8: sample pairs in the float2 slots
// (both control pointers = the one candidate); SMC_K2_SP=0 runs them one sample per lane.
// Ring sizes with instances below W (smallest R >= n is used): N = 5-6 in W = 8, 9-14 in 16,
// 17-28 in 32 -- the separation scan needs R/2 partner offsets instead of W/2.
static int ring_for(int W, int n) {
    if (!ring_enabled()) return W;
    static const int r8[] = {6}, r16[] = {10, 12, 14}, r32[] = {20, 24, 28};
    const int *r = W == 8 ? r8 : (W == 16 ? r16 : (W == 32 ? r32 : nullptr));
    const int m = W == 8 ? 1 : (W == 16 || W == 32 ? 3 : 0);
    for (int q = 0; q < m; ++q)
        if (n <= r[q]) return r[q];
    return W;
}

template <int W, int NC, bool DEBUG, bool SP>
static cudaError_t launch_ring(int R, const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    if constexpr (W == 8) {
        if (R == 6) return launch_w<8, NC, DEBUG, false, 6, SP>(sc, a, st);
    } else if constexpr (W == 16) {
        if (R == 10) return launch_w<16, NC, DEBUG, false, 10, SP>(sc, a, st);
        if (R == 12) return launch_w<16, NC, DEBUG, false, 12, SP>(sc, a, st);
        if (R == 14) return launch_w<16, NC, DEBUG, false, 14, SP>(sc, a, st);
    } else if constexpr (W == 32) {
        if (R == 20) return launch_w<32, NC, DEBUG, false, 20, SP>(sc, a, st);
        if (R == 24) return launch_w<32, NC, DEBUG, false, 24, SP>(sc, a, st);
        if (R == 28) return launch_w<32, NC, DEBUG, false, 28, SP>(sc, a, st);
    }
    return launch_w<W, NC, DEBUG, false, W, SP>(sc, a, st);
}

// Single-candidate launches on the 2x2x2 grid with W >= 8: sample pairs in the float2 slots
// (both control pointers = the one candidate); SMC_K2_SP=0 runs them one sample per lane.
static cudaError_t launch_sp(int W, const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    RolloutArgs b = a;
    b.ctrl[1] = a.ctrl[0];
    const int R = ring_for(W, sc.n);
    switch (W) {
        case 8: return launch_ring<8, 2, false, true>(R, sc, b, st);
        case 16: return launch_ring<16, 2, false, true>(R, sc, b, st);
        case 32: return launch_ring<32, 2, false, true>(R, sc, b, st);
    }
    return cudaErrorInvalidValue;
}

template <int NC, bool DEBUG>
static cudaError_t launch_nc(int W, bool dense, const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    if (dense) {
        switch (W) {     // dense grids: W >= 4 (shared-memory budget of the per-segment field)
            case 4: return launch_w<4, NC, DEBUG, true>(sc, a, st);
            case 8: return launch_w<8, NC, DEBUG, true>(sc, a, st);
            case 16: return launch_w<16, NC, DEBUG, true>(sc, a, st);
            case 32: return launch_w<32, NC, DEBUG, true>(sc, a, st);
        }
        return cudaErrorInvalidValue;
    }
    // separation rings smaller than the segment (SMC_K2_RING=0: off)
    const int R = ring_for(W, sc.n);
    switch (W) {
        case 1: return launch_w<1, NC, DEBUG, false>(sc, a, st);
        case 2: return launch_w<2, NC, DEBUG, false>(sc, a, st);
        case 4: return launch_w<4, NC, DEBUG, false>(sc, a, st);
        case 8: return launch_ring<8, NC, DEBUG, false>(R, sc, a, st);
        case 16: return launch_ring<16, NC, DEBUG, false>(R, sc, a, st);
        case 32: return launch_ring<32, NC, DEBUG, false>(R, sc, a, st);
    }
    return cudaErrorInvalidValue;
}

int segment_width(int n, bool dense) {
    int w = dense ? 4 : 1;
    while (w < n) w <<= 1;
    return w;
}

cudaError_t launch_rollout(const DevScen &sc, const RolloutArgs &a, int NC, bool debug, cudaStream_t st) {
    const bool dense = sc.wng > 8;
    const int W = segment_width(sc.n, dense);
    if (NC == 1 && !debug && !dense && W >= 8 && sp_enabled()) {
        // one candidate: four samples per lane in the two-chain kernel for 16-lane segments (flags:
        // 2 H <= 32 bits; Table-1 123.7 -> 112.8 ms), else sample pairs in the one-chain kernel
        // (flags: bit t; at W = 8 four samples per lane measured slower, c2's 1024 blocks filling
        // 2.3 waves)
        if (SMC_K2_SP4 && sc.H <= 16 && W == 16) {
            RolloutArgs b = a;
            b.ctrl[1] = a.ctrl[0];
            return launch_2s<true>(W, ring_for(W, sc.n), sc, b, st);
        }
        if (sc.H <= 32) return launch_sp(W, sc, a, st);
    }
    // two sample chains per lane where they measured faster (B200, K2 per MPC step, 2 interleaved repeats:
    // c5 2376 -> 2330 ms (21 rounds), c4 23.6 -> 22.3, c3 89.4 -> 83.6 (11 rounds); c2 (W = 8) 26.40 ->
    // 26.68: one chain)
    // the two-chain kernel: its per-step flag masks hold 2 H <= 32 bits; built to stage the noise
    // grid in shared memory (SMC_K2_POP_SMEM), a grid larger than kPopSmem padded entries takes the
    // one-chain kernel
    const bool pop_fits = !SMC_K2_POP_SMEM || !sc.has_noise || pop_smem_floats(sc.pop_nx + 1, sc.pop_ny + 1) > 0;
    if (NC == 2 && !debug && !dense && pop_fits && sc.H <= 16 && W >= SMC_K2_2S_MINW && ns2_enabled())
        return launch_2s<false>(W, ring_for(W, sc.n), sc, a, st);
    if (debug) return NC == 2 ? launch_nc<2, true>(W, dense, sc, a, st) : launch_nc<1, true>(W, dense, sc, a, st);
    return NC == 2 ? launch_nc<2, false>(W, dense, sc, a, st) : launch_nc<1, false>(W, dense, sc, a, st);
}

}  // namespace smc

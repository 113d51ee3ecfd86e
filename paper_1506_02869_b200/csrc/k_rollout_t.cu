// k_rollout_t.cu -- K2 (transposed layout): batched Monte Carlo evaluation
// (Alg.1 l.9-18) fused with the Metropolis-Hastings accept (R1).
//
// Mapping: a block evaluates PPB = 32/NC particles;
// warp i of the block is aircraft i, lane = (candidate c, particle p).  So
//  * every lane of a warp runs the same aircraft type and kind: the arrival /
//    departure cost code is warp-uniform (no predicated waste), and any N
//    uses exactly N warps (no power-of-two lane padding);
//  * the 2x2x2 wind field of particle p is produced once per step
//    by 4 Philox tasks and 16 mat-vec tasks spread over the whole block and
//    shared through shared memory by all N aircraft and both MH candidates
//    (common random numbers);
//  * separation (Eq. avoidance): positions published to shared
//    memory, each lane scans the other N-1 aircraft of its (particle,
//    candidate) with conflict-free lane-consecutive LDS.128.
// Per (sample, step): Philox + AR(1) -> barrier -> W = Qhat Z -> barrier ->
// dynamics / checks / geometry -> barrier -> separation / costs.
#include "smc_device.cuh"
#include "smc_kernels.h"

namespace smc {

namespace {

__device__ __forceinline__ float clamp01t(float v) { return fminf(fmaxf(v, 0.0f), 1.0f); }

__device__ __forceinline__ float rcp_a(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_a(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// atan2 on the MUFU reciprocal and a degree-15 odd polynomial (least-squares
// fit of atan(a)/a on [0,1] in a^2; |error| < 1.5e-7 rad in binary32).
__device__ __forceinline__ float atan2_p(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float a = mx > 0.0f ? mn * rcp_a(mx) : 0.0f;
    const float s = a * a;
    float p = -0.0040731243789196014f;
    p = fmaf(p, s, 0.021945973858237267f);
    p = fmaf(p, s, -0.056062303483486176f);
    p = fmaf(p, s, 0.0965619683265686f);
    p = fmaf(p, s, -0.13915780186653137f);
    p = fmaf(p, s, 0.19948504865169525f);
    p = fmaf(p, s, -0.3333010673522949f);
    p = fmaf(p, s, 0.999999463558197f);
    float r = p * a;
    r = ay > ax ? 1.57079632679489662f - r : r;
    r = x < 0.0f ? kPi - r : r;
    return copysignf(r, y);
}

__device__ __forceinline__ float popdense_t(const DevScen &sc, float x, float y) {
    float gx = (x - sc.pop_x0) * sc.pop_inv_dx, gy = (y - sc.pop_y0) * sc.pop_inv_dx;
    gx = fminf(fmaxf(gx, 0.0f), (float)(sc.pop_nx - 1));
    gy = fminf(fmaxf(gy, 0.0f), (float)(sc.pop_ny - 1));
    const int ix = min((int)gx, max(sc.pop_nx - 2, 0));
    const int iy = min((int)gy, max(sc.pop_ny - 2, 0));
    const float fx = sc.pop_nx > 1 ? gx - (float)ix : 0.0f;
    const float fy = sc.pop_ny > 1 ? gy - (float)iy : 0.0f;
    const int ix1 = sc.pop_nx > 1 ? ix + 1 : ix, iy1 = sc.pop_ny > 1 ? iy + 1 : iy;
    const float v00 = __ldg(&sc.pop[iy * sc.pop_nx + ix]), v10 = __ldg(&sc.pop[iy * sc.pop_nx + ix1]);
    const float v01 = __ldg(&sc.pop[iy1 * sc.pop_nx + ix]), v11 = __ldg(&sc.pop[iy1 * sc.pop_nx + ix1]);
    const float a = fmaf(fx, v10 - v00, v00), b = fmaf(fx, v11 - v01, v01);
    return fmaf(fy, b - a, a);
}

constexpr int kRow = 20;   // padded row of the 16 wind entries: conflict-free LDS.128 per lane
// Half pair scan (+1 barrier per step) measured slower than the full scan on
// B200 for c3 (N = 24: 1.55 s vs 1.42 s per MPC step); kept, disabled.
constexpr int kHalfScanN = 64;

}  // namespace

template <int NC, int MAXT, int MINB, bool DEBUG>
__global__ void __launch_bounds__(MAXT, MINB)
k_rollout_t(const DevScen sc, const RolloutArgs args) {
    constexpr int PPB = 32 / NC;                      // particles per block
    extern __shared__ __align__(16) float smem[];
    const int n = sc.n, H = sc.H;
    const int nthr = blockDim.x;                      // 32 n
    float4 *s_ctrl = reinterpret_cast<float4 *>(smem);              // [H][nthr]
    float *s_Z = reinterpret_cast<float *>(s_ctrl + H * nthr);      // [H][PPB][kRow] normals -> AR(1) state
    float *s_W = s_Z + H * PPB * kRow;                              // [H][PPB][kRow] wind at the nodes
    float4 *s_pos = reinterpret_cast<float4 *>(s_W + H * PPB * kRow); // [2][nthr] (x, y, z, present)
    float *s_Q = reinterpret_cast<float *>(s_pos + 2 * nthr);       // [8][9]
    unsigned char *s_flag = reinterpret_cast<unsigned char *>(s_Q + 72);   // [nthr][16] pair verdicts
    __shared__ double s_lam[32];
    __shared__ uint32_t s_dec[32];                 // survivor masks of the block's particles

    const int tid = threadIdx.x, lane = tid & 31, i = tid >> 5;
    const int p = lane % PPB, c = lane / PPB;
    const uint32_t pbase = blockIdx.x * PPB;
    const uint32_t lloc = pbase + p;
    const bool valid = lloc < args.L;
    const uint32_t l = args.l0 + lloc;
    const uint32_t k = args.k, mpc = *args.mpcp;

    for (int q = tid; q < 64; q += blockDim.x) s_Q[(q >> 3) * 9 + (q & 7)] = sc.Cq[q];   // trilinear-coefficient form
    reinterpret_cast<uint4 *>(s_flag)[tid] = make_uint4(0u, 0u, 0u, 0u);

    const DevAircraft *Ap = sc.ac + i;
    const int kind = Ap->kind, first = Ap->first_step;
    const float halfS = Ap->halfS, cd0 = Ap->cd0, cd2 = Ap->cd2, dt_eta = Ap->dt_eta;
    const float zmin = Ap->z_min, zmax = Ap->z_max, vmin = Ap->v_min, vmax = Ap->v_max, mempty = Ap->m_empty;
    const float gA = kind ? Ap->theta_F : Ap->beta_f;
    const float z_tf = Ap->z_tf, v_D = Ap->v_D;

    // controls -> (T, tan phi, sin gamma, cos gamma) in shared memory; envelope bits in a register
    uint32_t cbad = 0;
    {
        const float gmax = Ap->gamma_max, pmax = Ap->phi_max, Tmin = Ap->T_min, Tmax = Ap->T_max;
        const float *src = args.ctrl[c] + ((size_t)lloc * n + i) * H * 3;
        for (int t = 0; t < H; ++t) {
            float T = 0.f, ph = 0.f, ga = 0.f;
            if (valid) { T = src[3 * t]; ph = src[3 * t + 1]; ga = src[3 * t + 2]; }
            float sph, cph, sga, cga;
            sincosf(ph, &sph, &cph);
            sincosf(ga, &sga, &cga);
            s_ctrl[t * nthr + tid] = make_float4(T, sph / cph, sga, cga);
            const bool bad = (fabsf(ga) > gmax) || !(fabsf(ph) < pmax) || (T < Tmin) || (T > Tmax);
            cbad |= (bad ? 1u : 0u) << t;
        }
    }
    __syncthreads();

    float ell = args.ell0;
    const float dt = sc.dt, g = sc.g, dtg = dt * g;
    const float x0 = Ap->x0[0], y0 = Ap->x0[1], z0 = Ap->x0[2], v0 = Ap->x0[3], c0 = Ap->x0[4], m0 = Ap->x0[5];
    for (uint32_t s = 0; s < args.S; ++s) {
        float x = x0, y = y0, z = z0, v = v0, chi = c0, m = m0;
        float fuel = 0.f, sA = 0.f, sB = 0.f, sC = 0.f, sN = 0.f;
        bool landed = false, viol = false;
        float2 gust_odd = make_float2(0.f, 0.f);
        const uint32_t x1 = (s & 0xFFFFu) | (k << 16);
        // ---- 1. wind realisation of the whole horizon (Alg.1 l.10), block-wide:
        //      (a) Philox: 4 blocks x H steps per particle
        for (int task = tid; task < 4 * H * PPB; task += nthr) {
            const int q = task % PPB, b = (task / PPB) & 3, ts = task / (4 * PPB);
            const uint4 w = draw_ks(TAG_WIND, args.l0 + pbase + q, x1, (uint32_t)ts | ((uint32_t)b << 16), mpc, sc.ks);
            const float2 p0 = box_muller(w.x, w.y), p1 = box_muller(w.z, w.w);
            *reinterpret_cast<float4 *>(&s_Z[(ts * PPB + q) * kRow + 4 * b]) = make_float4(p0.x, p0.y, p1.x, p1.y);
        }
        __syncthreads();
        //      (b) AR(1) over t per (particle, entry), in place: Z(0) = v(0), Z(t) = a Z(t-1) + b v(t)
        for (int task = tid; task < 16 * PPB; task += nthr) {
            const int q = task % PPB, e = task / PPB;
            float zz = s_Z[q * kRow + e];
            for (int ts = 1; ts < H; ++ts) {
                float *zp = &s_Z[(ts * PPB + q) * kRow + e];
                zz = fmaf(sc.a, zz, sc.b * *zp);
                *zp = zz;
            }
        }
        __syncthreads();
        //      (c) W(t) = Qhat Z(t) per component
        for (int task = tid; task < 16 * H * PPB; task += nthr) {
            const int q = task % PPB, e = (task / PPB) & 15, ts = task / (16 * PPB);
            const int comp = e >> 3, node = e & 7;
            const float *zrow = &s_Z[(ts * PPB + q) * kRow + comp * 8];
            const float4 za = *reinterpret_cast<const float4 *>(zrow);
            const float4 zb = *reinterpret_cast<const float4 *>(zrow + 4);
            const float *qr = &s_Q[node * 9];
            float acc = qr[0] * za.x;
            acc = fmaf(qr[1], za.y, acc); acc = fmaf(qr[2], za.z, acc); acc = fmaf(qr[3], za.w, acc);
            acc = fmaf(qr[4], zb.x, acc); acc = fmaf(qr[5], zb.y, acc); acc = fmaf(qr[6], zb.z, acc);
            acc = fmaf(qr[7], zb.w, acc);
            s_W[(ts * PPB + q) * kRow + e] = acc;
        }
        __syncthreads();
        for (int t = 0; t < H; ++t) {
            float Wn[16];
            {
                const float4 *w4 = reinterpret_cast<const float4 *>(&s_W[(t * PPB + p) * kRow]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 a4 = w4[q];
                    Wn[4 * q] = a4.x; Wn[4 * q + 1] = a4.y; Wn[4 * q + 2] = a4.z; Wn[4 * q + 3] = a4.w;
                }
            }
            float gx = sc.nominal[0], gy = sc.nominal[1];
            if (sc.turb_sigma > 0.0f) {       // gusts (R15), shared by both candidates
                float2 gg;
                if ((t & 1) == 0) {
                    const uint4 w = draw_ks(TAG_TURB, l, x1, ((uint32_t)t >> 1) | ((uint32_t)i << 8), mpc, sc.ks);
                    gg = box_muller(w.x, w.y);
                    gust_odd = box_muller(w.z, w.w);
                } else {
                    gg = gust_odd;
                }
                gx = fmaf(sc.turb_sigma, gg.x, gx);
                gy = fmaf(sc.turb_sigma, gg.y, gy);
            }
            // ---- 2-3. Eq. hor, envelope, geometry, landing test
            const bool act = first <= t;
            const bool fly = act && !landed && !viol;
            const float4 cc = s_ctrl[t * nthr + tid];
            const float T = cc.x, tph = cc.y, sga = cc.z, cga = cc.w;
            const float fx = clamp01t((x - sc.wind_lo[0]) * sc.wind_inv_ext[0]);
            const float fy = clamp01t((y - sc.wind_lo[1]) * sc.wind_inv_ext[1]);
            const float fz = clamp01t((z - sc.wind_lo[2]) * sc.wind_inv_ext[2]);
            const float wx = tripoly(Wn, Wn[0] + gx, fx, fy, fz);
            const float wy = tripoly(Wn + 8, Wn[8] + gy, fx, fy, fz);
            float rho = sc.rho_const;
            if (sc.density_mode == 0) rho = 1.225f * ex2_a(4.2559f * __log2f(fmaxf(fmaf(-2.2558e-5f, z, 1.0f), 0.0f)));
            const float qd = rho * v * v * halfS;
            const float mgq = m * g * rcp_a(qd);
            const float D = qd * fmaf(cd2 * mgq * mgq, fmaf(tph, tph, 1.0f), cd0);
            const float chr = chi - kTwoPi * rintf(chi * (1.0f / kTwoPi));
            float sch, cch;
            __sincosf(chr, &sch, &cch);
            const float vcg = v * cga;
            const float nx = fmaf(dt, fmaf(vcg, cch, wx), x);
            const float ny = fmaf(dt, fmaf(vcg, sch, wy), y);
            const float nz = fmaf(dt * v, sga, z);
            const float nv = fmaf(dt, fmaf(T - D, rcp_a(m), -g * sga), v);
            const float nchi = fmaf(dtg * tph, rcp_a(v), chi);
            const float nm = fmaf(-dt_eta, T, m);
            bool vnow = (cbad >> t) & 1u;
            vnow |= !(nz >= zmin && nz <= zmax);
            vnow |= !(nv >= vmin && nv <= vmax);
            vnow |= !(nm >= mempty);
            // (x, y, chi stay finite whenever v, z, m and the controls pass: no extra test needed)
            const float th = atan2_p(ny, nx);
            float devA, devB;
            bool lnow = false;
            if (kind == 0) {                  // arrival (warp-uniform branch)
                const float r2 = fmaf(nx, nx, ny * ny);
                const float rh = r2 * rsqrtf(fmaxf(r2, 1e-30f));
                const float at = fabsf(th);
                const float sarc = at > 1e-4f ? rh * at * rcp_a(__sinf(at)) : rh;
                const float beta = atan2_p(nz, sarc);
                lnow = !landed && rh <= sc.P_runway && beta <= sc.P_beta && at <= sc.P_chi &&
                       angdist(nchi - kPi) <= sc.P_chi && nv <= sc.P_vs;
                devA = angdist(nchi - kPi - 2.0f * th);          // heading vs flow field (R8)
                devB = fabsf(beta - gA);                          // descent angle (R9)
            } else {
                devA = angdist(th - gA);                          // bearing (R22)
                devB = fabsf(z_tf - nz);
            }
            float4 *pos = s_pos + (t & 1) * nthr;          // double-buffered: one barrier per step
            pos[tid] = make_float4(nx, ny, nz, fly ? 1.0f : 0.0f);
            __syncthreads();
            // ---- 4. separation (Eq. avoidance) against the other aircraft of this (particle, candidate)
            if (n >= kHalfScanN) {
                // each unordered pair once: warp i checks aircraft i+d (mod n), d = 1..n/2, and leaves
                // the verdict in a per-(partner, d) byte the partner reads after one more barrier
                // (for even n the d = n/2 pair is checked by both warps and needs no hand-over)
                const int D = (n - 1) / 2;
                bool conf = false;
                for (int d = 1; d <= n / 2; ++d) {
                    int q = i + d;
                    q = q >= n ? q - n : q;
                    const float4 o = pos[q * 32 + lane];
                    const float dx = nx - o.x, dy = ny - o.y, dz = nz - o.z;
                    const bool hit = fly && (o.w != 0.0f) && (fmaf(dx, dx, dy * dy) < sc.twoPr2) && (fabsf(dz) < sc.twoPh);
                    conf = conf || hit;
                    if (d <= D) s_flag[(q * 32 + lane) * 16 + d - 1] = hit ? 1 : 0;
                }
                __syncthreads();
                const uint4 f = *reinterpret_cast<const uint4 *>(&s_flag[tid * 16]);
                vnow = vnow || conf || ((f.x | f.y | f.z | f.w) != 0u);
            } else {
                // small n: full scan; the own entry always hits itself when present
                int cnt = 0;
                for (int q = 0; q < n; ++q) {
                    const float4 o = pos[q * 32 + lane];
                    const float dx = nx - o.x, dy = ny - o.y, dz = nz - o.z;
                    cnt += ((o.w != 0.0f) && (fmaf(dx, dx, dy * dy) < sc.twoPr2) && (fabsf(dz) < sc.twoPh)) ? 1 : 0;
                }
                vnow = vnow || (cnt > 1);
            }
            // ---- 5. cost terms at j = t+1 and state update
            float nzs = 0.0f;
            if (sc.has_noise) {
                const float zz = nz * sc.inv_Ac;
                nzs = 1.0f - fmaxf(1.0f - zz * zz, 0.0f) * popdense_t(sc, nx, ny);
            }
            sA += fly ? devA : 0.0f;
            sB += fly ? devB : 0.0f;
            sC += fly ? fabsf(nv - v_D) : 0.0f;
            sN += fly ? nzs : ((act && landed) ? 1.0f : 0.0f);   // best cost after landing
            fuel += fly ? dt_eta * T : 0.0f;
            viol = viol || (fly && vnow);
            landed = landed || (fly && lnow);
            x = fly ? nx : x; y = fly ? ny : y; z = fly ? nz : z;
            v = fly ? nv : v; chi = fly ? nchi : chi; m = fly ? nm : m;
            if (DEBUG && c == 0 && valid && args.dbg_traj) {
                float *tr = args.dbg_traj + ((((size_t)lloc * args.S + s) * n + i) * (H + 1) + t + 1) * 6;
                tr[0] = x; tr[1] = y; tr[2] = z; tr[3] = v; tr[4] = chi; tr[5] = m;
                if (t == 0) {
                    tr[-6] = x0; tr[-5] = y0; tr[-4] = z0; tr[-3] = v0; tr[-2] = c0; tr[-1] = m0;
                }
            }
            if (DEBUG && c == 0 && valid && args.dbg_landed && lnow && fly)
                args.dbg_landed[((size_t)lloc * args.S + s) * n + i] = t + 1;
        }  // t

        // ---- utility J_T and weight
        float J = 1.0f, q0 = 1.f, q1 = 1.f, q2 = 1.f, q3 = 1.f;
        if (Ap->Ha > 0) {
            const float invHa = Ap->invHa;
            const float Jfuel = clamp01t(1.0f - fuel * Ap->invFmax);
            const float J1 = clamp01t(1.0f - sA * invHa * (1.0f / kPi));
            if (kind == 1) {
                q0 = J1;
                q1 = Jfuel;
                q2 = Ap->flagB ? 1.0f : clamp01t((Ap->supB - sB * invHa) * Ap->invDenB);
                q3 = clamp01t(1.0f - sC * invHa * Ap->invSupC);
                J = sc.alpha_dep[0] * q0 + sc.alpha_dep[1] * q1 + sc.alpha_dep[2] * q2 + sc.alpha_dep[3] * q3;
            } else {
                q0 = J1;
                q1 = clamp01t(1.0f - sB * invHa * Ap->invSupE);
                q2 = Jfuel;
                q3 = 0.0f;
                J = sc.alpha_arr[0] * q0 + sc.alpha_arr[1] * q1 + sc.alpha_arr[2] * q2;
            }
            if (sc.has_noise) J = (1.0f - sc.noise_w) * J + sc.noise_w * sN * invHa;
        }
        ell = (viol || !(J > 0.0f)) ? -INFINITY : ell + __log2f(J);
        if (DEBUG && c == 0 && valid) {
            const size_t o = ((size_t)lloc * args.S + s) * n + i;
            if (args.dbg_J) args.dbg_J[o] = J;
            if (args.dbg_viol) args.dbg_viol[o] = viol ? 1 : 0;
            if (args.dbg_fuel) args.dbg_fuel[o] = fuel;
            if (args.dbg_comp) { float *cp = args.dbg_comp + 4 * o; cp[0] = q0; cp[1] = q1; cp[2] = q2; cp[3] = q3; }
        }
    }  // s

    // ---- epilogue: lambda = sum_i ell (double, ascending i), MH (R1 / R46), survivors
    float *s_ell = reinterpret_cast<float *>(s_pos);              // reuse [nthr]
    const bool per_ac = (NC == 2) && args.mh_mode == 2;
    __syncthreads();
    s_ell[tid] = ell;
    if (tid < 32) s_dec[tid] = 0u;
    __syncthreads();
    if (per_ac) {                      // per-aircraft MH (R46): warp i decides for aircraft i
        const float e1 = __shfl_sync(0xffffffffu, ell, p + PPB);
        if (c == 0 && mh_decide_aircraft((double)ell, (double)e1, l, (uint32_t)i, k, mpc, sc.key0, sc.key1))
            atomicOr(&s_dec[p], 1u << i);
        __syncthreads();
    }
    if (i == 0) {
        double lam = 0.0;
        for (int a = 0; a < n; ++a) lam += (double)s_ell[a * 32 + lane];
        s_lam[lane] = lam;                                          // lane = (c, p)
        double lam_c0 = __shfl_sync(0xffffffffu, lam, p);
        double lam_c1 = __shfl_sync(0xffffffffu, lam, p + (NC - 1) * PPB);
        uint32_t mask = args.surv_single;
        double lam_s = lam_c0;
        if (per_ac) {
            mask = s_dec[p];
            lam_s = 0.0;
            for (int a = 0; a < n; ++a) lam_s += (double)s_ell[a * 32 + p + (((mask >> a) & 1u) ? PPB : 0)];
        } else if (NC == 2) {
            const bool acc = mh_decide(lam_c0, lam_c1, l, k, mpc, sc.key0, sc.key1);
            mask = acc ? 0xFFFFFFFFu : 0u;
            lam_s = acc ? lam_c1 : lam_c0;
        }
        __syncwarp();
        if (c == 0) {
            s_dec[p] = mask;
            if (valid) {
                args.lam_out[lloc] = lam_s;
                args.surv_out[lloc] = mask;
                if (args.lam_cand) {
                    args.lam_cand[lloc] = lam_c0;
                    args.lam_cand[args.L + lloc] = lam_c1;
                }
            }
        }
        if (NC == 2) {
            const unsigned mine = (c == 0 && valid) ? (per_ac ? __popc(mask) : (mask ? 1u : 0u)) : 0u;
            const unsigned cntv = __reduce_add_sync(0xffffffffu, mine);
            if (lane == 0 && cntv) atomicAdd(args.n_accept, (unsigned long long)cntv);
        }
        if (DEBUG && args.dbg_ell_c && valid)
            for (int a = 0; a < n; ++a) args.dbg_ell_c[((size_t)c * args.L + lloc) * n + a] = s_ell[a * 32 + lane];
    }
    __syncthreads();
    const uint32_t mbit = (s_dec[p] >> i) & 1u;
    const bool mine = (NC == 1) || ((uint32_t)c == mbit);
    if (valid && mine) args.ell_out[(size_t)i * args.L + lloc] = ell;
    // per-column max of the survivor log-weights (first half of the reduce, K3)
    const uint32_t key = (valid && mine) ? f2ord(ell) : 0u;
    const uint32_t mx = __reduce_max_sync(0xffffffffu, key);
    if (lane == 0 && mx) atomicMax(&args.colmax[i], mx);
}

size_t rollout_t_smem_bytes(int n, int H) {
    const int nthr = 32 * n;
    return sizeof(float4) * (size_t)H * nthr + sizeof(float) * 2 * (size_t)H * 32 * kRow + sizeof(float4) * 2 * nthr +
           sizeof(float) * 72 + 16 * (size_t)nthr + 16;
}

template <int NC, int MAXT, int MINB, bool DEBUG>
static cudaError_t launch_t(const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    const size_t smem = rollout_t_smem_bytes(sc.n, sc.H);
    auto kern = k_rollout_t<NC, MAXT, MINB, DEBUG>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    constexpr int PPB = 32 / NC;
    const unsigned grid = (a.L + PPB - 1) / PPB;
    if (grid == 0) return cudaSuccess;
    kern<<<grid, 32 * sc.n, smem, st>>>(sc, a);
    return cudaGetLastError();
}

template <int NC, bool DEBUG>
static cudaError_t launch_t_nc(const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    // register budget ~85 per thread for every block shape (MAXT * MINB <= 768 threads)
    if (sc.n <= 8) return launch_t<NC, 256, 3, DEBUG>(sc, a, st);
    if (sc.n <= 12) return launch_t<NC, 384, 2, DEBUG>(sc, a, st);
    if (sc.n <= 24) return launch_t<NC, 768, 1, DEBUG>(sc, a, st);
    return launch_t<NC, 1024, 1, DEBUG>(sc, a, st);
}

cudaError_t launch_rollout_t(const DevScen &sc, const RolloutArgs &a, int NC, bool debug, cudaStream_t st) {
    if (debug) return NC == 2 ? launch_t_nc<2, true>(sc, a, st) : launch_t_nc<1, true>(sc, a, st);
    return NC == 2 ? launch_t_nc<2, false>(sc, a, st) : launch_t_nc<1, false>(sc, a, st);
}

}  // namespace smc

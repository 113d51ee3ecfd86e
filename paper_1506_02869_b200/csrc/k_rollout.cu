// k_rollout.cu -- K2: batched Monte Carlo evaluation (Alg.1 l.9-18)
// fused with the Metropolis-Hastings accept step (R1).
//
// Mapping: one warp segment of W = next_pow2(N) lanes per
// particle l, lane = aircraft i.  Each lane keeps its aircraft's state for
// both MH candidates (c = 0: resampled x', c = 1: proposal x*) in registers;
// both candidates see the same wind realisation (common random numbers).
// Per step t the segment
//   1. draws the 16 normals of the 2x2x2 wind field (Philox, Box-Muller),
//      advances the AR(1) state Z and forms W = Qhat Z -- the 16
//      entries are distributed over the lanes and exchanged via shared memory;
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
#include "smc_device.cuh"
#include "smc_kernels.h"

namespace smc {

__device__ __forceinline__ float clamp01(float v) { return fminf(fmaxf(v, 0.0f), 1.0f); }

// popdense bilinear lookup on the 1 km grid, clamped at its edge.
__device__ __forceinline__ float popdense(const DevScen &sc, float x, float y) {
    float gx = (x - sc.pop_x0) * sc.pop_inv_dx, gy = (y - sc.pop_y0) * sc.pop_inv_dx;
    const float mx = (float)(sc.pop_nx - 1), my = (float)(sc.pop_ny - 1);
    gx = fminf(fmaxf(gx, 0.0f), mx);
    gy = fminf(fmaxf(gy, 0.0f), my);
    int ix = min((int)gx, max(sc.pop_nx - 2, 0));
    int iy = min((int)gy, max(sc.pop_ny - 2, 0));
    const float fx = sc.pop_nx > 1 ? gx - (float)ix : 0.0f;
    const float fy = sc.pop_ny > 1 ? gy - (float)iy : 0.0f;
    const int ix1 = sc.pop_nx > 1 ? ix + 1 : ix, iy1 = sc.pop_ny > 1 ? iy + 1 : iy;
    const float v00 = __ldg(&sc.pop[iy * sc.pop_nx + ix]), v10 = __ldg(&sc.pop[iy * sc.pop_nx + ix1]);
    const float v01 = __ldg(&sc.pop[iy1 * sc.pop_nx + ix]), v11 = __ldg(&sc.pop[iy1 * sc.pop_nx + ix1]);
    const float a = fmaf(fx, v10 - v00, v00), b = fmaf(fx, v11 - v01, v01);
    return fmaf(fy, b - a, a);
}

__device__ __forceinline__ float lerp(float a, float b, float t) { return fmaf(t, b - a, a); }

// Trilinear interpolation of one wind component (8 node values).
__device__ __forceinline__ float trilerp(const float *Wn, float fx, float fy, float fz) {
    const float a = lerp(Wn[0], Wn[1], fx), b = lerp(Wn[2], Wn[3], fx);
    const float c = lerp(Wn[4], Wn[5], fx), d = lerp(Wn[6], Wn[7], fx);
    return lerp(lerp(a, b, fy), lerp(c, d, fy), fz);
}

template <int W, int NC, bool DEBUG>
__global__ void __launch_bounds__(kBlock)
k_rollout(const DevScen sc, const RolloutArgs args) {
    constexpr int SEGS = kBlock / W;
    constexpr int E = (16 + W - 1) / W;           // wind-field entries owned per lane
    extern __shared__ __align__(16) float smem[];
    const int H = sc.H, n = sc.n;
    float *s_ctrl = smem;                                     // [H][NC][5][kBlock]
    float *s_V = s_ctrl + H * NC * 5 * kBlock;                // [SEGS][16] normals
    float *s_Z = s_V + SEGS * 16;                             // [SEGS][16] AR(1) state
    float *s_W = s_Z + SEGS * 16;                             // [SEGS][16] wind at nodes
    float4 *s_pos = reinterpret_cast<float4 *>(s_W + SEGS * 16);   // [NC][kBlock]
    float *s_Q = reinterpret_cast<float *>(s_pos + NC * kBlock);   // [8][9]

    const int tid = threadIdx.x, lane = tid % W, seg = tid / W;
    const uint32_t lloc = blockIdx.x * SEGS + seg;
    const bool valid = lloc < args.L;
    const uint32_t l = args.l0 + lloc;                         // global particle index
    const bool isac = lane < n;
    const uint32_t k = args.k, mpc = args.mpc;

    if (tid < 64) s_Q[(tid >> 3) * 9 + (tid & 7)] = sc.Qhat[tid];

    // ---- per-lane aircraft constants
    DevAircraft A;
    if (isac) A = sc.ac[lane];
    else { A = sc.ac[0]; A.first_step = 1 << 20; A.Ha = 0; }

    // ---- controls: derived trig terms to shared memory, envelope bits to registers
    uint32_t cbad[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        cbad[c] = 0;
        const float *src = args.ctrl[c] + ((size_t)lloc * n + lane) * H * 3;
        for (int t = 0; t < H; ++t) {
            float T = 0.f, ph = 0.f, ga = 0.f;
            if (isac && valid) { T = src[3 * t]; ph = src[3 * t + 1]; ga = src[3 * t + 2]; }
            float sph, cph, sga, cga;
            sincosf(ph, &sph, &cph);
            sincosf(ga, &sga, &cga);
            float *d = s_ctrl + ((t * NC + c) * 5) * kBlock + tid;
            d[0 * kBlock] = T;
            d[1 * kBlock] = sph / cph;          // tan(phi): turn rate g tan(phi)/v
            d[2 * kBlock] = 1.0f / cph;         // sec(phi): lift m g / cos(phi)
            d[3 * kBlock] = sga;
            d[4 * kBlock] = cga;
            const bool bad = (fabsf(ga) > A.gamma_max) || !(fabsf(ph) < A.phi_max) ||
                             (T < A.T_min) || (T > A.T_max);
            cbad[c] |= (bad ? 1u : 0u) << t;
        }
    }
    __syncthreads();

    float ell[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) ell[c] = args.ell0;

    const float dt = sc.dt, g = sc.g;
    for (uint32_t s = 0; s < args.S; ++s) {
        float x[NC], y[NC], z[NC], v[NC], chi[NC], m[NC], fuel[NC], sA[NC], sB[NC], sC[NC], sN[NC];
        bool landed[NC], viol[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            x[c] = A.x0[0]; y[c] = A.x0[1]; z[c] = A.x0[2]; v[c] = A.x0[3]; chi[c] = A.x0[4]; m[c] = A.x0[5];
            fuel[c] = sA[c] = sB[c] = sC[c] = sN[c] = 0.0f;
            landed[c] = false; viol[c] = false;
        }
        float Zr[E];
        float2 gust_odd = make_float2(0.f, 0.f);
        const uint32_t x1 = (s & 0xFFFFu) | (k << 16);

        for (int t = 0; t < H; ++t) {
            // ---------------- 1. wind realisation for step t (Alg.1 l.10)
            for (int b = lane; b < 4; b += W) {
                const uint4 w = draw(TAG_WIND, l, x1, (uint32_t)t | ((uint32_t)b << 16), mpc, sc.key0, sc.key1);
                const float2 p0 = box_muller(w.x, w.y), p1 = box_muller(w.z, w.w);
                *reinterpret_cast<float4 *>(&s_V[seg * 16 + 4 * b]) = make_float4(p0.x, p0.y, p1.x, p1.y);
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int e = lane + q * W;
                if (e < 16) {
                    const float ve = s_V[seg * 16 + e];
                    Zr[q] = (t == 0) ? ve : fmaf(sc.a, Zr[q], sc.b * ve);
                    s_Z[seg * 16 + e] = Zr[q];
                }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int e = lane + q * W;
                if (e < 16) {
                    const int comp = e >> 3, node = e & 7;
                    const float *zr = &s_Z[seg * 16 + comp * 8];
                    float acc = 0.0f;
#pragma unroll
                    for (int mm = 0; mm < 8; ++mm) acc = fmaf(s_Q[node * 9 + mm], zr[mm], acc);
                    s_W[seg * 16 + e] = acc;
                }
            }
            __syncwarp();
            float Wn[16];
            {
                const float4 *w4 = reinterpret_cast<const float4 *>(&s_W[seg * 16]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 a4 = w4[q];
                    Wn[4 * q] = a4.x; Wn[4 * q + 1] = a4.y; Wn[4 * q + 2] = a4.z; Wn[4 * q + 3] = a4.w;
                }
            }
            // gusts (R15): one Philox call covers steps 2u and 2u+1
            float gx = 0.0f, gy = 0.0f;
            if (sc.turb_sigma > 0.0f && isac) {
                if ((t & 1) == 0) {
                    const uint4 w = draw(TAG_TURB, l, x1, ((uint32_t)t >> 1) | ((uint32_t)lane << 8), mpc, sc.key0, sc.key1);
                    const float2 g0 = box_muller(w.x, w.y);
                    gust_odd = box_muller(w.z, w.w);
                    gx = g0.x; gy = g0.y;
                } else {
                    gx = gust_odd.x; gy = gust_odd.y;
                }
                gx *= sc.turb_sigma; gy *= sc.turb_sigma;
            }

            // ---------------- 2-3. dynamics and unary checks per candidate
            const bool act = isac && (A.first_step <= t);
            bool fly[NC], vnow[NC], lnow[NC];
            float nx[NC], ny[NC], nz[NC], nv[NC], nchi[NC], nm[NC], th[NC], beta[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                fly[c] = act && !landed[c] && !viol[c];
                nx[c] = x[c]; ny[c] = y[c]; nz[c] = z[c]; nv[c] = v[c]; nchi[c] = chi[c]; nm[c] = m[c];
                vnow[c] = false; lnow[c] = false; th[c] = 0.f; beta[c] = 0.f;
                if (fly[c]) {
                    const float *cc = s_ctrl + ((t * NC + c) * 5) * kBlock + tid;
                    const float T = cc[0], tph = cc[kBlock], sec = cc[2 * kBlock], sga = cc[3 * kBlock], cga = cc[4 * kBlock];
                    // wind at the pre-step position (trilinear, clamped to the box)
                    const float fx = clamp01((x[c] - sc.wind_lo[0]) * sc.wind_inv_ext[0]);
                    const float fy = clamp01((y[c] - sc.wind_lo[1]) * sc.wind_inv_ext[1]);
                    const float fz = clamp01((z[c] - sc.wind_lo[2]) * sc.wind_inv_ext[2]);
                    const float wx = trilerp(Wn, fx, fy, fz) + sc.nominal[0] + gx;
                    const float wy = trilerp(Wn + 8, fx, fy, fz) + sc.nominal[1] + gy;
                    // Eq. hor with coordinated-turn lift and parabolic drag (R12)
                    float rho = sc.rho_const;
                    if (sc.density_mode == 0)
                        rho = 1.225f * exp2f(4.2559f * __log2f(fmaxf(fmaf(-2.2558e-5f, z[c], 1.0f), 0.0f)));
                    const float qd = rho * v[c] * v[c] * A.halfS;
                    const float CL = __fdividef(m[c] * g * sec, qd);
                    const float D = qd * fmaf(A.cd2, CL * CL, A.cd0);
                    const float chr = chi[c] - kTwoPi * rintf(chi[c] * (1.0f / kTwoPi));
                    float sch, cch;
                    __sincosf(chr, &sch, &cch);
                    const float vcg = v[c] * cga;
                    nx[c] = x[c] + dt * fmaf(vcg, cch, wx);
                    ny[c] = y[c] + dt * fmaf(vcg, sch, wy);
                    nz[c] = z[c] + dt * v[c] * sga;
                    nv[c] = v[c] + dt * (__fdividef(T - D, m[c]) - g * sga);
                    nchi[c] = chi[c] + __fdividef(dt * g * tph, v[c]);
                    nm[c] = m[c] - A.dt_eta * T;
                    fuel[c] += A.dt_eta * T;
                    // envelope and mass at j = t+1 (R17)
                    bool bad = (cbad[c] >> t) & 1u;
                    bad |= !(nz[c] >= A.z_min && nz[c] <= A.z_max);
                    bad |= !(nv[c] >= A.v_min && nv[c] <= A.v_max);
                    bad |= !(nm[c] >= A.m_empty);
                    bad |= !(fabsf(nx[c]) <= 3.0e38f) || !(fabsf(ny[c]) <= 3.0e38f) || !(fabsf(nchi[c]) <= 3.0e38f);
                    vnow[c] = bad;
                    th[c] = atan2f(ny[c], nx[c]);
                    if (A.kind == 0) {
                        // descent angle on the flow-field arc (Eq. flow, R9) and landing test (R10)
                        const float rh = sqrtf(fmaf(nx[c], nx[c], ny[c] * ny[c]));
                        const float at = fabsf(th[c]);
                        const float sarc = at > 1e-4f ? __fdividef(rh * at, __sinf(at)) : rh;
                        beta[c] = atan2f(nz[c], sarc);
                        if (!landed[c])
                            lnow[c] = rh <= sc.P_runway && beta[c] <= sc.P_beta && at <= sc.P_chi &&
                                      angdist(nchi[c] - kPi) <= sc.P_chi && nv[c] <= sc.P_vs;
                    }
                }
                s_pos[c * kBlock + tid] = make_float4(nx[c], ny[c], nz[c], fly[c] ? 1.0f : 0.0f);
            }
            __syncwarp();
            // ---------------- 4. separation (Eq. avoidance) against every other lane
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (fly[c]) {
                    const float4 *P = s_pos + c * kBlock + seg * W;
                    bool conf = false;
                    for (int p = 0; p < n; ++p) {
                        const float4 q = P[p];
                        const float dx = nx[c] - q.x, dy = ny[c] - q.y, dz = nz[c] - q.z;
                        const bool hit = (q.w != 0.0f) && (fmaf(dx, dx, dy * dy) < sc.twoPr2) && (fabsf(dz) < sc.twoPh);
                        conf |= hit && (p != lane);
                    }
                    vnow[c] |= conf;
                }
            }
            // ---------------- 5. per-step cost terms at j = t+1
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (act) {
                    if (fly[c]) {
                        if (A.kind == 1) {
                            sA[c] += angdist(th[c] - A.theta_F);
                            sB[c] += fabsf(A.z_tf - nz[c]);
                            sC[c] += fabsf(nv[c] - A.v_D);
                        } else {
                            sA[c] += angdist(nchi[c] - kPi - 2.0f * th[c]);
                            sB[c] += fabsf(beta[c] - A.beta_f);
                        }
                        if (sc.has_noise) {
                            const float zz = nz[c] * sc.inv_Ac;
                            sN[c] += 1.0f - fmaxf(1.0f - zz * zz, 0.0f) * popdense(sc, nx[c], ny[c]);
                        }
                    } else if (landed[c]) {
                        sN[c] += 1.0f;      // "best possible cost, 1, for all remaining steps"
                    }
                }
                if (fly[c]) {
                    viol[c] = viol[c] || vnow[c];
                    landed[c] = landed[c] || lnow[c];
                    x[c] = nx[c]; y[c] = ny[c]; z[c] = nz[c]; v[c] = nv[c]; chi[c] = nchi[c]; m[c] = nm[c];
                }
                if (DEBUG && c == 0 && valid && isac && args.dbg_traj) {
                    float *tr = args.dbg_traj + ((((size_t)lloc * args.S + s) * n + lane) * (H + 1) + t + 1) * 6;
                    tr[0] = x[c]; tr[1] = y[c]; tr[2] = z[c]; tr[3] = v[c]; tr[4] = chi[c]; tr[5] = m[c];
                    if (t == 0) {
                        float *t0 = tr - 6;
                        for (int a = 0; a < 6; ++a) t0[a] = A.x0[a];
                    }
                }
                if (DEBUG && c == 0 && valid && isac && args.dbg_landed && lnow[c] && fly[c])
                    args.dbg_landed[((size_t)lloc * args.S + s) * n + lane] = t + 1;
            }
        }  // t

        // ---------------- utility J_T and weight
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            float J = 1.0f, c0 = 1.f, c1 = 1.f, c2 = 1.f, c3 = 1.f;
            if (A.Ha > 0) {
                const float Jfuel = clamp01(1.0f - fuel[c] * A.invFmax);
                if (A.kind == 1) {
                    c0 = clamp01(1.0f - sA[c] * A.invHa * (1.0f / kPi));
                    c1 = Jfuel;
                    c2 = A.flagB ? 1.0f : clamp01((A.supB - sB[c] * A.invHa) * A.invDenB);
                    c3 = clamp01(1.0f - sC[c] * A.invHa * A.invSupC);
                    J = sc.alpha_dep[0] * c0 + sc.alpha_dep[1] * c1 + sc.alpha_dep[2] * c2 + sc.alpha_dep[3] * c3;
                } else {
                    c0 = clamp01(1.0f - sA[c] * A.invHa * (1.0f / kPi));
                    c1 = clamp01(1.0f - sB[c] * A.invHa * A.invSupE);
                    c2 = Jfuel;
                    c3 = 0.0f;
                    J = sc.alpha_arr[0] * c0 + sc.alpha_arr[1] * c1 + sc.alpha_arr[2] * c2;
                }
                if (sc.has_noise) J = (1.0f - sc.noise_w) * J + sc.noise_w * sN[c] * A.invHa;
            }
            ell[c] = (viol[c] || !(J > 0.0f)) ? -INFINITY : ell[c] + log2f(J);
            if (DEBUG && c == 0 && valid && isac) {
                const size_t o = ((size_t)lloc * args.S + s) * n + lane;
                if (args.dbg_J) args.dbg_J[o] = J;
                if (args.dbg_viol) args.dbg_viol[o] = viol[c] ? 1 : 0;
                if (args.dbg_fuel) args.dbg_fuel[o] = fuel[c];
                if (args.dbg_comp) { float *cp = args.dbg_comp + 4 * o; cp[0] = c0; cp[1] = c1; cp[2] = c2; cp[3] = c3; }
            }
        }
    }  // s

    // ---------------- epilogue: lambda (double, ascending i), MH (R1), survivor
    __syncthreads();
    float *s_ell = reinterpret_cast<float *>(s_pos);          // reuse [NC][kBlock]
    int *s_dec = reinterpret_cast<int *>(s_V);                 // [SEGS]
#pragma unroll
    for (int c = 0; c < NC; ++c) s_ell[c * kBlock + tid] = ell[c];
    __syncwarp();
    double lam[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        lam[c] = 0.0;
        for (int i = 0; i < n; ++i) lam[c] += (double)s_ell[c * kBlock + seg * W + i];
    }
    int acc = args.surv_single;
    if (NC == 2) acc = mh_decide(lam[0], lam[1], l, k, mpc, sc.key0, sc.key1) ? 1 : 0;
    const float ell_s = (NC == 2 && acc) ? ell[NC - 1] : ell[0];
    const double lam_s = (NC == 2 && acc) ? lam[NC - 1] : lam[0];
    if (valid && isac) args.ell_out[(size_t)lane * args.L + lloc] = ell_s;
    if (valid && lane == 0) {
        args.lam_out[lloc] = lam_s;
        args.surv_out[lloc] = (uint8_t)acc;
        if (args.lam_cand) {
            args.lam_cand[lloc] = lam[0];
            args.lam_cand[args.L + lloc] = lam[NC - 1];
        }
        if (DEBUG && args.dbg_ell_c) {
            for (int c = 0; c < NC; ++c)
                for (int i = 0; i < n; ++i)
                    args.dbg_ell_c[((size_t)c * args.L + lloc) * n + i] = s_ell[c * kBlock + seg * W + i];
        }
    }
    if (lane == 0) s_dec[seg] = (valid && NC == 2) ? acc : 0;
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
    if (NC == 2 && tid == 0) {
        unsigned long long cnt = 0;
        for (int sg = 0; sg < SEGS; ++sg) cnt += s_dec[sg];
        if (cnt) atomicAdd(args.n_accept, cnt);
    }
}

size_t rollout_smem_bytes(int W, int NC, int H) {
    const int SEGS = kBlock / W;
    return sizeof(float) * ((size_t)H * NC * 5 * kBlock + 3 * SEGS * 16) + sizeof(float4) * NC * kBlock +
           sizeof(float) * 72 + 16;
}

template <int W, int NC, bool DEBUG>
static cudaError_t launch_w(const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    const size_t smem = rollout_smem_bytes(W, NC, sc.H);
    auto kern = k_rollout<W, NC, DEBUG>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int segs = kBlock / W;
    const unsigned grid = (a.L + segs - 1) / segs;
    if (grid == 0) return cudaSuccess;
    kern<<<grid, kBlock, smem, st>>>(sc, a);
    return cudaGetLastError();
}

template <int NC, bool DEBUG>
static cudaError_t launch_nc(int W, const DevScen &sc, const RolloutArgs &a, cudaStream_t st) {
    switch (W) {
        case 1: return launch_w<1, NC, DEBUG>(sc, a, st);
        case 2: return launch_w<2, NC, DEBUG>(sc, a, st);
        case 4: return launch_w<4, NC, DEBUG>(sc, a, st);
        case 8: return launch_w<8, NC, DEBUG>(sc, a, st);
        case 16: return launch_w<16, NC, DEBUG>(sc, a, st);
        case 32: return launch_w<32, NC, DEBUG>(sc, a, st);
    }
    return cudaErrorInvalidValue;
}

int segment_width(int n) {
    int w = 1;
    while (w < n) w <<= 1;
    return w;
}

cudaError_t launch_rollout(const DevScen &sc, const RolloutArgs &a, int NC, bool debug, cudaStream_t st) {
    const int W = segment_width(sc.n);
    if (debug) return NC == 2 ? launch_nc<2, true>(W, sc, a, st) : launch_nc<1, true>(W, sc, a, st);
    return NC == 2 ? launch_nc<2, false>(W, sc, a, st) : launch_nc<1, false>(W, sc, a, st);
}

}  // namespace smc

// smc_device.cuh -- device-side building blocks of libsmcatm (sm_100a).
//
// Independent of oracle/ (no shared code, headers or tables): every routine
// here is written from the paper / the DESIGN.md readings directly.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "smc_vec.cuh"

namespace smc {

constexpr int kMaxAc = 32;
constexpr int kMaxH = 32;
#ifndef SMC_K2_BLOCK
#define SMC_K2_BLOCK 128
#endif
constexpr int kBlock = SMC_K2_BLOCK;  // threads per rollout block (launch-geometry sweep: 64-512)
constexpr float kPi = 3.14159265358979323846f;
constexpr float kTwoPi = 6.28318530717958647692f;

// Stream tags of the counter-based generator (R37).
enum : uint32_t { TAG_INIT = 1, TAG_PERTURB = 2, TAG_WIND = 3, TAG_TURB = 4, TAG_MH = 5,
                  TAG_RESAMPLE = 6, TAG_PLANT_WIND = 7, TAG_PLANT_TURB = 8 };

// Per-aircraft constants, float, one entry per aircraft (lane-indexed).
struct DevAircraft {
    int kind, first_step, Ha, flagB;      // flagB: altitude term degenerate (sup-inf < 1 m) -> 1
    float x0[6];
    float theta_F, z_tf, v_D, beta_f;
    float halfS, cd0, cd2, dt_eta;        // 0.5 S, drag polar, dt * eta
    float m_empty, T_min, T_max, v_min, v_max, gamma_max, phi_max, z_min, z_max;
    float supB, invDenB, invSupC, invSupE, invFmax, invHa;
};

// Scenario constants, uniform over the grid: passed by value as a kernel parameter.
struct DevScen {
    int n, H, density_mode, has_noise;
    float dt, g, rho_const;
    float P_runway, P_beta, P_chi, P_vs, twoPr2, twoPh;
    float P_chi_west;                     // pi - P_chi: with chi in [-pi, pi], |wrap(chi - pi)| <= P_chi
                                          // (landing heading, Eq. TO_init) is |chi| >= pi - P_chi
    float alpha_dep[4], alpha_arr[3];
    float noise_w, inv_Ac;
    int pop_nx, pop_ny;
    float pop_x0, pop_y0, pop_inv_dx;
    float pop_ax, pop_bx, pop_ay, pop_by; // grid coordinate / (n - 1) = sat(a x + b) (0 for a 1-wide axis)
    float pop_mx, pop_my;                 // n - 1 per axis
    float wind_lo[3], wind_inv_ext[3];
    float Qhat[64];                       // lower-triangular, row-major
    float Cq[64];                         // M Qhat: row r gives coefficient r of the trilinear
                                          // polynomial of the node field (see tripoly)
    float a, b;                           // AR(1) coefficients
    float nominal[2], turb_sigma;
    uint32_t key0, key1;                  // Philox key = seed
    uint32_t ks[20];                      // Philox round keys (key0 + r W0, key1 + r W1), r = 0..9
    int wn[3], wng;                       // wind grid points per axis, wng = product
    const float *Qf;                      // [wng][wng] Qhat (FP32), read by the dense-grid path (wng > 8)
    const DevAircraft *ac;
    const float *pop;                     // [pop_ny][pop_nx] popdense grid
    const float *popp;                    // [pop_ny + 1][pop_nx + 1] the same, last row/column repeated
};

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al. (SC'11); constants M0, M1 (multipliers) and W0, W1 (Weyl key bumps).
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

// Same generator with the round keys precomputed (DevScen::ks, kernel-parameter
// space): the key XORs read them as constant-bank operands.
__device__ __forceinline__ uint4 philox_ks(uint4 c, const uint32_t *ks) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ ks[2 * r], lo1, hi0 ^ c.w ^ ks[2 * r + 1], lo0);
    }
    return c;
}

__device__ __forceinline__ uint4 draw(uint32_t tag, uint32_t x0, uint32_t x1, uint32_t x2,
                                      uint32_t mpc, uint32_t k0, uint32_t k1) {
    return philox(make_uint4(x0, x1, x2, (mpc & 0xFFFFFFu) | (tag << 24)), k0, k1);
}

__device__ __forceinline__ uint4 draw_ks(uint32_t tag, uint32_t x0, uint32_t x1, uint32_t x2, uint32_t mpc,
                                         const uint32_t *ks) {
    return philox_ks(make_uint4(x0, x1, x2, (mpc & 0xFFFFFFu) | (tag << 24)), ks);
}

// Trilinear interpolation in polynomial form: with c = M W (node n = ix + 2 iy + 4 iz)
//   f = c0 + c1 fx + c2 fy + c3 fz + c4 fx fy + c5 fx fz + c6 fy fz + c7 fx fy fz,
// algebraically the 7-lerp form; 7 FMAs (packed over the candidates when V = float2).  c0 is passed separately so a per-lane
// offset (nominal wind + gust) can be folded in once per step.
template <class V>
__device__ __forceinline__ V tripoly(const float *c, float c0, V fx, V fy, V fz) {
    const V A = vfma(fy, vfma(fz, c[7], c[4]), vfma(fz, c[5], c[1]));
    const V B = vfma(fy, vfma(fz, c[6], c[2]), vfma(fz, c[3], c0));
    return vfma(fx, A, B);
}

// The same with per-slot coefficients (sample pairs: slot a in .x, slot b in .y).
__device__ __forceinline__ float2 tripoly2(const float2 *c, float2 c0, float2 fx, float2 fy, float2 fz) {
    const float2 A = vfma(fy, vfma(fz, c[7], c[4]), vfma(fz, c[5], c[1]));
    const float2 B = vfma(fy, vfma(fz, c[6], c[2]), vfma(fz, c[3], c0));
    return vfma(fx, A, B);
}

// MUFU lg2 / rsqrt without the denormal-input fix-up (FSETP + two predicated ops) that __log2f and
// rsqrtf carry.  Every use has a normal input (uniforms >= 2^-24, -2 ln u >= 1.1e-7, clamps to
// >= 1e-30) or feeds ex2 of a large negative multiple (the ISA base), where a flushed denormal
// gives the same 0: results are bit-identical to the non-ftz forms.
__device__ __forceinline__ float lg2_approx(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Uniform (2k+1) 2^-24, k = w >> 9: exact in binary32 (R37).
__device__ __forceinline__ float unif(uint32_t w) {
    return __fmaf_rn(__uint2float_rn(w >> 9), 0x1.0p-23f, 0x1.0p-24f);
}

// Box-Muller (normal pair from two words).  angle 2 pi u2 is evaluated as
// pi + 2 pi (u2 - 1/2) so the fast sin/cos see an argument in [-pi, pi).
__device__ __forceinline__ float2 box_muller(uint32_t w0, uint32_t w1) {
    const float u1 = unif(w0), u2 = unif(w1);
    const float r2 = -2.0f * 0.69314718055994531f * lg2_approx(u1);
    const float r = r2 * rsqrt_approx(r2);
    float s, c;
    __sincosf(kTwoPi * (u2 - 0.5f), &s, &c);
    return make_float2(-r * c, -r * s);
}

// The two Box-Muller pairs of one Philox block, (w.x, w.y) -> (.x, .y) and (w.z, w.w) -> (.z, .w),
// evaluated as packed pairs; bit-identical to two box_muller calls (2 pi u2 - pi = 2 pi (u2 - 1/2)
// exactly: pi_f is half of (2 pi)_f and u2 - 1/2 is exact on the 2^-24 grid).
__device__ __forceinline__ float4 box_muller4(uint4 w) {
    const float2 u1 = vfma(make_float2(__uint2float_rn(w.x >> 9), __uint2float_rn(w.z >> 9)), 0x1.0p-23f, 0x1.0p-24f);
    const float2 u2 = vfma(make_float2(__uint2float_rn(w.y >> 9), __uint2float_rn(w.w >> 9)), 0x1.0p-23f, 0x1.0p-24f);
    const float2 r2 = make_float2(lg2_approx(u1.x), lg2_approx(u1.y)) * (-2.0f * 0.69314718055994531f);
    const float2 r = r2 * make_float2(rsqrt_approx(r2.x), rsqrt_approx(r2.y));
    const float2 ang = vfma(u2, kTwoPi, -kPi);
    float2 sn, cs;
    __sincosf(ang.x, &sn.x, &cs.x);
    __sincosf(ang.y, &sn.y, &cs.y);
    const float2 a = -r * cs, b = -r * sn;
    return make_float4(a.x, b.x, a.y, b.y);
}

__device__ __forceinline__ uint64_t r64(uint32_t tag, uint32_t x0, uint32_t k, uint32_t mpc,
                                        uint32_t k0, uint32_t k1) {
    const uint4 w = draw(tag, x0, k << 16, 0u, mpc, k0, k1);
    return (uint64_t)w.x | ((uint64_t)w.y << 32);
}

// ---------------------------------------------------------------- deterministic exp2 (R26)
// p(f) = sum_j c_j f^j, c_j = RN(ln2^j / j!), Horner with fma, then ldexp.
__device__ __forceinline__ double det_exp2(double y) {
    if (!(y >= -1022.0)) return 0.0;
    const double n = floor(y);
    const double f = y - n;
    double p = 0x1.38e89ae79f8b4p-53;
    p = fma(p, f, 0x1.c36e843b04022p-49);
    p = fma(p, f, 0x1.314964d5878a9p-44);
    p = fma(p, f, 0x1.816193166d0f9p-40);
    p = fma(p, f, 0x1.c3bd650fc2986p-36);
    p = fma(p, f, 0x1.e8cac7351bb25p-32);
    p = fma(p, f, 0x1.e4cf5158b8ecap-28);
    p = fma(p, f, 0x1.b5253d395e7c4p-24);
    p = fma(p, f, 0x1.62c0223a5c824p-20);
    p = fma(p, f, 0x1.ffcbfc588b0c7p-17);
    p = fma(p, f, 0x1.430912f86c787p-13);
    p = fma(p, f, 0x1.5d87fe78a6731p-10);
    p = fma(p, f, 0x1.3b2ab6fba4e77p-7);
    p = fma(p, f, 0x1.c6b08d704a0c0p-5);
    p = fma(p, f, 0x1.ebfbdff82c58fp-3);
    p = fma(p, f, 0x1.62e42fefa39efp-1);
    p = fma(p, f, 1.0);
    return ldexp(p, (int)n);
}

// Integer resampling weight: floor(2^(32 + d)) for d >= -32, else 0 (R25/R26).
__device__ __forceinline__ uint64_t det_quant(double d) {
    if (!(d >= -32.0)) return 0ull;
    return (uint64_t)floor(det_exp2(32.0 + d));
}

// MH decision for particle l in round k (R1): joint log2 weights.
__device__ __forceinline__ bool mh_decide(double lam_cur, double lam_prop, uint32_t l, uint32_t k,
                                          uint32_t mpc, uint32_t k0, uint32_t k1) {
    if (lam_cur == -INFINITY) return true;
    if (lam_prop == -INFINITY) return false;
    const double delta = lam_prop - lam_cur;
    if (delta >= 0.0) return true;
    const uint64_t r = r64(TAG_MH, l, k, mpc, k0, k1);
    const double u53 = (double)(r >> 11) * 0x1.0p-53;
    return u53 < det_exp2(delta);
}

// Per-aircraft MH decision (R46): the joint rules on one aircraft's log2 weights, uniform
// from the MH stream at counter (l, k<<16, i).
__device__ __forceinline__ bool mh_decide_aircraft(double ell_cur, double ell_prop, uint32_t l, uint32_t i,
                                                   uint32_t k, uint32_t mpc, uint32_t k0, uint32_t k1) {
    if (ell_cur == -INFINITY) return true;
    if (ell_prop == -INFINITY) return false;
    const double delta = ell_prop - ell_cur;
    if (delta >= 0.0) return true;
    const uint4 w = draw(TAG_MH, l, k << 16, i, mpc, k0, k1);
    const uint64_t r = (uint64_t)w.x | ((uint64_t)w.y << 32);
    const double u53 = (double)(r >> 11) * 0x1.0p-53;
    return u53 < det_exp2(delta);
}

// ---------------------------------------------------------------- angles
// |wrap(d)| in [0, pi].
__device__ __forceinline__ float angdist(float d) {
    const float r = d - kTwoPi * rintf(d * (1.0f / kTwoPi));
    return fabsf(r);
}

// Ordered encoding of floats for integer atomicMax.
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

}  // namespace smc

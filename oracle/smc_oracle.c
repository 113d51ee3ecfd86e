/*
 * smc_oracle.c -- TEST INFRASTRUCTURE ONLY (see smc_oracle.h).
 *
 * Plain FP64 CPU implementation of the hot path of Eele & Maciejowski (2015),
 * written step by step in the paper's order and notation.  No blocking,
 * fusion or reordering beyond what the paper's Algorithm 1 states.
 * OpenMP is used only across independent particles (Alg.1 l.8).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (no fused multiply-add except the explicit fma() calls det_exp2 requires).
 *
 * Parity status per function (DESIGN.md section 4 lists the pinning tests):
 *   philox, u24, box_muller, det_exp2, det_quant, derive (Rhat, Qhat, a, b,
 *   supB/infB), trilinear, popdense, density, lift_drag, step, unary/landing/
 *   pair checks, flow_heading, arc_length, beta, utilities (J1..J4, Jalt,
 *   Jfuel, noise), AR(1) propagation, weight recursion, mh_accept,
 *   resample_column, select, sample_schedule, init_population, perturb_row,
 *   plant_step, fuel estimates ........................................ pinned
 *   rolling-window averaging (R20), post-landing bonus (R18), constraint
 *   handling after a violation (Alg.1 l.11-13: the violator keeps flying and
 *   stays in every pair test), MH move semantics (R1) ............... pinned
 *   (conventions the paper states in prose only: pinned by invariants and
 *   closed forms in tests/test_oracle_conventions.py -- shorter-horizon
 *   equivalence, hand-computed post-landing means, a violator that later
 *   conflicts with a neighbour zeroes it, sigma = 0 reduction of the MH move
 *   to Alg.1 l.23)
 */
#include "smc_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------------ */
/* Counter-based streams (R37): Philox4x32-10 (Salmon et al., SC'11).        */
/* The paper used CURAND XORWOW with per-thread state; a stateless   */
/* counter-based generator keys every draw by (particle, sample, step, ...). */
/* ------------------------------------------------------------------------ */
enum { TAG_INIT = 1, TAG_PERTURB = 2, TAG_WIND = 3, TAG_TURB = 4, TAG_MH = 5,
       TAG_RESAMPLE = 6, TAG_PLANT_WIND = 7, TAG_PLANT_TURB = 8 };

void ora_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t y0 = hi1 ^ x1 ^ k0;
        uint32_t y1 = lo1;
        uint32_t y2 = hi0 ^ x3 ^ k1;
        uint32_t y3 = lo0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static void draw(uint32_t tag, uint32_t x0, uint32_t x1, uint32_t x2, uint32_t mpc,
                 uint64_t seed, uint32_t w[4])
{
    uint32_t ctr[4] = { x0, x1, x2, (mpc & 0xFFFFFFu) | (tag << 24) };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    ora_philox(ctr, key, w);
}

/* 23-bit uniform in (0,1): (2k+1) 2^-24 with k = w >> 9 < 2^23 has at most 24
 * significant bits, so it is exactly representable in binary32 and binary64
 * and both implementations see bit-identical uniforms (R37). */
double ora_u24(uint32_t w) { return ((double)(w >> 9) + 0.5) * (1.0 / 8388608.0); }

/* Box-Muller transform on one word pair. */
void ora_box_muller(uint32_t w0, uint32_t w1, double *n0, double *n1)
{
    double u1 = ora_u24(w0), u2 = ora_u24(w1);
    double r = sqrt(-2.0 * log(u1));
    *n0 = r * cos(2.0 * M_PI * u2);
    *n1 = r * sin(2.0 * M_PI * u2);
}

uint64_t ora_r64(uint32_t tag, uint32_t x0, uint32_t k, uint64_t seed, uint32_t mpc)
{
    uint32_t w[4];
    draw(tag, x0, k << 16, 0, mpc, seed, w);
    return (uint64_t)w[0] | ((uint64_t)w[1] << 32);
}

/* ------------------------------------------------------------------------ */
/* det_exp2 / det_quant (R26): 2^y from correctly rounded IEEE ops only, so  */
/* an independent implementation with the same op sequence agrees bit-exact. */
/* c_j = RN((ln 2)^j / j!), j = 0..16; Horner with fma; ldexp.               */
/* ------------------------------------------------------------------------ */
static const double DET_C[17] = {
    0x1.0000000000000p+0,  0x1.62e42fefa39efp-1, 0x1.ebfbdff82c58fp-3,
    0x1.c6b08d704a0c0p-5,  0x1.3b2ab6fba4e77p-7, 0x1.5d87fe78a6731p-10,
    0x1.430912f86c787p-13, 0x1.ffcbfc588b0c7p-17, 0x1.62c0223a5c824p-20,
    0x1.b5253d395e7c4p-24, 0x1.e4cf5158b8ecap-28, 0x1.e8cac7351bb25p-32,
    0x1.c3bd650fc2986p-36, 0x1.816193166d0f9p-40, 0x1.314964d5878a9p-44,
    0x1.c36e843b04022p-49, 0x1.38e89ae79f8b4p-53 };

const double *ora_det_coeffs(void) { return DET_C; }

double ora_det_exp2(double y)
{
    if (!(y >= -1022.0)) return 0.0;          /* keeps every result a normal number */
    double n = floor(y);
    double f = y - n;                          /* exact */
    double p = DET_C[16];
    for (int j = 15; j >= 0; --j) p = fma(p, f, DET_C[j]);
    return ldexp(p, (int)n);
}

uint64_t ora_det_quant(double d)
{
    if (!(d >= -32.0)) return 0;               /* also -inf and NaN */
    double v = ora_det_exp2(32.0 + d);
    return (uint64_t)floor(v);
}

/* ------------------------------------------------------------------------ */
/* Sample schedule: floor(3 + 5 e^{0.05 J}).                         */
/* ------------------------------------------------------------------------ */
int ora_sample_schedule(int J) { return (int)floor(3.0 + 5.0 * exp(0.05 * (double)J)); }

/* ------------------------------------------------------------------------ */
/* Scenario precompute                                                       */
/* ------------------------------------------------------------------------ */
/* Grid point n = ix + N_x (iy + N_y iz) of the N_x x N_y x N_z grid spanning
 * the box [wind_lo, wind_hi] evenly (the paper's runs use 2x2x2). */
static void node_pos(const ora_problem *p, const ora_derived *d, int n, double pos[3])
{
    int idx[3] = { n % d->nx, (n / d->nx) % d->ny, n / (d->nx * d->ny) };
    int cnt[3] = { d->nx, d->ny, d->nz };
    for (int a = 0; a < 3; ++a)
        pos[a] = p->wind_lo[a] + (p->wind_hi[a] - p->wind_lo[a]) * (double)idx[a] / (double)(cnt[a] - 1);
}

static double sigma_z(const ora_problem *p, double z)
{
    double fz = (z - p->wind_lo[2]) / (p->wind_hi[2] - p->wind_lo[2]);
    return p->sigma_lo + (p->sigma_hi - p->sigma_lo) * fz;
}

/* popdense: min(sum_i exp(-b_i^2/(2 c_i^2)) / (c_i sqrt(2 pi)), 1),
 * b_i, c_i in km (R23). */
double ora_popdense_point(const ora_problem *p, double x, double y)
{
    double sum = 0.0;
    for (int c = 0; c < p->n_centres; ++c) {
        double bx = (x - p->centres[3 * c + 0]) / 1000.0;
        double by = (y - p->centres[3 * c + 1]) / 1000.0;
        double ci = p->centres[3 * c + 2] / 1000.0;
        double b2 = bx * bx + by * by;
        sum += exp(-b2 / (2.0 * ci * ci)) / (ci * sqrt(2.0 * M_PI));
    }
    return sum < 1.0 ? sum : 1.0;
}

/* Cholesky factor L with L L^T = A (A SPD, row-major N x N). */
static int cholesky(const double *A, double *Lo, int N)
{
    memset(Lo, 0, (size_t)N * N * sizeof(double));
    for (int r = 0; r < N; ++r) {
        for (int c = 0; c <= r; ++c) {
            double s = A[r * N + c];
            for (int k = 0; k < c; ++k) s -= Lo[r * N + k] * Lo[c * N + k];
            if (r == c) {
                if (!(s > 0.0)) return -1;
                Lo[r * N + r] = sqrt(s);
            } else {
                Lo[r * N + c] = s / Lo[c * N + c];
            }
        }
    }
    return 0;
}

int ora_derive(const ora_problem *p, ora_derived *d)
{
    memset(d, 0, sizeof(*d));
    if (p->n < 0 || p->n > ORA_MAX_AC || p->H < 0 || p->H > 255) return -1;
    d->nx = p->wind_n[0] ? p->wind_n[0] : 2;
    d->ny = p->wind_n[1] ? p->wind_n[1] : 2;
    d->nz = p->wind_n[2] ? p->wind_n[2] : 2;
    if (d->nx < 2 || d->ny < 2 || d->nz < 2) return -3;
    d->ng = d->nx * d->ny * d->nz;
    if (d->ng > ORA_MAX_NODES) return -3;
    const int G = d->ng;
    /* Eq. cov, same-time entries of Rhat. */
    for (int n = 0; n < G; ++n) {
        double pn[3]; node_pos(p, d, n, pn);
        for (int m = 0; m < G; ++m) {
            double pm[3]; node_pos(p, d, m, pm);
            double dxy = sqrt((pn[0] - pm[0]) * (pn[0] - pm[0]) + (pn[1] - pm[1]) * (pn[1] - pm[1]));
            double dz = fabs(pn[2] - pm[2]);
            d->Rhat[n * G + m] = sigma_z(p, pn[2]) * sigma_z(p, pm[2])
                               * exp(-p->beta_w * dxy) * exp(-p->gamma_w * dz);
        }
    }
    /* Qhat Qhat^T = Rhat.  sigma == 0 gives a zero field. */
    int zero = 1;
    for (int n = 0; n < G * G; ++n) if (d->Rhat[n] != 0.0) zero = 0;
    if (!zero && cholesky(d->Rhat, d->Qhat, G) != 0) return -2;
    /* a = e^{-dt/G_t}, G_t = 1/lambda_t (R14); Q = sqrt(1-a^2) Qhat. */
    d->a = exp(-p->lambda_t * p->dt);
    d->b = sqrt(1.0 - d->a * d->a);
    /* Departure altitude term B: sup / inf by reachability with gamma_max, v_max (R21). */
    for (int i = 0; i < p->n; ++i) {
        int e = p->first_step[i];
        int Ha = p->H - e;
        double z0 = p->x0[6 * i + 2], zt = p->z_tf[i];
        double ssum = 0.0, isum = 0.0;
        for (int j = e + 1; j <= p->H; ++j) {
            double reach = (double)(j - e) * p->dt * p->v_max[i] * sin(p->gamma_max[i]);
            double lo = z0 - reach; if (lo < p->z_min[i]) lo = p->z_min[i];
            double hi = z0 + reach; if (hi > p->z_max[i]) hi = p->z_max[i];
            double sup = fabs(zt - lo) > fabs(zt - hi) ? fabs(zt - lo) : fabs(zt - hi);
            double nearest = zt < lo ? lo : (zt > hi ? hi : zt);
            ssum += sup;
            isum += fabs(zt - nearest);
        }
        d->supB[i] = Ha > 0 ? ssum / Ha : 0.0;
        d->infB[i] = Ha > 0 ? isum / Ha : 0.0;
    }
    /* 1 km population grid. */
    if (p->pop_nx > 0 && p->pop_ny > 0) {
        d->pop = (double *)malloc(sizeof(double) * (size_t)p->pop_nx * (size_t)p->pop_ny);
        for (int iy = 0; iy < p->pop_ny; ++iy)
            for (int ix = 0; ix < p->pop_nx; ++ix)
                d->pop[iy * p->pop_nx + ix] =
                    ora_popdense_point(p, p->pop_x0 + ix * p->pop_dx, p->pop_y0 + iy * p->pop_dx);
    }
    return 0;
}

void ora_free_derived(ora_derived *d) { free(d->pop); d->pop = NULL; }

/* Bilinear lookup on the 1 km grid, clamped at its edge (R23). */
double ora_popdense_grid(const ora_problem *p, const ora_derived *d, double x, double y)
{
    if (!d->pop) return 0.0;
    double gx = (x - p->pop_x0) / p->pop_dx, gy = (y - p->pop_y0) / p->pop_dx;
    double mx = (double)(p->pop_nx - 1), my = (double)(p->pop_ny - 1);
    if (!(gx > 0.0)) gx = 0.0;
    if (gx > mx) gx = mx;
    if (!(gy > 0.0)) gy = 0.0;
    if (gy > my) gy = my;
    int ix = (int)floor(gx), iy = (int)floor(gy);
    if (ix > p->pop_nx - 2) ix = p->pop_nx - 2;
    if (ix < 0) ix = 0;
    if (iy > p->pop_ny - 2) iy = p->pop_ny - 2;
    if (iy < 0) iy = 0;
    double fx = gx - ix, fy = gy - iy;
    if (p->pop_nx == 1) fx = 0.0;
    if (p->pop_ny == 1) fy = 0.0;
    int ix1 = p->pop_nx > 1 ? ix + 1 : ix, iy1 = p->pop_ny > 1 ? iy + 1 : iy;
    double v00 = d->pop[iy * p->pop_nx + ix], v10 = d->pop[iy * p->pop_nx + ix1];
    double v01 = d->pop[iy1 * p->pop_nx + ix], v11 = d->pop[iy1 * p->pop_nx + ix1];
    return (1 - fx) * (1 - fy) * v00 + fx * (1 - fy) * v10 + (1 - fx) * fy * v01 + fx * fy * v11;
}

/* "tri-linear interpolation between the grid points" of the grid
 * cell holding the position, clamped to the grid box (R14). */
void ora_trilinear(const ora_problem *p, const ora_derived *d, const double *W, const double pos[3], double *w)
{
    const int cnt[3] = { d->nx, d->ny, d->nz };
    int c0[3];
    double f[3];
    for (int a = 0; a < 3; ++a) {
        double t = (pos[a] - p->wind_lo[a]) / (p->wind_hi[a] - p->wind_lo[a]);
        if (!(t > 0.0)) t = 0.0;
        if (t > 1.0) t = 1.0;
        double g = t * (double)(cnt[a] - 1);          /* grid coordinate in [0, N-1] */
        int i0 = (int)floor(g);
        if (i0 > cnt[a] - 2) i0 = cnt[a] - 2;
        c0[a] = i0;
        f[a] = g - (double)i0;
    }
    double acc = 0.0;
    for (int corner = 0; corner < 8; ++corner) {
        int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
        double wx = dx ? f[0] : 1.0 - f[0];
        double wy = dy ? f[1] : 1.0 - f[1];
        double wz = dz ? f[2] : 1.0 - f[2];
        int node = (c0[0] + dx) + d->nx * ((c0[1] + dy) + d->ny * (c0[2] + dz));
        acc += wx * wy * wz * W[node];
    }
    *w = acc;
}

/* ------------------------------------------------------------------------ */
/* Aircraft model (Eq. hor)                                       */
/* ------------------------------------------------------------------------ */
static double density(const ora_problem *p, double z)
{
    if (p->density_mode == 1) return p->rho_const;
    double base = 1.0 - 2.2558e-5 * z;                   /* ISA troposphere (R12) */
    if (!(base > 0.0)) base = 0.0;
    return 1.225 * pow(base, 4.2559);
}

/* "Lift L and drag D are calculated using the standard aerodynamic relations"
 * -- read as coordinated-turn lift and a parabolic polar (R12). */
void ora_lift_drag(const ora_problem *p, int i, const double st[6], double phi,
                   double *lift, double *drag)
{
    double v = st[3], m = st[5];
    double rho = density(p, st[2]);
    double qd = 0.5 * rho * v * v * p->S[i];
    double L = m * p->g / cos(phi);
    double CL = L / qd;
    *lift = L;
    *drag = qd * (p->cd0[i] + p->cd2[i] * CL * CL);
}

/* Eq. hor, simultaneous explicit Euler (R41). st/out = x,y,z,v,chi,m. */
void ora_step(const ora_problem *p, int i, const double st[6], const double u[3],
              const double wind[2], double out[6])
{
    double T = u[0], phi = u[1], gam = u[2];
    double x = st[0], y = st[1], z = st[2], v = st[3], chi = st[4], m = st[5];
    double L, D;
    ora_lift_drag(p, i, st, phi, &L, &D);
    double dt = p->dt;
    out[0] = x + dt * (v * cos(chi) * cos(gam)) + wind[0] * dt;
    out[1] = y + dt * (v * sin(chi) * cos(gam)) + wind[1] * dt;
    out[2] = z + dt * (v * sin(gam));
    out[3] = v + dt * ((T - D) / m - p->g * sin(gam));
    out[4] = chi + dt * (L * sin(phi) / (m * v));
    out[5] = m - dt * (p->eta[i] * T);
}

/* |wrap(d)| in [0, pi] (R32). */
double ora_angdist(double d)
{
    double r = fmod(fabs(d), 2.0 * M_PI);
    return r > M_PI ? 2.0 * M_PI - r : r;
}

/* Flow-field heading (R8): the circle through the origin tangent to the
 * runway axis, flown so as to arrive heading West: chi_hat = pi + 2 theta. */
double ora_flow_heading(double x, double y) { return M_PI + 2.0 * atan2(y, x); }

/* "distance remaining on the arc of the flow field" (R9). */
double ora_arc_length(double x, double y)
{
    double rho = sqrt(x * x + y * y);
    double th = fabs(atan2(y, x));
    if (th == 0.0) return rho;
    return rho * th / sin(th);
}

/* Eq. flow with the arc length of R9. */
double ora_beta(double x, double y, double z) { return atan2(z, ora_arc_length(x, y)); }

/* Landing sector (Eq. TO_init; R10). */
int ora_landed(const ora_problem *p, const double st[6])
{
    double x = st[0], y = st[1], z = st[2], v = st[3], chi = st[4];
    double rho = sqrt(x * x + y * y);
    return rho <= p->P_runway
        && ora_beta(x, y, z) <= p->P_beta
        && fabs(atan2(y, x)) <= p->P_chi
        && ora_angdist(chi - M_PI) <= p->P_chi
        && v <= p->P_vs;
}

/* Unary constraints (R17): controls of the step and the new state. */
int ora_unary_violation(const ora_problem *p, int i, const double u[3], const double st[6])
{
    for (int a = 0; a < 6; ++a) if (!isfinite(st[a])) return 1;
    if (fabs(u[2]) > p->gamma_max[i]) return 1;
    if (!(fabs(u[1]) < p->phi_max[i])) return 1;
    if (u[0] < p->T_min[i] || u[0] > p->T_max[i]) return 1;
    if (st[2] < p->z_min[i] || st[2] > p->z_max[i]) return 1;
    if (st[3] < p->v_min[i] || st[3] > p->v_max[i]) return 1;
    if (st[5] < p->m_empty[i]) return 1;
    return 0;
}

/* Negation of Eq. avoidance: conflict iff both separations fail. */
int ora_pair_conflict(const ora_problem *p, const double a[6], const double b[6])
{
    double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
    double ok = (dx * dx + dy * dy >= (2.0 * p->P_r) * (2.0 * p->P_r)) || (fabs(dz) >= 2.0 * p->P_h);
    return !ok && isfinite(dx) && isfinite(dy) && isfinite(dz);
}

static double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

/* ------------------------------------------------------------------------ */
/* Decision margins (R30).  Every discrete decision of a rollout  */
/* is a Boolean combination of comparisons; comparison c holds iff mu_c >= 0 */
/* (mu_c > 0 for a strict bound), mu_c a relative distance to its threshold. */
/* An OR of conditions (a violation: any bound fails) changes outcome under  */
/* a perturbation smaller than e only if every failing condition flips (when */
/* it is true) or some condition flips (when it is false), so its margin is  */
/* max_{failing} |mu| if true, min_all |mu| if false.  An AND (landing, a    */
/* separation conflict) is the OR of the negations: the same formula with    */
/* "failing" read as "not holding".  Not-a-number never flips (margin inf).  */
/* ------------------------------------------------------------------------ */
typedef struct { int any; double true_max, all_min; } ora_or;

static void or_init(ora_or *o) { o->any = 0; o->true_max = 0.0; o->all_min = INFINITY; }

/* one member of an OR: val = its outcome, mu = its margin (>= 0) */
static void or_add(ora_or *o, int val, double mu)
{
    if (mu != mu) mu = INFINITY;
    if (mu < o->all_min) o->all_min = mu;
    if (val) { o->any = 1; if (mu > o->true_max) o->true_max = mu; }
}

static double or_margin(const ora_or *o) { return o->any ? o->true_max : o->all_min; }

/* a bound that must hold: fails iff !(mu >= 0) (strict: !(mu > 0)) */
static void or_fail_unless(ora_or *o, double mu, int strict)
{
    int holds = strict ? (mu > 0.0) : (mu >= 0.0);
    or_add(o, !holds, fabs(mu));
}

/* ------------------------------------------------------------------------ */
/* One rollout (Alg.1 l.10-16 for one particle, one sample)                  */
/* ------------------------------------------------------------------------ */
/* Alg.1 l.10-11 simulate ALL agents to the horizon and only then test the
 * constraints (l.12-14): a constraint failure sets the aircraft's
 * weight to 0 and does not change the simulation.  Every active
 * aircraft therefore flies its own controls to H and stays in every pair test
 * of Eq. avoidance ("for every time step in the MPC horizon ... for all
 * i != j") whether or not it has already failed a constraint; a
 * failing pair zeroes both aircraft.  Only landing removes an arrival
 * from the simulation ("future time steps within that horizon will not be
 * planned for that aircraft", R18).  A state that has left the model's
 * domain (v <= 0 in Eq. hor's L sin(phi)/(m v)) keeps being propagated
 * literally; once non-finite it fails the envelope and can no longer conflict
 * (a comparison with a non-finite coordinate is false). */
void ora_rollout_replay(const ora_problem *p, const ora_derived *d, const double *u,
                        uint32_t l, uint32_t s, uint32_t k, uint64_t seed, uint32_t mpc,
                        const ora_replay *rp, ora_rollout_out *out)
{
    const int n = p->n, H = p->H;
    double st[ORA_MAX_AC][6], nx[ORA_MAX_AC][6];
    double fuel[ORA_MAX_AC], sA[ORA_MAX_AC], sB[ORA_MAX_AC], sC[ORA_MAX_AC], sN[ORA_MAX_AC];
    double mland[ORA_MAX_AC];
    int landed[ORA_MAX_AC], fly[ORA_MAX_AC], replayed[ORA_MAX_AC];
    ora_or vio[ORA_MAX_AC];
    double Z[2][ORA_MAX_NODES], W[2][ORA_MAX_NODES];
    const int G = d->ng, nblk = (2 * d->ng + 3) / 4;

    for (int i = 0; i < n; ++i) {
        memcpy(st[i], &p->x0[6 * i], sizeof(st[i]));
        fuel[i] = sA[i] = sB[i] = sC[i] = sN[i] = 0.0;
        landed[i] = -1; mland[i] = INFINITY; replayed[i] = 0;
        or_init(&vio[i]);
        if (out && out->traj) memcpy(&out->traj[((size_t)i * (H + 1)) * 6], st[i], sizeof(st[i]));
    }
    const double twoPr2 = (2.0 * p->P_r) * (2.0 * p->P_r), twoPh = 2.0 * p->P_h;

    for (int t = 0; t < H; ++t) {
        /* Alg.1 l.10: disturbance realisation for step t:
         * W(0) = Qhat v(0); W(t) = a W(t-1) + Q v(t) with Q = b Qhat.
         * Normal e = 4 blk + j of step t: component e / ng (x, y), grid point e % ng. */
        double v[4 * ((2 * ORA_MAX_NODES + 3) / 4)];
        for (int blk = 0; blk < nblk; ++blk) {
            uint32_t w[4];
            draw(TAG_WIND, l, (s & 0xFFFFu) | (k << 16), (uint32_t)t | ((uint32_t)blk << 16), mpc, seed, w);
            ora_box_muller(w[0], w[1], &v[4 * blk + 0], &v[4 * blk + 1]);
            ora_box_muller(w[2], w[3], &v[4 * blk + 2], &v[4 * blk + 3]);
        }
        for (int c = 0; c < 2; ++c)
            for (int m = 0; m < G; ++m)
                Z[c][m] = (t == 0) ? v[G * c + m] : d->a * Z[c][m] + d->b * v[G * c + m];
        for (int c = 0; c < 2; ++c)
            for (int r = 0; r < G; ++r) {
                double acc = 0.0;
                for (int m = 0; m < G; ++m) acc += d->Qhat[r * G + m] * Z[c][m];
                W[c][r] = acc;
            }

        /* Alg.1 l.11: simulate every active, not yet landed aircraft at step t. */
        for (int i = 0; i < n; ++i) {
            fly[i] = (p->first_step[i] <= t) && landed[i] < 0;
            if (!fly[i]) { memcpy(nx[i], st[i], sizeof(nx[i])); continue; }
            double wind[2];
            ora_trilinear(p, d, W[0], st[i], &wind[0]);
            ora_trilinear(p, d, W[1], st[i], &wind[1]);
            wind[0] += p->nominal[0];
            wind[1] += p->nominal[1];
            if (p->turb_sigma > 0.0) {
                uint32_t w[4];
                draw(TAG_TURB, l, (s & 0xFFFFu) | (k << 16), ((uint32_t)t >> 1) | ((uint32_t)i << 8), mpc, seed, w);
                double g0, g1;
                if ((t & 1) == 0) ora_box_muller(w[0], w[1], &g0, &g1);
                else              ora_box_muller(w[2], w[3], &g0, &g1);
                wind[0] += p->turb_sigma * g0;
                wind[1] += p->turb_sigma * g1;
            }
            const double *ut = &u[((size_t)i * H + t) * 3];
            ora_step(p, i, st[i], ut, wind, nx[i]);
            fuel[i] += p->dt * p->eta[i] * ut[0];
        }

        /* Alg.1 l.12-14: constraints at the new state j = t+1, each bound a
         * member of the aircraft's violation OR with its margin. */
        for (int i = 0; i < n; ++i) {
            if (!fly[i]) continue;
            const double *ut = &u[((size_t)i * H + t) * 3];
            int finite = 1;
            for (int a = 0; a < 6; ++a) if (!isfinite(nx[i][a])) finite = 0;
            if (!finite) or_add(&vio[i], 1, INFINITY);
            const double zs = fmax(1.0, fabs(p->z_max[i])), Ts = fmax(1.0, fabs(p->T_max[i]));
            or_fail_unless(&vio[i], (p->gamma_max[i] - fabs(ut[2])) / p->gamma_max[i], 0);
            or_fail_unless(&vio[i], (p->phi_max[i] - fabs(ut[1])) / p->phi_max[i], 1);
            or_fail_unless(&vio[i], (ut[0] - p->T_min[i]) / Ts, 0);
            or_fail_unless(&vio[i], (p->T_max[i] - ut[0]) / Ts, 0);
            or_fail_unless(&vio[i], (nx[i][2] - p->z_min[i]) / zs, 0);
            or_fail_unless(&vio[i], (p->z_max[i] - nx[i][2]) / zs, 0);
            or_fail_unless(&vio[i], (nx[i][3] - p->v_min[i]) / p->v_max[i], 0);
            or_fail_unless(&vio[i], (p->v_max[i] - nx[i][3]) / p->v_max[i], 0);
            or_fail_unless(&vio[i], (nx[i][5] - p->m_empty[i]) / p->m_empty[i], 0);

            /* landing sector (Eq. TO_init), an AND of five bounds (R10) */
            if (p->kind[i] == 0 && landed[i] < 0) {
                double x = nx[i][0], y = nx[i][1];
                double rho = sqrt(x * x + y * y);
                ora_or miss;                      /* "not landed" = OR of the failing bounds */
                or_init(&miss);
                or_fail_unless(&miss, (p->P_runway - rho) / p->P_runway, 0);
                or_fail_unless(&miss, (p->P_beta - ora_beta(x, y, nx[i][2])) / p->P_beta, 0);
                or_fail_unless(&miss, (p->P_chi - fabs(atan2(y, x))) / p->P_chi, 0);
                or_fail_unless(&miss, (p->P_chi - ora_angdist(nx[i][4] - M_PI)) / p->P_chi, 0);
                or_fail_unless(&miss, (p->P_vs - nx[i][3]) / p->P_vs, 0);
                int ln = ora_landed(p, nx[i]);
                double mu = or_margin(&miss);
                if (mu < mland[i]) mland[i] = mu;
                if (rp && rp->landed_step && mu < rp->eps) {
                    ln = rp->landed_step[i] == t + 1;         /* decision replay (R30) */
                    replayed[i] |= 1;
                }
                if (ln) landed[i] = t + 1;
            }
        }
        /* Eq. avoidance for every pair of simulated aircraft: a conflict is the AND
         * of the two failed separations; both aircraft of a conflicting pair fail. */
        for (int i = 0; i < n; ++i) {
            if (!fly[i]) continue;
            for (int q = i + 1; q < n; ++q) {
                if (!fly[q]) continue;
                int conf = ora_pair_conflict(p, nx[i], nx[q]);
                double dx = nx[i][0] - nx[q][0], dy = nx[i][1] - nx[q][1], dz = nx[i][2] - nx[q][2];
                double mm = INFINITY;
                if (isfinite(dx) && isfinite(dy) && isfinite(dz)) {
                    ora_or sep;                   /* "separated" = OR of the two separations */
                    or_init(&sep);
                    or_add(&sep, !((dx * dx + dy * dy) < twoPr2), fabs((dx * dx + dy * dy) / twoPr2 - 1.0));
                    or_add(&sep, !(fabs(dz) < twoPh), fabs(fabs(dz) / twoPh - 1.0));
                    mm = or_margin(&sep);
                }
                or_add(&vio[i], conf, mm);
                or_add(&vio[q], conf, mm);
            }
        }

        /* Alg.1 l.15: per-step cost terms at j = t+1. */
        for (int i = 0; i < n; ++i) {
            if (p->first_step[i] > t) continue;
            if (fly[i]) {
                double x = nx[i][0], y = nx[i][1], z = nx[i][2];
                double th = atan2(y, x);
                if (p->kind[i] == 1) {
                    sA[i] += ora_angdist(th - p->theta_F[i]);
                    sB[i] += fabs(p->z_tf[i] - z);
                    sC[i] += fabs(nx[i][3] - p->v_D[i]);
                } else {
                    sA[i] += ora_angdist(nx[i][4] - ora_flow_heading(x, y));
                    sB[i] += fabs(ora_beta(x, y, z) - p->beta_f[i]);
                }
                if (p->noise_w > 0.0) {
                    double q = 1.0 - (z / p->A_c) * (z / p->A_c);
                    sN[i] += 1.0 - (q > 0.0 ? q : 0.0) * ora_popdense_grid(p, d, x, y);
                }
            } else if (landed[i] >= 0) {
                /* landed earlier: "best possible cost, 1, for all remaining steps" */
                sN[i] += 1.0;
            }
        }
        for (int i = 0; i < n; ++i) {
            memcpy(st[i], nx[i], sizeof(st[i]));
            if (out && out->traj) memcpy(&out->traj[((size_t)i * (H + 1) + t + 1) * 6], st[i], sizeof(st[i]));
        }
    }

    /* Objectives J^D_T and J^A_T in [0,1]; R4-R7, R21. */
    for (int i = 0; i < n; ++i) {
        int Ha = H - p->first_step[i];
        double J = 1.0, c4[4] = { 1.0, 1.0, 1.0, 1.0 };
        if (Ha > 0) {
            double Fmax = p->dt * Ha * p->T_max[i] * p->eta[i];
            double Jfuel = Fmax > 0.0 ? clamp01(1.0 - fuel[i] / Fmax) : 1.0;
            if (p->kind[i] == 1) {
                double J1 = clamp01(1.0 - (sA[i] / Ha) / M_PI);
                double den = d->supB[i] - d->infB[i];
                double J3 = den < 1.0 ? 1.0 : clamp01((d->supB[i] - sB[i] / Ha) / den);
                double supC = fmax(p->v_max[i] - p->v_D[i], p->v_D[i] - p->v_min[i]);
                double J4 = clamp01(1.0 - (sC[i] / Ha) / supC);
                J = p->alpha_dep[0] * J1 + p->alpha_dep[1] * Jfuel + p->alpha_dep[2] * J3 + p->alpha_dep[3] * J4;
                c4[0] = J1; c4[1] = Jfuel; c4[2] = J3; c4[3] = J4;
            } else {
                double J1 = clamp01(1.0 - (sA[i] / Ha) / M_PI);
                double supE = fmax(p->beta_f[i], M_PI / 2.0 - p->beta_f[i]);
                double Jalt = clamp01(1.0 - (sB[i] / Ha) / supE);
                J = p->alpha_arr[0] * J1 + p->alpha_arr[1] * Jalt + p->alpha_arr[2] * Jfuel;
                c4[0] = J1; c4[1] = Jalt; c4[2] = Jfuel; c4[3] = 0.0;
            }
            if (p->noise_w > 0.0) J = (1.0 - p->noise_w) * J + p->noise_w * (sN[i] / Ha);
        }
        int viol = vio[i].any;
        double mv = or_margin(&vio[i]);
        if (rp && rp->viol && mv < rp->eps) { viol = rp->viol[i] != 0; replayed[i] |= 2; }
        if (out) {
            if (out->J) out->J[i] = J;
            if (out->viol) out->viol[i] = viol;
            if (out->comp) memcpy(&out->comp[4 * i], c4, sizeof(c4));
            if (out->fuel) out->fuel[i] = fuel[i];
            if (out->landed_step) out->landed_step[i] = landed[i];
            if (out->margin) out->margin[i] = mv < mland[i] ? mv : mland[i];
            if (out->margin_land) out->margin_land[i] = mland[i];
            if (out->replayed) out->replayed[i] = replayed[i];
        }
    }
}

void ora_rollout(const ora_problem *p, const ora_derived *d, const double *u,
                 uint32_t l, uint32_t s, uint32_t k, uint64_t seed, uint32_t mpc,
                 ora_rollout_out *out)
{
    ora_rollout_replay(p, d, u, l, s, k, seed, mpc, NULL, out);
}

/* Alg.1 l.8-17: every particle, S samples, W <- W * J in log2 (R24).
 * margin (nullable) [L][n]: the smallest decision margin over the S samples that
 * can change ell[l][i] -- aircraft i's violation margin and the landing margin of
 * every aircraft (a landing freezes the lander, which every pair test sees). */
void ora_evaluate_margin(const ora_problem *p, const ora_derived *d, const double *ctrl,
                         uint32_t L, uint32_t S, uint32_t k, uint64_t seed, uint32_t mpc,
                         double *ell, double *margin, int nthreads)
{
    const int n = p->n;
    const size_t row = (size_t)n * p->H * 3;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t l = 0; l < (int64_t)L; ++l) {
        double J[ORA_MAX_AC], mg[ORA_MAX_AC], ml[ORA_MAX_AC];
        int32_t viol[ORA_MAX_AC];
        ora_rollout_out o;
        memset(&o, 0, sizeof(o));
        o.J = J; o.viol = viol;
        if (margin) {
            o.margin = mg; o.margin_land = ml;
            for (int i = 0; i < n; ++i) margin[(size_t)l * n + i] = INFINITY;
        }
        for (uint32_t s = 0; s < S; ++s) {
            ora_rollout(p, d, &ctrl[(size_t)l * row], (uint32_t)l, s, k, seed, mpc, &o);
            double lmin = INFINITY;
            if (margin) for (int i = 0; i < n; ++i) if (ml[i] < lmin) lmin = ml[i];
            for (int i = 0; i < n; ++i) {
                double *e = &ell[(size_t)l * n + i];
                if (viol[i] || !(J[i] > 0.0)) *e = -INFINITY;
                else *e += log2(J[i]);
                if (margin) {
                    double *m = &margin[(size_t)l * n + i];
                    double v = mg[i] < lmin ? mg[i] : lmin;
                    if (v < *m) *m = v;
                }
            }
        }
    }
}

void ora_evaluate(const ora_problem *p, const ora_derived *d, const double *ctrl,
                  uint32_t L, uint32_t S, uint32_t k, uint64_t seed, uint32_t mpc,
                  double *ell, int nthreads)
{
    ora_evaluate_margin(p, d, ctrl, L, S, k, seed, mpc, ell, NULL, nthreads);
}

/* Alg.1 l.3-5: uniform controls in [min, max]. */
void ora_init_population(const ora_problem *p, uint32_t L, uint64_t seed, uint32_t mpc, double *ctrl)
{
    const int n = p->n, H = p->H;
    for (uint32_t l = 0; l < L; ++l)
        for (int i = 0; i < n; ++i)
            for (int t = 0; t < H; ++t) {
                uint32_t w[4];
                draw(TAG_INIT, l, 0, (uint32_t)t | ((uint32_t)i << 8), mpc, seed, w);
                double *c = &ctrl[(((size_t)l * n + i) * H + t) * 3];
                c[0] = p->T_min[i] + (p->T_max[i] - p->T_min[i]) * ora_u24(w[0]);
                c[1] = -p->phi_max[i] + 2.0 * p->phi_max[i] * ora_u24(w[1]);
                c[2] = -p->gamma_max[i] + 2.0 * p->gamma_max[i] * ora_u24(w[2]);
            }
}

/* Per-aircraft MH acceptance (SURVEY Q1 variant / N2, reading R46): the
 * joint rules of ora_mh_accept applied to one aircraft's log2 weights, with
 * the uniform from the MH stream at counter (l, k<<16, i). */
int ora_mh_accept_aircraft(double ell_cur, double ell_prop, uint32_t l, uint32_t i, uint32_t k, uint64_t seed,
                           uint32_t mpc)
{
    if (ell_cur == -INFINITY) return 1;
    if (ell_prop == -INFINITY) return 0;
    double delta = ell_prop - ell_cur;
    if (delta >= 0.0) return 1;
    uint32_t w[4];
    draw(TAG_MH, l, k << 16, i, mpc, seed, w);
    uint64_t r = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    double u53 = (double)(r >> 11) * 0x1.0p-53;
    return u53 < ora_det_exp2(delta);
}

/* Warm start across MPC steps (reading R45): the previous
 * winner, shifted one step (row t <- row t+1, last row repeated), seeds the
 * first Lw particles of aircraft that were in the previous window; particle 0
 * takes it exactly, particles 1..Lw-1 add N(0, sigma^2) per component from the
 * INIT stream with x1 = 1<<16 (two Box-Muller pairs as in the proposal);
 * clamp as for proposals (R16).  Every other (particle, aircraft) row is the
 * fresh uniform draw of ora_init_population.
 * prev: [n][H][3] previous winner rows mapped to the current aircraft index;
 * has_prev[i] = 0 where aircraft i has none. */
void ora_init_population_warm(const ora_problem *p, uint32_t L, uint64_t seed, uint32_t mpc,
                              const double *prev, const int32_t *has_prev, uint32_t Lw,
                              const double sigma[3], int clamp, double *ctrl)
{
    const int n = p->n, H = p->H;
    ora_init_population(p, L, seed, mpc, ctrl);
    for (uint32_t l = 0; l < L && l < Lw; ++l)
        for (int i = 0; i < n; ++i) {
            if (!has_prev[i]) continue;
            for (int t = 0; t < H; ++t) {
                const double *base = &prev[((size_t)i * H + (t + 1 < H ? t + 1 : H - 1)) * 3];
                double *c = &ctrl[(((size_t)l * n + i) * H + t) * 3];
                if (l == 0) {
                    c[0] = base[0]; c[1] = base[1]; c[2] = base[2];
                    continue;
                }
                uint32_t w[4];
                draw(TAG_INIT, l, 1u << 16, (uint32_t)t | ((uint32_t)i << 8), mpc, seed, w);
                double z[4];
                ora_box_muller(w[0], w[1], &z[0], &z[1]);
                ora_box_muller(w[2], w[3], &z[2], &z[3]);
                for (int q = 0; q < 3; ++q) {
                    double v = base[q] + sigma[q] * z[q];
                    if (clamp) {
                        double lo = q == 0 ? p->T_min[i] : (q == 1 ? -p->phi_max[i] : -p->gamma_max[i]);
                        double hi = q == 0 ? p->T_max[i] : (q == 1 ? p->phi_max[i] : p->gamma_max[i]);
                        if (v < lo) v = lo;
                        if (v > hi) v = hi;
                    }
                    c[q] = v;
                }
            }
        }
}

/* MH accept/reject on the joint log2 weight (R1). */
int ora_mh_accept(double lam_cur, double lam_prop, uint32_t l, uint32_t k, uint64_t seed, uint32_t mpc)
{
    if (lam_cur == -INFINITY) return 1;
    if (lam_prop == -INFINITY) return 0;
    double delta = lam_prop - lam_cur;
    if (delta >= 0.0) return 1;
    uint64_t r = ora_r64(TAG_MH, l, k, seed, mpc);
    double u53 = (double)(r >> 11) * 0x1.0p-53;
    return u53 < ora_det_exp2(delta);
}

/* Systematic resampling of one aircraft column (K96; R25) into M
 * new particles: slot j in [0, M) takes min{ l : C_l > floor((j Q + R) / M) }
 * (M = L normally; M < L when the particle count shrinks over rounds). */
int ora_resample_column_m(const double *ell, uint32_t L, uint32_t M, uint32_t i, uint32_t k,
                          uint64_t seed, uint32_t mpc, int32_t *anc,
                          uint64_t *q_out, uint64_t *Q_out, uint64_t *R_out)
{
    double m = -INFINITY;
    for (uint32_t l = 0; l < L; ++l) if (ell[l] > m) m = ell[l];
    int infeasible = (m == -INFINITY);
    uint64_t *C = (uint64_t *)malloc(sizeof(uint64_t) * (L ? L : 1));
    uint64_t acc = 0;
    for (uint32_t l = 0; l < L; ++l) {
        uint64_t q = infeasible ? 1 : ora_det_quant(ell[l] - m);
        if (q_out) q_out[l] = q;
        acc += q;
        C[l] = acc;
    }
    uint64_t Q = acc;
    uint64_t r = ora_r64(TAG_RESAMPLE, i, k, seed, mpc);
    uint64_t R = (uint64_t)(((unsigned __int128)r * (unsigned __int128)Q) >> 64);
    uint32_t a = 0;
    for (uint32_t j = 0; j < M; ++j) {
        unsigned __int128 num = (unsigned __int128)j * Q + R;
        uint64_t tj = (uint64_t)(num / M);
        /* min{ l : C_l > t_j } by a forward scan: t_j is non-decreasing in j, so the
         * scan position never moves back; t_j < Q = C_{L-1} bounds it */
        while (C[a] <= tj) ++a;
        anc[j] = (int32_t)a;
    }
    if (Q_out) *Q_out = Q;
    if (R_out) *R_out = R;
    free(C);
    return infeasible;
}

int ora_resample_column(const double *ell, uint32_t L, uint32_t i, uint32_t k,
                        uint64_t seed, uint32_t mpc, int32_t *anc,
                        uint64_t *q_out, uint64_t *Q_out, uint64_t *R_out)
{
    return ora_resample_column_m(ell, L, L, i, k, seed, mpc, anc, q_out, Q_out, R_out);
}

/* Particle count of round k (R44): linear from L to L_final over K rounds,
 * exact integer arithmetic. */
uint32_t ora_particles_of(uint32_t L, uint32_t L_final, uint32_t K, uint32_t k)
{
    if (L_final == 0 || L_final >= L || K < 2) return L;
    return L - (uint32_t)(((uint64_t)(L - L_final) * k) / (K - 1));
}

/* Alg.1 l.23: controls + Gaussian white noise, sigma per
 * component; optional clamp to the envelope (R16). */
void ora_perturb_row(const ora_problem *p, int i, const double *parent_row, double *out_row,
                     uint32_t l, uint32_t k, uint64_t seed, uint32_t mpc,
                     const double sigma[3], int clamp)
{
    for (int t = 0; t < p->H; ++t) {
        uint32_t w[4];
        draw(TAG_PERTURB, l, k << 16, (uint32_t)t | ((uint32_t)i << 8), mpc, seed, w);
        double z[4];
        ora_box_muller(w[0], w[1], &z[0], &z[1]);
        ora_box_muller(w[2], w[3], &z[2], &z[3]);
        for (int c = 0; c < 3; ++c) {
            double v = parent_row[3 * t + c] + sigma[c] * z[c];
            if (clamp) {
                double lo = c == 0 ? p->T_min[i] : (c == 1 ? -p->phi_max[i] : -p->gamma_max[i]);
                double hi = c == 0 ? p->T_max[i] : (c == 1 ? p->phi_max[i] : p->gamma_max[i]);
                if (v < lo) v = lo;
                if (v > hi) v = hi;
            }
            out_row[3 * t + c] = v;
        }
    }
}

/* argmax_l prod_i W_il; a zero weight disqualifies; ties -> lowest l (R27). */
int64_t ora_select(const double *lam, uint32_t L)
{
    int64_t best = -1;
    for (uint32_t l = 0; l < L; ++l) {
        if (lam[l] == -INFINITY) continue;
        if (best < 0 || lam[l] > lam[best]) best = l;
    }
    return best;
}

static double lambda_of(const double *ell_row, int n)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += ell_row[i];
    return s;
}

/* Algorithm 1 with the MH move of R1. */
int ora_run_smc(const ora_problem *p, const ora_smc_cfg *cfg, double *best_ctrl,
                double *best_lambda, int64_t *best_index, double *stats)
{
    ora_derived d;
    if (ora_derive(p, &d) != 0) return -1;
    const uint32_t L = cfg->L;
    const int n = p->n, H = p->H;
    const size_t row = (size_t)n * H * 3;
    double *cur = (double *)calloc(L * row + 1, sizeof(double));   /* x'  */
    double *prop = (double *)calloc(L * row + 1, sizeof(double));  /* x*  */
    double *surv = (double *)calloc(L * row + 1, sizeof(double));
    double *ell_c = (double *)malloc(sizeof(double) * (L * (size_t)n + 1));
    double *ell_p = (double *)malloc(sizeof(double) * (L * (size_t)n + 1));
    double *ell_s = (double *)malloc(sizeof(double) * (L * (size_t)n + 1));
    double *lam = (double *)malloc(sizeof(double) * (L + 1));
    double *lam_c = (double *)malloc(sizeof(double) * (L + 1));
    double *lam_p = (double *)malloc(sizeof(double) * (L + 1));
    double *col = (double *)malloc(sizeof(double) * (L + 1));
    int32_t *anc = (int32_t *)malloc(sizeof(int32_t) * ((size_t)L * n + 1));

    ora_init_population(p, L, cfg->seed, cfg->mpc, cur);           /* Alg.1 l.1-5 */
    uint32_t Lk = L;
    for (uint32_t k = 0; k < cfg->K; ++k) {
        uint32_t S = cfg->sched_paper ? (uint32_t)ora_sample_schedule((int)k) : cfg->S;
        Lk = ora_particles_of(L, cfg->L_final, cfg->K, k);
        const uint32_t Ln = ora_particles_of(L, cfg->L_final, cfg->K, k + 1);
        const double ell0 = -log2((double)Lk);
        uint64_t accepted = 0;
        if (k == 0) {
            for (size_t e = 0; e < Lk * (size_t)n; ++e) ell_s[e] = ell0;
            ora_evaluate(p, &d, cur, Lk, S, k, cfg->seed, cfg->mpc, ell_s, cfg->nthreads);
            memcpy(surv, cur, sizeof(double) * Lk * row);
        } else if (!cfg->mh) {                                      /* paper-literal: x* replaces x' */
            for (size_t e = 0; e < Lk * (size_t)n; ++e) ell_s[e] = ell0;
            ora_evaluate(p, &d, prop, Lk, S, k, cfg->seed, cfg->mpc, ell_s, cfg->nthreads);
            memcpy(surv, prop, sizeof(double) * Lk * row);
            accepted = Lk;
        } else if (cfg->mh == 2) {                                  /* per-aircraft MH (R46) */
            for (size_t e = 0; e < Lk * (size_t)n; ++e) { ell_c[e] = ell0; ell_p[e] = ell0; }
            ora_evaluate(p, &d, cur, Lk, S, k, cfg->seed, cfg->mpc, ell_c, cfg->nthreads);
            ora_evaluate(p, &d, prop, Lk, S, k, cfg->seed, cfg->mpc, ell_p, cfg->nthreads);
            for (uint32_t l = 0; l < Lk; ++l) {
                lam_c[l] = lambda_of(&ell_c[(size_t)l * n], n);
                lam_p[l] = lambda_of(&ell_p[(size_t)l * n], n);
                for (int i = 0; i < n; ++i) {
                    const size_t e = (size_t)l * n + i;
                    int acc = ora_mh_accept_aircraft(ell_c[e], ell_p[e], l, (uint32_t)i, k, cfg->seed, cfg->mpc);
                    accepted += acc;
                    const size_t o = (size_t)l * row + (size_t)i * H * 3;
                    memcpy(&surv[o], acc ? &prop[o] : &cur[o], sizeof(double) * H * 3);
                    ell_s[e] = acc ? ell_p[e] : ell_c[e];
                }
            }
        } else {
            for (size_t e = 0; e < Lk * (size_t)n; ++e) { ell_c[e] = ell0; ell_p[e] = ell0; }
            ora_evaluate(p, &d, cur, Lk, S, k, cfg->seed, cfg->mpc, ell_c, cfg->nthreads);
            ora_evaluate(p, &d, prop, Lk, S, k, cfg->seed, cfg->mpc, ell_p, cfg->nthreads);
            for (uint32_t l = 0; l < Lk; ++l) {
                double lc = lambda_of(&ell_c[(size_t)l * n], n);
                double lp = lambda_of(&ell_p[(size_t)l * n], n);
                int acc = ora_mh_accept(lc, lp, l, k, cfg->seed, cfg->mpc);
                accepted += acc;
                const double *src = acc ? &prop[l * row] : &cur[l * row];
                memcpy(&surv[l * row], src, sizeof(double) * row);
                memcpy(&ell_s[(size_t)l * n], acc ? &ell_p[(size_t)l * n] : &ell_c[(size_t)l * n], sizeof(double) * n);
            }
        }
        for (uint32_t l = 0; l < Lk; ++l) lam[l] = lambda_of(&ell_s[(size_t)l * n], n);
        double ess_min = INFINITY;
        int n_inf = 0;
        if (k + 1 < cfg->K) {
            /* Alg.1 l.22: per-aircraft resampling */
            for (int i = 0; i < n; ++i) {
                for (uint32_t l = 0; l < Lk; ++l) col[l] = ell_s[(size_t)l * n + i];
                n_inf += ora_resample_column_m(col, Lk, Ln, (uint32_t)i, k, cfg->seed, cfg->mpc,
                                               &anc[(size_t)i * L], NULL, NULL, NULL);
            }
            /* recombine and perturb (Alg.1 l.23); weights reset happens at evaluation */
            double sig[3];
            double f = pow(cfg->anneal, (double)k);
            for (int c = 0; c < 3; ++c) sig[c] = cfg->sigma[c] * f;
            for (uint32_t j = 0; j < Ln; ++j)
                for (int i = 0; i < n; ++i) {
                    int32_t a = anc[(size_t)i * L + j];
                    const double *src = &surv[(size_t)a * row + (size_t)i * H * 3];
                    double *dst = &cur[(size_t)j * row + (size_t)i * H * 3];
                    memcpy(dst, src, sizeof(double) * H * 3);
                    ora_perturb_row(p, i, dst, &prop[(size_t)j * row + (size_t)i * H * 3],
                                    j, k, cfg->seed, cfg->mpc, sig, (int)cfg->clamp);
                }
        }
        for (int i = 0; i < n; ++i) {
            double mx = -INFINITY, s1 = 0.0, s2 = 0.0;
            for (uint32_t l = 0; l < Lk; ++l) if (ell_s[(size_t)l * n + i] > mx) mx = ell_s[(size_t)l * n + i];
            if (mx == -INFINITY) { ess_min = 0.0; continue; }
            for (uint32_t l = 0; l < Lk; ++l) {
                double w = exp2(ell_s[(size_t)l * n + i] - mx);
                s1 += w; s2 += w * w;
            }
            double ess = s1 * s1 / s2;
            if (ess < ess_min) ess_min = ess;
        }
        if (stats) {
            int64_t b = ora_select(lam, Lk);
            stats[4 * k + 0] = b >= 0 ? lam[b] : -INFINITY;
            stats[4 * k + 1] = k == 0 ? 1.0 : (double)accepted / ((double)Lk * (cfg->mh == 2 ? n : 1));
            stats[4 * k + 2] = ess_min;
            stats[4 * k + 3] = (double)n_inf;
        }
    }
    int64_t b;
    if (cfg->mh == 2 && cfg->K >= 2) {
        /* per-aircraft survivors mix two joint evaluations; the pick is made over
         * the jointly evaluated candidates of the last round: lambda of x'_l and x*_l, ties ->
         * lowest l, then x' before x* (R46) */
        int64_t bc = -1;
        double bl = -INFINITY;
        for (uint32_t l = 0; l < Lk; ++l)
            for (int c = 0; c < 2; ++c) {
                double v = c ? lam_p[l] : lam_c[l];
                if (v == -INFINITY) continue;
                if (bc < 0 || v > bl) { bl = v; bc = 2 * (int64_t)l + c; }
            }
        b = bc >= 0 ? bc / 2 : -1;
        if (best_index) *best_index = b;
        if (best_lambda) *best_lambda = bl;
        if (best_ctrl && bc >= 0) memcpy(best_ctrl, (bc & 1) ? &prop[(size_t)b * row] : &cur[(size_t)b * row],
                                         sizeof(double) * row);
    } else {
        b = ora_select(lam, Lk);                                     /* Alg.1 l.27 */
        if (best_index) *best_index = b;
        if (best_lambda) *best_lambda = b >= 0 ? lam[b] : -INFINITY;
        if (best_ctrl && b >= 0) memcpy(best_ctrl, &surv[(size_t)b * row], sizeof(double) * row);
    }
    free(cur); free(prop); free(surv); free(ell_c); free(ell_p); free(ell_s);
    free(lam); free(lam_c); free(lam_p); free(col); free(anc);
    ora_free_derived(&d);
    return b >= 0 ? 0 : 2;
}

/* MPC apply: first control of the winner, realised wind (PLANT streams). */
void ora_plant_step(const ora_problem *p, const ora_derived *d, const double *states,
                    const double *u0, uint64_t seed, uint32_t mpc, double *Zplant,
                    int32_t *zinit, double *next, int32_t *flags)
{
    const int G = d->ng, nblk = (2 * d->ng + 3) / 4;
    double v[4 * ((2 * ORA_MAX_NODES + 3) / 4)], W[2][ORA_MAX_NODES];
    for (int blk = 0; blk < nblk; ++blk) {
        uint32_t w[4];
        draw(TAG_PLANT_WIND, 0, 0, (uint32_t)blk << 16, mpc, seed, w);
        ora_box_muller(w[0], w[1], &v[4 * blk + 0], &v[4 * blk + 1]);
        ora_box_muller(w[2], w[3], &v[4 * blk + 2], &v[4 * blk + 3]);
    }
    for (int e = 0; e < 2 * G; ++e) Zplant[e] = *zinit ? d->a * Zplant[e] + d->b * v[e] : v[e];
    *zinit = 1;
    for (int c = 0; c < 2; ++c)
        for (int r = 0; r < G; ++r) {
            double acc = 0.0;
            for (int m = 0; m < G; ++m) acc += d->Qhat[r * G + m] * Zplant[G * c + m];
            W[c][r] = acc;
        }
    for (int i = 0; i < p->n; ++i) {
        const double *st = &states[6 * i];
        flags[i] = 0;
        if (p->first_step[i] != 0) { memcpy(&next[6 * i], st, 6 * sizeof(double)); continue; }
        double wind[2];
        ora_trilinear(p, d, W[0], st, &wind[0]);
        ora_trilinear(p, d, W[1], st, &wind[1]);
        wind[0] += p->nominal[0];
        wind[1] += p->nominal[1];
        if (p->turb_sigma > 0.0) {
            uint32_t w[4];
            double g0, g1;
            draw(TAG_PLANT_TURB, 0, 0, (uint32_t)i << 8, mpc, seed, w);
            ora_box_muller(w[0], w[1], &g0, &g1);
            wind[0] += p->turb_sigma * g0;
            wind[1] += p->turb_sigma * g1;
        }
        ora_step(p, i, st, &u0[3 * i], wind, &next[6 * i]);
        const double *nx = &next[6 * i];
        if (p->kind[i] == 0 && ora_landed(p, nx)) flags[i] |= 1;
        if (p->kind[i] == 1 && sqrt(nx[0] * nx[0] + nx[1] * nx[1]) >= p->tma_radius) flags[i] |= 2;
        if (ora_unary_violation(p, i, &u0[3 * i], nx)) flags[i] |= 4;
    }
}

/* ------------------------------------------------------------------------ */
/* Fuel estimates from recorded traces (section 5).    */
/* ------------------------------------------------------------------------ */
static double clamp_gamma(double sg, double gmax, int *flag)
{
    /* gamma = asin(dz / (dt v)); |sin gamma| > 1 (degenerate data) -> +-gamma_max (R47) */
    if (sg > 1.0 || sg < -1.0 || sg != sg) { *flag = 1; return sg > 0.0 ? gmax : -gmax; }
    return asin(sg);
}

static double wrap_pi(double d) { return d - 2.0 * M_PI * floor((d + M_PI) / (2.0 * M_PI)); }

/* Fuel estimate 1: fly the recorded heading, match the next
 * airspeed; the position mismatch is the wind residual.  Mass runs forward
 * with eta = Cf1 (1 + v / Cf2) and T from the airspeed change (bank 0);
 * negative burn is clamped to 0.  Returns flags (bit0 gamma clamped). */
int ora_fuel_estimate1(const ora_problem *p, int i, const double *Cf, const double *trace, int K, double dt,
                       double m1, double *m_out, double *w_out)
{
    int flags = 0;
    double m = m1;
    m_out[0] = m;
    for (int k = 0; k + 1 < K; ++k) {
        const double *a = &trace[5 * k], *b = &trace[5 * (k + 1)];
        double vs = a[3];
        double eta = Cf[0] * (1.0 + vs / Cf[1]);
        int fl = 0;
        double gam = clamp_gamma((b[2] - a[2]) / (dt * vs), p->gamma_max[i], &fl);
        flags |= fl;
        w_out[2 * k] = (b[0] - a[0]) / dt - vs * cos(a[4]) * cos(gam);
        w_out[2 * k + 1] = (b[1] - a[1]) / dt - vs * sin(a[4]) * cos(gam);
        double st[6] = { a[0], a[1], a[2], vs, a[4], m };
        double L, D;
        ora_lift_drag(p, i, st, 0.0, &L, &D);
        double T = m * (b[3] - vs) / dt + D + m * p->g * sin(gam);
        double burn = dt * eta * T;
        if (!(burn > 0.0)) burn = 0.0;                 /* negative or undefined (R47): none */
        m -= burn;
        m_out[k + 1] = m;
    }
    if (K >= 1) { w_out[2 * (K - 1)] = 0.0; w_out[2 * (K - 1) + 1] = 0.0; }
    return flags;
}

/* Fuel estimate 2: dead reckoning, no wind.  Airspeed from the
 * 3-D distance, track angle from the two positions, bank from the heading
 * change; T from the airspeed change to the next sample.  A zero-distance
 * interval burns nothing and is flagged (bit1).  Returns flags. */
int ora_fuel_estimate2(const ora_problem *p, int i, const double *Cf, const double *trace, int K, double dt,
                       double m1, double *m_out)
{
    int flags = 0;
    double m = m1;
    m_out[0] = m;
    for (int k = 0; k + 1 < K; ++k) {
        const double *a = &trace[5 * k], *b = &trace[5 * (k + 1)];
        double dx = b[0] - a[0], dy = b[1] - a[1], dz = b[2] - a[2];
        double d = sqrt(dx * dx + dy * dy + dz * dz);
        if (!(d > 0.0)) { flags |= 2; m_out[k + 1] = m; continue; }
        double vh = d / dt;
        double eta = Cf[0] * (1.0 + vh / Cf[1]);
        int fl = 0;
        double gam = clamp_gamma(dz / (dt * vh), p->gamma_max[i], &fl);
        flags |= fl;
        double chih = atan2(dy, dx);                   /* tan^-1(dy/dx) on the full circle (R47) */
        double dchi = wrap_pi(chih - a[4]);
        double phi = atan(dchi * vh / (p->g * dt));
        double st[6] = { a[0], a[1], a[2], vh, a[4], m };
        double L, D;
        ora_lift_drag(p, i, st, phi, &L, &D);
        double T = m * (b[3] - vh) / dt + D + m * p->g * sin(gam);
        double burn = dt * eta * T;
        if (!(burn > 0.0)) burn = 0.0;                 /* negative or undefined (R47): none */
        m -= burn;
        m_out[k + 1] = m;
    }
    return flags;
}

/*
 * smc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, FP64 CPU oracle for the SMC-in-MPC hot path of
 * Eele & Maciejowski, "Sequential Monte Carlo Optimisation for Air Traffic
 * Management", CUED/F-INFENG/TR.693 (arxiv 1506.02869).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1506_02869_b200/, libsmcatm) never includes, links or calls it;
 * the two implementations share no code, headers or tables.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation named
 * beside it).  Readings of silent or garbled passages are numbered R1..Rn and
 * listed in DESIGN.md section 3.
 */
#ifndef SMC_ORACLE_H
#define SMC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORA_MAX_AC 64
#define ORA_MAX_NODES 64            /* wind-grid points N_x N_y N_z */

/* One planning problem: N aircraft, horizon H, plus every
 * constant the method needs.  Per-aircraft arrays have length n. */
typedef struct {
    int32_t n, H;
    double dt, g;
    int32_t density_mode;           /* 0: ISA troposphere, 1: constant rho_const (R12) */
    double rho_const;
    /* per aircraft */
    const int32_t *kind;            /* 0 arrival, 1 departure */
    const int32_t *first_step;      /* e_i in [0,H]  (rolling window) */
    const double *x0;               /* [n][6] = x, y, z, v, chi, m */
    const double *theta_F, *z_tf, *v_D;   /* departure goals */
    const double *beta_f;           /* arrival nominal descent angle */
    /* aircraft-type constants, expanded per aircraft */
    const double *S, *cd0, *cd2, *eta, *m_empty;
    const double *T_min, *T_max, *v_min, *v_max, *gamma_max, *phi_max, *z_min, *z_max;
    /* landing envelope (Eq. TO_init) and separation cylinder */
    double P_runway, P_beta, P_chi, P_vs, P_r, P_h;
    /* objective weights (Table coeff) */
    double alpha_dep[4];            /* bearing A, fuel, altitude B, speed C */
    double alpha_arr[3];            /* heading D, altitude E, fuel */
    /* noise extension */
    double noise_w, A_c;
    int32_t n_centres;
    const double *centres;          /* [n_centres][3] = x_m, y_m, radius_m */
    int32_t pop_nx, pop_ny;
    double pop_x0, pop_y0, pop_dx;  /* grid origin / spacing in metres */
    /* wind model */
    double wind_lo[3], wind_hi[3];  /* grid box corners */
    double sigma_lo, sigma_hi;      /* sigma(z) at wind_lo[2] / wind_hi[2], linear */
    double beta_w, gamma_w, lambda_t;
    double nominal[2];              /* forecast (nominal) wind */
    double turb_sigma;              /* R15 */
    double tma_radius;              /* D_TMA */
    int32_t wind_n[3];              /* grid points per axis N_x, N_y, N_z; 0 -> 2 (the
                                       paper's eight-point grid) */
} ora_problem;

/* Derived, per-problem constants: Qhat = chol(Rhat), a, b,
 * departure B normalisers, population grid. */
typedef struct {
    int32_t nx, ny, nz, ng;         /* grid points per axis, ng = nx ny nz */
    double Rhat[ORA_MAX_NODES * ORA_MAX_NODES], Qhat[ORA_MAX_NODES * ORA_MAX_NODES];   /* [ng][ng] */
    double a, b;
    double supB[ORA_MAX_AC], infB[ORA_MAX_AC];
    double *pop;                    /* [pop_ny][pop_nx] owned */
} ora_derived;

/* ---- counter-based random streams (R37) ---- */
void     ora_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double   ora_u24(uint32_t w);
void     ora_box_muller(uint32_t w0, uint32_t w1, double *n0, double *n1);
uint64_t ora_r64(uint32_t tag, uint32_t x0, uint32_t k, uint64_t seed, uint32_t mpc);

/* ---- deterministic exp2 / weight quantiser (R26) ---- */
double   ora_det_exp2(double y);
uint64_t ora_det_quant(double d);

/* ---- scenario precompute ---- */
int    ora_derive(const ora_problem *p, ora_derived *d);
void   ora_free_derived(ora_derived *d);
double ora_popdense_point(const ora_problem *p, double x, double y);
double ora_popdense_grid(const ora_problem *p, const ora_derived *d, double x, double y);
void   ora_trilinear(const ora_problem *p, const ora_derived *d, const double *W /*[ng]*/,
                     const double pos[3], double *w);
int    ora_sample_schedule(int J);

/* ---- models ---- */
void ora_lift_drag(const ora_problem *p, int i, const double st[6], double phi,
                   double *lift, double *drag);
void ora_step(const ora_problem *p, int i, const double st[6], const double u[3],
              const double wind[2], double out[6]);
int  ora_landed(const ora_problem *p, const double st[6]);
int  ora_unary_violation(const ora_problem *p, int i, const double u[3], const double st[6]);
int  ora_pair_conflict(const ora_problem *p, const double a[6], const double b[6]);
double ora_flow_heading(double x, double y);
double ora_arc_length(double x, double y);
double ora_beta(double x, double y, double z);
double ora_angdist(double d);

/* ---- one rollout: particle l, sample s of round k, candidate controls u ----
 * u: [n][H][3] (T, phi, gamma).  Outputs per aircraft (any may be NULL):
 *   J[n]      utility J_T in [0,1] (meaningless if viol)
 *   viol[n]   1 if any constraint failed in this sample
 *   comp[n][4] components (dep: J1,Jfuel,J3,J4; arr: J1,Jalt,Jfuel,0)
 *   traj[n][H+1][6] states, fuel[n], landed_step[n] (-1 if not landed)
 *   margin[n]  decision margin of the aircraft's outcome (R30): the smaller of
 *              its violation margin and its landing margin; a perturbation of
 *              every compared quantity by less than this relative amount cannot
 *              change viol[i] or landed_step[i]
 *   margin_land[n] the landing margin alone (inf for departures)
 *   replayed[n] bit0: a landing decision was replayed, bit1: viol was replayed */
typedef struct {
    double *J, *comp, *traj, *fuel, *margin, *margin_land;
    int32_t *viol, *landed_step, *replayed;
} ora_rollout_out;

/* Decision replay (R30): where the oracle's own margin of a
 * decision is below eps, it takes the decision another implementation made
 * (landed_step[n], viol[n]; either may be NULL) and computes every continuous
 * quantity from there.  Decisions with margin >= eps are never replayed. */
typedef struct {
    const int32_t *landed_step;
    const int32_t *viol;
    double eps;
} ora_replay;

void ora_rollout(const ora_problem *p, const ora_derived *d, const double *u,
                 uint32_t l, uint32_t s, uint32_t k, uint64_t seed, uint32_t mpc,
                 ora_rollout_out *out);
void ora_rollout_replay(const ora_problem *p, const ora_derived *d, const double *u,
                        uint32_t l, uint32_t s, uint32_t k, uint64_t seed, uint32_t mpc,
                        const ora_replay *rp, ora_rollout_out *out);

/* Alg.1 l.9-18 for a whole population: ell[l][i] += sum_s log2 J (or -inf).
 * ell must be pre-set by the caller (normally -log2 L).  margin
 * (nullable, [L][n]): smallest margin over the samples of the decisions that
 * can change ell[l][i] (aircraft i's violation, every aircraft's landing). */
void ora_evaluate(const ora_problem *p, const ora_derived *d, const double *ctrl,
                  uint32_t L, uint32_t S, uint32_t k, uint64_t seed, uint32_t mpc,
                  double *ell, int nthreads);
void ora_evaluate_margin(const ora_problem *p, const ora_derived *d, const double *ctrl,
                         uint32_t L, uint32_t S, uint32_t k, uint64_t seed, uint32_t mpc,
                         double *ell, double *margin, int nthreads);

/* Population init, Alg.1 l.1-5: ctrl[L][n][H][3]. */
void ora_init_population(const ora_problem *p, uint32_t L, uint64_t seed, uint32_t mpc,
                         double *ctrl);

/* Per-aircraft MH acceptance (R46): joint rules on one aircraft's log2 weights,
 * uniform from the MH stream at counter (l, k<<16, i). Returns 1 = accept x*_i. */
int ora_mh_accept_aircraft(double ell_cur, double ell_prop, uint32_t l, uint32_t i, uint32_t k, uint64_t seed,
                           uint32_t mpc);

/* Warm start (R45): first Lw particles from the shifted previous winner. */
void ora_init_population_warm(const ora_problem *p, uint32_t L, uint64_t seed, uint32_t mpc,
                              const double *prev, const int32_t *has_prev, uint32_t Lw,
                              const double sigma[3], int clamp, double *ctrl);

/* MH accept for particle l in round k (R1). Returns 1 = accept proposal. */
int ora_mh_accept(double lam_cur, double lam_prop, uint32_t l, uint32_t k,
                  uint64_t seed, uint32_t mpc);

/* Per-aircraft systematic resampling of one column (R25).
 * ell[L] (log2 weights) -> anc[L].  Returns 1 if the column was all -inf. */
int ora_resample_column(const double *ell, uint32_t L, uint32_t i, uint32_t k,
                        uint64_t seed, uint32_t mpc, int32_t *anc,
                        uint64_t *q_out, uint64_t *Q_out, uint64_t *R_out);

int ora_resample_column_m(const double *ell, uint32_t L, uint32_t M, uint32_t i, uint32_t k,
                          uint64_t seed, uint32_t mpc, int32_t *anc,
                          uint64_t *q_out, uint64_t *Q_out, uint64_t *R_out);
uint32_t ora_particles_of(uint32_t L, uint32_t L_final, uint32_t K, uint32_t k);

/* Gaussian perturbation of one control row (Alg.1 l.23). */
void ora_perturb_row(const ora_problem *p, int i, const double *parent_row /*[H][3]*/,
                     double *out_row, uint32_t l, uint32_t k, uint64_t seed, uint32_t mpc,
                     const double sigma[3], int clamp);

/* Final selection: argmax_l lam, ties -> lowest l; -1 if none finite. */
int64_t ora_select(const double *lam, uint32_t L);

/* Full Alg.1 (+ MH move, R1) for K rounds.  best_ctrl: [n][H][3].
 * stats (nullable): per round {best_lambda, accept_rate, ess_min, n_infeasible}. */
typedef struct {
    uint32_t L, S, K, sched_paper, mh, clamp;   /* mh: 0 paper Alg.1, 1 joint MH (R1), 2 per-aircraft (R46) */
    double sigma[3], anneal;
    uint64_t seed;
    uint32_t mpc;
    int nthreads;
    uint32_t L_final;               /* particle count of the last round (0 = constant L) */
} ora_smc_cfg;

int ora_run_smc(const ora_problem *p, const ora_smc_cfg *cfg, double *best_ctrl,
                double *best_lambda, int64_t *best_index, double *stats);

/* Plant advance for one MPC step: applies u0[n][3] to aircraft with
 * first_step == 0, realised wind from the PLANT streams (Z carried in
 * Zplant[2][ng], *zinit = 0 on the first call).  flags: bit0 landed, bit1 exited. */
void ora_plant_step(const ora_problem *p, const ora_derived *d, const double *states,
                    const double *u0, uint64_t seed, uint32_t mpc, double *Zplant,
                    int32_t *zinit, double *next, int32_t *flags);

/* Fuel estimates on a recorded trace (section 5): trace [K][5] =
 * x, y, z, v_s, chi per sample at spacing dt, aircraft constants of problem
 * aircraft i (drag polar, gamma_max, density), Cf = {Cf1, Cf2}.  m_out [K]
 * mass series; w_out [K][2] wind residuals of estimate 1 (last row 0).
 * Return flags: bit0 gamma clamped, bit1 zero-distance interval (estimate 2). */
int ora_fuel_estimate1(const ora_problem *p, int i, const double *Cf, const double *trace, int K, double dt,
                       double m1, double *m_out, double *w_out);
int ora_fuel_estimate2(const ora_problem *p, int i, const double *Cf, const double *trace, int K, double dt,
                       double m1, double *m_out);

#ifdef __cplusplus
}
#endif
#endif

/*
 * smcatm.h -- C ABI of libsmcatm, the B200-native (sm_100a) hot path of
 * Eele & Maciejowski, "Sequential Monte Carlo Optimisation for Air Traffic
 * Management", CUED/F-INFENG/TR.693, 2015 (arxiv 1506.02869).
 *
 * Citations: P:n = line n of the paper's text; R<n> = reading n in
 * DESIGN.md section 3 (how a silent / garbled passage is interpreted).
 *
 * Conventions for every entry point
 *   - All functions return smc_status; nothing throws across the ABI.  On a
 *     non-OK status, smc_last_error(ctx) holds a one-line message.
 *   - Host arrays are owned by the caller; the library copies what it needs
 *     during the call and never retains a host pointer.
 *   - Device memory: the caller provides ONE device workspace of
 *     smc_workspace_bytes(cfg) bytes (e.g. a torch uint8 CUDA tensor) that
 *     must outlive the context.  The library allocates no device memory.
 *   - Streams: every call is ordered on cfg.stream (a cudaStream_t; NULL =
 *     legacy default stream).  Calls that return host data synchronise it;
 *     asynchronous CUDA errors surface at the next synchronising call as
 *     SMC_ECUDA.
 *   - One host thread per context at a time.  One context per GPU rank.
 *   - Units are SI; angles in radians; x East, y North, chi measured
 *     counter-clockwise from +x (the form of Eq. hor); runway at
 *     the origin, landings heading West.
 */
#ifndef SMCATM_H
#define SMCATM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct smc_ctx smc_ctx;

typedef enum {
    SMC_OK = 0,
    SMC_EINVAL = 1,       /* bad configuration / scenario / argument            */
    SMC_EINFEASIBLE = 2,  /* no particle without a zero weight   */
    SMC_ECUDA = 3,        /* CUDA runtime error (message in smc_last_error)     */
    SMC_ENCCL = 4,        /* NCCL error (multi-GPU)                             */
    SMC_ENOMEM = 5,       /* workspace too small                                */
    SMC_ESTATE = 6        /* call order violated (e.g. iterate before scenario) */
} smc_status;

enum { SMC_ARRIVAL = 0, SMC_DEPARTURE = 1 };
enum { SMC_SCHED_CONST = 0, SMC_SCHED_PAPER = 1 };   /* S_k const or floor(3+5e^{0.05k}) */
enum { SMC_DENSITY_ISA = 0, SMC_DENSITY_CONST = 1 }; /* R12 */
enum { SMC_FLAG_LANDED = 1, SMC_FLAG_EXITED = 2, SMC_FLAG_VIOLATED = 4 };

/* Aircraft state (order R29). */
typedef struct { double x, y, z, v, chi, m; } smc_state;

/* Control per aircraft per step: thrust T [N], bank phi [rad], climb gamma [rad]. */
typedef struct { float thrust, bank, climb; } smc_control;

/* Aircraft-type constants: drag polar (R12), fuel coefficient eta
 * (constant, R13) and the flight envelope. */
typedef struct {
    double S, cd0, cd2, eta, m_empty;
    double T_min, T_max, v_min, v_max, gamma_max, phi_max, z_min, z_max;
} smc_aircraft_type;

/* One aircraft in the planning problem. first_step = e in [0, H]: the
 * aircraft is simulated on horizon steps [e, H) only (rolling window, P:428;
 * R20).  Departures use theta_F / z_tf / v_D, arrivals beta_f. */
typedef struct {
    uint32_t kind;        /* SMC_ARRIVAL or SMC_DEPARTURE */
    uint32_t type;        /* index into smc_scenario.types */
    uint32_t first_step;
    uint32_t id;          /* persistent aircraft identifier: matches rows of the previous
                             winner to this window for warm starts (R45); else unused */
    smc_state x0;         /* state at entry (shared by all particles) */
    double theta_F, z_tf, v_D, beta_f;
} smc_aircraft;

/* The planning problem and every model constant. */
typedef struct {
    uint32_t n_aircraft;  /* N, 1..32 */
    uint32_t n_types;
    const smc_aircraft *aircraft;          /* [n_aircraft] */
    const smc_aircraft_type *types;        /* [n_types] */
    uint32_t horizon;     /* H, 1..32 */
    int32_t density_mode; /* SMC_DENSITY_* */
    double dt, g, rho_const;               /* delta t, gravity, rho for CONST mode */
    double P_runway, P_beta, P_chi, P_vs;  /* landing sector (Eq. TO_init) */
    double P_r, P_h;                       /* separation cylinder (Eq. avoidance) */
    double alpha_dep[4];                   /* bearing A, fuel, altitude B, speed C */
    double alpha_arr[3];                   /* heading D, altitude E, fuel (R7) */
    double noise_w, A_c;                   /* noise weight and altitude cut-off */
    uint32_t n_centres;                    /* population centres */
    const double *centres;                 /* [n_centres][3] = x, y, radius (m) */
    uint32_t pop_nx, pop_ny;               /* popdense grid; 0 = no grid */
    double pop_x0, pop_y0, pop_dx;
    double wind_lo[3], wind_hi[3];         /* wind-grid box */
    double sigma_lo, sigma_hi;             /* sigma(z) at the box bottom / top */
    double beta_w, gamma_w, lambda_t;      /* Eq. cov decay rates (R14) */
    double nominal[2];                     /* forecast wind */
    double turb_sigma;                     /* per-aircraft gust std (R15), 0 = off */
    double tma_radius;                     /* D_TMA */
    uint32_t wind_n[3];                    /* wind grid points per axis N_x, N_y, N_z, evenly spaced
                                              over the box; 0 = 2; product <= 64.  The
                                              paper's runs use 2 x 2 x 2 */
} smc_scenario;

/* Host-side collectives (optional; a test shim for world_size > 1 without NCCL, e.g. two
 * processes sharing one GPU over a CPU process group).  Each call is collective over the
 * world_size ranks and operates on HOST buffers the library owns for the call: the library
 * synchronises its stream, copies the device operand to the host, calls the function and
 * copies the result back.  allreduce_max_u32: element-wise maximum of `count` words in
 * place.  allgather: rank r's `bytes` bytes land at recv + r * bytes on every rank.  Return
 * 0 on success.  Incompatible with use_graph (a captured graph cannot call the host). */
typedef struct {
    void *user;
    int (*allreduce_max_u32)(void *user, uint32_t *buf, size_t count);
    int (*allgather)(void *user, const void *send, void *recv, size_t bytes);
} smc_host_collectives;

/* Solver configuration. */
typedef struct {
    uint32_t n_particles;      /* L, global over all ranks; L < 2^30 and
                                  L * max_aircraft < 2^31, else SMC_EINVAL           */
    uint32_t n_samples;        /* S per round for SMC_SCHED_CONST (Alg.1 l.7)         */
    uint32_t schedule;         /* SMC_SCHED_*                                         */
    uint32_t n_rounds;         /* K rounds per mpc_step (J_max + 1)     */
    uint32_t mh;               /* 0: Alg.1 l.23 as printed; 1: joint Metropolis-Hastings
                                  move (R1); 2: per-aircraft acceptance (R46) with the
                                  final pick over the jointly evaluated candidates     */
    uint32_t clamp_proposals;  /* 1: clamp perturbed controls to the envelope (R16)   */
    double sigma[3];           /* perturbation std (T, phi, gamma)     */
    double anneal;             /* sigma_k = sigma * anneal^k                          */
    uint64_t seed;             /* Philox key                                          */
    int32_t device;            /* CUDA device ordinal                                 */
    int32_t rank, world_size;  /* particle sharding (1 = single GPU)                  */
    const void *nccl_unique_id;/* 128-byte ncclUniqueId from rank 0; NULL if world 1  */
    void *workspace;           /* caller-owned device memory                          */
    size_t workspace_bytes;
    void *stream;              /* cudaStream_t                                        */
    uint32_t max_aircraft;     /* capacity (<= 32)                                    */
    uint32_t max_horizon;      /* capacity (<= 32)                                    */
    uint32_t use_graph;        /* 1: replay the round loop as a CUDA graph            */
    uint32_t profile;          /* 1: time each phase with CUDA events (smc_phase_times) */
    uint32_t virtual_world;    /* test mode (world_size 1): run the multi-GPU resampling and
                                  selection path -- per-shard CDFs, survivor exchange layout,
                                  shard-aware gather, record merge -- for this many virtual
                                  ranks on one GPU; results are bit-identical to 1 / 0 */
    uint32_t n_particles_final;/* particle count of the last round, decreasing linearly
                                  L_k = L - (L - L_final) k / (K - 1) (integer);
                                  0 = constant L.  Single-rank contexts only. */
    double warm_fraction;      /* warm start (R45): the first floor(warm_fraction L) particles of
                                  each solve start from the previous solve's winner shifted one
                                  step (aircraft matched by smc_aircraft.id; particle 0 exact, the
                                  others + N(0, sigma^2)); 0 = fresh uniform init */
    const smc_host_collectives *host_coll; /* NULL: NCCL (world_size > 1 needs nccl_unique_id) */
} smc_config;

/* Per-round diagnostics (smc_iterate). */
typedef struct {
    double best_lambda;        /* max_l sum_i log2 W_il over survivors        */
    double accept_rate;        /* MH acceptances / L (1.0 in round 0)                 */
    double ess_min;            /* min_i (sum w)^2 / sum w^2, diagnostic       */
    uint32_t infeasible_lo;    /* bit i: column i all-zero (resampled uniformly, R25) */
    uint32_t infeasible_hi;
    uint32_t n_samples;        /* S_k used in this round                              */
    uint32_t round;            /* k                                                   */
} smc_round_stats;

/* Bytes of device workspace needed for cfg (uses n_particles, world_size,
 * max_aircraft, max_horizon).  0 on invalid cfg. */
size_t smc_workspace_bytes(const smc_config *cfg);

/* Create a context.  Validates cfg, carves the workspace, creates events.
 * With world_size > 1 also joins the NCCL communicator (R43; or uses
 * cfg.host_coll): rank r owns the global particles [L r / G, L (r+1) / G);
 * every random stream is keyed by the global particle index, so rollouts, MH
 * decisions and ancestors are identical for any world size.  Each round then
 * exchanges the column maxima (all-reduce MAX, N words) and the per-rank
 * column totals of the integer weights (all-gather, N uint64 per rank) on
 * cfg.stream; each rank's gather searches the owning rank's CDF and reads its
 * parents' control rows where their owner keeps them (peer mode, the
 * default): smc_init exports the allocation holding cfg.workspace as a CUDA
 * IPC handle, all-gathers the handles and maps every peer's workspace
 * (NVLink/NVSwitch loads; the mappings are closed by smc_destroy, so every
 * rank's workspace must outlive every rank's context).  If a mapping cannot
 * be opened, or with the environment variable SMC_P2P=0 (read by
 * smc_workspace_bytes and smc_init alike), the per-rank CDFs and compacted
 * survivor rows are all-gathered instead (the workspace size accounts for
 * both).  Selection all-gathers per-rank winners. */
smc_status smc_init(const smc_config *cfg, smc_ctx **out);

/* Copy the scenario, precompute (Qhat = chol(Rhat) P:463-465, normalisers
 * P:336, population grid P:1131-1133) and draw the initial population
 * (Alg.1 l.1-5).  Resets the round counter k to 0. */
smc_status smc_set_scenario(smc_ctx *ctx, const smc_scenario *scn);

/* Run n_rounds SMC rounds (Alg.1 l.6-24).  Round k: evaluate every particle
 * over S_k wind samples (l.9-18; with MH both the resampled particle and its
 * perturbation, common random numbers), MH-select (R1), reduce the log2
 * weights, per-aircraft systematic resampling (l.22, R25) and propose
 * (l.23).  stats: nullable, n_rounds entries (synchronises if non-NULL). */
smc_status smc_iterate(smc_ctx *ctx, uint32_t n_rounds, smc_round_stats *stats);

/* Final sample selection (Alg.1 l.27): the survivor of the last
 * evaluated round with the greatest prod_i W_il; ties -> lowest global index.
 * out: host [N][H] controls.  Returns SMC_EINFEASIBLE if every particle has
 * a zero weight.  Synchronises. */
smc_status smc_best_controls(smc_ctx *ctx, smc_control *out, double *lambda, int64_t *particle);

/* One MPC update: x0 := measured (host [N]), fresh population,
 * n_rounds rounds, selection, apply the t=0 control of the winner (applied,
 * host [N]) and advance the plant one dt with the realised wind (next, host
 * [N]); flags[N] = SMC_FLAG_* (landed Eq. TO_init, exited D_TMA P:257).
 * Aircraft with first_step > 0 are not advanced.  Increments the MPC step
 * index that keys every random stream.  Synchronises. */
smc_status mpc_step(smc_ctx *ctx, const smc_state *measured, smc_control *applied,
                    smc_state *next, uint32_t *flags);

/* Device-resident MPC update: fresh population from the current x0, n_rounds
 * rounds, selection and (advance_plant != 0) the plant step on the device
 * copy of the plant state, all enqueued on cfg.stream with no host copy and
 * no synchronisation.  The plant state is the scenario's x0 after
 * smc_set_scenario / the last mpc_step's next state.  Infeasible solves leave
 * the plant state unchanged and set SMC_FLAG_VIOLATED in the device flags. */
smc_status smc_solve(smc_ctx *ctx, uint32_t advance_plant);

/* Accumulated device time per phase since the last call (requires
 * cfg.profile = 1; synchronises): ms[0] rollout+MH (K2), ms[1] reduce +
 * resampling scans (K4a, K4b, K5), ms[2] gather + propose (K6), ms[3] other
 * (init, select, plant).  launches[4] = kernel launches per phase. */
smc_status smc_phase_times(smc_ctx *ctx, double ms[4], uint64_t launches[4]);

const char *smc_last_error(const smc_ctx *ctx);
void smc_destroy(smc_ctx *ctx);

/* Set / read the MPC step index (keys all streams; mpc_step increments it). */
smc_status smc_set_mpc_index(smc_ctx *ctx, uint32_t mpc_index);
uint32_t smc_get_mpc_index(const smc_ctx *ctx);

/* Peer-mode test hooks.  smc_ipc_record writes the 128-byte record a rank
 * publishes in peer mode (CUDA IPC handle of the allocation holding the
 * workspace + the workspace's offset in it).  smc_ipc_peek, called in ANOTHER
 * process, maps such a record, copies `bytes` bytes from workspace offset
 * `offset` to host_out and unmaps.  SMC_ECUDA on any CUDA IPC failure. */
smc_status smc_ipc_record(const smc_ctx *ctx, void *out128);
smc_status smc_ipc_peek(const void *rec128, uint64_t offset, void *host_out, size_t bytes);

/* 128-byte NCCL unique id for a multi-GPU context (call on rank 0, share
 * with every rank, pass as smc_config.nccl_unique_id).  SMC_ENCCL if NCCL
 * cannot be loaded. */
smc_status smc_nccl_unique_id(void *out128);

/* Number of kernel launches the library issued since smc_init. */
uint64_t smc_launch_count(const smc_ctx *ctx);

/* Host->device and device->host bytes the production entry points copied since
 * the last call (debug hooks excluded); resets the counters. */
void smc_io_bytes(smc_ctx *ctx, uint64_t *h2d_bytes, uint64_t *d2h_bytes);

/* ---------------- parity / test hooks (stream-synchronising) -------------- */

/* Roll out caller-given controls (host [L][N][H][3], particle l = global
 * index l0 + l) for S samples of round k, through the production rollout
 * code.  Outputs per (l, s, i) (host, nullable): J [L][S][N], viol
 * [L][S][N] (uint8), comp [L][S][N][4], fuel [L][S][N], landed
 * [L][S][N] (int32, -1 = not landed), traj [L][S][N][H+1][6] (float). */
smc_status smc_debug_rollout(smc_ctx *ctx, const float *controls, uint32_t L, uint32_t l0,
                             uint32_t S, uint32_t k, float *J, uint8_t *viol, float *comp,
                             float *fuel, int32_t *landed, float *traj);

/* Evaluate (Alg.1 l.9-18) caller-given controls with the production kernel:
 * ell[L][N] (host float) = -log2(L_global) + sum_s log2 J (or -inf). */
smc_status smc_debug_evaluate(smc_ctx *ctx, const float *controls, uint32_t L, uint32_t S,
                              uint32_t k, float *ell);

/* The same through the two-candidate production kernel (both MH candidates = controls, so the
 * survivor's weights are the candidates' whatever MH decides): the kernel of rounds k >= 1. */
smc_status smc_debug_evaluate2(smc_ctx *ctx, const float *controls, uint32_t L, uint32_t S,
                               uint32_t k, float *ell);

/* MH decisions (R1) for injected joint log2 weights: acc[l] = 1 accept. */
smc_status smc_debug_mh(smc_ctx *ctx, const double *lam_cur, const double *lam_prop, uint32_t L,
                        uint32_t k, uint8_t *acc);

/* Per-aircraft MH decisions (R46) on injected log2 weights ell_cur / ell_prop
 * [L][N] (host float) with the production device function -> mask[L] (bit i =
 * accept x*_i). */
smc_status smc_debug_mh_aircraft(smc_ctx *ctx, const float *ell_cur, const float *ell_prop, uint32_t L,
                                 uint32_t N, uint32_t k, uint32_t *mask);

/* Per-aircraft systematic resampling (R25) of injected log2 weights
 * ell[N][L] (host float) into M new particles (M = 0 means L) with the
 * production kernels -> anc[N][M] (host int32).  Q[N] (nullable) receives the
 * integer weight totals. */
smc_status smc_debug_resample(smc_ctx *ctx, const float *ell, uint32_t N, uint32_t L, uint32_t M, uint32_t k,
                              int32_t *anc, uint64_t *Q);

/* Gather + propose (Alg.1 l.22-23) on injected survivors: surv_ctrl [L][N][H][3]
 * (host), anc [N][L] -> xp (resampled, = parent rows) and xs (perturbed),
 * both host [L][N][H][3], with sigma_k = sigma * anneal^k. */
smc_status smc_debug_propose(smc_ctx *ctx, const float *surv_ctrl, const int32_t *anc, uint32_t L,
                             uint32_t k, float *xp, float *xs);

/* Device population after the last call, packed for the Lk particles the
 * last round evaluated (Lk = L unless n_particles_final shrinks it; written
 * to *n_eval, nullable; buffers are sized for L): ctrl_cur / ctrl_prop
 * [Lk][N][H][3] of the last evaluated pair, surv[Lk] survivor masks (bit i
 * set = aircraft i's row is the proposal x*; joint MH: all bits alike), ell_surv[N][Lk], lam_surv[Lk], lam_cand[2][Lk]
 * (joint log2 weight of both MH candidates as the kernel computed them;
 * round 0 / mh=0: only [0] is meaningful).  Any pointer may be NULL. */
smc_status smc_debug_population(smc_ctx *ctx, float *ctrl_cur, float *ctrl_prop, uint32_t *surv,
                                float *ell_surv, double *lam_surv, double *lam_cand, uint32_t *n_eval);

/* ---------------- multi-GPU partition helpers (pure host, no GPU) ---------- */

/* Particles [begin, end) owned by rank (contiguous block sharding). */
void smc_shard_range(uint32_t L, int32_t world_size, int32_t rank, uint32_t *begin, uint32_t *end);

/* Given every rank's per-column integer weight totals Q_all[world][N]
 * (allgathered), the exclusive CDF offset of `rank` per column and the
 * global totals. */
void smc_shard_offsets(uint32_t N, int32_t world_size, int32_t rank, const uint64_t *Q_all,
                       uint64_t *offset, uint64_t *Q_total);

/* Number of systematic slots j in [0, L) with floor((j Q + R) / L) < C
 * (exact integer arithmetic): the slot boundary of CDF value C (R25). */
uint64_t smc_slot_count(uint64_t C, uint64_t Q, uint64_t R, uint32_t L);

/* ---------------- fuel estimates on recorded traces (section 5) ---------------- */
/* Aircraft constants of one trace: drag polar (R12), fuel-flow coefficients
 * eta = Cf1 (1 + v / Cf2) in kg/(N s) and m/s, and the |gamma|
 * clamp for degenerate intervals (R47). */
typedef struct {
    double S, cd0, cd2, Cf1, Cf2, gamma_max;
} smc_fuel_type;

/* A batch of traces, every pointer DEVICE memory owned by the caller.
 * trace[n][max_len][5] = x, y, z, v_s, chi per sample at spacing dt; len[n]
 * samples used (>= 1).  Outputs: m1 / m2 [n][max_len] mass series of
 * estimate 1 / 2, wres[n][max_len][2] estimate-1 wind
 * residuals (0 in the last sample), fuel[n][2] total burn, flags[n] (bit0
 * gamma clamped, bit1 zero-distance interval in estimate 2).  Negative burn is
 * clamped to 0. */
typedef struct {
    uint32_t n_traces, max_len;
    const uint32_t *len;
    const double *trace;
    const double *m0;
    const smc_fuel_type *type;
    double dt, g;
    int32_t density_mode;      /* SMC_DENSITY_* */
    double rho_const;
    double *m1, *m2, *wres, *fuel;
    uint32_t *flags;
} smc_fuel_args;

/* One thread per trace (sequential in time, independent across aircraft),
 * FP64; ordered on `stream` (cudaStream_t, NULL = legacy default).  Errors:
 * SMC_EINVAL for a NULL pointer or zero sizes, SMC_ECUDA on launch failure. */
smc_status smc_fuel_estimates(const smc_fuel_args *args, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SMCATM_H */

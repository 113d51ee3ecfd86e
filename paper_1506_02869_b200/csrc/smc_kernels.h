// smc_kernels.h -- launch interface between the host orchestrator (capi.cu)
// and the kernels (k_rollout.cu, k_population.cu).  Internal to libsmcatm.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace smc {

struct DevScen;

struct RolloutArgs {
    const float *ctrl[2];      // candidate buffers [L][n][H][3]: 0 = x' (resampled), 1 = x* (proposal)
    uint32_t L, l0, S, k;      // local particles, global offset, samples, round
    const uint32_t *mpcp;      // device: MPC step index (keys every stream)
    float ell0;                // -log2(L_global)  (W^0 = 1/L)
    uint32_t surv_single;      // survivor mask written when only one candidate is evaluated (0 or ~0)
    int mh_mode;               // 1: joint MH on lambda (R1); 2: per-aircraft MH (R46)
    float *ell_out;            // [n][L] survivor log2 weights (column-major per aircraft)
    double *lam_out;           // [L] survivor joint log2 weight
    double *lam_cand;          // [2][L] both candidates' joint log2 weights (nullable)
    uint32_t *surv_out;        // [L] survivor mask: bit i set = aircraft i's row comes from x*
    uint32_t *colmax;          // [n] ordered-float max of ell_out (atomicMax)
    unsigned long long *n_accept;
    // debug outputs (candidate 0), per (l, s, i)
    float *dbg_J, *dbg_comp, *dbg_fuel, *dbg_traj, *dbg_ell_c;
    uint8_t *dbg_viol;
    int32_t *dbg_landed;
};

constexpr int kMaxWindNodes = 64;   // N_x N_y N_z
int segment_width(int n, bool dense = false);
size_t rollout_smem_bytes(int W, int NC, int H, int ng = 8, bool sp = false);
cudaError_t launch_rollout(const DevScen &sc, const RolloutArgs &a, int NC, bool debug, cudaStream_t st);

struct PopArgs {
    int n, H;
    uint32_t L, l0, k, key0, key1;
    const uint32_t *mpcp;
    // warm start (R45): particles l < Lw of aircraft with warm_map[i] >= 0 start from the
    // previous winner's row warm_map[i] (shifted one step) when *warm_ok >= 0
    uint32_t Lw;
    const float *warm_row;      // [n_prev][H][3]
    const long long *warm_ok;   // previous winner index (< 0: none)
    const int32_t *warm_map;    // [n]
    float sig[3];
    int clamp;
    const float *lo3, *hi3;
};

// K1: uniform initial controls (Alg.1 l.3-5)
cudaError_t launch_init_population(const DevScen &sc, const PopArgs &p, float *ctrl, cudaStream_t st);

// Resampling (R25): K4b decoupled look-back scan of the integer
// weights -> CDF C and (Q, R); ancestors by bisection (in K6 or k_ancestors).
// K4a (k_qsum) computes totals and ESS for diagnostics only.
struct ResampleArgs {
    int n;
    uint32_t L;                 // particles (local == global when single GPU)
    uint32_t k, key0, key1;
    const uint32_t *mpcp;
    const float *ell;           // [n][ell_stride]
    uint32_t ell_stride;        // row stride of ell (0 = L)
    const uint32_t *colmax;     // [n] ordered max
    unsigned long long *Q;      // [n] totals (nullable)
    double *ess;                // [2n] sum w, sum w^2 (diagnostic)
    unsigned long long *status; // [n][ntiles] look-back words
    uint32_t *tile_ctr;         // [n] dynamic tile counters
    unsigned long long *C;      // [n][Cstride] inclusive integer CDF
    uint32_t Cstride;           // row stride of C (0 = L)
    unsigned long long *QR;     // [n][2] (Q, R)
    int32_t *anc;               // [n][M] (K5 ancestors only)
    uint32_t M;                 // new particles drawn (K5 ancestors only)
    uint32_t *splits;           // [n][mp_split_words(L, M)] K5 merge-path split points
    unsigned long long *Cs;     // [n][Cs_stride] every kCdfSample-th inclusive prefix (nullable):
    uint32_t Cs_stride;         //   Cs[g] = C[min(16 g + 15, L - 1)], for K6's two-level search
    int32_t *inf_round;         // [n] first round whose column had no nonzero weight (-1: none; nullable)
};
constexpr int kCdfSample = 16;
__host__ __device__ inline uint32_t cdf_samples(uint32_t L) { return (L + kCdfSample - 1) / kCdfSample; }
int scan_tiles(uint32_t L);
int scan_tiles_max(uint32_t L);    // upper bound over all tile sizes (status allocation)
cudaError_t launch_qsum(const ResampleArgs &r, cudaStream_t st);
cudaError_t launch_scan(const ResampleArgs &r, cudaStream_t st);
// single-pass scan by one 8-CTA cluster per column (DSMEM exchange of CTA totals), L <= 65536
bool cluster_scan_fits(uint32_t L);
cudaError_t launch_scan_cluster(const ResampleArgs &r, cudaStream_t st);
cudaError_t launch_ancestors(const ResampleArgs &r, cudaStream_t st);          // K5 merge path (needs r.splits)
size_t mp_split_words(uint32_t L, uint32_t M);
cudaError_t launch_ancestors_bisect(const ResampleArgs &r, cudaStream_t st);   // one bisection per slot
cudaError_t launch_ancestors_two_level(const ResampleArgs &r, cudaStream_t st); // K6's search (needs r.Cs)

// K6: gather survivors' rows by ancestor, Gaussian proposal (Alg.1 l.22-23)
struct ProposeArgs {
    int n, H;
    uint32_t L, l0, k, key0, key1;
    const uint32_t *mpcp;
    const float *src[2];        // survivor pair: [0] x', [1] x*
    const uint32_t *surv;       // [L] survivor masks: bit i = buffer holding aircraft i's row
    uint32_t Lsrc;              // particles evaluated this round (CDF length); L = new particles
    const int32_t *anc;         // [n][L] explicit ancestors (debug) or NULL -> bisection of C
    const unsigned long long *C, *QR;
    const unsigned long long *Cs;   // [n][Cs_stride] CDF samples (nullable: plain bisection)
    uint32_t Cs_stride;
    // per-round accumulators zeroed here for the next round (stream-ordered after K2 and K4)
    uint32_t *reset_colmax, *reset_tiles;   // [reset_n] each
    unsigned long long *reset_accept;
    unsigned long long *reset_status;       // [reset_status_n] look-back words
    size_t reset_status_n;
    int reset_n;
    float *xp, *xs;             // outputs [L][n][H][3]
    uint32_t ks[20];            // Philox round keys of (key0, key1) (nullable use: all zero -> computed)
    float sig[3];
    int clamp;
    const float *lo3, *hi3;     // per aircraft [n][3] envelope for clamping
};
cudaError_t launch_gather_propose(const ProposeArgs &p, cudaStream_t st);

// Multi-GPU gather + propose
struct MultiArgs {
    ProposeArgs p;              // p.L = local new particles, p.l0 = global offset of this rank
    uint32_t Lg;                // global particles
    int G;                      // ranks (<= 8)
    const unsigned long long *Qall;     // [G][Qstride] per-rank column totals (all-gathered)
    uint32_t Qstride;
    // rank r's local inclusive CDF [n][Cstride] and its every-16th samples [n][Cs_stride]
    // (NULL: plain bisection) -- NVLink peer mappings, all-gathered copies or buffer slices
    const unsigned long long *peer_C[8], *peer_Cs[8];
    uint32_t Cstride, Cs_stride;
    uint32_t len[8];            // particles of rank r
    // parents' survivor rows: rank r's pair at peer_ctrl[r] (+ prow: x*), masks peer_surv[r]
    // (peer mode), or the all-gathered compacted rows Sall [G][Lmax][n][H][3] (all-gather mode)
    const float *peer_ctrl[8];
    const uint32_t *peer_surv[8];
    size_t prow;
    const float *Sall;
    uint32_t Lmax;
};
cudaError_t launch_compact_survivors(const float *xp, const float *xs, const uint32_t *surv, uint32_t Lloc, int n,
                                     int rowlen, float *out, cudaStream_t st);
cudaError_t launch_gather_propose_multi(const MultiArgs &m, cudaStream_t st);
cudaError_t launch_select_merge(const unsigned char *recs, int G, size_t rec_bytes, int rowlen, unsigned char *out,
                                cudaStream_t st);

// K7: final selection + winner row copy
struct SelectArgs {
    uint32_t L, l0;
    int n, H;
    const double *lam;
    const uint32_t *surv;
    const float *src[2];
    double *part_lam;           // [nblocks]
    long long *part_idx;        // [nblocks]
    unsigned int *done_ctr;
    double *best_lam;           // [1]
    long long *best_idx;        // [1]  (-1 if infeasible)
    float *best_row;            // [n][H][3]
    const double *lam2;         // [2][lam2_stride] candidates' joint lambdas (per-aircraft MH pick) or NULL
    uint32_t lam2_stride;
};
int select_blocks(uint32_t L);
cudaError_t launch_select(const SelectArgs &s, cudaStream_t st);

// K8: plant advance in FP64
struct PlantArgs {
    int n;
    uint32_t key0, key1;
    const uint32_t *mpcp;
    const double *states;       // [n][6]
    const float *best_row;      // [n][H][3] (t = 0 is applied)
    int H;
    double *Z;                  // [16] realised AR(1) state
    int *zinit;
    double *next;               // [n][6]
    int *flags;                 // [n]
    float *applied;             // [n][3]
    const long long *best_idx;  // [1] winner (-1: infeasible -> plant state unchanged)
};
struct PlantScen {              // FP64 constants for the plant
    const double *Qd;           // [ng][ng] Qhat (FP64)
    int wn[3], ng;
    double a, b, dt, g, rho_const;
    double wind_lo[3], wind_hi[3], nominal[2], turb_sigma, tma_radius;
    double P_runway, P_beta, P_chi, P_vs;
    int density_mode;
    int kind[32], first_step[32];
    double halfS[32], cd0[32], cd2[32], eta[32];
    double m_empty[32], T_min[32], T_max[32], v_min[32], v_max[32], gamma_max[32], phi_max[32], z_min[32], z_max[32];
};
cudaError_t launch_plant(const PlantScen &ps, const PlantArgs &p, cudaStream_t st);

// popdense grid, computed in FP64 on the device: out [ny][nx], and outp [ny + 1][nx + 1]
// with the last row and column repeated (K2's cell lookup needs no index clamp)
cudaError_t launch_popgrid(const double *centres, int n_centres, int nx, int ny, double x0, double y0,
                           double dx, float *out, float *outp, cudaStream_t st);

// MH decisions for injected lambdas (debug hook)
cudaError_t launch_mh_debug(const double *lc, const double *lp, uint32_t L, uint32_t k, const uint32_t *mpcp,
                            uint32_t key0, uint32_t key1, uint8_t *acc, cudaStream_t st);
// per-aircraft MH decisions on injected float log2 weights [L][n] -> masks (debug hook)
cudaError_t launch_mh_aircraft_debug(const float *ec, const float *ep, uint32_t L, int n, uint32_t k,
                                     const uint32_t *mpcp, uint32_t key0, uint32_t key1, uint32_t *mask,
                                     cudaStream_t st);

__host__ __device__ uint64_t slot_count(uint64_t C, uint64_t Q, uint64_t R, uint32_t L);
cudaError_t launch_colmax(const float *ell, int n, uint32_t L, uint32_t *colmax, cudaStream_t st);

}  // namespace smc

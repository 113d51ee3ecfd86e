// capi.cu -- C ABI and host orchestrator of libsmcatm (include/smcatm.h).
//
// The host side only validates, packs constants, carves the caller's device
// workspace and sequences kernels on the caller's stream; every per-particle
// step of the path runs in the kernels of k_rollout.cu / k_population.cu.
// Scenario precompute that is O(1) in the particle count (the 8x8 Cholesky of
// Rhat; the departure altitude normalisers) is host FP64.
#include <dlfcn.h>

#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: host ranges for nsys / ncu --nvtx (no-op untraced)

#include "../../include/smcatm.h"
#include "smc_device.cuh"
#include "smc_kernels.h"

using namespace smc;

static void ipc_release(void *mapping);

namespace {

// ---- NCCL, loaded at run time (only multi-GPU contexts need it; the ABI types are stable)
typedef int ncclResult_t;
struct ncclUniqueId { char internal[128]; };
typedef void *ncclComm_t;
enum { ncclUint8_ = 1, ncclUint32_ = 3, ncclUint64_ = 5, ncclFloat32_ = 7 };
enum { ncclMax_ = 2 };
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi *nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
            api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
            if (api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather)
                api.h = h;
        }
    }
    return api.h ? &api : nullptr;
}

constexpr uint32_t kPopCap = 256 * 256;
constexpr uint32_t kCentreCap = 256;
constexpr size_t kIpcRec = 128;     // cudaIpcMemHandle_t (64 B) + workspace offset in its allocation

size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

struct Layout {
    size_t ctrl, ell, lam, lam2, surv, colmax, Q, ess, status, tiles, C, QR, anc, splits, Cs, accept, mpc, dac, pop, popp, centres,
        part_lam, part_idx, done, best_lam, best_idx, best_row, Call, Qall, Csall, Sc, Sall, survp, ipc, pZ, pzi, pstates,
        pnext, pflags, papplied, lohi, wmap, flag, infround, infcol,
        qf, qd, total;
};

// Bump-allocate every device buffer from the caller's workspace.
size_t record_bytes(int nmax, int Hmax) { return (16 + (size_t)nmax * Hmax * 12 + 15) & ~(size_t)15; }

// world: real ranks (Lloc = this rank's share); vworld: virtual ranks inside one context
// (test mode, Lloc = L).  G = ranks whose CDFs / survivors / records are exchanged.
// Multi-rank exchange of parent rows: in place from the owner (peer mode: NVLink reads
// through CUDA IPC mappings, or slices of one buffer for virtual ranks -- the default), or
// an all-gather of every rank's compacted survivor rows (SMC_P2P=0).
bool p2p_mode() {
    const char *e = getenv("SMC_P2P");
    return !(e && strcmp(e, "0") == 0);
}

Layout layout(uint32_t Lloc, int nmax, int Hmax, int world = 1, int vworld = 1) {
    const bool p2p = p2p_mode();
    const int G = world > 1 ? world : vworld;
    const uint32_t Lx = world > 1 ? Lloc : (Lloc + vworld - 1) / vworld;   // per-rank stride
    Layout o{};
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t at = off; off += align_up(bytes); return at; };
    const size_t row = (size_t)Lloc * nmax * Hmax * 3 * sizeof(float);
    o.ctrl = take(4 * row);
    o.ell = take((size_t)nmax * Lloc * sizeof(float));
    o.lam = take((size_t)Lloc * sizeof(double));
    o.lam2 = take(2 * (size_t)Lloc * sizeof(double));
    o.surv = take((size_t)Lloc * sizeof(uint32_t));
    o.colmax = take(nmax * sizeof(uint32_t));
    o.Q = take(nmax * sizeof(unsigned long long));
    o.ess = take(2 * nmax * sizeof(double));
    o.status = take((size_t)nmax * scan_tiles_max(Lloc) * 8);
    o.tiles = take(2 * nmax * sizeof(uint32_t));
    o.C = take((size_t)nmax * Lloc * sizeof(unsigned long long));
    o.QR = take(2 * nmax * sizeof(unsigned long long));
    o.anc = take(world > 1 ? 0 : (size_t)nmax * Lloc * sizeof(int32_t));   // K5 ancestors (single rank)
    o.splits = take(world > 1 ? 0 : (size_t)nmax * mp_split_words(Lloc, Lloc) * sizeof(uint32_t));
    o.Cs = take((size_t)nmax * cdf_samples(Lloc) * sizeof(unsigned long long));   // CDF samples (stride cdf_samples(Lloc))
    o.accept = take(8);
    o.mpc = take(sizeof(uint32_t));
    o.dac = take(nmax * sizeof(DevAircraft));
    o.pop = take(kPopCap * sizeof(float));
    o.popp = take((2 * kPopCap + 2) * sizeof(float));           // (nx + 1)(ny + 1) <= 2 nx ny + 2
    o.centres = take(kCentreCap * 3 * sizeof(double));
    o.part_lam = take(512 * sizeof(double));
    o.part_idx = take(512 * sizeof(long long));
    o.done = take(sizeof(unsigned));
    o.best_lam = take(record_bytes(nmax, Hmax));               // local selection record
    o.best_idx = take(record_bytes(nmax, Hmax));               // final (merged) record
    o.best_row = take(G > 1 ? record_bytes(nmax, Hmax) * G : 0);           // all-gathered records
    // multi-rank exchange: per-rank CDFs (all-gather mode / virtual ranks), column totals, CDF samples
    // (virtual ranks), compacted survivor rows; real ranks reserve the all-gather buffers even in peer
    // mode, which falls back to them when an IPC mapping cannot be opened
    o.Call = take(G > 1 ? (size_t)G * nmax * Lx * 8 : 0);
    o.Qall = take(G > 1 ? (size_t)G * nmax * 8 : 0);
    o.Csall = take(world == 1 && G > 1 ? (size_t)G * nmax * cdf_samples(Lx) * 8 : 0);
    o.Sc = take(world > 1 ? (size_t)Lloc * nmax * Hmax * 3 * sizeof(float) : 0);
    o.Sall = take((world > 1 || (G > 1 && !p2p)) ? (size_t)G * Lx * nmax * Hmax * 3 * sizeof(float) : 0);
    o.survp = take(world > 1 ? 2 * (size_t)Lloc * sizeof(uint32_t) : 0);   // published masks, by round parity
    o.ipc = take(world > 1 ? (size_t)(G + 1) * kIpcRec : 0);              // IPC handle exchange
    o.flag = take(16);
    o.infround = take(nmax * sizeof(int32_t));
    o.infcol = take(nmax * sizeof(uint32_t));
    o.pZ = take(2 * kMaxWindNodes * sizeof(double));
    o.pzi = take(sizeof(int));
    o.pstates = take(nmax * 6 * sizeof(double));
    o.pnext = take(nmax * 6 * sizeof(double));
    o.pflags = take(nmax * sizeof(int));
    o.papplied = take(nmax * 3 * sizeof(float));
    o.lohi = take(nmax * 6 * sizeof(float));
    o.qf = take(kMaxWindNodes * kMaxWindNodes * sizeof(float));
    o.qd = take(kMaxWindNodes * kMaxWindNodes * sizeof(double));
    o.wmap = take(nmax * sizeof(int32_t));
    o.total = off;
    return o;
}

uint32_t local_count(uint32_t L, int world, int rank) {
    uint32_t b, e;
    smc_shard_range(L, world, rank, &b, &e);
    return e - b;
}

uint32_t max_local(uint32_t L, int world) {
    uint32_t m = 0;
    for (int r = 0; r < world; ++r) m = std::max(m, local_count(L, world, r));
    return m;
}

}  // namespace

struct smc_ctx {
    smc_config cfg{};
    cudaStream_t st = nullptr;
    uint32_t Lg = 0, Lloc = 0, l0 = 0;
    int nmax = 0, Hmax = 0;
    char *ws = nullptr;
    Layout lay{};
    float *ctrl[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    float *ell = nullptr;
    int nsm = 148;
    double *lam = nullptr, *lam2 = nullptr;
    uint32_t *surv = nullptr;          // survivor masks (bit i: aircraft i's row from x*)
    int last_nc = 1;                   // candidates evaluated by the last round
    uint32_t *colmax = nullptr, *tiles = nullptr;
    unsigned long long *Q = nullptr, *status = nullptr, *accept = nullptr, *C = nullptr, *QR = nullptr;
    double *ess = nullptr;
    uint32_t *mpc_dev = nullptr;
    DevAircraft *dac = nullptr;
    float *pop = nullptr, *popp = nullptr, *best_row = nullptr, *papplied = nullptr, *lohi = nullptr;
    double *centres = nullptr, *part_lam = nullptr, *best_lam = nullptr, *pZ = nullptr, *pstates = nullptr,
           *pnext = nullptr;
    long long *part_idx = nullptr, *best_idx = nullptr;
    unsigned *done = nullptr;
    int *pzi = nullptr, *pflags = nullptr;
    // selection records {lambda, index, row}: local (K7) and final (merged across ranks)
    unsigned char *rec_local = nullptr, *rec_final = nullptr, *rec_all = nullptr;
    size_t rec_bytes = 0;
    double *sel_lam = nullptr;
    long long *sel_idx = nullptr;
    float *sel_row = nullptr;
    // multi-GPU
    int world = 1, rank = 0, vworld = 1;
    uint32_t Lfinal = 0, Leval = 0;     // shrinking populations: final count, last evaluated
    // warm start (R45): ids of the current window and of the last solved one; device map
    uint32_t Lw = 0;
    int32_t *wmap = nullptr;
    // wind grid Qhat on the device (FP32 for K2's dense path, FP64 for the plant); host copy
    // of the last upload so unchanged grids are not re-sent every MPC step
    float *qf = nullptr;
    double *qd = nullptr;
    std::vector<double> qd_h;
    std::vector<uint32_t> cur_ids, solved_ids, wmap_h;
    uint32_t solved_H = 0;
    uint32_t Lmax = 0;
    ncclComm_t comm = nullptr;
    unsigned long long *Call = nullptr, *Qall = nullptr, *Csall = nullptr;
    float *Sc = nullptr, *Sall = nullptr;
    uint32_t *dflag = nullptr;
    int32_t *inf_round = nullptr;       // [nmax] first round with an all-zero column (-1: none)
    uint32_t *infcol = nullptr;         // [nmax] scratch: column maxima for the EINFEASIBLE report
    const smc_host_collectives *hcoll = nullptr;   // host-side collectives (test shim) instead of NCCL
    // peer mode (world > 1): every rank's population buffers mapped into this process
    bool p2p = false;
    uint32_t *survp = nullptr;                 // [2][Lmax] this rank's published survivor masks
    const float *peer_ctrl[8] = {};            // rank r's control buffers (4 x prow floats)
    const uint32_t *peer_survp[8] = {};        // rank r's published masks
    const unsigned long long *peer_C[8] = {}, *peer_Cs[8] = {};   // rank r's CDF and CDF samples
    void *peer_open[8] = {};                   // IPC mappings to close

    bool have_scn = false;
    DevScen dsc{};
    PlantScen psc{};
    std::vector<smc_aircraft> ac;
    std::vector<smc_aircraft_type> types;
    std::vector<double> centres_h;
    smc_scenario scn{};
    uint32_t k = 0, mpc = 0, mpc_stage = 0;
    bool acc_clean = false;            // per-round accumulators already zero
    bool mpc_dirty = true;
    int cur = 0, last_eval = -1;
    uint64_t launches = 0;
    uint64_t io_h2d = 0, io_d2h = 0;   // host<->device bytes of the production path
    int anc_mode = -1;                 // SMC_ANC: 1 merge-path K5, 0 bisection in K6, -1 by size
    int32_t *anc = nullptr;            // [n][Lloc] K5 ancestors
    uint32_t *splits = nullptr;        // K5 merge-path split points
    unsigned long long *Cs = nullptr;  // [n][cdf_samples(Lmax)] CDF samples for K6's two-level search
    bool cdf_sample = true;            // SMC_CDF_SAMPLE=0: plain bisection in K6
    bool scan_cluster = true;          // SMC_SCAN=lookback: decoupled look-back scan only
    std::string err;
    // phase timing (cfg.profile): event pairs per phase, summed on request
    std::vector<cudaEvent_t> ev_free;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used[4];
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_graph[4];   // timing nodes inside the captured graph
    double phase_ms_acc[4] = {0, 0, 0, 0};
    uint64_t phase_launches[4] = {0, 0, 0, 0};
    // CUDA graph of one device-resident MPC update (smc_solve)
    bool capturing = false, graph_ok = false;
    int graph_adv = -1;
    uint32_t graph_K = 0, g_k = 0;
    int g_cur = 0, g_last = -1;
    uint64_t g_launches = 0, g_phase_launches[4] = {0, 0, 0, 0};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    void drop_graph() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        gexec = nullptr; graph = nullptr; graph_ok = false;
        for (auto &v : ev_graph) {
            for (auto &p : v) { ev_free.push_back(p.first); ev_free.push_back(p.second); }
            v.clear();
        }
    }
    ~smc_ctx() {
        drop_graph();
        for (void *p : peer_open)
            if (p) ipc_release(p);
        if (comm && nccl_api()) nccl_api()->CommDestroy(comm);
        for (auto &v : ev_used)
            for (auto &p : v) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
        for (auto e : ev_free) cudaEventDestroy(e);
    }
    cudaEvent_t get_event() {
        if (!ev_free.empty()) { cudaEvent_t e = ev_free.back(); ev_free.pop_back(); return e; }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
};

static smc_status fail(smc_ctx *c, smc_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return s;
}

struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static cudaError_t h2d(smc_ctx *c, void *dst, const void *src, size_t bytes) {
    c->io_h2d += bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->st);
}
static cudaError_t d2h(smc_ctx *c, void *dst, const void *src, size_t bytes) {
    c->io_d2h += bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->st);
}

#define CK(expr)                                                                                   \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) return fail(ctx, SMC_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)
#define NCK(expr)                                                                                  \
    do {                                                                                           \
        ++ctx->launches;                                                                           \
        ncclResult_t _r = (expr);                                                                  \
        if (_r != 0) return fail(ctx, SMC_ENCCL, "%s: %s", #expr,                                  \
                                 nccl_api()->GetErrorString ? nccl_api()->GetErrorString(_r) : "nccl error"); \
    } while (0)
#define LAUNCHP(phase, expr)                                                                       \
    do {                                                                                           \
        ++ctx->launches;                                                                           \
        ++ctx->phase_launches[phase];                                                              \
        cudaEvent_t _e0 = nullptr, _e1 = nullptr;                                                  \
        if (ctx->cfg.profile) { _e0 = ctx->get_event(); _e1 = ctx->get_event();                   \
                                CK(cudaEventRecordWithFlags(_e0, ctx->st, ctx->capturing ? cudaEventRecordExternal : 0)); } \
        CK(expr);                                                                                  \
        if (ctx->cfg.profile) { CK(cudaEventRecordWithFlags(_e1, ctx->st, ctx->capturing ? cudaEventRecordExternal : 0)); \
                                (ctx->capturing ? ctx->ev_graph[phase] : ctx->ev_used[phase]).push_back({_e0, _e1}); } \
    } while (0)
#define LAUNCH(expr) LAUNCHP(3, expr)
enum { PH_ROLLOUT = 0, PH_RESAMPLE = 1, PH_PROPOSE = 2, PH_OTHER = 3 };

// ---------------------------------------------------------------- collectives
// NCCL on the context's communicator, or the host-side shim (cfg.host_coll: test mode, the
// operands round-trip through the host around the caller's collective).
static smc_status coll_allreduce_max_u32(smc_ctx *ctx, uint32_t *dev, size_t count) {
    if (ctx->hcoll) {
        std::vector<uint32_t> h(count);
        CK(cudaMemcpyAsync(h.data(), dev, 4 * count, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        if (ctx->hcoll->allreduce_max_u32(ctx->hcoll->user, h.data(), count) != 0)
            return fail(ctx, SMC_ENCCL, "host all-reduce failed");
        CK(cudaMemcpyAsync(dev, h.data(), 4 * count, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        ++ctx->launches;
        return SMC_OK;
    }
    NCK(nccl_api()->AllReduce(dev, dev, count, ncclUint32_, ncclMax_, ctx->comm, ctx->st));
    return SMC_OK;
}

static smc_status coll_allgather(smc_ctx *ctx, const void *dev_send, void *dev_recv, size_t bytes) {
    if (ctx->hcoll) {
        std::vector<unsigned char> hs(bytes), hr(bytes * (size_t)ctx->world);
        CK(cudaMemcpyAsync(hs.data(), dev_send, bytes, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        if (ctx->hcoll->allgather(ctx->hcoll->user, hs.data(), hr.data(), bytes) != 0)
            return fail(ctx, SMC_ENCCL, "host all-gather failed");
        CK(cudaMemcpyAsync(dev_recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        ++ctx->launches;
        return SMC_OK;
    }
    NCK(nccl_api()->AllGather(dev_send, dev_recv, bytes, ncclUint8_, ctx->comm, ctx->st));
    return SMC_OK;
}

#define COLL(expr)                                                                                 \
    do {                                                                                           \
        smc_status _s = (expr);                                                                    \
        if (_s != SMC_OK) return _s;                                                               \
    } while (0)

// ---------------------------------------------------------------- partition helpers
extern "C" void smc_shard_range(uint32_t L, int32_t world, int32_t rank, uint32_t *begin, uint32_t *end) {
    if (world < 1) world = 1;
    const uint64_t b = (uint64_t)L * (uint64_t)rank / (uint64_t)world;
    const uint64_t e = (uint64_t)L * (uint64_t)(rank + 1) / (uint64_t)world;
    *begin = (uint32_t)b;
    *end = (uint32_t)e;
}

extern "C" void smc_shard_offsets(uint32_t N, int32_t world, int32_t rank, const uint64_t *Q_all, uint64_t *offset,
                                  uint64_t *Q_total) {
    for (uint32_t i = 0; i < N; ++i) {
        uint64_t off = 0, tot = 0;
        for (int r = 0; r < world; ++r) {
            if (r < rank) off += Q_all[(size_t)r * N + i];
            tot += Q_all[(size_t)r * N + i];
        }
        if (offset) offset[i] = off;
        if (Q_total) Q_total[i] = tot;
    }
}

extern "C" uint64_t smc_slot_count(uint64_t C, uint64_t Q, uint64_t R, uint32_t L) { return slot_count(C, Q, R, L); }

// ---------------------------------------------------------------- lifecycle
extern "C" size_t smc_workspace_bytes(const smc_config *cfg) {
    if (!cfg || cfg->n_particles == 0 || cfg->max_aircraft == 0 || cfg->max_aircraft > 32 || cfg->max_horizon == 0 ||
        cfg->max_horizon > 32)
        return 0;
    const int world = cfg->world_size < 1 ? 1 : cfg->world_size;
    const int vw = (world == 1 && cfg->virtual_world > 1) ? (int)cfg->virtual_world : 1;
    return layout(max_local(cfg->n_particles, world), cfg->max_aircraft, cfg->max_horizon, world, vw).total;
}

// Peer mode: export this rank's workspace allocation as a CUDA IPC handle, all-gather the
// handles (NCCL, through the ipc scratch), and map every other rank's allocation.  The
// workspace is a sub-range of a caller (torch) allocation, so each record carries the
// workspace's offset from its allocation base (driver cuMemGetAddressRange).
static cudaError_t ipc_record(const void *ws, unsigned char rec[kIpcRec]) {
    typedef int (*GetRange)(unsigned long long *, size_t *, unsigned long long);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (h) get_range = (GetRange)dlsym(h, "cuMemGetAddressRange_v2");
    }
    if (!get_range) return cudaErrorNotSupported;
    unsigned long long base = 0;
    size_t bytes = 0;
    if (get_range(&base, &bytes, (unsigned long long)(uintptr_t)ws) != 0) return cudaErrorInvalidDevicePointer;
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
    if (e != cudaSuccess) return e;
    const uint64_t off = (uint64_t)((uintptr_t)ws - base);
    memset(rec, 0, kIpcRec);
    memcpy(rec, &h, sizeof(h));
    memcpy(rec + sizeof(h), &off, sizeof(off));
    return cudaSuccess;
}

// A handle may be opened once per process: mappings are shared and reference-counted
// (two contexts -- e.g. bench.py's timed and profiled solvers -- may map the same peer
// allocation when the peer's caching allocator placed both workspaces in one segment).
struct IpcMapping { cudaIpcMemHandle_t h; void *p; int refs; };
static std::vector<IpcMapping> &ipc_cache() { static std::vector<IpcMapping> c; return c; }

// Map a peer's record: *mapping = the opened allocation (to release), *ws = its workspace.
static cudaError_t ipc_open(const unsigned char *rec, void **mapping, char **ws) {
    cudaIpcMemHandle_t h;
    uint64_t off;
    memcpy(&h, rec, sizeof(h));
    memcpy(&off, rec + sizeof(h), sizeof(off));
    for (auto &m : ipc_cache())
        if (memcmp(&m.h, &h, sizeof(h)) == 0) {
            ++m.refs;
            *mapping = m.p;
            *ws = (char *)m.p + off;
            return cudaSuccess;
        }
    void *p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return e;
    ipc_cache().push_back({h, p, 1});
    *mapping = p;
    *ws = (char *)p + off;
    return cudaSuccess;
}

static void ipc_release(void *mapping) {
    auto &c = ipc_cache();
    for (size_t q = 0; q < c.size(); ++q)
        if (c[q].p == mapping) {
            if (--c[q].refs == 0) {
                cudaIpcCloseMemHandle(mapping);
                c.erase(c.begin() + (long)q);
            }
            return;
        }
}

// Peer mode: every rank maps every other rank's workspace.  A rank that cannot open a mapping
// reports it through an all-reduce, and then every rank falls back to the all-gather exchange
// (the modes must agree: they issue different collectives).
static smc_status map_peers(smc_ctx *ctx) {
    unsigned char rec[kIpcRec];
    const int G = ctx->world;
    uint32_t bad = ipc_record(ctx->ws, rec) == cudaSuccess ? 0u : 1u;
    unsigned char *dipc = (unsigned char *)ctx->ws + ctx->lay.ipc;
    CK(cudaMemcpyAsync(dipc + (size_t)G * kIpcRec, rec, kIpcRec, cudaMemcpyHostToDevice, ctx->st));
    COLL(coll_allgather(ctx, dipc + (size_t)G * kIpcRec, dipc, kIpcRec));
    std::vector<unsigned char> all((size_t)G * kIpcRec);
    CK(cudaMemcpyAsync(all.data(), dipc, all.size(), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    for (int r = 0; r < G && !bad; ++r) {
        char *pws = (char *)ctx->ws;
        if (r != ctx->rank && ipc_open(all.data() + (size_t)r * kIpcRec, &ctx->peer_open[r], &pws) != cudaSuccess) {
            cudaGetLastError();
            bad = 1u;
            break;
        }
        // every rank carves the same layout (same config), so offsets agree
        ctx->peer_ctrl[r] = (const float *)(pws + ctx->lay.ctrl);
        ctx->peer_survp[r] = (const uint32_t *)(pws + ctx->lay.survp);
        ctx->peer_C[r] = (const unsigned long long *)(pws + ctx->lay.C);
        ctx->peer_Cs[r] = (const unsigned long long *)(pws + ctx->lay.Cs);
    }
    CK(cudaMemcpyAsync(ctx->dflag, &bad, 4, cudaMemcpyHostToDevice, ctx->st));
    COLL(coll_allreduce_max_u32(ctx, ctx->dflag, 1));
    CK(cudaMemcpyAsync(&bad, ctx->dflag, 4, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (bad) {                                       // some rank could not map a peer: all-gather mode
        for (void *&m : ctx->peer_open)
            if (m) { ipc_release(m); m = nullptr; }
        ctx->p2p = false;
    }
    return SMC_OK;
}

// Test hooks of the peer mapping (one GPU, two processes, no kernel waits on another).
extern "C" smc_status smc_ipc_record(const smc_ctx *ctx, void *out128) {
    if (!ctx || !out128) return SMC_EINVAL;
    return ipc_record(ctx->ws, (unsigned char *)out128) == cudaSuccess ? SMC_OK : SMC_ECUDA;
}

extern "C" smc_status smc_ipc_peek(const void *rec128, uint64_t offset, void *host_out, size_t bytes) {
    if (!rec128 || !host_out) return SMC_EINVAL;
    void *map = nullptr;
    char *ws = nullptr;
    if (ipc_open((const unsigned char *)rec128, &map, &ws) != cudaSuccess) return SMC_ECUDA;
    const cudaError_t e = cudaMemcpy(host_out, ws + offset, bytes, cudaMemcpyDeviceToHost);
    ipc_release(map);
    return e == cudaSuccess ? SMC_OK : SMC_ECUDA;
}

extern "C" smc_status smc_init(const smc_config *cfg, smc_ctx **out) {
    if (!cfg || !out) return SMC_EINVAL;
    *out = nullptr;
    smc_ctx *ctx = new smc_ctx();
    ctx->cfg = *cfg;
    const int world = cfg->world_size < 1 ? 1 : cfg->world_size;
    if (world > 8 || cfg->rank < 0 || cfg->rank >= world || (world > 1 && !cfg->nccl_unique_id && !cfg->host_coll) ||
        cfg->n_particles < (uint32_t)world || (cfg->host_coll && cfg->use_graph) ||
        (cfg->host_coll && (!cfg->host_coll->allreduce_max_u32 || !cfg->host_coll->allgather))) {
        delete ctx;
        return SMC_EINVAL;
    }
    ctx->world = world;
    ctx->rank = cfg->rank;
    if (cfg->n_particles == 0 || cfg->max_aircraft == 0 || cfg->max_aircraft > 32 || cfg->max_horizon == 0 ||
        cfg->max_horizon > 32 || cfg->n_samples == 0 || cfg->n_samples > 65535 || cfg->n_particles >= (1u << 30) ||
        (uint64_t)cfg->n_particles * cfg->max_aircraft >= (1ull << 31) || cfg->mh > 2) {
        delete ctx;
        return SMC_EINVAL;
    }
    {
        // ancestors: merge-path K5 + K6 reading them ("mp"), or bisection inside K6 ("bisect");
        // default by population size
        const char *sm = getenv("SMC_SCAN");
        ctx->scan_cluster = !(sm && strcmp(sm, "lookback") == 0);
        const char *cs = getenv("SMC_CDF_SAMPLE");          // K6 two-level search (default on)
        ctx->cdf_sample = !(cs && strcmp(cs, "0") == 0);
        const char *am = getenv("SMC_ANC");
        // "bisect2": debug_resample runs K6's two-level search (production default below 2^17)
        ctx->anc_mode = am ? (strcmp(am, "mp") == 0 ? 1 : (strcmp(am, "bisect") == 0 ? 0 :
                                                          (strcmp(am, "bisect2") == 0 ? 2 : -1))) : -1;
    }
    ctx->Lg = cfg->n_particles;
    smc_shard_range(ctx->Lg, world, cfg->rank, &ctx->l0, &ctx->Lloc);
    ctx->Lloc -= ctx->l0;
    ctx->nmax = (int)cfg->max_aircraft;
    ctx->Hmax = (int)cfg->max_horizon;
    ctx->vworld = (world == 1 && cfg->virtual_world > 1) ? (int)cfg->virtual_world : 1;
    ctx->Lfinal = (cfg->n_particles_final && cfg->n_particles_final < cfg->n_particles) ? cfg->n_particles_final : 0;
    if (ctx->Lfinal && (world > 1 || ctx->vworld > 1)) { delete ctx; return SMC_EINVAL; }
    if (ctx->vworld > 8 || ctx->Lg < (uint32_t)ctx->vworld) { delete ctx; return SMC_EINVAL; }
    ctx->lay = layout(max_local(ctx->Lg, world), ctx->nmax, ctx->Hmax, world, ctx->vworld);
    if (!cfg->workspace || cfg->workspace_bytes < ctx->lay.total) {
        delete ctx;
        return SMC_ENOMEM;
    }
    cudaError_t e = cudaSetDevice(cfg->device);
    if (e != cudaSuccess) {
        delete ctx;
        return SMC_ECUDA;
    }
    ctx->st = (cudaStream_t)cfg->stream;
    char *ws = (char *)cfg->workspace;
    ctx->ws = ws;
    const Layout &L = ctx->lay;
    const size_t row = (size_t)ctx->Lloc * ctx->nmax * ctx->Hmax * 3;
    (void)row;
    const size_t prow = (size_t)max_local(ctx->Lg, world) * ctx->nmax * ctx->Hmax * 3;
    float *cb = (float *)(ws + L.ctrl);
    ctx->ctrl[0][0] = cb;
    ctx->ctrl[0][1] = cb + prow;
    ctx->ctrl[1][0] = cb + 2 * prow;
    ctx->ctrl[1][1] = cb + 3 * prow;
    ctx->ell = (float *)(ws + L.ell);
    cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, cfg->device);
    ctx->lam = (double *)(ws + L.lam);
    ctx->lam2 = (double *)(ws + L.lam2);
    ctx->surv = (uint32_t *)(ws + L.surv);
    ctx->colmax = (uint32_t *)(ws + L.colmax);
    ctx->Q = (unsigned long long *)(ws + L.Q);
    ctx->ess = (double *)(ws + L.ess);
    ctx->status = (unsigned long long *)(ws + L.status);
    ctx->tiles = (uint32_t *)(ws + L.tiles);
    ctx->C = (unsigned long long *)(ws + L.C);
    ctx->QR = (unsigned long long *)(ws + L.QR);
    ctx->anc = (int32_t *)(ws + L.anc);
    ctx->splits = (uint32_t *)(ws + L.splits);
    ctx->Cs = (unsigned long long *)(ws + L.Cs);
    ctx->accept = (unsigned long long *)(ws + L.accept);
    ctx->mpc_dev = (uint32_t *)(ws + L.mpc);
    ctx->dac = (DevAircraft *)(ws + L.dac);
    ctx->pop = (float *)(ws + L.pop);
    ctx->popp = (float *)(ws + L.popp);
    ctx->centres = (double *)(ws + L.centres);
    ctx->part_lam = (double *)(ws + L.part_lam);
    ctx->part_idx = (long long *)(ws + L.part_idx);
    ctx->done = (unsigned *)(ws + L.done);
    ctx->rec_bytes = record_bytes(ctx->nmax, ctx->Hmax);
    ctx->rec_local = (unsigned char *)(ws + L.best_lam);
    ctx->rec_final = (world > 1 || ctx->vworld > 1) ? (unsigned char *)(ws + L.best_idx) : ctx->rec_local;
    ctx->rec_all = (unsigned char *)(ws + L.best_row);
    ctx->sel_lam = (double *)ctx->rec_local;
    ctx->sel_idx = (long long *)(ctx->rec_local + 8);
    ctx->sel_row = (float *)(ctx->rec_local + 16);
    ctx->best_lam = (double *)ctx->rec_final;
    ctx->best_idx = (long long *)(ctx->rec_final + 8);
    ctx->best_row = (float *)(ctx->rec_final + 16);
    ctx->Lmax = world > 1 ? max_local(ctx->Lg, world) : max_local(ctx->Lg, ctx->vworld);
    ctx->Call = (unsigned long long *)(ws + L.Call);
    ctx->Qall = (unsigned long long *)(ws + L.Qall);
    ctx->Csall = (unsigned long long *)(ws + L.Csall);
    ctx->dflag = (uint32_t *)(ws + L.flag);
    ctx->inf_round = (int32_t *)(ws + L.infround);
    ctx->infcol = (uint32_t *)(ws + L.infcol);
    ctx->hcoll = world > 1 ? cfg->host_coll : nullptr;
    ctx->Sc = (float *)(ws + L.Sc);
    ctx->Sall = (float *)(ws + L.Sall);
    ctx->p2p = p2p_mode() && (world > 1 || ctx->vworld > 1);
    ctx->survp = (uint32_t *)(ws + L.survp);
    ctx->pZ = (double *)(ws + L.pZ);
    ctx->pzi = (int *)(ws + L.pzi);
    ctx->pstates = (double *)(ws + L.pstates);
    ctx->pnext = (double *)(ws + L.pnext);
    ctx->pflags = (int *)(ws + L.pflags);
    ctx->papplied = (float *)(ws + L.papplied);
    ctx->lohi = (float *)(ws + L.lohi);
    ctx->wmap = (int32_t *)(ws + L.wmap);
    ctx->qf = (float *)(ws + L.qf);
    ctx->qd = (double *)(ws + L.qd);
    if (cfg->warm_fraction > 0.0) {
        const double w = cfg->warm_fraction < 1.0 ? cfg->warm_fraction : 1.0;
        ctx->Lw = (uint32_t)std::floor(w * (double)ctx->Lg);
    }
    e = cudaMemsetAsync(ws, 0, L.total, ctx->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->wmap, 0xFF, L.total - L.wmap, ctx->st);   // map = -1
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    if (e != cudaSuccess) {
        delete ctx;
        return SMC_ECUDA;
    }
    ctx->wmap_h.assign(ctx->nmax, 0xFFFFFFFFu);
    if (world > 1) {
        if (!ctx->hcoll) {
            NcclApi *api = nccl_api();
            if (!api) { delete ctx; return SMC_ENCCL; }
            ncclUniqueId id;
            memcpy(&id, cfg->nccl_unique_id, sizeof(id));
            if (api->CommInitRank(&ctx->comm, world, id, cfg->rank) != 0) { ctx->comm = nullptr; delete ctx; return SMC_ENCCL; }
        }
        if (ctx->p2p) {
            const smc_status s = map_peers(ctx);
            if (s != SMC_OK) { delete ctx; return s; }
        }
    }
    *out = ctx;
    return SMC_OK;
}

extern "C" smc_status smc_nccl_unique_id(void *out128) {
    NcclApi *api = nccl_api();
    if (!api || !out128) return SMC_ENCCL;
    ncclUniqueId id;
    if (api->GetUniqueId(&id) != 0) return SMC_ENCCL;
    memcpy(out128, &id, sizeof(id));
    return SMC_OK;
}

extern "C" void smc_destroy(smc_ctx *ctx) { delete ctx; }
extern "C" const char *smc_last_error(const smc_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }
extern "C" uint64_t smc_launch_count(const smc_ctx *ctx) { return ctx ? ctx->launches : 0; }
extern "C" void smc_io_bytes(smc_ctx *ctx, uint64_t *h2d_bytes, uint64_t *d2h_bytes) {
    if (!ctx) return;
    if (h2d_bytes) *h2d_bytes = ctx->io_h2d;
    if (d2h_bytes) *d2h_bytes = ctx->io_d2h;
    ctx->io_h2d = ctx->io_d2h = 0;
}
extern "C" uint32_t smc_get_mpc_index(const smc_ctx *ctx) { return ctx ? ctx->mpc : 0; }
extern "C" smc_status smc_set_mpc_index(smc_ctx *ctx, uint32_t m) {
    if (!ctx) return SMC_EINVAL;
    if (m >= (1u << 24)) return fail(ctx, SMC_EINVAL, "mpc index must be < 2^24");
    ctx->mpc = m;
    ctx->mpc_dirty = true;
    return SMC_OK;
}

// The MPC step index keys every stream; kernels read it from device memory so
// a captured graph stays valid across MPC steps.
static smc_status sync_mpc(smc_ctx *ctx) {
    if (!ctx->mpc_dirty) return SMC_OK;
    ctx->mpc_stage = ctx->mpc;
    CK(h2d(ctx, ctx->mpc_dev, &ctx->mpc_stage, sizeof(uint32_t)));
    ctx->mpc_dirty = false;
    return SMC_OK;
}

// ---------------------------------------------------------------- scenario precompute (host FP64)
// Cholesky factor Lo Lo^T = A of an SPD N x N matrix (row-major).
static int cholesky(const double *A, double *Lo, int N) {
    for (int q = 0; q < N * N; ++q) Lo[q] = 0.0;
    for (int j = 0; j < N; ++j) {
        double d = A[j * N + j];
        for (int p = 0; p < j; ++p) d -= Lo[j * N + p] * Lo[j * N + p];
        if (!(d > 0.0)) return -1;
        Lo[j * N + j] = std::sqrt(d);
        for (int r = j + 1; r < N; ++r) {
            double s = A[r * N + j];
            for (int p = 0; p < j; ++p) s -= Lo[r * N + p] * Lo[j * N + p];
            Lo[r * N + j] = s / Lo[j * N + j];
        }
    }
    return 0;
}

static int wind_axis(uint32_t v) { return v ? (int)v : 2; }

static smc_status build_constants(smc_ctx *ctx) {
    const smc_scenario &s = ctx->scn;
    const int n = (int)s.n_aircraft, H = (int)s.horizon;
    DevScen &d = ctx->dsc;
    PlantScen &p = ctx->psc;
    d = DevScen{};
    p = PlantScen{};
    d.n = n; d.H = H; d.density_mode = s.density_mode;
    d.dt = (float)s.dt; d.g = (float)s.g; d.rho_const = (float)s.rho_const;
    d.P_runway = (float)s.P_runway; d.P_beta = (float)s.P_beta; d.P_chi = (float)s.P_chi; d.P_vs = (float)s.P_vs;
    d.P_chi_west = (float)(3.14159265358979323846 - s.P_chi);
    d.twoPr2 = (float)((2.0 * s.P_r) * (2.0 * s.P_r));
    d.twoPh = (float)(2.0 * s.P_h);
    for (int q = 0; q < 4; ++q) d.alpha_dep[q] = (float)s.alpha_dep[q];
    for (int q = 0; q < 3; ++q) d.alpha_arr[q] = (float)s.alpha_arr[q];
    d.has_noise = s.noise_w > 0.0 && s.pop_nx > 0 && s.pop_ny > 0;
    d.noise_w = (float)s.noise_w;
    d.inv_Ac = (float)(1.0 / s.A_c);
    d.pop_nx = (int)s.pop_nx; d.pop_ny = (int)s.pop_ny;
    d.pop_x0 = (float)s.pop_x0; d.pop_y0 = (float)s.pop_y0; d.pop_inv_dx = (float)(1.0 / s.pop_dx);
    {
        const double mx = s.pop_nx > 1 ? (double)(s.pop_nx - 1) : 0.0, my = s.pop_ny > 1 ? (double)(s.pop_ny - 1) : 0.0;
        d.pop_mx = (float)mx; d.pop_my = (float)my;
        d.pop_ax = mx > 0 ? (float)(1.0 / (s.pop_dx * mx)) : 0.0f; d.pop_bx = mx > 0 ? (float)(-s.pop_x0 / (s.pop_dx * mx)) : 0.0f;
        d.pop_ay = my > 0 ? (float)(1.0 / (s.pop_dx * my)) : 0.0f; d.pop_by = my > 0 ? (float)(-s.pop_y0 / (s.pop_dx * my)) : 0.0f;
    }
    for (int a = 0; a < 3; ++a) {
        d.wind_lo[a] = (float)s.wind_lo[a];
        d.wind_inv_ext[a] = (float)(1.0 / (s.wind_hi[a] - s.wind_lo[a]));
    }
    // Eq. cov between the N_x N_y N_z grid points (same time),
    // evenly spaced over the wind box, node = ix + N_x (iy + N_y iz)
    const int wnx = wind_axis(s.wind_n[0]), wny = wind_axis(s.wind_n[1]), wnz = wind_axis(s.wind_n[2]);
    const int G = wnx * wny * wnz;
    std::vector<double> Rh((size_t)G * G), Qh((size_t)G * G, 0.0), pos((size_t)G * 3);
    for (int a = 0; a < G; ++a) {
        const int idx[3] = {a % wnx, (a / wnx) % wny, a / (wnx * wny)}, cnt[3] = {wnx, wny, wnz};
        for (int c = 0; c < 3; ++c)
            pos[3 * a + c] = s.wind_lo[c] + (s.wind_hi[c] - s.wind_lo[c]) * (double)idx[c] / (double)(cnt[c] - 1);
    }
    const double ext = s.wind_hi[2] - s.wind_lo[2];
    for (int a = 0; a < G; ++a)
        for (int b = 0; b < G; ++b) {
            const double *pa = &pos[3 * a], *pb = &pos[3 * b];
            const double sa = s.sigma_lo + (s.sigma_hi - s.sigma_lo) * (pa[2] - s.wind_lo[2]) / ext;
            const double sb = s.sigma_lo + (s.sigma_hi - s.sigma_lo) * (pb[2] - s.wind_lo[2]) / ext;
            Rh[(size_t)a * G + b] = sa * sb * std::exp(-s.beta_w * std::hypot(pa[0] - pb[0], pa[1] - pb[1])) *
                                    std::exp(-s.gamma_w * std::fabs(pa[2] - pb[2]));
        }
    bool zero = true;
    for (double v : Rh) zero = zero && v == 0.0;
    if (!zero && cholesky(Rh.data(), Qh.data(), G) != 0)
        return fail(ctx, SMC_EINVAL, "wind covariance not positive definite");
    d.wn[0] = wnx; d.wn[1] = wny; d.wn[2] = wnz; d.wng = G;
    p.wn[0] = wnx; p.wn[1] = wny; p.wn[2] = wnz; p.ng = G;
    d.Qf = ctx->qf; p.Qd = ctx->qd;
    if (Qh != ctx->qd_h) {                 // upload only when the grid constants change
        std::vector<float> qf(Qh.size());
        for (size_t q = 0; q < Qh.size(); ++q) qf[q] = (float)Qh[q];
        CK(h2d(ctx, ctx->qd, Qh.data(), sizeof(double) * Qh.size()));
        CK(h2d(ctx, ctx->qf, qf.data(), sizeof(float) * qf.size()));
        CK(cudaMemsetAsync(ctx->pzi, 0, sizeof(int), ctx->st));   // new grid: plant field restarts
        CK(cudaStreamSynchronize(ctx->st));  // host vectors go out of scope
        ctx->qd_h = Qh;
    }
    if (G == 8)
        for (int q = 0; q < 64; ++q) d.Qhat[q] = (float)Qh[q];
    // trilinear basis change (tripoly): coefficient r = sum_n M[r][n] W_n
    static const int Mtri[8][8] = {{1, 0, 0, 0, 0, 0, 0, 0},   {-1, 1, 0, 0, 0, 0, 0, 0},
                                   {-1, 0, 1, 0, 0, 0, 0, 0},  {-1, 0, 0, 0, 1, 0, 0, 0},
                                   {1, -1, -1, 1, 0, 0, 0, 0}, {1, -1, 0, 0, -1, 1, 0, 0},
                                   {1, 0, -1, 0, -1, 0, 1, 0}, {-1, 1, 1, -1, 1, -1, -1, 1}};
    for (int r = 0; r < 8; ++r)
        for (int m = 0; m < 8; ++m) {
            double acc = 0.0;
            if (G == 8)
                for (int nn = 0; nn < 8; ++nn) acc += Mtri[r][nn] * Qh[nn * 8 + m];
            d.Cq[r * 8 + m] = (float)acc;
        }
    p.a = std::exp(-s.lambda_t * s.dt);
    p.b = std::sqrt(1.0 - p.a * p.a);
    d.a = (float)p.a; d.b = (float)p.b;
    d.nominal[0] = (float)s.nominal[0]; d.nominal[1] = (float)s.nominal[1];
    d.turb_sigma = (float)s.turb_sigma;
    d.key0 = (uint32_t)ctx->cfg.seed; d.key1 = (uint32_t)(ctx->cfg.seed >> 32);
    for (int r = 0; r < 10; ++r) {
        d.ks[2 * r] = d.key0 + (uint32_t)r * 0x9E3779B9u;
        d.ks[2 * r + 1] = d.key1 + (uint32_t)r * 0xBB67AE85u;
    }
    d.ac = ctx->dac;
    d.pop = ctx->pop;
    d.popp = ctx->popp;
    p.dt = s.dt; p.g = s.g; p.rho_const = s.rho_const; p.density_mode = s.density_mode;
    for (int a = 0; a < 3; ++a) { p.wind_lo[a] = s.wind_lo[a]; p.wind_hi[a] = s.wind_hi[a]; }
    p.nominal[0] = s.nominal[0]; p.nominal[1] = s.nominal[1];
    p.turb_sigma = s.turb_sigma; p.tma_radius = s.tma_radius;
    p.P_runway = s.P_runway; p.P_beta = s.P_beta; p.P_chi = s.P_chi; p.P_vs = s.P_vs;

    std::vector<DevAircraft> hac(n);
    std::vector<float> lohi(6 * n);
    for (int i = 0; i < n; ++i) {
        const smc_aircraft &a = ctx->ac[i];
        const smc_aircraft_type &ty = ctx->types[a.type];
        DevAircraft &A = hac[i];
        A.kind = (int)a.kind;
        A.first_step = (int)a.first_step;
        A.Ha = H - (int)a.first_step;
        const double x0[6] = {a.x0.x, a.x0.y, a.x0.z, a.x0.v, a.x0.chi, a.x0.m};
        for (int q = 0; q < 6; ++q) A.x0[q] = (float)x0[q];
        A.x0[4] = (float)std::remainder(x0[4], 2.0 * 3.14159265358979323846);   // K2 keeps chi in [-pi, pi]
        A.theta_F = (float)a.theta_F; A.z_tf = (float)a.z_tf; A.v_D = (float)a.v_D; A.beta_f = (float)a.beta_f;
        A.halfS = (float)(0.5 * ty.S); A.cd0 = (float)ty.cd0; A.cd2 = (float)ty.cd2; A.dt_eta = (float)(s.dt * ty.eta);
        A.m_empty = (float)ty.m_empty; A.T_min = (float)ty.T_min; A.T_max = (float)ty.T_max;
        A.v_min = (float)ty.v_min; A.v_max = (float)ty.v_max; A.gamma_max = (float)ty.gamma_max;
        A.phi_max = (float)ty.phi_max; A.z_min = (float)ty.z_min; A.z_max = (float)ty.z_max;
        // altitude term B: sup / inf by reachability with gamma_max, v_max (R21)
        double ssum = 0.0, isum = 0.0;
        for (int j = (int)a.first_step + 1; j <= H; ++j) {
            const double reach = (double)(j - (int)a.first_step) * s.dt * ty.v_max * std::sin(ty.gamma_max);
            const double lo = std::max(ty.z_min, a.x0.z - reach), hi = std::min(ty.z_max, a.x0.z + reach);
            ssum += std::max(std::fabs(a.z_tf - lo), std::fabs(a.z_tf - hi));
            const double near = std::min(std::max(a.z_tf, lo), hi);
            isum += std::fabs(a.z_tf - near);
        }
        const double supB = A.Ha > 0 ? ssum / A.Ha : 0.0, infB = A.Ha > 0 ? isum / A.Ha : 0.0;
        A.supB = (float)supB;
        A.flagB = (supB - infB) < 1.0 ? 1 : 0;
        A.invDenB = A.flagB ? 0.0f : (float)(1.0 / (supB - infB));
        A.invSupC = (float)(1.0 / std::max(ty.v_max - a.v_D, a.v_D - ty.v_min));
        A.invSupE = (float)(1.0 / std::max(a.beta_f, 1.5707963267948966 - a.beta_f));
        const double Fmax = s.dt * A.Ha * ty.T_max * ty.eta;
        A.invFmax = Fmax > 0.0 ? (float)(1.0 / Fmax) : 0.0f;
        A.invHa = A.Ha > 0 ? (float)(1.0 / A.Ha) : 0.0f;
        lohi[6 * i + 0] = (float)ty.T_min; lohi[6 * i + 1] = (float)-ty.phi_max; lohi[6 * i + 2] = (float)-ty.gamma_max;
        lohi[6 * i + 3] = (float)ty.T_max; lohi[6 * i + 4] = (float)ty.phi_max; lohi[6 * i + 5] = (float)ty.gamma_max;
        p.kind[i] = A.kind; p.first_step[i] = A.first_step;
        p.halfS[i] = 0.5 * ty.S; p.cd0[i] = ty.cd0; p.cd2[i] = ty.cd2; p.eta[i] = ty.eta;
        p.m_empty[i] = ty.m_empty; p.T_min[i] = ty.T_min; p.T_max[i] = ty.T_max; p.v_min[i] = ty.v_min;
        p.v_max[i] = ty.v_max; p.gamma_max[i] = ty.gamma_max; p.phi_max[i] = ty.phi_max;
        p.z_min[i] = ty.z_min; p.z_max[i] = ty.z_max;
    }
    CK(h2d(ctx, ctx->dac, hac.data(), sizeof(DevAircraft) * n));
    // lohi: stored as [n][3] lo followed by [n][3] hi
    std::vector<float> lo3(3 * n), hi3(3 * n);
    for (int i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) { lo3[3 * i + c] = lohi[6 * i + c]; hi3[3 * i + c] = lohi[6 * i + 3 + c]; }
    CK(h2d(ctx, ctx->lohi, lo3.data(), sizeof(float) * 3 * n));
    CK(h2d(ctx, ctx->lohi + 3 * ctx->nmax, hi3.data(), sizeof(float) * 3 * n));
    CK(cudaStreamSynchronize(ctx->st));   // host staging vectors go out of scope
    return SMC_OK;
}

// Warm start (R45): map aircraft of this window to rows of the last solved window's
// winner by id (host-side; uploaded only when it changes, outside any graph).
static smc_status warm_prepare(smc_ctx *ctx) {
    if (!ctx->Lw) return SMC_OK;
    const int n = ctx->dsc.n;
    std::vector<uint32_t> m(ctx->nmax, 0xFFFFFFFFu);
    if (ctx->solved_H == (uint32_t)ctx->dsc.H)
        for (int i = 0; i < n; ++i)
            for (size_t j = 0; j < ctx->solved_ids.size(); ++j)
                if (ctx->solved_ids[j] == ctx->cur_ids[i]) { m[i] = (uint32_t)j; break; }
    if (m != ctx->wmap_h) {
        ctx->wmap_h = m;
        CK(h2d(ctx, ctx->wmap, m.data(), sizeof(int32_t) * ctx->nmax));
    }
    return SMC_OK;
}

static void warm_solved(smc_ctx *ctx) {
    ctx->solved_ids = ctx->cur_ids;
    ctx->solved_H = (uint32_t)ctx->dsc.H;
}

static smc_status init_population(smc_ctx *ctx) {
    smc_status s0 = sync_mpc(ctx);
    if (s0 != SMC_OK) return s0;
    if (!ctx->capturing) {                 // graph replays: smc_solve prepares the map first
        s0 = warm_prepare(ctx);
        if (s0 != SMC_OK) return s0;
    }
    PopArgs pa{};
    pa.n = ctx->dsc.n; pa.H = ctx->dsc.H; pa.L = ctx->Lloc; pa.l0 = ctx->l0; pa.k = 0u;
    pa.key0 = ctx->dsc.key0; pa.key1 = ctx->dsc.key1; pa.mpcp = ctx->mpc_dev;
    pa.Lw = ctx->Lw; pa.warm_row = ctx->best_row; pa.warm_ok = ctx->best_idx; pa.warm_map = ctx->wmap;
    for (int c = 0; c < 3; ++c) pa.sig[c] = (float)ctx->cfg.sigma[c];
    pa.clamp = (int)ctx->cfg.clamp_proposals;
    pa.lo3 = ctx->lohi; pa.hi3 = ctx->lohi + 3 * ctx->nmax;
    LAUNCH(launch_init_population(ctx->dsc, pa, ctx->ctrl[0][0], ctx->st));
    CK(cudaMemsetAsync(ctx->inf_round, 0xFF, sizeof(int32_t) * ctx->nmax, ctx->st));
    ctx->k = 0;
    ctx->cur = 0;
    ctx->last_eval = -1;
    ctx->acc_clean = false;            // round 0 zeroes the accumulators itself (also inside graphs)
    return SMC_OK;
}

extern "C" smc_status smc_set_scenario(smc_ctx *ctx, const smc_scenario *scn) {
    if (!ctx || !scn) return SMC_EINVAL;
    const uint32_t n = scn->n_aircraft, H = scn->horizon;
    if (n == 0 || n > (uint32_t)ctx->nmax) return fail(ctx, SMC_EINVAL, "n_aircraft %u outside [1, %d]", n, ctx->nmax);
    if (H == 0 || H > (uint32_t)ctx->Hmax) return fail(ctx, SMC_EINVAL, "horizon %u outside [1, %d]", H, ctx->Hmax);
    if (!scn->aircraft || !scn->types || scn->n_types == 0) return fail(ctx, SMC_EINVAL, "aircraft/types missing");
    if (!(scn->dt > 0.0) || !(scn->A_c > 0.0)) return fail(ctx, SMC_EINVAL, "dt and A_c must be positive");
    for (int a = 0; a < 3; ++a)
        if (!(scn->wind_hi[a] > scn->wind_lo[a])) return fail(ctx, SMC_EINVAL, "empty wind box");
    if ((size_t)scn->pop_nx * scn->pop_ny > kPopCap) return fail(ctx, SMC_EINVAL, "population grid too large");
    if (scn->n_centres > kCentreCap) return fail(ctx, SMC_EINVAL, "too many population centres");
    if (scn->pop_nx * scn->pop_ny > 0 && !(scn->pop_dx > 0.0)) return fail(ctx, SMC_EINVAL, "pop_dx must be > 0");
    for (int a = 0; a < 3; ++a)
        if (scn->wind_n[a] == 1 || scn->wind_n[a] > (uint32_t)kMaxWindNodes)
            return fail(ctx, SMC_EINVAL, "wind grid: %u points on axis %d", scn->wind_n[a], a);
    if (wind_axis(scn->wind_n[0]) * wind_axis(scn->wind_n[1]) * wind_axis(scn->wind_n[2]) > kMaxWindNodes)
        return fail(ctx, SMC_EINVAL, "wind grid: more than %d points", kMaxWindNodes);
    for (uint32_t i = 0; i < n; ++i) {
        const smc_aircraft &a = scn->aircraft[i];
        if (a.type >= scn->n_types) return fail(ctx, SMC_EINVAL, "aircraft %u: bad type", i);
        if (a.first_step > H) return fail(ctx, SMC_EINVAL, "aircraft %u: first_step > H", i);
        if (a.kind > 1) return fail(ctx, SMC_EINVAL, "aircraft %u: bad kind", i);
    }
    ctx->ac.assign(scn->aircraft, scn->aircraft + n);
    ctx->cur_ids.resize(n);
    for (uint32_t i = 0; i < n; ++i) ctx->cur_ids[i] = scn->aircraft[i].id;
    ctx->types.assign(scn->types, scn->types + scn->n_types);
    ctx->centres_h.assign(scn->centres, scn->centres + 3 * (size_t)scn->n_centres);
    ctx->scn = *scn;
    ctx->scn.aircraft = ctx->ac.data();
    ctx->scn.types = ctx->types.data();
    ctx->scn.centres = ctx->centres_h.data();
    smc_status s = build_constants(ctx);
    if (s != SMC_OK) return s;
    if (scn->n_centres) {
        CK(h2d(ctx, ctx->centres, scn->centres, sizeof(double) * 3 * scn->n_centres));
    }
    LAUNCH(launch_popgrid(ctx->centres, (int)scn->n_centres, (int)scn->pop_nx, (int)scn->pop_ny, scn->pop_x0,
                          scn->pop_y0, scn->pop_dx, ctx->pop, ctx->popp, ctx->st));
    ctx->drop_graph();            // (the realised plant wind persists across scenarios: mpc loop)
    ctx->have_scn = true;
    return init_population(ctx);
}

// ---------------------------------------------------------------- one SMC round
static smc_status select_best(smc_ctx *ctx);

// Particle count of round k: linear from L to L_final over the K rounds of a solve.
static uint32_t particles_of(const smc_ctx *ctx, uint32_t k) {
    const uint32_t K = ctx->cfg.n_rounds;
    if (!ctx->Lfinal || K < 2) return ctx->Lloc;
    if (k >= K) k = K - 1;
    return ctx->Lloc - (uint32_t)(((uint64_t)(ctx->Lloc - ctx->Lfinal) * k) / (K - 1));
}

static uint32_t samples_of(const smc_ctx *ctx, uint32_t k) {
    if (ctx->cfg.schedule == SMC_SCHED_PAPER) return (uint32_t)std::floor(3.0 + 5.0 * std::exp(0.05 * (double)k));
    return ctx->cfg.n_samples;
}

// Merge-path ancestors (K5) pay once the CDF no longer sits in L2 and a bisection per
// slot turns into DRAM misses; below that the extra launch costs more than it saves.
// Cluster scan (one 8-CTA cluster per column, DSMEM) up to 65 536 particles, else the
// decoupled look-back scan; SMC_SCAN=lookback forces the latter.
static bool use_cluster_scan(const smc_ctx *ctx, uint32_t Lk) {
    return ctx->scan_cluster && cluster_scan_fits(Lk);
}

static bool use_merge_path(const smc_ctx *ctx, uint32_t Lk) {
    if (ctx->anc_mode == 0 || ctx->anc_mode == 1) return ctx->anc_mode == 1;
    if (ctx->anc_mode == 2) return false;
    return Lk >= (1u << 17);
}

static smc_status run_round(smc_ctx *ctx, bool tail, smc_round_stats *stats) {
    NvtxRange nvtx_round("smc_round");
    const uint32_t k = ctx->k;
    const int n = ctx->dsc.n, H = ctx->dsc.H;
    const int P = ctx->cur;
    smc_status s0 = sync_mpc(ctx);
    if (s0 != SMC_OK) return s0;
    const uint32_t S = samples_of(ctx, k);
    if (!ctx->acc_clean) {                 // normally zeroed by the previous round's K6
        CK(cudaMemsetAsync(ctx->colmax, 0, sizeof(uint32_t) * n, ctx->st));
        CK(cudaMemsetAsync(ctx->accept, 0, 8, ctx->st));
        CK(cudaMemsetAsync(ctx->status, 0, 8 * (size_t)scan_tiles(ctx->Lloc) * n, ctx->st));
        CK(cudaMemsetAsync(ctx->tiles, 0, 4 * n, ctx->st));
    }
    ctx->acc_clean = false;
    RolloutArgs ra{};
    int NC;
    if (k == 0) {
        NC = 1; ra.ctrl[0] = ctx->ctrl[P][0]; ra.ctrl[1] = nullptr; ra.surv_single = 0u;
    } else if (ctx->cfg.mh) {
        NC = 2; ra.ctrl[0] = ctx->ctrl[P][0]; ra.ctrl[1] = ctx->ctrl[P][1]; ra.surv_single = 0u;
    } else {
        NC = 1; ra.ctrl[0] = ctx->ctrl[P][1]; ra.ctrl[1] = nullptr; ra.surv_single = 0xFFFFFFFFu;
    }
    ra.mh_mode = ctx->cfg.mh == 2 ? 2 : 1;
    ctx->last_nc = NC;
    const uint32_t Lk = particles_of(ctx, k), Ln = particles_of(ctx, k + 1);
    ra.L = Lk; ra.l0 = ctx->l0; ra.S = S; ra.k = k; ra.mpcp = ctx->mpc_dev;
    ra.ell0 = (float)(-std::log2((double)(ctx->Lfinal ? Lk : ctx->Lg)));
    ra.ell_out = ctx->ell; ra.lam_out = ctx->lam; ra.surv_out = ctx->surv; ra.colmax = ctx->colmax;
    ra.n_accept = ctx->accept; ra.lam_cand = ctx->lam2;
    LAUNCHP(PH_ROLLOUT, launch_rollout(ctx->dsc, ra, NC, false, ctx->st));
    ctx->last_eval = P;
    ctx->Leval = Lk;
    if (ctx->world > 1 && ctx->p2p && tail)
        // publish this round's survivor masks for the peers' gathers (by round parity: a peer
        // may still read the previous round's copy; the one before is fenced by this round's
        // all-reduce, which no peer passes before finishing its previous gather)
        CK(cudaMemcpyAsync(ctx->survp + (size_t)(k & 1) * ctx->Lmax, ctx->surv, 4 * (size_t)ctx->Lloc,
                           cudaMemcpyDeviceToDevice, ctx->st));
    if (ctx->world > 1)                    // global column maxima (reduce step 1)
        COLL(coll_allreduce_max_u32(ctx, ctx->colmax, (size_t)n));
    ResampleArgs rs{};
    rs.n = n; rs.L = Lk; rs.k = k; rs.key0 = ctx->dsc.key0; rs.key1 = ctx->dsc.key1; rs.mpcp = ctx->mpc_dev;
    rs.ell = ctx->ell; rs.colmax = ctx->colmax; rs.Q = ctx->Q; rs.ess = ctx->ess; rs.status = ctx->status;
    rs.tile_ctr = ctx->tiles; rs.C = ctx->C; rs.QR = ctx->QR; rs.Cstride = ctx->world > 1 ? ctx->Lmax : 0;
    rs.inf_round = ctx->inf_round;
    uint32_t cm[32];
    double ess[64];
    unsigned long long acc = 0;
    if (stats) {
        CK(cudaMemsetAsync(ctx->ess, 0, 16 * n, ctx->st));
        CK(cudaMemsetAsync(ctx->Q, 0, 8 * n, ctx->st));
        rs.Q = ctx->Q;
        LAUNCHP(PH_RESAMPLE, launch_qsum(rs, ctx->st));
        // read the round's accumulators before K6 zeroes them for the next round
        CK(d2h(ctx, cm, ctx->colmax, 4 * n));
        CK(d2h(ctx, ess, ctx->ess, 16 * n));
        CK(d2h(ctx, &acc, ctx->accept, 8));
        CK(cudaStreamSynchronize(ctx->st));
    }
    if (tail) {
        // look-back status words the next round's scan (over Ln particles) will read
        const size_t nt = (size_t)std::max(scan_tiles(Lk), scan_tiles(Ln));
        rs.Q = nullptr;
        const bool single = ctx->world == 1 && ctx->vworld == 1, mp = single && use_merge_path(ctx, Lk);
        // bisection in K6 / the multi-rank gather: K4 also writes every 16th prefix (two-level search)
        const bool two_level = !mp && ctx->cdf_sample;
        if (two_level) { rs.Cs = ctx->Cs; rs.Cs_stride = cdf_samples(single ? Lk : ctx->Lmax); }
        if (ctx->world > 1) rs.Q = ctx->Q;     // this rank's column totals, all-gathered below
        if (ctx->vworld == 1)
            LAUNCHP(PH_RESAMPLE, use_cluster_scan(ctx, Lk) ? launch_scan_cluster(rs, ctx->st) : launch_scan(rs, ctx->st));
        ProposeArgs pa{};
        pa.n = n; pa.H = H; pa.L = Ln; pa.Lsrc = Lk; pa.l0 = ctx->l0; pa.k = k; pa.mpcp = ctx->mpc_dev;
        pa.key0 = ctx->dsc.key0; pa.key1 = ctx->dsc.key1;
        pa.src[0] = ctx->ctrl[P][0]; pa.src[1] = ctx->ctrl[P][1];
        pa.surv = ctx->surv; pa.anc = nullptr; pa.C = ctx->C; pa.QR = ctx->QR;
        if (two_level && single) { pa.Cs = ctx->Cs; pa.Cs_stride = cdf_samples(Lk); }
        if (mp) {
            rs.anc = ctx->anc; rs.M = Ln; rs.splits = ctx->splits;
            LAUNCHP(PH_RESAMPLE, launch_ancestors(rs, ctx->st));
            pa.anc = ctx->anc;
        }
        pa.xp = ctx->ctrl[P ^ 1][0]; pa.xs = ctx->ctrl[P ^ 1][1];
        const double f = std::pow(ctx->cfg.anneal, (double)k);
        for (int c = 0; c < 3; ++c) pa.sig[c] = (float)(ctx->cfg.sigma[c] * f);
        pa.clamp = (int)ctx->cfg.clamp_proposals;
        pa.lo3 = ctx->lohi; pa.hi3 = ctx->lohi + 3 * ctx->nmax;
        pa.reset_n = n; pa.reset_colmax = ctx->colmax; pa.reset_tiles = ctx->tiles; pa.reset_accept = ctx->accept;
        pa.reset_status = ctx->status; pa.reset_status_n = nt * n;
        const int rowlen = n * H * 3;
        if (ctx->vworld > 1) {
            // virtual ranks (test mode): the multi-GPU path with the exchange done in place -- rank r's
            // CDF, CDF samples and column totals in its slices of Call / Csall / Qall, its rows a row
            // slice of this context's buffers (peer mode) or compacted into Sall (all-gather mode)
            const int G = ctx->vworld;
            const uint32_t css = cdf_samples(ctx->Lmax);
            const size_t ntv = (size_t)scan_tiles(ctx->Lmax);
            MultiArgs ma{};
            ma.Lg = ctx->Lg; ma.G = G; ma.Qall = ctx->Qall; ma.Qstride = (uint32_t)ctx->nmax;
            ma.Cstride = ctx->Lmax; ma.Cs_stride = css; ma.Lmax = ctx->Lmax;
            ma.prow = (size_t)(ctx->ctrl[P][1] - ctx->ctrl[P][0]);
            ma.Sall = ctx->p2p ? nullptr : ctx->Sall;
            for (int r = 0; r < G; ++r) {
                uint32_t b, e;
                smc_shard_range(ctx->Lg, G, r, &b, &e);
                ResampleArgs rr = rs;
                rr.L = e - b; rr.ell = ctx->ell + b; rr.ell_stride = ctx->Lloc;
                rr.C = ctx->Call + (size_t)r * n * ctx->Lmax; rr.Cstride = ctx->Lmax;
                rr.Q = ctx->Qall + (size_t)r * ctx->nmax;
                rr.Cs = two_level ? ctx->Csall + (size_t)r * n * css : nullptr; rr.Cs_stride = css;
                CK(cudaMemsetAsync(ctx->status, 0, 8 * ntv * n, ctx->st));
                CK(cudaMemsetAsync(ctx->tiles, 0, 4 * n, ctx->st));
                LAUNCHP(PH_RESAMPLE, launch_scan(rr, ctx->st));
                if (!ctx->p2p)
                    LAUNCHP(PH_PROPOSE, launch_compact_survivors(ctx->ctrl[P][0] + (size_t)b * rowlen,
                                                                 ctx->ctrl[P][1] + (size_t)b * rowlen, ctx->surv + b, e - b,
                                                                 n, rowlen, ctx->Sall + (size_t)r * ctx->Lmax * rowlen,
                                                                 ctx->st));
                ma.peer_C[r] = rr.C;
                ma.peer_Cs[r] = rr.Cs;
                ma.len[r] = e - b;
                ma.peer_ctrl[r] = ctx->ctrl[P][0] + (size_t)b * rowlen;
                ma.peer_surv[r] = ctx->surv + b;
            }
            for (int r = 0; r < G; ++r) {
                uint32_t b, e;
                smc_shard_range(ctx->Lg, G, r, &b, &e);
                MultiArgs mr = ma;
                mr.p = pa;
                mr.p.L = e - b; mr.p.l0 = b;
                mr.p.xp = ctx->ctrl[P ^ 1][0] + (size_t)b * rowlen; mr.p.xs = ctx->ctrl[P ^ 1][1] + (size_t)b * rowlen;
                mr.p.reset_status_n = 0;
                LAUNCHP(PH_PROPOSE, launch_gather_propose_multi(mr, ctx->st));
            }
            CK(cudaMemsetAsync(ctx->status, 0, 8 * nt * n, ctx->st));
            CK(cudaMemsetAsync(ctx->tiles, 0, 4 * n, ctx->st));
        } else if (ctx->world > 1) {
            // exchange: all-gather of the per-rank column totals (N uint64 per
            // rank); the owner's CDF is searched in place through the IPC mappings (peer mode), or the
            // per-rank CDFs and compacted survivor rows are all-gathered (all-gather mode)
            COLL(coll_allgather(ctx, ctx->Q, ctx->Qall, sizeof(unsigned long long) * ctx->nmax));
            MultiArgs ma{};
            ma.p = pa;
            ma.Lg = ctx->Lg; ma.G = ctx->world; ma.Qall = ctx->Qall; ma.Qstride = (uint32_t)ctx->nmax;
            ma.Cstride = ctx->Lmax; ma.Cs_stride = cdf_samples(ctx->Lmax); ma.Lmax = ctx->Lmax;
            for (int r = 0; r < ctx->world; ++r) ma.len[r] = local_count(ctx->Lg, ctx->world, r);
            if (ctx->p2p) {
                // parents read in place over NVLink: rank r's current pair, published masks and CDF
                const size_t prow = (size_t)(ctx->ctrl[0][1] - ctx->ctrl[0][0]);
                ma.prow = prow;
                for (int r = 0; r < ctx->world; ++r) {
                    ma.peer_ctrl[r] = ctx->peer_ctrl[r] + (size_t)(2 * P) * prow;
                    ma.peer_surv[r] = ctx->peer_survp[r] + (size_t)(k & 1) * ctx->Lmax;
                    ma.peer_C[r] = ctx->peer_C[r];
                    ma.peer_Cs[r] = two_level ? ctx->peer_Cs[r] : nullptr;
                }
            } else {
                COLL(coll_allgather(ctx, ctx->C, ctx->Call, sizeof(unsigned long long) * n * ctx->Lmax));
                LAUNCHP(PH_PROPOSE, launch_compact_survivors(ctx->ctrl[P][0], ctx->ctrl[P][1], ctx->surv, ctx->Lloc, n,
                                                             rowlen, ctx->Sc, ctx->st));
                COLL(coll_allgather(ctx, ctx->Sc, ctx->Sall, sizeof(float) * ctx->Lmax * rowlen));
                ma.Sall = ctx->Sall;
                ma.Cstride = ctx->Lmax;
                for (int r = 0; r < ctx->world; ++r) {
                    ma.peer_C[r] = ctx->Call + (size_t)r * n * ctx->Lmax;
                    ma.peer_Cs[r] = nullptr;
                }
            }
            LAUNCHP(PH_PROPOSE, launch_gather_propose_multi(ma, ctx->st));
        } else {
            LAUNCHP(PH_PROPOSE, launch_gather_propose(pa, ctx->st));
        }
        ctx->cur = P ^ 1;
        ctx->acc_clean = true;
    }
    if (stats) {
        smc_status s2 = select_best(ctx);
        if (s2 != SMC_OK) return s2;
        double bl;
        CK(d2h(ctx, &bl, ctx->best_lam, 8));
        CK(cudaStreamSynchronize(ctx->st));
        stats->best_lambda = bl;
        stats->accept_rate = (k == 0) ? 1.0 : (ctx->cfg.mh ? (double)acc / ((double)Lk * (ctx->cfg.mh == 2 ? n : 1)) : 1.0);
        double em = INFINITY;
        uint32_t lo = 0, hi = 0;
        for (int i = 0; i < n; ++i) {
            const bool inf = cm[i] == 0u || cm[i] == 0x007FFFFFu;
            if (inf) { if (i < 32) lo |= 1u << i; em = 0.0; continue; }
            const double e = ess[2 * i] * ess[2 * i] / ess[2 * i + 1];
            em = std::min(em, e);
        }
        stats->ess_min = em;
        stats->infeasible_lo = lo;
        stats->infeasible_hi = hi;
        stats->n_samples = S;
        stats->round = k;
    }
    ctx->k = k + 1;
    return SMC_OK;
}

extern "C" smc_status smc_iterate(smc_ctx *ctx, uint32_t n_rounds, smc_round_stats *stats) {
    if (!ctx) return SMC_EINVAL;
    if (!ctx->have_scn) return fail(ctx, SMC_ESTATE, "smc_iterate before smc_set_scenario");
    for (uint32_t r = 0; r < n_rounds; ++r) {
        if (ctx->k >= 65535) return fail(ctx, SMC_EINVAL, "round index exceeds 2^16");
        smc_status s = run_round(ctx, true, stats ? &stats[r] : nullptr);
        if (s != SMC_OK) return s;
    }
    return SMC_OK;
}

static smc_status select_best(smc_ctx *ctx) {
    if (ctx->last_eval < 0) return fail(ctx, SMC_ESTATE, "no evaluated population");
    const int P = ctx->last_eval;
    // per-aircraft MH (R46): survivors mix two joint evaluations -> pick among the candidates
    const bool cand = ctx->cfg.mh == 2 && ctx->last_nc == 2;
    if (ctx->vworld > 1) {                // virtual ranks: per-shard records, then the multi-GPU merge
        const int rowlen = ctx->dsc.n * ctx->dsc.H * 3;
        for (int r = 0; r < ctx->vworld; ++r) {
            uint32_t b, e;
            smc_shard_range(ctx->Lg, ctx->vworld, r, &b, &e);
            unsigned char *rec = ctx->rec_all + (size_t)r * ctx->rec_bytes;
            SelectArgs sr{e - b, b, ctx->dsc.n, ctx->dsc.H, ctx->lam + b, ctx->surv + b,
                          {ctx->ctrl[P][0] + (size_t)b * rowlen, ctx->ctrl[P][1] + (size_t)b * rowlen},
                          ctx->part_lam, ctx->part_idx, ctx->done, (double *)rec, (long long *)(rec + 8),
                          (float *)(rec + 16), cand ? ctx->lam2 + b : nullptr, ctx->Lloc};
            LAUNCH(launch_select(sr, ctx->st));
        }
        LAUNCH(launch_select_merge(ctx->rec_all, ctx->vworld, ctx->rec_bytes, rowlen, ctx->rec_final, ctx->st));
        return SMC_OK;
    }
    SelectArgs sa{ctx->Leval ? ctx->Leval : ctx->Lloc, ctx->l0, ctx->dsc.n, ctx->dsc.H, ctx->lam, ctx->surv,
                  {ctx->ctrl[P][0], ctx->ctrl[P][1]},
                  ctx->part_lam, ctx->part_idx, ctx->done, ctx->sel_lam, ctx->sel_idx, ctx->sel_row,
                  cand ? ctx->lam2 : nullptr, ctx->Leval ? ctx->Leval : ctx->Lloc};
    LAUNCH(launch_select(sa, ctx->st));
    if (ctx->world > 1) {                 // all-gather the per-rank records, merge on every rank
        COLL(coll_allgather(ctx, ctx->rec_local, ctx->rec_all, ctx->rec_bytes));
        LAUNCH(launch_select_merge(ctx->rec_all, ctx->world, ctx->rec_bytes, ctx->dsc.n * ctx->dsc.H * 3,
                                   ctx->rec_final, ctx->st));
    }
    return SMC_OK;
}

// SMC_EINFEASIBLE report: which aircraft has no nonzero weight in any particle
// of the last evaluated round (column maxima of the survivor weights), and the first round in
// which each such column was all zero (recorded by K4).  Synchronises; failure path only.
static smc_status infeasible(smc_ctx *ctx, const char *what) {
    const int n = ctx->dsc.n;
    const uint32_t Lk = ctx->Leval ? ctx->Leval : ctx->Lloc;
    uint32_t cm[32];
    int32_t fr[32];
    if (cudaMemsetAsync(ctx->infcol, 0, 4 * n, ctx->st) == cudaSuccess &&
        launch_colmax(ctx->ell, n, Lk, ctx->infcol, ctx->st) == cudaSuccess &&
        cudaMemcpyAsync(cm, ctx->infcol, 4 * n, cudaMemcpyDeviceToHost, ctx->st) == cudaSuccess &&
        cudaMemcpyAsync(fr, ctx->inf_round, 4 * n, cudaMemcpyDeviceToHost, ctx->st) == cudaSuccess &&
        cudaStreamSynchronize(ctx->st) == cudaSuccess) {
        std::string msg;
        char buf[96];
        for (int i = 0; i < n; ++i)
            if (cm[i] == 0u || cm[i] == 0x007FFFFFu) {      // ordered -inf (or nothing written)
                snprintf(buf, sizeof buf, "%saircraft %d (index in the scenario) zero in every particle", msg.empty() ? "" : "; ", i);
                msg += buf;
                if (fr[i] >= 0) { snprintf(buf, sizeof buf, " since round %d", fr[i]); msg += buf; }
                else { snprintf(buf, sizeof buf, " in the last round %u", ctx->k ? ctx->k - 1 : 0); msg += buf; }
            }
        if (msg.empty()) msg = "no single aircraft is zero everywhere, but every particle has a zero-weight aircraft";
        return fail(ctx, SMC_EINFEASIBLE, "%s: every particle has a zero weight (P:423): %s", what, msg.c_str());
    }
    cudaGetLastError();
    return fail(ctx, SMC_EINFEASIBLE, "%s: every particle has a zero weight (P:423)", what);
}

extern "C" smc_status smc_best_controls(smc_ctx *ctx, smc_control *out, double *lambda, int64_t *particle) {
    if (!ctx) return SMC_EINVAL;
    NvtxRange nvtx_sel("smc_best_controls");
    if (!ctx->have_scn) return fail(ctx, SMC_ESTATE, "no scenario");
    smc_status s = select_best(ctx);
    if (s != SMC_OK) return s;
    double bl;
    long long bi;
    const int n = ctx->dsc.n, H = ctx->dsc.H;
    CK(d2h(ctx, &bl, ctx->best_lam, 8));
    CK(d2h(ctx, &bi, ctx->best_idx, 8));
    if (out) CK(d2h(ctx, out, ctx->best_row, sizeof(float) * 3 * n * H));
    CK(cudaStreamSynchronize(ctx->st));
    if (lambda) *lambda = bl;
    if (particle) *particle = bi;
    if (bi < 0) return infeasible(ctx, "selection");
    return SMC_OK;
}

static smc_status solve_body(smc_ctx *ctx, uint32_t advance_plant) {
    smc_status s = init_population(ctx);                       // fresh population (R31)
    if (s != SMC_OK) return s;
    const uint32_t K = ctx->cfg.n_rounds ? ctx->cfg.n_rounds : 1;
    for (uint32_t r = 0; r < K; ++r) {
        s = run_round(ctx, r + 1 < K, nullptr);                // last round: no resample/propose
        if (s != SMC_OK) return s;
    }
    s = select_best(ctx);
    if (s != SMC_OK) return s;
    if (advance_plant) {
        PlantArgs pa{ctx->dsc.n, ctx->dsc.key0, ctx->dsc.key1, ctx->mpc_dev, ctx->pstates, ctx->best_row, ctx->dsc.H,
                     ctx->pZ, ctx->pzi, ctx->pnext, ctx->pflags, ctx->papplied, ctx->best_idx};
        LAUNCH(launch_plant(ctx->psc, pa, ctx->st));
    }
    return SMC_OK;
}

extern "C" smc_status smc_solve(smc_ctx *ctx, uint32_t advance_plant) {
    if (!ctx) return SMC_EINVAL;
    NvtxRange nvtx_solve("smc_solve");
    if (!ctx->have_scn) return fail(ctx, SMC_ESTATE, "smc_solve before smc_set_scenario");
    if (!ctx->cfg.use_graph || ctx->st == nullptr) {
        smc_status s = solve_body(ctx, advance_plant);
        if (s == SMC_OK) warm_solved(ctx);
        return s;
    }
    smc_status s = sync_mpc(ctx);                              // outside the graph: mpc is read from device memory
    if (s != SMC_OK) return s;
    s = warm_prepare(ctx);
    if (s != SMC_OK) return s;
    const uint32_t K = ctx->cfg.n_rounds ? ctx->cfg.n_rounds : 1;
    if (!ctx->graph_ok || ctx->graph_adv != (int)advance_plant || ctx->graph_K != K) {
        ctx->drop_graph();
        const uint64_t l0 = ctx->launches;
        uint64_t p0[4];
        for (int q = 0; q < 4; ++q) p0[q] = ctx->phase_launches[q];
        CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
        ctx->capturing = true;
        s = solve_body(ctx, advance_plant);
        ctx->capturing = false;
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->st, &g);
        if (s != SMC_OK) { if (g) cudaGraphDestroy(g); return s; }
        if (e != cudaSuccess) return fail(ctx, SMC_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        ctx->graph = g;
        CK(cudaGraphInstantiate(&ctx->gexec, g, 0));
        ctx->g_k = ctx->k; ctx->g_cur = ctx->cur; ctx->g_last = ctx->last_eval;
        ctx->g_launches = ctx->launches - l0;
        ctx->launches = l0;
        for (int q = 0; q < 4; ++q) { ctx->g_phase_launches[q] = ctx->phase_launches[q] - p0[q]; ctx->phase_launches[q] = p0[q]; }
        ctx->graph_ok = true; ctx->graph_adv = (int)advance_plant; ctx->graph_K = K;
    }
    CK(cudaGraphLaunch(ctx->gexec, ctx->st));
    warm_solved(ctx);
    ctx->k = ctx->g_k; ctx->cur = ctx->g_cur; ctx->last_eval = ctx->g_last;
    ctx->launches += ctx->g_launches;
    for (int q = 0; q < 4; ++q) ctx->phase_launches[q] += ctx->g_phase_launches[q];
    if (ctx->cfg.profile) {                                    // read the graph's timing nodes now (they are reused)
        CK(cudaStreamSynchronize(ctx->st));
        for (int q = 0; q < 4; ++q)
            for (auto &pr : ctx->ev_graph[q]) {
                float t = 0.f;
                CK(cudaEventElapsedTime(&t, pr.first, pr.second));
                ctx->phase_ms_acc[q] += t;
            }
    }
    return SMC_OK;
}

extern "C" smc_status mpc_step(smc_ctx *ctx, const smc_state *measured, smc_control *applied, smc_state *next,
                               uint32_t *flags) {
    if (!ctx || !measured) return SMC_EINVAL;
    NvtxRange nvtx_step("mpc_step");
    if (!ctx->have_scn) return fail(ctx, SMC_ESTATE, "mpc_step before smc_set_scenario");
    const int n = ctx->dsc.n;
    for (int i = 0; i < n; ++i) ctx->ac[i].x0 = measured[i];
    smc_status s = build_constants(ctx);
    if (s != SMC_OK) return s;
    CK(h2d(ctx, ctx->pstates, measured, sizeof(double) * 6 * n));
    s = smc_solve(ctx, 1);
    if (s != SMC_OK) return s;
    long long bi;
    int fl[32];
    CK(d2h(ctx, &bi, ctx->best_idx, 8));
    if (next) CK(d2h(ctx, next, ctx->pnext, sizeof(double) * 6 * n));
    if (applied) CK(d2h(ctx, applied, ctx->papplied, sizeof(float) * 3 * n));
    CK(d2h(ctx, fl, ctx->pflags, sizeof(int) * n));
    CK(cudaStreamSynchronize(ctx->st));
    if (flags)
        for (int i = 0; i < n; ++i) flags[i] = (uint32_t)fl[i];
    const uint32_t m = ctx->mpc;
    ctx->mpc += 1;
    ctx->mpc_dirty = true;
    if (bi < 0) {
        char what[48];
        snprintf(what, sizeof what, "MPC step %u", m);
        return infeasible(ctx, what);
    }
    return SMC_OK;
}

extern "C" smc_status smc_phase_times(smc_ctx *ctx, double ms[4], uint64_t launches[4]) {
    if (!ctx) return SMC_EINVAL;
    CK(cudaStreamSynchronize(ctx->st));
    for (int p = 0; p < 4; ++p) {
        double tot = 0.0;
        for (auto &pr : ctx->ev_used[p]) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, pr.first, pr.second));
            tot += t;
            ctx->ev_free.push_back(pr.first);
            ctx->ev_free.push_back(pr.second);
        }
        ctx->ev_used[p].clear();
        tot += ctx->phase_ms_acc[p];
        ctx->phase_ms_acc[p] = 0.0;
        if (ms) ms[p] = tot;
        if (launches) launches[p] = ctx->phase_launches[p];
        ctx->phase_launches[p] = 0;
    }
    return SMC_OK;
}

// ---------------------------------------------------------------- debug hooks
namespace {
struct DevTmp {
    std::vector<void *> ptrs;
    ~DevTmp() { for (void *p : ptrs) cudaFree(p); }
    template <class T>
    T *alloc(size_t count) {
        void *p = nullptr;
        if (cudaMalloc(&p, count * sizeof(T) + 16) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return (T *)p;
    }
};
}  // namespace

static smc_status debug_rollout_impl(smc_ctx *ctx, const float *controls, uint32_t L, uint32_t l0, uint32_t S,
                                     uint32_t k, bool debug, float *J, uint8_t *viol, float *comp, float *fuel,
                                     int32_t *landed, float *traj, float *ell, int nc = 1) {
    if (!ctx || !controls || L == 0 || S == 0) return SMC_EINVAL;
    if (!ctx->have_scn) return fail(ctx, SMC_ESTATE, "no scenario");
    const int n = ctx->dsc.n, H = ctx->dsc.H;
    DevTmp tmp;
    const size_t nrow = (size_t)L * n * H * 3;
    float *dctrl = tmp.alloc<float>(nrow);
    float *dell = tmp.alloc<float>((size_t)n * L);
    double *dlam = tmp.alloc<double>(L);
    uint32_t *dsurv = tmp.alloc<uint32_t>(L);
    uint32_t *dcm = tmp.alloc<uint32_t>(n);
    unsigned long long *dacc = tmp.alloc<unsigned long long>(1);
    const size_t nu = (size_t)L * S * n;
    float *dJ = debug ? tmp.alloc<float>(nu) : nullptr, *dcomp = debug ? tmp.alloc<float>(4 * nu) : nullptr;
    float *dfuel = debug ? tmp.alloc<float>(nu) : nullptr;
    uint8_t *dviol = debug ? tmp.alloc<uint8_t>(nu) : nullptr;
    int32_t *dland = debug ? tmp.alloc<int32_t>(nu) : nullptr;
    float *dtraj = (debug && traj) ? tmp.alloc<float>(nu * (H + 1) * 6) : nullptr;
    if (!dctrl || !dell || !dlam || !dsurv || !dcm || !dacc) return fail(ctx, SMC_ECUDA, "debug allocation failed");
    CK(cudaMemcpyAsync(dctrl, controls, sizeof(float) * nrow, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemsetAsync(dcm, 0, 4 * n, ctx->st));
    if (dland) CK(cudaMemsetAsync(dland, 0xFF, sizeof(int32_t) * nu, ctx->st));
    RolloutArgs ra{};
    smc_status s0 = sync_mpc(ctx);
    if (s0 != SMC_OK) return s0;
    ra.ctrl[0] = dctrl; ra.L = L; ra.l0 = l0; ra.S = S; ra.k = k; ra.mpcp = ctx->mpc_dev;
    ra.ell0 = (float)(-std::log2((double)L));
    ra.ell_out = dell; ra.lam_out = dlam; ra.surv_out = dsurv; ra.colmax = dcm; ra.n_accept = dacc;
    ra.dbg_J = dJ; ra.dbg_comp = dcomp; ra.dbg_fuel = dfuel; ra.dbg_traj = dtraj; ra.dbg_viol = dviol;
    ra.dbg_landed = dland;
    if (nc == 2) ra.ctrl[1] = dctrl;          // both candidates alike: the survivor's weights are theirs
    LAUNCH(launch_rollout(ctx->dsc, ra, nc, debug, ctx->st));
    if (debug) {
        if (J) CK(cudaMemcpyAsync(J, dJ, sizeof(float) * nu, cudaMemcpyDeviceToHost, ctx->st));
        if (viol) CK(cudaMemcpyAsync(viol, dviol, nu, cudaMemcpyDeviceToHost, ctx->st));
        if (comp) CK(cudaMemcpyAsync(comp, dcomp, sizeof(float) * 4 * nu, cudaMemcpyDeviceToHost, ctx->st));
        if (fuel) CK(cudaMemcpyAsync(fuel, dfuel, sizeof(float) * nu, cudaMemcpyDeviceToHost, ctx->st));
        if (landed) CK(cudaMemcpyAsync(landed, dland, sizeof(int32_t) * nu, cudaMemcpyDeviceToHost, ctx->st));
        if (traj) CK(cudaMemcpyAsync(traj, dtraj, sizeof(float) * nu * (H + 1) * 6, cudaMemcpyDeviceToHost, ctx->st));
    }
    if (ell) {
        // device layout [n][L] -> host [L][n]
        std::vector<float> tmpe((size_t)n * L);
        CK(cudaMemcpyAsync(tmpe.data(), dell, sizeof(float) * n * L, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        for (uint32_t l = 0; l < L; ++l)
            for (int i = 0; i < n; ++i) ell[(size_t)l * n + i] = tmpe[(size_t)i * L + l];
    }
    CK(cudaStreamSynchronize(ctx->st));
    return SMC_OK;
}

extern "C" smc_status smc_debug_rollout(smc_ctx *ctx, const float *controls, uint32_t L, uint32_t l0, uint32_t S,
                                        uint32_t k, float *J, uint8_t *viol, float *comp, float *fuel, int32_t *landed,
                                        float *traj) {
    return debug_rollout_impl(ctx, controls, L, l0, S, k, true, J, viol, comp, fuel, landed, traj, nullptr);
}

extern "C" smc_status smc_debug_evaluate(smc_ctx *ctx, const float *controls, uint32_t L, uint32_t S, uint32_t k,
                                         float *ell) {
    return debug_rollout_impl(ctx, controls, L, 0, S, k, false, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                              ell);
}

extern "C" smc_status smc_debug_evaluate2(smc_ctx *ctx, const float *controls, uint32_t L, uint32_t S, uint32_t k,
                                          float *ell) {
    return debug_rollout_impl(ctx, controls, L, 0, S, k, false, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                              ell, 2);
}

extern "C" smc_status smc_debug_mh(smc_ctx *ctx, const double *lam_cur, const double *lam_prop, uint32_t L, uint32_t k,
                                   uint8_t *acc) {
    if (!ctx || !lam_cur || !lam_prop || !acc) return SMC_EINVAL;
    DevTmp tmp;
    double *a = tmp.alloc<double>(L), *b = tmp.alloc<double>(L);
    uint8_t *o = tmp.alloc<uint8_t>(L);
    if (!a || !b || !o) return fail(ctx, SMC_ECUDA, "debug allocation failed");
    CK(cudaMemcpyAsync(a, lam_cur, 8 * (size_t)L, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(b, lam_prop, 8 * (size_t)L, cudaMemcpyHostToDevice, ctx->st));
    const uint32_t key0 = (uint32_t)ctx->cfg.seed, key1 = (uint32_t)(ctx->cfg.seed >> 32);
    smc_status s0 = sync_mpc(ctx);
    if (s0 != SMC_OK) return s0;
    LAUNCH(launch_mh_debug(a, b, L, k, ctx->mpc_dev, key0, key1, o, ctx->st));
    CK(cudaMemcpyAsync(acc, o, L, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SMC_OK;
}

extern "C" smc_status smc_debug_mh_aircraft(smc_ctx *ctx, const float *ell_cur, const float *ell_prop, uint32_t L,
                                            uint32_t N, uint32_t k, uint32_t *mask) {
    if (!ctx || !ell_cur || !ell_prop || !mask || N == 0 || N > 32) return SMC_EINVAL;
    DevTmp tmp;
    float *a = tmp.alloc<float>((size_t)L * N), *b = tmp.alloc<float>((size_t)L * N);
    uint32_t *o = tmp.alloc<uint32_t>(L);
    if (!a || !b || !o) return fail(ctx, SMC_ECUDA, "debug allocation failed");
    CK(cudaMemcpyAsync(a, ell_cur, sizeof(float) * L * N, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(b, ell_prop, sizeof(float) * L * N, cudaMemcpyHostToDevice, ctx->st));
    const uint32_t key0 = (uint32_t)ctx->cfg.seed, key1 = (uint32_t)(ctx->cfg.seed >> 32);
    smc_status s0 = sync_mpc(ctx);
    if (s0 != SMC_OK) return s0;
    LAUNCH(launch_mh_aircraft_debug(a, b, L, (int)N, k, ctx->mpc_dev, key0, key1, o, ctx->st));
    CK(cudaMemcpyAsync(mask, o, sizeof(uint32_t) * L, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SMC_OK;
}

extern "C" smc_status smc_debug_resample(smc_ctx *ctx, const float *ell, uint32_t N, uint32_t L, uint32_t M,
                                         uint32_t k, int32_t *anc, uint64_t *Q) {
    if (!ctx || !ell || !anc || N == 0 || N > 32 || L == 0 || L >= (1u << 30)) return SMC_EINVAL;
    if (M == 0) M = L;
    smc_status s0 = sync_mpc(ctx);
    if (s0 != SMC_OK) return s0;
    DevTmp tmp;
    const int nt = scan_tiles(L);
    float *dell = tmp.alloc<float>((size_t)N * L);
    uint32_t *dcm = tmp.alloc<uint32_t>(N);
    unsigned long long *dQ = tmp.alloc<unsigned long long>(N);
    unsigned long long *dQR = tmp.alloc<unsigned long long>(2 * N);
    unsigned long long *dC = tmp.alloc<unsigned long long>((size_t)N * L);
    double *dess = tmp.alloc<double>(2 * N);
    unsigned long long *st1 = tmp.alloc<unsigned long long>((size_t)N * nt);
    unsigned long long *dCs = tmp.alloc<unsigned long long>((size_t)N * cdf_samples(L));
    uint32_t *tiles = tmp.alloc<uint32_t>(2 * N);
    int32_t *danc = tmp.alloc<int32_t>((size_t)N * M);
    uint32_t *dspl = tmp.alloc<uint32_t>((size_t)N * mp_split_words(L, M));
    if (!dell || !dcm || !dQ || !dQR || !dC || !dess || !st1 || !tiles || !danc || !dspl)
        return fail(ctx, SMC_ECUDA, "debug allocation failed");
    CK(cudaMemcpyAsync(dell, ell, sizeof(float) * N * (size_t)L, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemsetAsync(dcm, 0, 4 * N, ctx->st));
    CK(cudaMemsetAsync(dQ, 0, 8 * N, ctx->st));
    CK(cudaMemsetAsync(st1, 0, 8 * (size_t)N * nt, ctx->st));
    CK(cudaMemsetAsync(tiles, 0, 8 * N, ctx->st));
    LAUNCH(launch_colmax(dell, (int)N, L, dcm, ctx->st));
    ResampleArgs rs{};
    rs.n = (int)N; rs.L = L; rs.k = k; rs.mpcp = ctx->mpc_dev;
    rs.key0 = (uint32_t)ctx->cfg.seed; rs.key1 = (uint32_t)(ctx->cfg.seed >> 32);
    rs.ell = dell; rs.colmax = dcm; rs.Q = dQ; rs.ess = dess; rs.status = st1;
    rs.tile_ctr = tiles; rs.C = dC; rs.QR = dQR; rs.anc = danc; rs.M = M; rs.splits = dspl;
    if (ctx->anc_mode == 2) { rs.Cs = dCs; rs.Cs_stride = cdf_samples(L); }
    LAUNCH(use_cluster_scan(ctx, L) ? launch_scan_cluster(rs, ctx->st) : launch_scan(rs, ctx->st));
    LAUNCH(ctx->anc_mode == 0 ? launch_ancestors_bisect(rs, ctx->st)
                              : (ctx->anc_mode == 2 ? launch_ancestors_two_level(rs, ctx->st) : launch_ancestors(rs, ctx->st)));
    CK(cudaMemcpyAsync(anc, danc, 4 * (size_t)N * M, cudaMemcpyDeviceToHost, ctx->st));
    if (Q) CK(cudaMemcpyAsync(Q, dQ, 8 * N, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SMC_OK;
}

extern "C" smc_status smc_debug_propose(smc_ctx *ctx, const float *surv_ctrl, const int32_t *anc, uint32_t L,
                                        uint32_t k, float *xp, float *xs) {
    if (!ctx || !surv_ctrl || !anc || !xp || !xs) return SMC_EINVAL;
    if (!ctx->have_scn) return fail(ctx, SMC_ESTATE, "no scenario");
    const int n = ctx->dsc.n, H = ctx->dsc.H;
    const size_t nrow = (size_t)L * n * H * 3;
    DevTmp tmp;
    float *src = tmp.alloc<float>(nrow), *dxp = tmp.alloc<float>(nrow), *dxs = tmp.alloc<float>(nrow);
    int32_t *danc = tmp.alloc<int32_t>((size_t)n * L);
    uint32_t *dsurv = tmp.alloc<uint32_t>(L);
    if (!src || !dxp || !dxs || !danc || !dsurv) return fail(ctx, SMC_ECUDA, "debug allocation failed");
    CK(cudaMemcpyAsync(src, surv_ctrl, sizeof(float) * nrow, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemcpyAsync(danc, anc, sizeof(int32_t) * n * (size_t)L, cudaMemcpyHostToDevice, ctx->st));
    CK(cudaMemsetAsync(dsurv, 0, sizeof(uint32_t) * L, ctx->st));
    ProposeArgs pa{};
    smc_status s0 = sync_mpc(ctx);
    if (s0 != SMC_OK) return s0;
    pa.n = n; pa.H = H; pa.L = L; pa.Lsrc = L; pa.l0 = 0; pa.k = k; pa.mpcp = ctx->mpc_dev;
    pa.key0 = ctx->dsc.key0; pa.key1 = ctx->dsc.key1;
    pa.src[0] = src; pa.src[1] = src; pa.surv = dsurv; pa.anc = danc; pa.xp = dxp; pa.xs = dxs;
    const double f = std::pow(ctx->cfg.anneal, (double)k);
    for (int c = 0; c < 3; ++c) pa.sig[c] = (float)(ctx->cfg.sigma[c] * f);
    pa.clamp = (int)ctx->cfg.clamp_proposals;
    pa.lo3 = ctx->lohi; pa.hi3 = ctx->lohi + 3 * ctx->nmax;
    LAUNCH(launch_gather_propose(pa, ctx->st));
    CK(cudaMemcpyAsync(xp, dxp, sizeof(float) * nrow, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaMemcpyAsync(xs, dxs, sizeof(float) * nrow, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SMC_OK;
}

extern "C" smc_status smc_debug_population(smc_ctx *ctx, float *ctrl_cur, float *ctrl_prop, uint32_t *surv,
                                           float *ell_surv, double *lam_surv, double *lam_cand, uint32_t *n_eval) {
    if (!ctx) return SMC_EINVAL;
    if (!ctx->have_scn) return fail(ctx, SMC_ESTATE, "no scenario");
    const int n = ctx->dsc.n, H = ctx->dsc.H;
    const int P = ctx->last_eval >= 0 ? ctx->last_eval : ctx->cur;
    const size_t Lk = (ctx->last_eval >= 0 && ctx->Leval) ? ctx->Leval : ctx->Lloc;
    const size_t nrow = Lk * n * H * 3;
    if (n_eval) *n_eval = (uint32_t)Lk;
    if (ctrl_cur) CK(cudaMemcpyAsync(ctrl_cur, ctx->ctrl[P][0], sizeof(float) * nrow, cudaMemcpyDeviceToHost, ctx->st));
    if (ctrl_prop) CK(cudaMemcpyAsync(ctrl_prop, ctx->ctrl[P][1], sizeof(float) * nrow, cudaMemcpyDeviceToHost, ctx->st));
    if (surv) CK(cudaMemcpyAsync(surv, ctx->surv, sizeof(uint32_t) * Lk, cudaMemcpyDeviceToHost, ctx->st));
    if (ell_surv) CK(cudaMemcpyAsync(ell_surv, ctx->ell, sizeof(float) * n * Lk, cudaMemcpyDeviceToHost, ctx->st));
    if (lam_surv) CK(cudaMemcpyAsync(lam_surv, ctx->lam, sizeof(double) * Lk, cudaMemcpyDeviceToHost, ctx->st));
    if (lam_cand) CK(cudaMemcpyAsync(lam_cand, ctx->lam2, 2 * sizeof(double) * Lk, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return SMC_OK;
}

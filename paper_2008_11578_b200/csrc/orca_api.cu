// orca_api.cu -- host side of the C ABI declared in include/orca_b200.h.
//
// No CPU fallback lives here: every entry point either launches the sm_100a
// kernels of orca_kernels.cuh / orca_lp_batch.cuh or fails with an error code.
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <pthread.h>
#include <new>
#include <vector>

#include "orca_kernels.cuh"
#include "orca_cert.cuh"
#include "orca_lp_batch.cuh"

using namespace orca;

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------

struct orca_sim {
    int device = 0;
    int precision = ORCA_F32;
    int64_t capacity = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    orca_params params{};
    bool have_params = false;
    bool loaded = false;
    int64_t frame = 0;   // frames completed (host mirror)
    int64_t n_bound = 0; // host-side upper bound on resident rows (owned + ghost)
    int64_t n_pre = 0;   // n_bound before the last step (parity taps)

    // state, storage-row order
    void *pv[3] = {nullptr, nullptr, nullptr}; // (x, y, vx, vy)
    int cur = 0;                               // pv[cur] is the current snapshot
    int pre = 0;                               // pv[pre] is the pre-step snapshot of the last step
    void *goalpref[2] = {nullptr, nullptr};    // (gx, gy, pref_speed, goal_tol)
    void *radmax[2] = {nullptr, nullptr};      // (radius, max_speed)
    i64 *ids[2] = {nullptr, nullptr};
    u8 *cls[2] = {nullptr, nullptr};
    i8 *status[2] = {nullptr, nullptr};
    i8 *failed[2] = {nullptr, nullptr};
    float *hint[2] = {nullptr, nullptr};       // radius that held last step's neighbour list
    // Physical rows may be stored in a different order than the reference's (logical) rows:
    // lrow[.][p] is the logical row of physical row p (identity until the first reordering).
    // Every host-facing copy goes through it; the kernels of the step never need it.
    int *lrow[2] = {nullptr, nullptr};
    Attr64 *a64[2] = {nullptr, nullptr};       // float64 attributes as uploaded (FP32-state modes only)
    int *lkeep = nullptr, *lscan = nullptr;    // compaction: keep flags / new rows in logical order
    bool rows_permuted = false;
    bool reorder_due = false;                  // lay the rows out in cell order at the next step
    int reorder_every = 32;                    // ORCA_REORDER_EVERY: frames between reorderings (0: never);
                                               // 1500-step run at 1 M agents: 32 -> 0.954 ms, 128 -> 0.963, 512 -> 0.986, once -> 1.006
    int64_t since_reorder = 0;
    int apre = 0;                              // attribute buffer index before the last step's compaction
    int acur = 0;
    u8 *arrived = nullptr;
    int *keep = nullptr, *dst_idx = nullptr;
    int *sel = nullptr, *sel_idx = nullptr; // strip selection flags and their scan
    int64_t ghost_bound = 0;                // ghost rows currently appended (upper bound)
    // device-side frame log (orca_run_logged)
    int log_mode = 0;                       // 0 off, 1 records, 2 records + trajectories
    orca_frame_record *log_rec = nullptr;
    int log_cap = 0;
    double4 *log_traj = nullptr;
    int64_t log_traj_cap = 0;
    i64 *arr_ids = nullptr, *arr_frames = nullptr; // arrivals since the upload (capacity rows)
    int64_t arr_read = 0;                          // ... of which the host has fetched this many
    // strip decomposition without host round trips (orca_strip_configure / _step)
    bool strip_on = false;
    int64_t strip_slack = 0;                // rows the host's launch bound keeps above the last known count
    bool strip_ghosts = false;              // ghost rows are resident (the host does not know how many)
    double strip_lo = -INFINITY, strip_hi = INFINITY;
    void *mig_slab[2] = {nullptr, nullptr}; // migrant slabs of the running orca_strip_step
    int64_t mig_cap = 0;
    // the exchange through peer memory (orca_strip_window_*)
    unsigned char *win = nullptr;           // this handle's window: [flag line x 2][side x parity receive buffers]
    int64_t win_side_bytes = 0, win_stride = 0;
    unsigned char *win_peer[2] = {nullptr, nullptr}; // the neighbours' windows as mapped here
    bool win_peer_ipc[2] = {false, false};           // ... through cudaIpcOpenMemHandle (to be closed)
    unsigned *win_done = nullptr;                    // block counter of k_window_push
    int64_t win_pushed[2] = {0, 0}, win_waited[2] = {0, 0}; // next exchange index per side
    unsigned long long win_timeout_ns = 20000000000ULL;

    // per-step scratch
    int max_cells = 0;
    int *cell_of = nullptr, *rank_of = nullptr, *cell_count = nullptr, *cell_start = nullptr,
        *block_sums = nullptr;
    void *s_xy = nullptr, *s_nr = nullptr, *s_dm = nullptr; // s_nr: NbRec<S>, 8 storage words per slot
    int *s_row = nullptr, *s_cell = nullptr;
    int *nb = nullptr;
    u8 *nb_cnt = nullptr;
    int *fq = nullptr;
    void *fq_state = nullptr;
    // half-planes (R4 x MAXN) and insertion order (u8 x MAXN) of the queued agents, written by the
    // solve kernels, read by k_fallback_coop; sized by orca_set_params for the max_neighbors in use
    void *fq_cons = nullptr;
    u8 *fq_perm = nullptr;
    u8 *s_perm = nullptr; // insertion order per sorted slot (k_shuffle -> k_solve_group), spill_maxn bytes each
    int spill_maxn = 0;
    int *cq = nullptr; // ORCA_CERT32: agents whose FP32 solve was not certified (solved in FP64)
    // ORCA_CERT32 takes the certified path only where it pays -- large crowds in which most LPs are
    // feasible (the count is the last one the host saw) -- and the FP64 kernels of ORCA_MIXED
    // otherwise; the results are the same bits either way, so this is a performance choice only
    bool cert_active = false;
    bool cert_force = false;   // ORCA_CERT_FORCE=1: always the certified path (tests: small and jammed crowds)
    int64_t cert_seen_frame = -1;
    int *gq = nullptr; // agents queued for the exact ring search
    GridPlan *plan = nullptr;
    GridPlan *h_plan = nullptr; // pinned mirror

    // float64 staging in the reference's host layout
    double *stg = nullptr;
    size_t stg_bytes = 0;
    double *dbg = nullptr;
    size_t dbg_bytes = 0;

    int64_t binned_frame = -1; // the sorted arrays describe the state after this many frames
    int64_t bbox_frame = -1;   // frame whose positions k_count's per-block boxes describe (-1: none)
    double4 *box_part = nullptr; // one bounding box per k_count block of the last bin build
    int box_parts = 0;
    int64_t launches = 0;      // kernels launched by this handle since creation
    double occ_target = 4.0;   // mean agents per search cell the plan aims for (ORCA_OCC_TARGET; results are
                               //  invariant under it, tests/test_gpu_step.py)
    int solve_gl = 2;          // lanes per agent in the LP kernel: 2 with FP64 arithmetic, 1 with FP32 (measured)
    bool use_graph = true;     // ORCA_GRAPH=0: launch the step's kernels one by one
    cudaStream_t aux_stream = nullptr; // copy stream of orca_advance_host
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // gather + solve + fallback are issued per CHUNK of sorted slots on two streams (solve_stage)
    int chunks = 0;                    // 0: chosen from the crowd size; ORCA_CHUNKS forces 1..ORCA_MAX_CHUNKS
    cudaStream_t chunk_stream = nullptr;
    cudaEvent_t ev_cfork = nullptr, ev_cjoin = nullptr, ev_patched = nullptr;
    // orca_advance_host: copies overlapped with the step (see there)
    cudaEvent_t ev_vel = nullptr, ev_state = nullptr, ev_dl = nullptr;
    bool split_vel = false;             // velocities arrive on aux_stream; patched in before k_solve
    double *early_pos = nullptr, *early_vel = nullptr; // host targets of the early download

    // CUDA graphs of one whole step, keyed by everything the launch sequence depends on
    struct StepGraph {
        int cur, acur;             // key: buffer rotation state before the step
        int64_t n_bound;           // key: launch grid sizes
        bool had_bins;             // key: sorted arrays already valid (metrics mode)
        int bbox_gap;              // key: which bounding-box path the bin build takes (-1: k_bbox)
        int log_mode;              // key: the frame-log kernels are part of the sequence
        void *mig0, *mig1;         // key: migrant slabs of orca_strip_step (null outside strips)
        int64_t mig_cap;
        bool strip_ghosts;         // key: the compaction that drops ghosts is part of the sequence
        bool cert_active;          // key: which solve kernels run (ORCA_CERT32)
        int bbox_rel;              // bbox_frame - frame after the step
        cudaGraphExec_t exec;
        int new_cur, new_acur, new_pre; // host state after the step
        bool leaves_bins;
        int64_t launches;
    };
    std::vector<StepGraph> graphs;
    void drop_graphs()
    {
        for (auto &g : graphs) cudaGraphExecDestroy(g.exec);
        graphs.clear();
    }

    // optional per-stage timing (orca_profile_stages)
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool; // ORCA_N_STAGES + 1 events per profiled step
    size_t ev_used = 0;
    char err[512] = {0};

    void mark()
    {
        if (!profiling) return;
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return;
            ev_pool.push_back(e);
        }
        cudaEventRecord(ev_pool[ev_used++], stream);
    }
};

static thread_local char g_err[512] = {0};

static int fail(orca_sim *sim, int code, const char *fmt, ...)
{
    char *dst = sim ? sim->err : g_err;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(dst, 512, fmt, ap);
    va_end(ap);
    if (sim) memcpy(g_err, sim->err, 512);
    return code;
}

#define CK(sim, call)                                                                             \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(sim, ORCA_ECUDA, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),      \
                        __FILE__, __LINE__, cudaGetErrorString(e_));                              \
    } while (0)

#define CKL(sim) CK(sim, cudaGetLastError())

template <typename T> static cudaError_t dalloc(T **p, size_t count)
{
    return cudaMalloc(reinterpret_cast<void **>(p), (count ? count : 1) * sizeof(T));
}

static constexpr int pick_threads(int bytes_per_thread)
{
    return bytes_per_thread * 128 <= 72 * 1024 ? 128 : (bytes_per_thread * 64 <= 72 * 1024 ? 64 : 32);
}

template <typename R, int MAXN> struct KCfg {
    typedef typename Vec<R>::T4 R4;
    static constexpr int solve_bpt = (int)sizeof(R4) * MAXN + MAXN;
    static constexpr int solve_threads = pick_threads(solve_bpt);
    static constexpr int fb_bpt = 2 * (int)sizeof(R4) * MAXN + 2 * MAXN; // per ACTIVE thread
#ifndef ORCA_FB_THREADS
#define ORCA_FB_THREADS 128
#endif
    static constexpr int fb_threads = ORCA_FB_THREADS;
};

extern "C" int orca_abi_version(void) { return ORCA_ABI_VERSION; }

extern "C" const char *orca_last_error(const orca_sim *sim) { return sim ? sim->err : g_err; }

// ---------------------------------------------------------------------------
// create / destroy
// ---------------------------------------------------------------------------

template <typename S, typename R, int MAXN> static cudaError_t set_smem_attrs()
{
    typedef KCfg<R, MAXN> C;
    cudaError_t e = cudaFuncSetAttribute(k_solve<S, R, MAXN, C::solve_threads>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::solve_bpt * C::solve_threads);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_solve_group<S, R, MAXN, 128, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::solve_bpt * 64);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_solve_group<S, R, MAXN, 128, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::solve_bpt * 64);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_solve_group_queue<S, R, MAXN, 128, ORCA_QUEUE_GL, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, C::solve_bpt * (128 / ORCA_QUEUE_GL));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_fallback_coop<S, R, MAXN, C::fb_threads, ORCA_GL_SHORT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::fb_bpt * (C::fb_threads / ORCA_GL_SHORT));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_fallback_coop<S, R, MAXN, C::fb_threads, ORCA_GL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::fb_bpt * (C::fb_threads / ORCA_GL));
}

extern "C" void orca_destroy(orca_sim *sim)
{
    if (!sim) return;
    cudaSetDevice(sim->device);
    if (sim->stream) cudaStreamSynchronize(sim->stream);
    orca_strip_window_close(sim);
    for (int i = 0; i < 3; ++i) cudaFree(sim->pv[i]);
    for (int i = 0; i < 2; ++i) {
        cudaFree(sim->goalpref[i]);
        cudaFree(sim->radmax[i]);
        cudaFree(sim->ids[i]);
        cudaFree(sim->cls[i]);
        cudaFree(sim->status[i]);
        cudaFree(sim->failed[i]);
        cudaFree(sim->hint[i]);
    }
    cudaFree(sim->arrived);
    cudaFree(sim->keep);
    cudaFree(sim->dst_idx);
    cudaFree(sim->sel);
    cudaFree(sim->sel_idx);
    cudaFree(sim->box_part);
    cudaFree(sim->lrow[0]);
    cudaFree(sim->lrow[1]);
    cudaFree(sim->a64[0]);
    cudaFree(sim->a64[1]);
    cudaFree(sim->log_rec);
    cudaFree(sim->log_traj);
    cudaFree(sim->arr_ids);
    cudaFree(sim->arr_frames);
    cudaFree(sim->lkeep);
    cudaFree(sim->lscan);
    cudaFree(sim->cell_of);
    cudaFree(sim->rank_of);
    cudaFree(sim->cell_count);
    cudaFree(sim->cell_start);
    cudaFree(sim->block_sums);
    cudaFree(sim->s_xy);
    cudaFree(sim->s_nr);
    cudaFree(sim->s_dm);
    cudaFree(sim->s_row);
    cudaFree(sim->s_cell);
    cudaFree(sim->nb);
    cudaFree(sim->nb_cnt);
    cudaFree(sim->fq);
    cudaFree(sim->fq_state);
    cudaFree(sim->fq_cons);
    cudaFree(sim->fq_perm);
    cudaFree(sim->s_perm);
    cudaFree(sim->gq);
    cudaFree(sim->cq);
    cudaFree(sim->plan);
    cudaFree(sim->stg);
    cudaFree(sim->dbg);
    sim->drop_graphs();
    for (cudaEvent_t e : sim->ev_pool) cudaEventDestroy(e);
    if (sim->h_plan) cudaFreeHost(sim->h_plan);
    if (sim->own_stream) cudaStreamDestroy(sim->own_stream);
    if (sim->aux_stream) cudaStreamDestroy(sim->aux_stream);
    if (sim->chunk_stream) cudaStreamDestroy(sim->chunk_stream);
    if (sim->ev_cfork) cudaEventDestroy(sim->ev_cfork);
    if (sim->ev_cjoin) cudaEventDestroy(sim->ev_cjoin);
    if (sim->ev_patched) cudaEventDestroy(sim->ev_patched);
    if (sim->ev_fork) cudaEventDestroy(sim->ev_fork);
    if (sim->ev_join) cudaEventDestroy(sim->ev_join);
    if (sim->ev_vel) cudaEventDestroy(sim->ev_vel);
    if (sim->ev_state) cudaEventDestroy(sim->ev_state);
    if (sim->ev_dl) cudaEventDestroy(sim->ev_dl);
    delete sim;
}

extern "C" int orca_create(orca_sim **out, int device, int64_t capacity, int precision)
{
    if (!out) return fail(nullptr, ORCA_EINVAL, "orca_create: out is NULL");
    *out = nullptr;
    if (capacity < 0 || capacity > 0x3FFFFFFF)
        return fail(nullptr, ORCA_EINVAL, "orca_create: capacity %lld out of range", (long long)capacity);
    if (precision != ORCA_F32 && precision != ORCA_F64 && precision != ORCA_MIXED && precision != ORCA_CERT32)
        return fail(nullptr, ORCA_EINVAL, "orca_create: unknown precision %d", precision);
    int ndev = 0;
    CK(nullptr, cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(nullptr, ORCA_EINVAL, "orca_create: device %d not available (%d visible)", device, ndev);
    CK(nullptr, cudaSetDevice(device));

    orca_sim *sim = new (std::nothrow) orca_sim();
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_create: out of host memory");
    sim->device = device;
    sim->precision = precision;
    sim->capacity = capacity;
    if (const char *occ = getenv("ORCA_OCC_TARGET")) {
        const double v = atof(occ);
        if (v > 0.0) sim->occ_target = v;
    }
    sim->solve_gl = precision == ORCA_F32 ? 1 : 2;
    if (const char *re = getenv("ORCA_REORDER_EVERY")) sim->reorder_every = std::max(0, atoi(re));
    if (const char *gr = getenv("ORCA_GRAPH")) sim->use_graph = atoi(gr) != 0;
    if (const char *cf = getenv("ORCA_CERT_FORCE")) sim->cert_force = atoi(cf) != 0;
    if (const char *ch = getenv("ORCA_CHUNKS")) sim->chunks = std::min(ORCA_MAX_CHUNKS, std::max(0, atoi(ch)));
    const size_t cap = (size_t)(capacity > 0 ? capacity : 1);
    const size_t rs = precision == ORCA_F64 ? sizeof(double) : sizeof(float); // storage type S
    const size_t as = precision == ORCA_F32 ? sizeof(float) : sizeof(double); // arithmetic type R
    sim->max_cells = (int)(2 * cap + 1024);

#define CKC(call)                                                                                 \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            int rc_ = fail(nullptr, ORCA_ECUDA, "orca_create: %s: %s", #call, cudaGetErrorString(e_)); \
            orca_destroy(sim);                                                                    \
            return rc_;                                                                           \
        }                                                                                         \
    } while (0)

    CKC(cudaStreamCreateWithFlags(&sim->own_stream, cudaStreamNonBlocking));
    sim->stream = sim->own_stream;
    CKC(cudaStreamCreateWithFlags(&sim->aux_stream, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&sim->chunk_stream, cudaStreamNonBlocking));
    CKC(cudaEventCreateWithFlags(&sim->ev_cfork, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&sim->ev_cjoin, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&sim->ev_patched, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&sim->ev_fork, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&sim->ev_join, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&sim->ev_vel, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&sim->ev_state, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&sim->ev_dl, cudaEventDisableTiming));
    for (int i = 0; i < 3; ++i) CKC(cudaMalloc(&sim->pv[i], cap * 4 * rs));
    for (int i = 0; i < 2; ++i) {
        CKC(cudaMalloc(&sim->goalpref[i], cap * 4 * rs));
        CKC(cudaMalloc(&sim->radmax[i], cap * 2 * rs));
        CKC(dalloc(&sim->ids[i], cap));
        CKC(dalloc(&sim->cls[i], cap));
        CKC(dalloc(&sim->status[i], cap));
        CKC(dalloc(&sim->failed[i], cap));
        CKC(dalloc(&sim->hint[i], cap));
    }
    CKC(dalloc(&sim->arrived, cap));
    CKC(dalloc(&sim->keep, cap + 1));
    CKC(dalloc(&sim->dst_idx, cap + 1));
    CKC(dalloc(&sim->sel, cap + 1));
    CKC(dalloc(&sim->sel_idx, cap + 1));
    CKC(dalloc(&sim->box_part, (size_t)((std::max<int64_t>(cap, 1) + 255) / 256)));
    CKC(dalloc(&sim->lrow[0], cap));
    CKC(dalloc(&sim->lrow[1], cap));
    if (precision != ORCA_F64) {
        CKC(dalloc(&sim->a64[0], cap));
        CKC(dalloc(&sim->a64[1], cap));
    }
    CKC(dalloc(&sim->lkeep, cap + 1));
    CKC(dalloc(&sim->lscan, cap + 1));
    CKC(dalloc(&sim->cell_of, cap));
    CKC(dalloc(&sim->rank_of, cap));
    CKC(dalloc(&sim->cell_count, (size_t)sim->max_cells + 1));
    CKC(dalloc(&sim->cell_start, (size_t)sim->max_cells + 1));
    CKC(dalloc(&sim->block_sums, (size_t)sim->max_cells / SCAN_TILE + 2));
    CKC(cudaMalloc(&sim->s_xy, cap * 2 * rs));
    CKC(cudaMalloc(&sim->s_nr, cap * 8 * rs));
    CKC(cudaMalloc(&sim->s_dm, cap * 4 * as));
    CKC(dalloc(&sim->s_row, cap));
    CKC(dalloc(&sim->s_cell, cap));
    CKC(dalloc(&sim->nb, cap * ORCA_MAX_NEIGHBORS));
    CKC(dalloc(&sim->nb_cnt, cap));
    CKC(dalloc(&sim->fq, cap));
    CKC(cudaMalloc(&sim->fq_state, cap * 4 * as));
    CKC(dalloc(&sim->gq, cap));
    if (precision == ORCA_CERT32) CKC(dalloc(&sim->cq, cap));
    CKC(dalloc(&sim->plan, 1));
    CKC(cudaMallocHost(reinterpret_cast<void **>(&sim->h_plan), sizeof(GridPlan)));
    sim->stg_bytes = cap * 12 * sizeof(double);
    CKC(cudaMalloc(reinterpret_cast<void **>(&sim->stg), sim->stg_bytes));
    CKC(cudaMemset(sim->plan, 0, sizeof(GridPlan)));
    CKC((set_smem_attrs<float, float, 16>()));
    CKC((set_smem_attrs<float, float, 32>()));
    CKC((set_smem_attrs<float, double, 16>()));
    CKC((set_smem_attrs<float, double, 32>()));
    CKC((set_smem_attrs<double, double, 16>()));
    CKC((set_smem_attrs<double, double, 32>()));
    CKC(cudaFuncSetAttribute(k_solve_cert<16, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 18 * 16 * 128));
    CKC(cudaFuncSetAttribute(k_solve_cert<32, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 18 * 32 * 128));
#undef CKC
    *out = sim;
    return ORCA_OK;
}

extern "C" int orca_set_stream(orca_sim *sim, void *cuda_stream)
{
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_set_stream: sim is NULL");
    CK(sim, cudaSetDevice(sim->device));
    CK(sim, cudaStreamSynchronize(sim->stream));
    sim->stream = cuda_stream ? reinterpret_cast<cudaStream_t>(cuda_stream) : sim->own_stream;
    sim->drop_graphs();
    return ORCA_OK;
}

extern "C" int orca_set_params(orca_sim *sim, const orca_params *p)
{
    if (!sim || !p) return fail(sim, ORCA_EINVAL, "orca_set_params: NULL argument");
    if (!(p->dt > 0.0) || !std::isfinite(p->dt))
        return fail(sim, ORCA_EINVAL, "dt must be positive, got %g", p->dt);
    if (!(p->tau > 0.0) || !std::isfinite(p->tau))
        return fail(sim, ORCA_EINVAL, "tau must be positive, got %g", p->tau);
    if (!(p->neighbor_radius > 0.0) || !std::isfinite(p->neighbor_radius))
        return fail(sim, ORCA_EINVAL, "neighbor_radius must be positive, got %g", p->neighbor_radius);
    if (p->max_neighbors < 0)
        return fail(sim, ORCA_EINVAL, "max_neighbors must be >= 0, got %d", p->max_neighbors);
    if (p->max_neighbors > ORCA_MAX_NEIGHBORS)
        return fail(sim, ORCA_EUNSUPPORTED, "max_neighbors %d exceeds ORCA_MAX_NEIGHBORS (%d)",
                    p->max_neighbors, ORCA_MAX_NEIGHBORS);
    if (!sim->have_params || memcmp(&sim->params, p, sizeof(orca_params)) != 0) sim->drop_graphs();
    const int maxn = p->max_neighbors <= 16 ? 16 : 32; // the MAXN the step's kernels are instantiated for
    if (maxn > sim->spill_maxn) {
        CK(sim, cudaSetDevice(sim->device));
        CK(sim, cudaStreamSynchronize(sim->stream));
        sim->drop_graphs(); // captured launches hold the old pointers
        cudaFree(sim->fq_cons);
        cudaFree(sim->fq_perm);
        cudaFree(sim->s_perm);
        sim->fq_cons = nullptr;
        sim->fq_perm = nullptr;
        sim->s_perm = nullptr;
        sim->spill_maxn = 0;
        const size_t cap = (size_t)(sim->capacity > 0 ? sim->capacity : 1);
        const size_t as = sim->precision == ORCA_F32 ? sizeof(float) : sizeof(double);
        CK(sim, cudaMalloc(&sim->fq_cons, cap * maxn * 4 * as));
        CK(sim, dalloc(&sim->fq_perm, cap * maxn));
        CK(sim, dalloc(&sim->s_perm, cap * maxn));
        sim->spill_maxn = maxn;
    }
    sim->params = *p;
    sim->have_params = true;
    sim->binned_frame = -1;
    return ORCA_OK;
}

// ---------------------------------------------------------------------------
// upload / download
// ---------------------------------------------------------------------------

static inline dim3 grid_for(int64_t n, int threads) { return dim3((unsigned)std::max<int64_t>(1, (n + threads - 1) / threads)); }

template <typename R>
static int upload_pv_impl(orca_sim *sim, int64_t n, const double *positions, const double *velocities)
{
    typedef typename Vec<R>::T4 R4;
    double *d_pos = sim->stg, *d_vel = sim->stg + 2 * n;
    CK(sim, cudaMemcpyAsync(d_pos, positions, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, sim->stream));
    CK(sim, cudaMemcpyAsync(d_vel, velocities, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, sim->stream));
    k_import_pv<R><<<grid_for(n, 256), 256, 0, sim->stream>>>(
        (int)n, d_pos, d_vel, reinterpret_cast<R4 *>(sim->pv[sim->cur]), sim->lrow[sim->acur]);
    CKL(sim);
    return ORCA_OK;
}

template <typename R>
static int upload_attrs_impl(orca_sim *sim, int64_t n, const double *radii, const double *pref,
                             const double *maxs, const double *goals, const double *gtol,
                             const int64_t *cls)
{
    typedef typename Vec<R>::T4 R4;
    typedef typename Vec<R>::T2 R2;
    double *b = sim->stg + 4 * n;
    double *d_rad = b, *d_pref = b + n, *d_max = b + 2 * n, *d_goal = b + 3 * n, *d_gtol = b + 5 * n;
    i64 *d_cls = reinterpret_cast<i64 *>(b + 6 * n);
    cudaStream_t st = sim->stream;
    CK(sim, cudaMemcpyAsync(d_rad, radii, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(sim, cudaMemcpyAsync(d_pref, pref, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(sim, cudaMemcpyAsync(d_max, maxs, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(sim, cudaMemcpyAsync(d_goal, goals, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, st));
    CK(sim, cudaMemcpyAsync(d_gtol, gtol, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(sim, cudaMemcpyAsync(d_cls, cls, sizeof(i64) * n, cudaMemcpyHostToDevice, st));
    k_import_attrs<R><<<grid_for(n, 256), 256, 0, st>>>(
        (int)n, d_rad, d_pref, d_max, d_goal, d_gtol, d_cls,
        reinterpret_cast<R4 *>(sim->goalpref[sim->acur]), reinterpret_cast<R2 *>(sim->radmax[sim->acur]),
        sim->cls[sim->acur], sim->hint[sim->acur], sim->plan, sim->a64[sim->acur]);
    CKL(sim);
    return ORCA_OK;
}

static int reset_plan(orca_sim *sim, int64_t n, int64_t frame)
{
    GridPlan h;
    memset(&h, 0, sizeof(h));
    h.n = (int)n;
    h.n_owned = (int)n;
    h.n_after = (int)n;
    h.n_pre = (int)n;
    h.err_pair = ORCA_NO_ERR;
    h.err_frame = -1;
    h.frame = frame;
    h.min_sep_enc = enc_double(INFINITY);
    h.vmax_enc = enc_double(0.0);
    h.rmax_enc = enc_double(0.0);
    h.sep_ub_enc = enc_double(INFINITY);
    *sim->h_plan = h;
    CK(sim, cudaMemcpyAsync(sim->plan, sim->h_plan, sizeof(GridPlan), cudaMemcpyHostToDevice, sim->stream));
    // the pinned mirror is reused by later reads; make sure this copy has left it
    CK(sim, cudaStreamSynchronize(sim->stream));
    return ORCA_OK;
}

extern "C" int orca_upload(orca_sim *sim, int64_t n, int64_t frame, const int64_t *ids,
                           const double *positions, const double *velocities, const double *radii,
                           const double *pref_speeds, const double *max_speeds, const double *goals,
                           const double *goal_tols, const int64_t *class_codes)
{
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_upload: sim is NULL");
    if (n < 0) return fail(sim, ORCA_EINVAL, "orca_upload: n = %lld", (long long)n);
    if (n > sim->capacity)
        return fail(sim, ORCA_ECAPACITY, "orca_upload: %lld agents exceed the handle capacity %lld",
                    (long long)n, (long long)sim->capacity);
    if (n > 0 && (!ids || !positions || !velocities || !radii || !pref_speeds || !max_speeds || !goals ||
                  !goal_tols || !class_codes))
        return fail(sim, ORCA_EINVAL, "orca_upload: NULL array");
    CK(sim, cudaSetDevice(sim->device));
    sim->cur = 0;
    sim->pre = 0;
    sim->acur = 0;
    int rc = reset_plan(sim, n, frame);
    if (rc) return rc;
    sim->rows_permuted = false;
    sim->reorder_due = sim->reorder_every > 0;
    sim->since_reorder = 0;
    sim->apre = 0;
    sim->drop_graphs(); // captured compactions assume the row-order state they were recorded in
    sim->arr_read = 0;
    if (n > 0) {
        k_iota<<<grid_for(n, 256), 256, 0, sim->stream>>>((int)n, sim->lrow[0]);
        CK(sim, cudaMemcpyAsync(sim->ids[0], ids, sizeof(i64) * n, cudaMemcpyHostToDevice, sim->stream));
        CK(sim, cudaMemsetAsync(sim->status[0], 0, n, sim->stream));
        CK(sim, cudaMemsetAsync(sim->failed[0], 0xFF, n, sim->stream));
        rc = sim->precision != ORCA_F64 ? upload_pv_impl<float>(sim, n, positions, velocities)
                                        : upload_pv_impl<double>(sim, n, positions, velocities);
        if (rc) return rc;
        rc = sim->precision != ORCA_F64 ? upload_attrs_impl<float>(sim, n, radii, pref_speeds, max_speeds, goals, goal_tols, class_codes)
                 : upload_attrs_impl<double>(sim, n, radii, pref_speeds, max_speeds, goals, goal_tols, class_codes);
        if (rc) return rc;
    }
    sim->frame = frame;
    sim->n_bound = n;
    sim->n_pre = n;
    sim->ghost_bound = 0;
    sim->strip_on = false;
    sim->strip_ghosts = false;
    sim->cert_active = sim->precision == ORCA_CERT32 && (sim->cert_force || n >= ORCA_CERT_MIN_AGENTS); // until a fallback count is seen
    sim->cert_seen_frame = frame;
    sim->loaded = true;
    sim->binned_frame = -1;
    sim->bbox_frame = -1;
    return ORCA_OK;
}

static int fetch_plan(orca_sim *sim);

extern "C" int orca_upload_pv(orca_sim *sim, int64_t n, int64_t frame, const double *positions,
                              const double *velocities)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_upload_pv: no resident state");
    if (sim->strip_on) { // the host bound has slack: ask the device
        int rc = fetch_plan(sim);
        if (rc) return rc;
        if (n != sim->h_plan->n_owned || sim->strip_ghosts)
            return fail(sim, ORCA_EINVAL, "orca_upload_pv: n = %lld but %d owned rows are resident%s", (long long)n,
                        sim->h_plan->n_owned, sim->strip_ghosts ? " (and ghosts)" : "");
    } else if (n != sim->n_bound)
        return fail(sim, ORCA_EINVAL, "orca_upload_pv: n = %lld but %lld rows are resident", (long long)n,
                    (long long)sim->n_bound);
    if (n > 0 && (!positions || !velocities)) return fail(sim, ORCA_EINVAL, "orca_upload_pv: NULL array");
    CK(sim, cudaSetDevice(sim->device));
    sim->frame = frame;
    sim->binned_frame = -1;
    sim->bbox_frame = -1; // positions replaced from outside
    k_set_frame<<<1, 1, 0, sim->stream>>>(sim->plan, frame);
    CKL(sim);
    if (n == 0) return ORCA_OK;
    return sim->precision != ORCA_F64 ? upload_pv_impl<float>(sim, n, positions, velocities)
                                      : upload_pv_impl<double>(sim, n, positions, velocities);
}

// copy the device plan to the pinned mirror and wait
static int fetch_plan(orca_sim *sim)
{
    CK(sim, cudaSetDevice(sim->device));
    CK(sim, cudaMemcpyAsync(sim->h_plan, sim->plan, sizeof(GridPlan), cudaMemcpyDeviceToHost, sim->stream));
    CK(sim, cudaStreamSynchronize(sim->stream));
    const GridPlan &h = *sim->h_plan;
    // strips: the launch bound stays FIXED between two synchronisations (so one captured graph
    // serves every frame in between) and therefore keeps room for what may arrive until the next
    // (rounded up to 32,768 rows so that the bound -- a graph key -- changes rarely)
    sim->n_bound = sim->strip_on ? std::min<int64_t>(sim->capacity, (((int64_t)h.n + sim->strip_slack + 32767) >> 15) << 15)
                                 : h.n;
    if (sim->precision == ORCA_CERT32 && h.frame > sim->cert_seen_frame) {
        int64_t fb = 0;
        for (int c = 0; c < ORCA_MAX_CHUNKS; ++c) fb += h.fq_count[c];
        sim->cert_active = sim->cert_force || (h.n_owned >= ORCA_CERT_MIN_AGENTS &&
                                               fb * 100 < (int64_t)h.n_owned * ORCA_CERT_MAX_FALLBACK_PCT);
        sim->cert_seen_frame = h.frame;
    }
    if (h.err_range) return fail(sim, ORCA_ERANGE, "agent position out of indexable grid range");
    if (h.err_capacity)
        return fail(sim, ORCA_ECAPACITY, "strip exchange: a slab or the handle capacity (%lld rows) overflowed",
                    (long long)sim->capacity);
    if (h.err_window)
        return fail(sim, ORCA_ETIMEOUT, "strip exchange: a neighbouring strip's slabs did not arrive within %.1f s",
                    (double)sim->win_timeout_ns * 1e-9);
    if (h.err_pair != ORCA_NO_ERR)
        return fail(sim, ORCA_ECOINCIDENT,
                    "frame %lld: agents %lld and %lld have exactly coincident centers; "
                    "avoidance direction is undefined",
                    (long long)h.err_frame, (long long)h.err_id_i, (long long)h.err_id_j);
    return ORCA_OK;
}

extern "C" int orca_sync(orca_sim *sim)
{
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_sync: sim is NULL");
    return fetch_plan(sim);
}

extern "C" int orca_get_info(orca_sim *sim, orca_info *info)
{
    if (!sim || !info) return fail(sim, ORCA_EINVAL, "orca_get_info: NULL argument");
    int rc = fetch_plan(sim);
    const GridPlan &h = *sim->h_plan;
    info->frame = h.frame;
    info->active_agents = h.n_owned;
    info->lp_fallbacks = 0;
    info->gather_queue = 0;
    info->solve_queue = 0;
    for (int c = 0; c < ORCA_MAX_CHUNKS; ++c) {
        info->lp_fallbacks += h.fq_count[c];
        info->gather_queue += h.gq_count[c];
        info->solve_queue += h.cq_count[c];
    }
    info->removed_agents = h.removed;
    info->collision_count = (int64_t)h.collisions;
    info->min_separation = dec_double(h.min_sep_enc);
    info->grid_nx = h.nx;
    info->grid_ny = h.ny;
    info->grid_cell = h.cell;
    info->kernel_launches = sim->launches;
    return rc;
}

template <typename R>
static int download_pv_impl(orca_sim *sim, int64_t n, double *positions, double *velocities, int lidx = -1)
{
    typedef typename Vec<R>::T4 R4;
    double *d_pos = sim->stg, *d_vel = sim->stg + 2 * n;
    k_export_pv<R><<<grid_for(n, 256), 256, 0, sim->stream>>>(
        (int)n, reinterpret_cast<const R4 *>(sim->pv[sim->cur]), d_pos, d_vel,
        sim->lrow[lidx < 0 ? sim->acur : lidx]);
    CKL(sim);
    if (positions)
        CK(sim, cudaMemcpyAsync(positions, d_pos, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, sim->stream));
    if (velocities)
        CK(sim, cudaMemcpyAsync(velocities, d_vel, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, sim->stream));
    return ORCA_OK;
}

template <typename R>
static int download_attrs_impl(orca_sim *sim, int64_t n, double *radii, double *pref, double *maxs,
                               double *goals, double *gtol, int64_t *cls)
{
    typedef typename Vec<R>::T4 R4;
    typedef typename Vec<R>::T2 R2;
    double *b = sim->stg + 4 * n;
    double *d_rad = b, *d_pref = b + n, *d_max = b + 2 * n, *d_goal = b + 3 * n, *d_gtol = b + 5 * n;
    i64 *d_cls = reinterpret_cast<i64 *>(b + 6 * n);
    cudaStream_t st = sim->stream;
    k_export_attrs<R><<<grid_for(n, 256), 256, 0, st>>>(
        (int)n, reinterpret_cast<const R4 *>(sim->goalpref[sim->acur]),
        reinterpret_cast<const R2 *>(sim->radmax[sim->acur]), sim->cls[sim->acur], d_rad, d_pref, d_max,
        d_goal, d_gtol, d_cls, sim->lrow[sim->acur], sim->a64[sim->acur]);
    CKL(sim);
    if (radii) CK(sim, cudaMemcpyAsync(radii, d_rad, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    if (pref) CK(sim, cudaMemcpyAsync(pref, d_pref, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    if (maxs) CK(sim, cudaMemcpyAsync(maxs, d_max, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    if (goals) CK(sim, cudaMemcpyAsync(goals, d_goal, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
    if (gtol) CK(sim, cudaMemcpyAsync(gtol, d_gtol, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    if (cls) CK(sim, cudaMemcpyAsync(cls, d_cls, sizeof(i64) * n, cudaMemcpyDeviceToHost, st));
    return ORCA_OK;
}

extern "C" int orca_download(orca_sim *sim, int64_t *ids, double *positions, double *velocities,
                             double *radii, double *pref_speeds, double *max_speeds, double *goals,
                             double *goal_tols, int64_t *class_codes)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_download: no resident state");
    int rc = fetch_plan(sim);
    if (rc) return rc;
    const int64_t n = sim->h_plan->n_owned;
    if (n == 0) return ORCA_OK;
    if (ids) {
        i64 *d_ids = reinterpret_cast<i64 *>(sim->stg + 11 * n);
        k_export_i64<<<grid_for(n, 256), 256, 0, sim->stream>>>((int)n, sim->ids[sim->acur], d_ids,
                                                                sim->lrow[sim->acur]);
        CKL(sim);
        CK(sim, cudaMemcpyAsync(ids, d_ids, sizeof(i64) * n, cudaMemcpyDeviceToHost, sim->stream));
    }
    if (positions || velocities) {
        rc = sim->precision != ORCA_F64 ? download_pv_impl<float>(sim, n, positions, velocities)
                                        : download_pv_impl<double>(sim, n, positions, velocities);
        if (rc) return rc;
    }
    if (radii || pref_speeds || max_speeds || goals || goal_tols || class_codes) {
        rc = sim->precision != ORCA_F64 ? download_attrs_impl<float>(sim, n, radii, pref_speeds, max_speeds, goals, goal_tols, class_codes)
                 : download_attrs_impl<double>(sim, n, radii, pref_speeds, max_speeds, goals, goal_tols, class_codes);
        if (rc) return rc;
    }
    CK(sim, cudaStreamSynchronize(sim->stream));
    return ORCA_OK;
}

extern "C" int orca_download_last_step_pv(orca_sim *sim, int64_t n, double *positions, double *velocities)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_download_last_step_pv: no resident state");
    int rc = fetch_plan(sim);
    if (rc) return rc;
    // (the device knows how many rows the last step had even after graph replays with removal)
    if (sim->frame > 0 || sim->h_plan->n_pre > 0) sim->n_pre = sim->h_plan->n_pre;
    if (n != sim->n_pre)
        return fail(sim, ORCA_EINVAL, "orca_download_last_step_pv: n = %lld, last step had %lld rows",
                    (long long)n, (long long)sim->n_pre);
    if (n == 0) return ORCA_OK;
    // the step wrote pv[(pre+1)%3]; arrival removal compacts into a third buffer and leaves it intact
    const int keep_cur = sim->cur;
    sim->cur = (sim->pre + 1) % 3;
    rc = sim->precision != ORCA_F64 ? download_pv_impl<float>(sim, n, positions, velocities, sim->apre)
                                    : download_pv_impl<double>(sim, n, positions, velocities, sim->apre);
    sim->cur = keep_cur;
    if (rc) return rc;
    CK(sim, cudaStreamSynchronize(sim->stream));
    return ORCA_OK;
}

extern "C" int orca_download_last_step_kept(orca_sim *sim, int64_t n, uint8_t *kept)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_download_last_step_kept: no resident state");
    int rc = fetch_plan(sim);
    if (rc) return rc;
    if (sim->frame > 0 || sim->h_plan->n_pre > 0) sim->n_pre = sim->h_plan->n_pre;
    if (n != sim->n_pre)
        return fail(sim, ORCA_EINVAL, "orca_download_last_step_kept: n = %lld, last step had %lld rows",
                    (long long)n, (long long)sim->n_pre);
    if (n == 0) return ORCA_OK;
    if (!kept) return fail(sim, ORCA_EINVAL, "orca_download_last_step_kept: kept is NULL");
    u8 *d = reinterpret_cast<u8 *>(sim->stg);
    if (!sim->params.remove_arrivals) { // nothing is ever removed: no compaction ran, no flags exist
        CK(sim, cudaMemsetAsync(d, 1, (size_t)n, sim->stream));
    } else {
        // the flags of the step's compaction, in the physical row order of the pre-compaction arrays
        k_export_keep<<<grid_for(n, 256), 256, 0, sim->stream>>>((int)n, sim->keep, sim->lrow[sim->apre], d);
        CKL(sim);
    }
    CK(sim, cudaMemcpyAsync(kept, d, (size_t)n, cudaMemcpyDeviceToHost, sim->stream));
    CK(sim, cudaStreamSynchronize(sim->stream));
    return ORCA_OK;
}

extern "C" int orca_download_pv(orca_sim *sim, double *positions, double *velocities)
{
    return orca_download(sim, nullptr, positions, velocities, nullptr, nullptr, nullptr, nullptr, nullptr,
                         nullptr);
}

// ---------------------------------------------------------------------------
// the step
// ---------------------------------------------------------------------------

static StepParams make_params(const orca_sim *sim)
{
    StepParams P;
    const orca_params &p = sim->params;
    P.dt = p.dt;
    P.tau = p.tau;
    P.nr = p.neighbor_radius;
    P.rad2 = p.neighbor_radius * p.neighbor_radius; // engine.py:213
    P.half_margin = 0.5 * p.avoidance_margin;       // engine.py:227
    for (int i = 0; i < 4; ++i) P.fmat[i] = p.fmat[i];
    P.max_n = p.max_neighbors;
    P.stride = (int)(sim->capacity > 0 ? sim->capacity : 1);
    P.max_cells = (int)std::min<int64_t>(sim->max_cells, 2 * sim->n_bound + 1024);
    P.occ_target = sim->occ_target;
    return P;
}

// K0 + K1: bounding box, plan, histogram, scan, scatter of pv[cur]
template <typename S, typename R> static int bin_build(orca_sim *sim, const StepParams &P)
{
    typedef typename Vec<S>::T4 S4;
    typedef typename Vec<S>::T2 S2;
    typedef typename Vec<R>::T4 R4;
    cudaStream_t st = sim->stream;
    const int64_t n = sim->n_bound;
    const S4 *pv = reinterpret_cast<const S4 *>(sim->pv[sim->cur]);
    CK(sim, cudaMemsetAsync(sim->cell_count, 0, sizeof(int) * ((size_t)P.max_cells + 1), st));
    // the box of the previous build (k_count accumulated it), grown by the frames since, or a
    // fresh reduction over the positions when they were replaced from outside
    const int64_t gap = sim->bbox_frame < 0 ? -1 : sim->frame - sim->bbox_frame;
    if (gap < 0 || gap > 1) {
        const int bbox_blocks = (int)std::min<int64_t>(148 * 4, std::max<int64_t>(1, (n + 255) / 256));
        k_begin_bins<<<1, 1, 0, st>>>(sim->plan);
        k_bbox<S><<<bbox_blocks, 256, 0, st>>>(sim->plan, pv);
        k_plan<<<1, 1, 0, st>>>(sim->plan, P, -1.0);
        sim->launches += 2;
    } else {
        k_plan<<<1, 1, 0, st>>>(sim->plan, P, (double)gap);
    }
    sim->bbox_frame = sim->frame;
    sim->box_parts = (int)std::max<int64_t>(1, (n + 255) / 256);
    k_count<S><<<grid_for(n, 256), 256, 0, st>>>(sim->plan, pv, sim->cell_of, sim->rank_of, sim->cell_count, P.nr,
                                                sim->box_part);
    const int scan_blocks = (P.max_cells + 1 + SCAN_TILE - 1) / SCAN_TILE;
    if (P.max_cells <= ORCA_SCAN_SMALL_CELLS) { // ncells <= max_cells: at most 33 tiles, typically a few
        k_scan_small<<<1, SCAN_THREADS, 0, st>>>(&sim->plan->ncells, 1, sim->cell_count, sim->cell_start);
        sim->launches -= 2;
    } else {
        k_scan_reduce<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->ncells, 1, sim->cell_count, sim->block_sums);
        k_scan_top<<<1, SCAN_THREADS, 0, st>>>(&sim->plan->ncells, 1, sim->block_sums);
        k_scan_apply<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->ncells, 1, sim->cell_count,
                                                           sim->block_sums, sim->cell_start);
    }
    k_scatter<S, R><<<grid_for(n, 256), 256, 0, st>>>(
        sim->plan, P, pv, reinterpret_cast<const S4 *>(sim->goalpref[sim->acur]),
        reinterpret_cast<const S2 *>(sim->radmax[sim->acur]), sim->cls[sim->acur], sim->cell_of, sim->rank_of,
        sim->cell_start, reinterpret_cast<S2 *>(sim->s_xy), reinterpret_cast<NbRec<S> *>(sim->s_nr),
        reinterpret_cast<R4 *>(sim->s_dm), sim->s_row, sim->s_cell);
    CKL(sim);
    sim->launches += 6;
    sim->binned_frame = sim->frame;
    return ORCA_OK;
}

// K2 for the sorted slots [s0, s1) = chunk c: certified fast pass for everyone, exact ring
// search for the agents it queued (queue segment gq + s0, counter gq_count[c])
template <typename S, int MAXN>
static int gather_stage(orca_sim *sim, const StepParams &P, cudaStream_t st, int s0, int s1, int c)
{
    typedef typename Vec<S>::T2 S2;
    const int64_t m = s1 - s0;
    const int a = sim->acur;
    k_gather_fast32<S, MAXN, 48><<<grid_for(m, 128), 128, 0, st>>>(
        sim->plan, P, reinterpret_cast<const S2 *>(sim->s_xy), sim->cell_start, sim->s_cell, sim->s_row,
        reinterpret_cast<const S2 *>(sim->radmax[a]), sim->hint[a], sim->nb, sim->nb_cnt, sim->gq + s0,
        &sim->plan->gq_count[c], s0, s1);
    const int gq_blocks = (int)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (m + 127) / 128));
    k_gather<S, MAXN><<<gq_blocks, 128, 0, st>>>(
        sim->plan, P, reinterpret_cast<const S2 *>(sim->s_xy), sim->cell_start, sim->s_cell, sim->s_row,
        sim->ids[a], sim->hint[a], sim->nb, sim->nb_cnt, sim->gq + s0, &sim->plan->gq_count[c]);
    CKL(sim);
    sim->launches += 2;
    return ORCA_OK;
}

// K3 for chunk c: insertion orders, half-planes + LP (k_solve_group / k_solve / k_solve_cert + the
// FP64 pass over what it could not certify), least-penetration queue
template <typename S, typename R, int MAXN>
static int solve_chunk(orca_sim *sim, const StepParams &P, int out_idx, cudaStream_t st, int s0, int s1, int c,
                       bool mark)
{
    typedef typename Vec<S>::T4 S4;
    typedef typename Vec<R>::T4 R4;
    typedef KCfg<R, MAXN> C;
    const int64_t m = s1 - s0;
    const int64_t n = sim->n_bound;
    const int a = sim->acur;
    int *fq_cnt = &sim->plan->fq_count[c];
    // queue segments of this chunk: at most m entries each, so they start at its first slot
    int *fq = sim->fq + s0;
    R4 *fq_state = reinterpret_cast<R4 *>(sim->fq_state) + s0;
    R4 *fq_cons = reinterpret_cast<R4 *>(sim->fq_cons) + (size_t)s0 * MAXN;
    u8 *fq_perm = sim->fq_perm + (size_t)s0 * MAXN;
#define ORCA_SOLVE_ARGS                                                                                    \
    sim->plan, P, reinterpret_cast<const NbRec<S> *>(sim->s_nr), reinterpret_cast<const R4 *>(sim->s_dm),  \
        sim->s_row, sim->ids[a], sim->nb, sim->nb_cnt,            \
        reinterpret_cast<const S4 *>(sim->goalpref[a]), reinterpret_cast<S4 *>(sim->pv[out_idx]),          \
        sim->status[a], sim->failed[a], sim->arrived, fq, fq_state, s0, s1, sim->lrow[a], fq_cons, fq_perm
    // below ~64 k agents the step is launch-latency bound and the extra launch costs more than the
    // idle lanes of the in-kernel shuffle (16,640 agents: +1.8 us)
    const bool cert = sim->precision == ORCA_CERT32 && sim->cert_active;
    const bool preshuffle = ORCA_PRESHUFFLE && sim->solve_gl >= 2 && (cert || n >= ORCA_PRESHUFFLE_MIN_AGENTS);
    const uint32_t *s_perm = preshuffle ? reinterpret_cast<const uint32_t *>(sim->s_perm) : nullptr;
    if (preshuffle) {
        k_shuffle<MAXN><<<grid_for(m, 128), 128, 0, st>>>(sim->plan, sim->s_row, sim->ids[a], sim->nb_cnt,
                                                         reinterpret_cast<uint4 *>(sim->s_perm), s0, s1);
        sim->launches += 1;
    }
    if (cert) {
        // FP32 solve with a certificate for everyone, the FP64 kernel for the agents it queued
        if constexpr (Fmt<S>::is_f32 && !Fmt<R>::is_f32) {
            k_solve_cert<MAXN, 128><<<grid_for(m, 128), 128, 18 * MAXN * 128, st>>>(
                sim->plan, P, reinterpret_cast<const NbRec<float> *>(sim->s_nr),
                reinterpret_cast<const double4 *>(sim->s_dm), sim->s_row, sim->nb, sim->nb_cnt,
                reinterpret_cast<const float4 *>(sim->goalpref[a]), reinterpret_cast<float4 *>(sim->pv[out_idx]),
                sim->status[a], sim->failed[a], sim->arrived, sim->cq + s0, s_perm, &sim->plan->cq_count[c], s0, s1);
            // (4x the resident blocks: a typical queue -- the ~6 % of a sparse crowd -- is ONE chunk per
            //  block, spread over every SM at once; blocks beyond the queue exit at their first test)
            constexpr int QNG = 128 / ORCA_QUEUE_GL; // agents per block of the queue pass
            const int qblocks = (int)std::min<int64_t>(148 * ORCA_SG_BLOCKS * 4 * (ORCA_QUEUE_GL / 2),
                                                       std::max<int64_t>(1, (m + QNG - 1) / QNG));
            k_solve_group_queue<S, R, MAXN, 128, ORCA_QUEUE_GL, true><<<qblocks, 128, C::solve_bpt * QNG, st>>>(
                ORCA_SOLVE_ARGS, s_perm, fq_cnt, sim->cq + s0, &sim->plan->cq_count[c]);
            sim->launches += 1;
        }
    } else if (sim->solve_gl == 2 && preshuffle)
        k_solve_group<S, R, MAXN, 128, 2, true><<<grid_for(m, 64), 128, C::solve_bpt * 64, st>>>(
            ORCA_SOLVE_ARGS, s_perm, fq_cnt);
    else if (sim->solve_gl == 2 && ORCA_SMALL_SOLVE_GL != 2 && n <= ORCA_SMALL_SOLVE_AGENTS)
        // a small crowd is one wave whose time is ONE agent's chain of half-planes: more lanes per agent
        k_solve_group<S, R, MAXN, 128, ORCA_SMALL_SOLVE_GL, false>
            <<<grid_for(m, 128 / ORCA_SMALL_SOLVE_GL), 128, C::solve_bpt * (128 / ORCA_SMALL_SOLVE_GL), st>>>(
                ORCA_SOLVE_ARGS, s_perm, fq_cnt);
    else if (sim->solve_gl == 2)
        k_solve_group<S, R, MAXN, 128, 2, false><<<grid_for(m, 64), 128, C::solve_bpt * 64, st>>>(
            ORCA_SOLVE_ARGS, s_perm, fq_cnt);
    else
        k_solve<S, R, MAXN, C::solve_threads><<<grid_for(m, C::solve_threads), C::solve_threads,
                                                C::solve_bpt * C::solve_threads, st>>>(ORCA_SOLVE_ARGS, fq_cnt);
#undef ORCA_SOLVE_ARGS
    sim->launches += 1;
    if (mark) sim->mark();
    {
#define ORCA_FB_ARGS                                                                                       \
    sim->plan, P, reinterpret_cast<const NbRec<S> *>(sim->s_nr), reinterpret_cast<const R4 *>(sim->s_dm),  \
        sim->s_row, sim->ids[a], sim->nb, sim->nb_cnt,            \
        reinterpret_cast<const S4 *>(sim->goalpref[a]), reinterpret_cast<S4 *>(sim->pv[out_idx]),          \
        sim->arrived, fq, fq_state, fq_cons, fq_perm, fq_cnt
        // long-queue and short-queue instance; the device-side queue length decides which one works
        const int ng = C::fb_threads / ORCA_GL; // agents per block and pass
        const int fb_blocks = (int)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (m + ng - 1) / ng));
        if (ORCA_GL_SHORT == ORCA_GL || m > ORCA_FB_SHORT_QUEUE) { // a queue of <= m entries is never "long"
            k_fallback_coop<S, R, MAXN, C::fb_threads, ORCA_GL><<<fb_blocks, C::fb_threads, C::fb_bpt * ng, st>>>(
                ORCA_FB_ARGS);
            sim->launches += 1;
        }
        if (ORCA_GL_SHORT != ORCA_GL) {
            const int ngs = C::fb_threads / ORCA_GL_SHORT;
            const int64_t qmax = std::min<int64_t>(m, ORCA_FB_SHORT_QUEUE);
            const int sb = (int)std::max<int64_t>(1, (qmax + ngs - 1) / ngs);
            k_fallback_coop<S, R, MAXN, C::fb_threads, ORCA_GL_SHORT><<<sb, C::fb_threads, C::fb_bpt * ngs, st>>>(
                ORCA_FB_ARGS);
            sim->launches += 1;
        }
#undef ORCA_FB_ARGS
    }
    CKL(sim);
    return ORCA_OK;
}

// K2 + K3. The stage is a pipeline over CHUNKS of sorted slots on two streams: the exact-search
// queue, the FP64 pass of ORCA_CERT32 and the least-penetration queue serve a few percent of the
// agents at a few percent of the machine's warp slots and take as long as one dependent chain;
// issued per chunk, those latency-bound kernels of one chunk run under the throughput-bound
// kernels (fast gather, LP) of the next. Chunks own disjoint sorted slots, queue segments and
// queue counters, and results do not depend on the number of chunks (tests/test_gpu_step.py).
template <typename S, typename R, int MAXN> static int solve_stage(orca_sim *sim, const StepParams &P, int out_idx)
{
    typedef typename Vec<S>::T4 S4;
    cudaStream_t st = sim->stream;
    const int64_t n = sim->n_bound;
    const int a = sim->acur;
    if (sim->spill_maxn < MAXN || !sim->fq_cons || !sim->fq_perm)
        return fail(sim, ORCA_EINVAL, "solve_stage: no spill buffers for max_neighbors %d", P.max_n);
    int chunks = sim->chunks > 0 ? sim->chunks : (n >= ORCA_CHUNK_MIN_AGENTS ? ORCA_CHUNKS_DEFAULT : 1);
    if (sim->profiling) chunks = 1; // per-stage events need the stages one after the other
    chunks = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, n / 1024));
    const int64_t per = ((n + chunks - 1) / chunks + 127) / 128 * 128;
    if (chunks == 1) {
        int rc = gather_stage<S, MAXN>(sim, P, st, 0, (int)n, 0);
        if (rc) return rc;
        sim->mark();
        if (sim->split_vel) {
            // the velocities were still in flight while the bins and the neighbour lists
            // were built from the positions; they are needed from here on
            CK(sim, cudaStreamWaitEvent(st, sim->ev_vel, 0));
            k_patch_vel<S><<<grid_for(n, 256), 256, 0, st>>>(
                sim->plan, sim->stg + 2 * n, reinterpret_cast<S4 *>(sim->pv[sim->cur]),
                reinterpret_cast<NbRec<S> *>(sim->s_nr), sim->cell_of, sim->rank_of, sim->cell_start, sim->lrow[a]);
            sim->launches += 1;
        }
        rc = solve_chunk<S, R, MAXN>(sim, P, out_idx, st, 0, (int)n, 0, true);
        if (rc) return rc;
        sim->mark();
        return ORCA_OK;
    }
    // fork: even chunks on the handle's stream, odd chunks on the second one
    cudaStream_t s2 = sim->chunk_stream;
    CK(sim, cudaEventRecord(sim->ev_cfork, st));
    CK(sim, cudaStreamWaitEvent(s2, sim->ev_cfork, 0));
    for (int c = 0; c < chunks; ++c) {
        cudaStream_t cs = (c & 1) ? s2 : st;
        const int s0 = (int)std::min<int64_t>(n, c * per), s1 = (int)std::min<int64_t>(n, (c + 1) * per);
        if (s1 <= s0) continue;
        int rc = gather_stage<S, MAXN>(sim, P, cs, s0, s1, c);
        if (rc) return rc;
        if (sim->split_vel) {
            if (c == 0) { // one patch of all rows, after the first chunk's gather; the others wait for it
                CK(sim, cudaStreamWaitEvent(cs, sim->ev_vel, 0));
                k_patch_vel<S><<<grid_for(n, 256), 256, 0, cs>>>(
                    sim->plan, sim->stg + 2 * n, reinterpret_cast<S4 *>(sim->pv[sim->cur]),
                    reinterpret_cast<NbRec<S> *>(sim->s_nr), sim->cell_of, sim->rank_of, sim->cell_start,
                    sim->lrow[a]);
                sim->launches += 1;
                CK(sim, cudaEventRecord(sim->ev_patched, cs));
            } else {
                CK(sim, cudaStreamWaitEvent(cs, sim->ev_patched, 0));
            }
        }
        rc = solve_chunk<S, R, MAXN>(sim, P, out_idx, cs, s0, s1, c, false);
        if (rc) return rc;
    }
    CK(sim, cudaEventRecord(sim->ev_cjoin, s2));
    CK(sim, cudaStreamWaitEvent(st, sim->ev_cjoin, 0));
    for (int i = 0; i < 3; ++i) sim->mark(); // (not reached while profiling; keeps the event count per step fixed)
    return ORCA_OK;
}

// A strip's removal of rows after a step, in place (k_strip_holes): emigrants into the slabs,
// arrivals and ghosts dropped, the tail's survivors moved into the holes. pv_idx: the buffer the
// step wrote (it stays the current one).
template <typename R> static int strip_fill_stage(orca_sim *sim, int pv_idx)
{
    typedef typename Vec<R>::T4 R4;
    typedef typename Vec<R>::T2 R2;
    cudaStream_t st = sim->stream;
    const int64_t n = sim->n_bound;
    const int a = sim->acur;
    orca_slab_header *hl = reinterpret_cast<orca_slab_header *>(sim->mig_slab[0]);
    orca_slab_header *hr = reinterpret_cast<orca_slab_header *>(sim->mig_slab[1]);
    k_strip_keep_flags<R><<<grid_for(n + 1, 256), 256, 0, st>>>(
        sim->plan, sim->arrived, sim->keep, sim->params.remove_arrivals, reinterpret_cast<const R4 *>(sim->pv[pv_idx]),
        reinterpret_cast<const R4 *>(sim->goalpref[a]), reinterpret_cast<const R2 *>(sim->radmax[a]), sim->ids[a],
        sim->cls[a], sim->strip_lo, sim->strip_hi, hl, hl ? reinterpret_cast<orca_agent_record *>(hl + 1) : nullptr, hr,
        hr ? reinterpret_cast<orca_agent_record *>(hr + 1) : nullptr, (int)sim->mig_cap, sim->a64[a]);
    k_strip_holes<<<grid_for(n, 256), 256, 0, st>>>(sim->plan, sim->keep, sim->sel, sim->sel_idx);
    // (holes are at most the emigrant slabs' capacity plus the arrivals; the grid covers every row
    //  all the same -- surplus threads leave at once)
    k_strip_fill<R><<<grid_for(n, 256), 256, 0, st>>>(
        sim->plan, sim->sel, sim->sel_idx, reinterpret_cast<R4 *>(sim->pv[pv_idx]),
        reinterpret_cast<R4 *>(sim->goalpref[a]), reinterpret_cast<R2 *>(sim->radmax[a]), sim->ids[a], sim->cls[a],
        sim->status[a], sim->failed[a], sim->hint[a], sim->lrow[a], sim->a64[a]);
    k_after_strip_fill<<<1, 1, 0, st>>>(sim->plan);
    CKL(sim);
    sim->launches += 4;
    return ORCA_OK;
}

// Order-preserving removal of rows: arrivals and ghosts after a step (from_sel == false)
// or the rows orca_strip_pack selected (from_sel == true).
template <typename R> static int compact_stage(orca_sim *sim, int src_idx, int dst_pv_idx, bool from_sel = false)
{
    typedef typename Vec<R>::T4 R4;
    typedef typename Vec<R>::T2 R2;
    cudaStream_t st = sim->stream;
    const int64_t n = sim->n_bound;
    const int a = sim->acur, b = 1 - a;
    const int *lscan = nullptr;
    // (a strip's storage order means nothing to the host -- agents come and go with every
    //  migration -- so there the survivors are simply renumbered in their new physical order)
    const bool logical = sim->rows_permuted && !sim->strip_on;
    if (!from_sel && n + 1 <= ORCA_SMALL_ROWS) {
        // a small crowd's frame is a chain of dependent launches: all four passes in one block
        k_removal_scans_small<<<1, SCAN_THREADS, 0, st>>>(sim->plan, sim->arrived, sim->params.remove_arrivals, sim->keep,
                                                          sim->dst_idx, logical ? sim->lrow[a] : nullptr, sim->lkeep,
                                                          sim->lscan);
        sim->launches -= 3;
        if (logical) lscan = sim->lscan;
    } else {
        if (from_sel)
            k_keep_unselected<<<grid_for(n + 1, 256), 256, 0, st>>>(sim->plan, sim->sel, sim->keep);
        else
            k_keep_flags<<<grid_for(n + 1, 256), 256, 0, st>>>(sim->plan, sim->arrived, sim->keep,
                                                               sim->params.remove_arrivals);
        const int scan_blocks = (int)((n + 1 + SCAN_TILE - 1) / SCAN_TILE);
        k_scan_reduce<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->keep, sim->block_sums);
        k_scan_top<<<1, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->block_sums);
        k_scan_apply<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->keep, sim->block_sums,
                                                           sim->dst_idx);
        if (logical) {
            // survivors keep the reference's relative order: new logical row = rank among the
            // surviving logical rows
            k_keep_by_logical<<<grid_for(n + 1, 256), 256, 0, st>>>(sim->plan, sim->keep, sim->lrow[a], sim->lkeep);
            k_scan_reduce<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->lkeep, sim->block_sums);
            k_scan_top<<<1, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->block_sums);
            k_scan_apply<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->lkeep, sim->block_sums,
                                                               sim->lscan);
            sim->launches += 4;
            lscan = sim->lscan;
        }
    }
    k_compact<R><<<grid_for(n, 256), 256, 0, st>>>(
        sim->plan, sim->keep, sim->dst_idx, reinterpret_cast<const R4 *>(sim->pv[src_idx]),
        reinterpret_cast<R4 *>(sim->pv[dst_pv_idx]), reinterpret_cast<const R4 *>(sim->goalpref[a]),
        reinterpret_cast<R4 *>(sim->goalpref[b]), reinterpret_cast<const R2 *>(sim->radmax[a]),
        reinterpret_cast<R2 *>(sim->radmax[b]), sim->ids[a], sim->ids[b], sim->cls[a], sim->cls[b],
        sim->status[a], sim->status[b], sim->failed[a], sim->failed[b], sim->hint[a], sim->hint[b],
        sim->lrow[a], sim->lrow[b], lscan, sim->a64[a], sim->a64[b],
        sim->log_mode && !from_sel ? sim->arr_ids : nullptr, sim->arr_frames, (int)sim->capacity);
    k_after_compact<<<1, 1, 0, st>>>(sim->plan, sim->dst_idx);
    CKL(sim);
    sim->launches += 6;
    sim->acur = b;
    return ORCA_OK;
}

template <typename R> static int metrics_stage(orca_sim *sim, const StepParams &P)
{
    typedef typename Vec<R>::T2 R2;
    const int64_t n = sim->n_bound;
    k_min_sep_bound<R><<<grid_for(n, 128), 128, 0, sim->stream>>>(
        sim->plan, P, reinterpret_cast<const R2 *>(sim->s_xy), sim->cell_start, sim->s_cell, sim->s_row,
        reinterpret_cast<const R2 *>(sim->radmax[sim->acur]));
    k_min_sep<R><<<grid_for(n, 128), 128, 0, sim->stream>>>(
        sim->plan, P, reinterpret_cast<const R2 *>(sim->s_xy), sim->cell_start, sim->s_cell, sim->s_row,
        sim->ids[sim->acur], reinterpret_cast<const R2 *>(sim->radmax[sim->acur]), 1e-6 /* engine.py:36 */);
    CKL(sim);
    sim->launches += 2;
    return ORCA_OK;
}

// Lay the rows out in the cell-sorted order of a fresh bin build (k_permute_rows).
template <typename S, typename R> static int reorder_rows(orca_sim *sim, const StepParams &P)
{
    typedef typename Vec<S>::T4 S4;
    typedef typename Vec<S>::T2 S2;
    const int64_t n = sim->n_bound;
    int rc = bin_build<S, R>(sim, P);
    if (rc) return rc;
    const int a = sim->acur, b = 1 - a, dst = (sim->cur + 1) % 3;
    k_permute_rows<S><<<grid_for(n, 256), 256, 0, sim->stream>>>(
        sim->plan, sim->s_row, reinterpret_cast<const S4 *>(sim->pv[sim->cur]), reinterpret_cast<S4 *>(sim->pv[dst]),
        reinterpret_cast<const S4 *>(sim->goalpref[a]), reinterpret_cast<S4 *>(sim->goalpref[b]),
        reinterpret_cast<const S2 *>(sim->radmax[a]), reinterpret_cast<S2 *>(sim->radmax[b]), sim->ids[a],
        sim->ids[b], sim->cls[a], sim->cls[b], sim->status[a], sim->status[b], sim->failed[a], sim->failed[b],
        sim->hint[a], sim->hint[b], sim->lrow[a], sim->lrow[b], sim->a64[a], sim->a64[b]);
    CKL(sim);
    sim->launches += 1;
    if (sim->strip_on) { // a strip's logical rows are its physical rows (strip_fill_stage relies on it)
        k_iota<<<grid_for(n, 256), 256, 0, sim->stream>>>((int)n, sim->lrow[b]);
        CKL(sim);
        sim->launches += 1;
    }
    sim->cur = dst;
    sim->acur = b;
    sim->rows_permuted = true;
    sim->binned_frame = -1; // the sorted arrays refer to the old rows
    return ORCA_OK;
}

template <typename S, typename R> static int step_impl(orca_sim *sim)
{
    StepParams P = make_params(sim);
    int rc;
    const int64_t n = sim->n_bound;
    sim->n_pre = n;
    if (sim->reorder_due && sim->ghost_bound == 0 && !sim->strip_on && n > 1) { // (strips: the driver reorders)
        rc = reorder_rows<S, R>(sim, P);
        if (rc) return rc;
        sim->reorder_due = false;
        sim->since_reorder = 0;
    }
    sim->mark(); // stage boundaries: bins | gather | solve | fallback | finish+compact | metrics
    k_begin_step<<<1, 1, 0, sim->stream>>>(sim->plan);
    sim->launches += 1;
    if (n == 0) { // engine.py:202-209
        k_finish<<<1, 1, 0, sim->stream>>>(sim->plan, sim->params.remove_arrivals, nullptr, nullptr);
        if (sim->log_mode)
            k_log_frame<<<1, 1, 0, sim->stream>>>(sim->plan, sim->log_rec, sim->log_cap, sim->log_mode == 2);
        CKL(sim);
        sim->launches += 1 + (sim->log_mode ? 1 : 0);
        for (int i = 0; i < ORCA_N_STAGES; ++i) sim->mark();
        sim->frame += 1;
        return ORCA_OK;
    }
    if (sim->binned_frame != sim->frame) {
        rc = bin_build<S, R>(sim, P);
        if (rc) return rc;
    }
    sim->mark();
    const int out_idx = (sim->cur + 1) % 3;
    rc = P.max_n <= 16 ? solve_stage<S, R, 16>(sim, P, out_idx) : solve_stage<S, R, 32>(sim, P, out_idx);
    if (rc) return rc;
    k_finish<<<1, 1, 0, sim->stream>>>(sim->plan, sim->params.remove_arrivals, sim->ids[sim->acur],
                                       sim->lrow[sim->acur]);
    CKL(sim);
    sim->launches += 1;
    sim->pre = sim->cur;
    sim->apre = sim->acur;
    if (sim->reorder_every > 0 && ++sim->since_reorder >= sim->reorder_every) sim->reorder_due = true;
    if (sim->params.remove_arrivals || sim->ghost_bound > 0 || sim->strip_ghosts || sim->mig_cap > 0) {
        if (sim->mig_cap > 0) { // a strip: in place
            rc = strip_fill_stage<S>(sim, out_idx);
            if (rc) return rc;
            sim->cur = out_idx;
        } else {
            const int dst = (sim->cur + 2) % 3;
            rc = compact_stage<S>(sim, out_idx, dst);
            if (rc) return rc;
            sim->cur = dst;
        }
        sim->n_bound -= sim->ghost_bound; // ghosts never survive a step
        sim->ghost_bound = 0;             // (strips: the bound is fixed and ghost_bound stays 0)
        sim->strip_ghosts = false;
    } else {
        sim->cur = out_idx;
    }
    sim->mark();
    sim->frame += 1;
    sim->binned_frame = -1;
    if (sim->early_pos || sim->early_vel) {
        // the step's result is final here: ship it to the host on the copy stream while
        // this stream goes on with the metrics
        typedef typename Vec<S>::T4 S4;
        const int64_t m = sim->n_pre; // rows beyond the kept ones are don't-care
        CK(sim, cudaEventRecord(sim->ev_state, sim->stream));
        CK(sim, cudaStreamWaitEvent(sim->aux_stream, sim->ev_state, 0));
        // (only the surviving rows: the export scatters by logical row, and rows beyond them
        //  hold stale mappings)
        k_export_pv<S><<<grid_for(m, 256), 256, 0, sim->aux_stream>>>(
            (int)m, reinterpret_cast<const S4 *>(sim->pv[sim->cur]), sim->stg, sim->stg + 2 * m,
            sim->lrow[sim->acur], &sim->plan->n_owned);
        CKL(sim);
        if (sim->early_pos)
            CK(sim, cudaMemcpyAsync(sim->early_pos, sim->stg, sizeof(double) * 2 * m, cudaMemcpyDeviceToHost,
                                    sim->aux_stream));
        if (sim->early_vel)
            CK(sim, cudaMemcpyAsync(sim->early_vel, sim->stg + 2 * m, sizeof(double) * 2 * m,
                                    cudaMemcpyDeviceToHost, sim->aux_stream));
        CK(sim, cudaEventRecord(sim->ev_dl, sim->aux_stream));
        sim->launches += 1;
    }
    if (sim->params.compute_metrics) {
        // engine.py:270-286: metrics of the post-step, post-removal positions. The bin
        // build it needs is the one the next step would do anyway, so it is kept.
        StepParams P2 = make_params(sim);
        rc = bin_build<S, R>(sim, P2);
        if (rc) return rc;
        rc = metrics_stage<S>(sim, P2);
        if (rc) return rc;
    }
    if (sim->log_mode) {
        if (sim->log_mode == 2) {
            typedef typename Vec<S>::T4 S4;
            k_log_traj<S><<<grid_for(n, 256), 256, 0, sim->stream>>>(
                sim->plan, reinterpret_cast<const S4 *>(sim->pv[out_idx]), sim->lrow[sim->apre], sim->log_traj,
                (i64)sim->log_traj_cap);
            sim->launches += 1;
        }
        k_log_frame<<<1, 1, 0, sim->stream>>>(sim->plan, sim->log_rec, sim->log_cap, sim->log_mode == 2);
        CKL(sim);
        sim->launches += 1;
    }
    sim->mark();
    return ORCA_OK;
}

static int step_plain(orca_sim *sim)
{
    switch (sim->precision) {
    case ORCA_F32: return step_impl<float, float>(sim);
    case ORCA_MIXED:
    case ORCA_CERT32: return step_impl<float, double>(sim);
    default: return step_impl<double, double>(sim);
    }
}

// Replay (or capture on first use) the CUDA graph of one step. The launch sequence of a
// step depends only on the buffer rotation state, the launch bound n_bound and whether
// the bins are already valid; everything else the kernels need (n, frame, grid plan,
// queues) lives in device memory.
static int step_graphed(orca_sim *sim)
{
    const bool had_bins = sim->binned_frame == sim->frame;
    const int64_t gap64 = sim->bbox_frame < 0 ? -1 : sim->frame - sim->bbox_frame;
    const int bbox_gap = gap64 < 0 || gap64 > 1 ? -1 : (int)gap64;
    for (auto &g : sim->graphs) {
        if (g.cur == sim->cur && g.acur == sim->acur && g.n_bound == sim->n_bound && g.had_bins == had_bins &&
            g.bbox_gap == bbox_gap && g.log_mode == sim->log_mode && g.mig0 == sim->mig_slab[0] &&
            g.mig1 == sim->mig_slab[1] && g.mig_cap == sim->mig_cap && g.strip_ghosts == sim->strip_ghosts &&
            g.cert_active == sim->cert_active) {
            CK(sim, cudaGraphLaunch(g.exec, sim->stream));
            sim->n_pre = sim->n_bound;
            sim->apre = g.acur;
            if (sim->reorder_every > 0 && ++sim->since_reorder >= sim->reorder_every) sim->reorder_due = true;
            sim->pre = g.new_pre;
            sim->cur = g.new_cur;
            sim->acur = g.new_acur;
            sim->frame += 1;
            sim->bbox_frame = sim->frame + g.bbox_rel;
            sim->binned_frame = g.leaves_bins ? sim->frame : -1;
            sim->launches += g.launches;
            sim->strip_ghosts = false;
            return ORCA_OK;
        }
    }
    if (sim->graphs.size() >= 16) sim->drop_graphs(); // n_bound kept shrinking: start over
    orca_sim::StepGraph g{};
    g.cur = sim->cur;
    g.acur = sim->acur;
    g.n_bound = sim->n_bound;
    g.had_bins = had_bins;
    g.bbox_gap = bbox_gap;
    g.log_mode = sim->log_mode;
    g.mig0 = sim->mig_slab[0];
    g.mig1 = sim->mig_slab[1];
    g.mig_cap = sim->mig_cap;
    g.strip_ghosts = sim->strip_ghosts;
    g.cert_active = sim->cert_active;
    const int64_t l0 = sim->launches;
    if (cudaStreamBeginCapture(sim->stream, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
        cudaGetLastError();
        return step_plain(sim);
    }
    const int rc = step_plain(sim); // records the launches, advances the host-side state
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(sim->stream, &graph);
    if (rc != ORCA_OK || e != cudaSuccess || !graph) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        sim->use_graph = false; // fall back to plain launches for good
        return rc != ORCA_OK ? rc : fail(sim, ORCA_ECUDA, "CUDA graph capture failed: %s", cudaGetErrorString(e));
    }
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        sim->use_graph = false;
        return fail(sim, ORCA_ECUDA, "cudaGraphInstantiate failed: %s", cudaGetErrorString(e));
    }
    g.new_cur = sim->cur;
    g.new_acur = sim->acur;
    g.new_pre = sim->pre;
    g.leaves_bins = sim->binned_frame == sim->frame;
    g.bbox_rel = (int)(sim->bbox_frame - sim->frame);
    g.launches = sim->launches - l0;
    sim->graphs.push_back(g);
    CK(sim, cudaGraphLaunch(g.exec, sim->stream)); // the capture itself executed nothing
    return ORCA_OK;
}

// graph replay whenever the launch sequence is a function of the key (see step_graphed); in a
// strip the launch bound is fixed between synchronisations and the driver does the reordering,
// so frames with ghost rows resident replay too
static int step_dispatch(orca_sim *sim)
{
    const bool plain_state = sim->ghost_bound == 0 && (sim->strip_on || !sim->reorder_due);
    if (sim->use_graph && !sim->profiling && plain_state && sim->n_bound > 0) return step_graphed(sim);
    return step_plain(sim);
}

extern "C" int orca_step(orca_sim *sim)
{
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_step: sim is NULL");
    if (!sim->loaded) return fail(sim, ORCA_EINVAL, "orca_step: no state uploaded");
    if (!sim->have_params) return fail(sim, ORCA_EINVAL, "orca_step: orca_set_params was not called");
    CK(sim, cudaSetDevice(sim->device));
    return step_dispatch(sim);
}

// Lay the resident rows out in cell-sorted order now. orca_step does this by
// itself after an upload and every ORCA_REORDER_EVERY frames when no ghost rows are resident;
// the strip-decomposed driver, which always steps with ghosts appended, calls it explicitly
// between migration and the next halo exchange. Nothing the host can observe changes.
extern "C" int orca_reorder_rows(orca_sim *sim)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_reorder_rows: no resident state");
    if (!sim->have_params) return fail(sim, ORCA_EINVAL, "orca_reorder_rows: orca_set_params was not called");
    if (sim->ghost_bound > 0 || sim->strip_ghosts)
        return fail(sim, ORCA_EINVAL, "orca_reorder_rows: ghost rows are resident (drop them first)");
    CK(sim, cudaSetDevice(sim->device));
    if (sim->n_bound < 2) return ORCA_OK;
    const StepParams P = make_params(sim);
    int rc;
    if (!sim->rows_permuted) sim->drop_graphs(); // graphs captured with identity row order are stale now
    switch (sim->precision) {
    case ORCA_F32: rc = reorder_rows<float, float>(sim, P); break;
    case ORCA_MIXED:
    case ORCA_CERT32: rc = reorder_rows<float, double>(sim, P); break;
    default: rc = reorder_rows<double, double>(sim, P); break;
    }
    sim->reorder_due = false;
    sim->since_reorder = 0;
    return rc;
}

extern "C" int orca_profile_stages(orca_sim *sim, int enable)
{
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_profile_stages: sim is NULL");
    CK(sim, cudaSetDevice(sim->device));
    CK(sim, cudaStreamSynchronize(sim->stream));
    sim->profiling = enable != 0;
    sim->ev_used = 0;
    return ORCA_OK;
}

extern "C" int orca_get_stage_ms(orca_sim *sim, double *ms, int64_t *steps)
{
    if (!sim || !ms) return fail(sim, ORCA_EINVAL, "orca_get_stage_ms: NULL argument");
    CK(sim, cudaSetDevice(sim->device));
    CK(sim, cudaStreamSynchronize(sim->stream));
    for (int i = 0; i < ORCA_N_STAGES; ++i) ms[i] = 0.0;
    const size_t per = ORCA_N_STAGES + 1;
    const size_t nsteps = sim->ev_used / per;
    for (size_t k = 0; k < nsteps; ++k)
        for (int i = 0; i < ORCA_N_STAGES; ++i) {
            float t = 0.f;
            CK(sim, cudaEventElapsedTime(&t, sim->ev_pool[k * per + i], sim->ev_pool[k * per + i + 1]));
            ms[i] += (double)t;
        }
    if (steps) *steps = (int64_t)nsteps;
    sim->ev_used = 0;
    return ORCA_OK;
}

extern "C" int orca_run(orca_sim *sim, int64_t steps)
{
    for (int64_t i = 0; i < steps; ++i) {
        int rc = orca_step(sim);
        if (rc) return rc;
    }
    return ORCA_OK;
}

extern "C" int orca_run_logged(orca_sim *sim, int64_t steps, orca_frame_record *records, int64_t *n_records,
                               double *traj, int64_t traj_cap_rows, int64_t *traj_rows, int64_t *arr_ids,
                               int64_t *arr_frames, int64_t arr_cap, int64_t *n_arrivals)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_run_logged: no resident state");
    if (!sim->have_params) return fail(sim, ORCA_EINVAL, "orca_run_logged: orca_set_params was not called");
    if (steps < 0 || steps > 0x3FFFFFFF || (steps > 0 && !records) || !n_records ||
        (traj && (traj_cap_rows < 0 || !traj_rows)) || arr_cap < 0 || (arr_cap > 0 && (!arr_ids || !arr_frames)) ||
        !n_arrivals)
        return fail(sim, ORCA_EINVAL, "orca_run_logged: bad arguments");
    if (sim->ghost_bound > 0 || sim->strip_on)
        return fail(sim, ORCA_EINVAL, "orca_run_logged: not available on a strip / with ghost rows resident");
    CK(sim, cudaSetDevice(sim->device));
    *n_records = 0;
    *n_arrivals = 0;
    if (traj_rows) *traj_rows = 0;
    if (steps == 0) return ORCA_OK;
    // device-side log buffers (grown on demand; a new buffer invalidates captured launches)
    if (sim->log_cap < steps) {
        CK(sim, cudaStreamSynchronize(sim->stream));
        sim->drop_graphs();
        cudaFree(sim->log_rec);
        sim->log_rec = nullptr;
        sim->log_cap = 0;
        CK(sim, dalloc(&sim->log_rec, (size_t)steps));
        sim->log_cap = (int)steps;
    }
    if (traj && sim->log_traj_cap < traj_cap_rows) {
        CK(sim, cudaStreamSynchronize(sim->stream));
        sim->drop_graphs();
        cudaFree(sim->log_traj);
        sim->log_traj = nullptr;
        sim->log_traj_cap = 0;
        CK(sim, dalloc(&sim->log_traj, (size_t)std::max<int64_t>(traj_cap_rows, 1)));
        sim->log_traj_cap = traj_cap_rows;
    }
    if (!sim->arr_ids) {
        const size_t cap = (size_t)std::max<int64_t>(sim->capacity, 1);
        CK(sim, dalloc(&sim->arr_ids, cap));
        CK(sim, dalloc(&sim->arr_frames, cap));
    }
    k_log_reset<<<1, 1, 0, sim->stream>>>(sim->plan, 1);
    CKL(sim);
    sim->launches += 1;
    sim->log_mode = traj ? 2 : 1;
    int rc = ORCA_OK;
    for (int64_t i = 0; i < steps && rc == ORCA_OK; ++i) rc = orca_step(sim);
    sim->log_mode = 0;
    // ONE synchronisation: the plan (counters, sticky errors), then the logs it describes
    const int rc_plan = fetch_plan(sim);
    const GridPlan h = *sim->h_plan;
    k_log_reset<<<1, 1, 0, sim->stream>>>(sim->plan, 0);
    sim->launches += 1;
    if (rc) return rc;
    if (rc_plan) return rc_plan;
    // idle steps (nobody left) did not advance the device's frame counter: follow it
    sim->frame = h.frame;
    sim->bbox_frame = -1;
    sim->binned_frame = -1;
    const int64_t nrec = std::min<int64_t>(h.log_count, steps);
    if (nrec > 0)
        CK(sim, cudaMemcpyAsync(records, sim->log_rec, sizeof(orca_frame_record) * nrec, cudaMemcpyDeviceToHost,
                                sim->stream));
    *n_records = nrec;
    if (traj) {
        if (h.traj_rows > traj_cap_rows)
            return fail(sim, ORCA_ECAPACITY, "orca_run_logged: %lld trajectory rows, buffer holds %lld",
                        (long long)h.traj_rows, (long long)traj_cap_rows);
        if (h.traj_rows > 0)
            CK(sim, cudaMemcpyAsync(traj, sim->log_traj, sizeof(double4) * h.traj_rows, cudaMemcpyDeviceToHost,
                                    sim->stream));
        *traj_rows = h.traj_rows;
    }
    const int64_t fresh = (int64_t)h.arr_count - sim->arr_read;
    if (fresh > arr_cap)
        return fail(sim, ORCA_ECAPACITY, "orca_run_logged: %lld arrivals, buffers hold %lld", (long long)fresh,
                    (long long)arr_cap);
    if (fresh > 0) {
        CK(sim, cudaMemcpyAsync(arr_ids, sim->arr_ids + sim->arr_read, sizeof(i64) * fresh, cudaMemcpyDeviceToHost,
                                sim->stream));
        CK(sim, cudaMemcpyAsync(arr_frames, sim->arr_frames + sim->arr_read, sizeof(i64) * fresh,
                                cudaMemcpyDeviceToHost, sim->stream));
    }
    *n_arrivals = fresh;
    sim->arr_read = h.arr_count;
    CK(sim, cudaStreamSynchronize(sim->stream));
    return ORCA_OK;
}

extern "C" int orca_step_host(orca_sim *sim, int64_t n, int64_t frame, const double *positions,
                              const double *velocities, double *new_positions, double *new_velocities,
                              int64_t *out_status)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_step_host: no resident state");
    if (sim->params.remove_arrivals)
        return fail(sim, ORCA_EINVAL, "orca_step_host requires remove_arrivals == 0");
    int rc = orca_upload_pv(sim, n, frame, positions, velocities);
    if (rc) return rc;
    rc = orca_step(sim);
    if (rc) return rc;
    if (n > 0) {
        rc = sim->precision != ORCA_F64 ? download_pv_impl<float>(sim, n, new_positions, new_velocities)
                                        : download_pv_impl<double>(sim, n, new_positions, new_velocities);
        if (rc) return rc;
        if (out_status) {
            i64 *d = reinterpret_cast<i64 *>(sim->stg + 4 * n);
            k_export_i8<<<grid_for(n, 256), 256, 0, sim->stream>>>((int)n, sim->status[sim->acur], d,
                                                                   sim->lrow[sim->acur]);
            CKL(sim);
            CK(sim, cudaMemcpyAsync(out_status, d, sizeof(i64) * n, cudaMemcpyDeviceToHost, sim->stream));
        }
    }
    return fetch_plan(sim);
}

// engine._advance through host buffers with the copies overlapped (engine.py:194-295 with
// the static attributes resident): positions go up first and the bin build + neighbour
// gather start on them while the velocities are still on the wire; the new positions and
// velocities go down on the copy stream while the metrics of the new state are computed.
// Rows [0, info->active_agents) of new_positions / new_velocities are the new state (the
// buffers must hold n rows). Same results as orca_upload_pv + orca_step + orca_download_pv.
extern "C" int orca_advance_host(orca_sim *sim, int64_t n, int64_t frame, const double *positions,
                                 const double *velocities, double *new_positions, double *new_velocities,
                                 orca_info *info)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_advance_host: no resident state");
    if (!sim->have_params) return fail(sim, ORCA_EINVAL, "orca_advance_host: orca_set_params was not called");
    if (sim->strip_on) return fail(sim, ORCA_EINVAL, "orca_advance_host: not available on a strip");
    if (n != sim->n_bound || sim->ghost_bound != 0)
        return fail(sim, ORCA_EINVAL, "orca_advance_host: n = %lld but %lld rows are resident", (long long)n,
                    (long long)sim->n_bound);
    if (!info || (n > 0 && (!positions || !velocities || !new_positions || !new_velocities)))
        return fail(sim, ORCA_EINVAL, "orca_advance_host: NULL argument");
    CK(sim, cudaSetDevice(sim->device));
    sim->frame = frame;
    sim->binned_frame = -1;
    sim->bbox_frame = -1; // positions replaced from outside
    k_set_frame<<<1, 1, 0, sim->stream>>>(sim->plan, frame);
    CKL(sim);
    int rc = ORCA_OK;
    if (n > 0) {
        cudaStream_t st = sim->stream, cp = sim->aux_stream;
        double *d_pos = sim->stg, *d_vel = sim->stg + 2 * n;
        // earlier work on the main stream (a previous download) may still read the staging area
        CK(sim, cudaEventRecord(sim->ev_fork, st));
        CK(sim, cudaStreamWaitEvent(cp, sim->ev_fork, 0));
        CK(sim, cudaMemcpyAsync(d_pos, positions, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, st));
        CK(sim, cudaMemcpyAsync(d_vel, velocities, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, cp));
        CK(sim, cudaEventRecord(sim->ev_vel, cp));
        if (sim->precision != ORCA_F64)
            k_import_pos<float><<<grid_for(n, 256), 256, 0, st>>>(
                (int)n, d_pos, reinterpret_cast<float4 *>(sim->pv[sim->cur]), sim->lrow[sim->acur]);
        else
            k_import_pos<double><<<grid_for(n, 256), 256, 0, st>>>(
                (int)n, d_pos, reinterpret_cast<double4 *>(sim->pv[sim->cur]), sim->lrow[sim->acur]);
        CKL(sim);
        sim->split_vel = true;
        sim->early_pos = new_positions;
        sim->early_vel = new_velocities;
        rc = step_plain(sim);
        sim->split_vel = false;
        sim->early_pos = sim->early_vel = nullptr;
        if (rc) return rc;
        CK(sim, cudaStreamWaitEvent(st, sim->ev_dl, 0)); // fetch_plan's sync then covers the copies
    } else {
        rc = step_plain(sim);
        if (rc) return rc;
    }
    return orca_get_info(sim, info);
}

// ---------------------------------------------------------------------------
// strip decomposition
// ---------------------------------------------------------------------------

template <typename S>
static int strip_pack_impl(orca_sim *sim, double x_lo, double x_hi, int remove, orca_agent_record *records,
                           int64_t cap, int64_t *count_out)
{
    typedef typename Vec<S>::T4 S4;
    typedef typename Vec<S>::T2 S2;
    cudaStream_t st = sim->stream;
    const int64_t n = sim->n_bound;
    const int a = sim->acur;
    const S4 *pv = reinterpret_cast<const S4 *>(sim->pv[sim->cur]);
    k_strip_flags<S><<<grid_for(n + 1, 256), 256, 0, st>>>(sim->plan, pv, x_lo, x_hi, sim->sel);
    const int scan_blocks = (int)((n + 1 + SCAN_TILE - 1) / SCAN_TILE);
    k_scan_reduce<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->sel, sim->block_sums);
    k_scan_top<<<1, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->block_sums);
    k_scan_apply<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->sel, sim->block_sums, sim->sel_idx);
    k_strip_pack<S><<<grid_for(std::max<int64_t>(n, 1), 256), 256, 0, st>>>(
        sim->plan, sim->sel, sim->sel_idx, pv, reinterpret_cast<const S4 *>(sim->goalpref[a]),
        reinterpret_cast<const S2 *>(sim->radmax[a]), sim->ids[a], sim->cls[a], records, cap, sim->a64[a]);
    CKL(sim);
    sim->launches += 5;
    int rc = fetch_plan(sim);
    if (rc) return rc;
    const int64_t count = sim->h_plan->pack_count;
    if (count_out) *count_out = count;
    if (count > cap)
        return fail(sim, ORCA_ECAPACITY, "orca_strip_pack: %lld agents selected, buffer holds %lld",
                    (long long)count, (long long)cap);
    if (remove && count > 0) {
        // compaction of the CURRENT snapshot into a spare pv buffer
        const int dst = (sim->cur + 1) % 3;
        rc = compact_stage<S>(sim, sim->cur, dst, true);
        if (rc) return rc;
        sim->cur = dst;
        sim->n_bound -= count;
        sim->binned_frame = -1;
    }
    return ORCA_OK;
}

extern "C" int orca_strip_pack(orca_sim *sim, double x_lo, double x_hi, int remove,
                               orca_agent_record *records, int64_t cap, int64_t *count_out)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_pack: no resident state");
    if (cap < 0 || (cap > 0 && !records)) return fail(sim, ORCA_EINVAL, "orca_strip_pack: bad buffer");
    if (sim->strip_on)
        return fail(sim, ORCA_EINVAL, "orca_strip_pack: the handle runs the slab protocol (orca_strip_configure)");
    if (remove && sim->ghost_bound > 0)
        return fail(sim, ORCA_EINVAL, "orca_strip_pack: cannot remove rows while ghosts are resident");
    CK(sim, cudaSetDevice(sim->device));
    return sim->precision == ORCA_F64 ? strip_pack_impl<double>(sim, x_lo, x_hi, remove, records, cap, count_out)
                                      : strip_pack_impl<float>(sim, x_lo, x_hi, remove, records, cap, count_out);
}

template <typename S> static int strip_append_impl(orca_sim *sim, const orca_agent_record *records, int64_t count, int ghost)
{
    typedef typename Vec<S>::T4 S4;
    typedef typename Vec<S>::T2 S2;
    const int a = sim->acur;
    k_strip_append<S><<<grid_for(count, 256), 256, 0, sim->stream>>>(
        sim->plan, records, (int)count, reinterpret_cast<S4 *>(sim->pv[sim->cur]),
        reinterpret_cast<S4 *>(sim->goalpref[a]), reinterpret_cast<S2 *>(sim->radmax[a]), sim->ids[a],
        sim->cls[a], sim->status[a], sim->failed[a], sim->hint[a], sim->lrow[a], sim->a64[a]);
    k_after_append<<<1, 1, 0, sim->stream>>>(sim->plan, (int)count, ghost);
    CKL(sim);
    sim->launches += 2;
    return ORCA_OK;
}

extern "C" int orca_strip_append(orca_sim *sim, const orca_agent_record *records, int64_t count, int ghost)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_append: no resident state");
    if (count < 0 || (count > 0 && !records)) return fail(sim, ORCA_EINVAL, "orca_strip_append: bad arguments");
    if (sim->strip_on)
        return fail(sim, ORCA_EINVAL, "orca_strip_append: the handle runs the slab protocol (orca_strip_configure)");
    if (!ghost && sim->ghost_bound > 0)
        return fail(sim, ORCA_EINVAL, "orca_strip_append: owned rows cannot follow ghost rows");
    if (sim->n_bound + count > sim->capacity)
        return fail(sim, ORCA_ECAPACITY, "orca_strip_append: %lld + %lld agents exceed the handle capacity %lld",
                    (long long)sim->n_bound, (long long)count, (long long)sim->capacity);
    if (count == 0) return ORCA_OK;
    CK(sim, cudaSetDevice(sim->device));
    int rc = sim->precision == ORCA_F64 ? strip_append_impl<double>(sim, records, count, ghost)
                                        : strip_append_impl<float>(sim, records, count, ghost);
    if (rc) return rc;
    sim->n_bound += count;
    if (ghost) sim->ghost_bound += count;
    sim->binned_frame = -1;
    sim->bbox_frame = -1; // rows appended from outside
    return ORCA_OK;
}

extern "C" int orca_strip_drop_ghosts(orca_sim *sim)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_drop_ghosts: no resident state");
    CK(sim, cudaSetDevice(sim->device));
    k_drop_ghosts<<<1, 1, 0, sim->stream>>>(sim->plan);
    CKL(sim);
    sim->launches += 1;
    sim->n_bound -= sim->ghost_bound;
    sim->ghost_bound = 0;
    sim->binned_frame = -1;
    return ORCA_OK;
}

// ---- the protocol with the counts kept on the device (see include/orca_b200.h) ----------

extern "C" int64_t orca_strip_halo_record_bytes(const orca_sim *sim)
{
    return sim && sim->precision == ORCA_F64 ? (int64_t)sizeof(orca_halo_record_f64)
                                             : (int64_t)sizeof(orca_halo_record_f32);
}

extern "C" int orca_strip_configure(orca_sim *sim, double x_lo, double x_hi, double vmax_floor, int64_t slack_rows)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_configure: no resident state");
    if (slack_rows < 0) return fail(sim, ORCA_EINVAL, "orca_strip_configure: slack_rows = %lld", (long long)slack_rows);
    if (sim->ghost_bound > 0) return fail(sim, ORCA_EINVAL, "orca_strip_configure: ghost rows are resident");
    if (!(x_lo < x_hi)) return fail(sim, ORCA_EINVAL, "orca_strip_configure: empty strip [%g, %g)", x_lo, x_hi);
    if (!(vmax_floor >= 0.0) || !std::isfinite(vmax_floor))
        return fail(sim, ORCA_EINVAL, "orca_strip_configure: vmax_floor = %g", vmax_floor);
    CK(sim, cudaSetDevice(sim->device));
    {   // exact row count now, launch bound = count + slack from here on (see fetch_plan)
        sim->strip_on = false;
        int rc = fetch_plan(sim);
        if (rc) return rc;
    }
    sim->strip_on = true;
    sim->strip_slack = slack_rows;
    sim->n_bound = std::min<int64_t>(sim->capacity, ((sim->n_bound + slack_rows + 32767) >> 15) << 15);
    sim->drop_graphs();
    sim->strip_lo = x_lo;
    sim->strip_hi = x_hi;
    k_strip_configure<<<1, 1, 0, sim->stream>>>(sim->plan, vmax_floor);
    CKL(sim);
    sim->launches += 1;
    return ORCA_OK;
}

extern "C" int orca_strip_pack_halo(orca_sim *sim, double reach, void *slab_left, void *slab_right, int64_t cap)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_pack_halo: no resident state");
    if (!sim->strip_on) return fail(sim, ORCA_EINVAL, "orca_strip_pack_halo: orca_strip_configure was not called");
    if (cap < 0 || cap > 0x7FFFFFFF || !(reach >= 0.0)) return fail(sim, ORCA_EINVAL, "orca_strip_pack_halo: bad arguments");
    if (sim->strip_ghosts) return fail(sim, ORCA_EINVAL, "orca_strip_pack_halo: ghost rows are resident");
    CK(sim, cudaSetDevice(sim->device));
    cudaStream_t st = sim->stream;
    orca_slab_header *hl = reinterpret_cast<orca_slab_header *>(slab_left);
    orca_slab_header *hr = reinterpret_cast<orca_slab_header *>(slab_right);
    if (hl) CK(sim, cudaMemsetAsync(hl, 0, sizeof(orca_slab_header), st));
    if (hr) CK(sim, cudaMemsetAsync(hr, 0, sizeof(orca_slab_header), st));
    if (!hl && !hr) return ORCA_OK;
    const int64_t n = sim->n_bound;
    const int a = sim->acur;
    const double le = sim->strip_lo + reach, re = sim->strip_hi - reach;
    if (sim->precision == ORCA_F64)
        k_strip_pack_halo<double><<<grid_for(n, 256), 256, 0, st>>>(
            sim->plan, reinterpret_cast<const double4 *>(sim->pv[sim->cur]),
            reinterpret_cast<const double2 *>(sim->radmax[a]), sim->ids[a], sim->cls[a], le, re, hl,
            hl ? reinterpret_cast<HaloRec<double> *>(hl + 1) : nullptr, hr,
            hr ? reinterpret_cast<HaloRec<double> *>(hr + 1) : nullptr, (int)cap);
    else
        k_strip_pack_halo<float><<<grid_for(n, 256), 256, 0, st>>>(
            sim->plan, reinterpret_cast<const float4 *>(sim->pv[sim->cur]),
            reinterpret_cast<const float2 *>(sim->radmax[a]), sim->ids[a], sim->cls[a], le, re, hl,
            hl ? reinterpret_cast<HaloRec<float> *>(hl + 1) : nullptr, hr,
            hr ? reinterpret_cast<HaloRec<float> *>(hr + 1) : nullptr, (int)cap);
    CKL(sim);
    sim->launches += 1;
    return ORCA_OK;
}

template <typename S> static int strip_append_slab_impl(orca_sim *sim, const void *slab, int64_t cap, int ghost)
{
    typedef typename Vec<S>::T4 S4;
    typedef typename Vec<S>::T2 S2;
    const int a = sim->acur;
    const orca_slab_header *hdr = reinterpret_cast<const orca_slab_header *>(slab);
    cudaStream_t st = sim->stream;
    const int cap_rows = (int)sim->n_bound; // the launch bound: rows beyond it would never be visited
    if (ghost == 1)
        k_strip_append_halo<S><<<grid_for(cap, 256), 256, 0, st>>>(
            sim->plan, hdr, reinterpret_cast<const HaloRec<S> *>(hdr + 1), (int)cap, cap_rows,
            reinterpret_cast<S4 *>(sim->pv[sim->cur]), reinterpret_cast<S4 *>(sim->goalpref[a]),
            reinterpret_cast<S2 *>(sim->radmax[a]), sim->ids[a], sim->cls[a], sim->status[a], sim->failed[a],
            sim->hint[a], sim->lrow[a], sim->a64[a]);
    else
        k_strip_append_slab<S><<<grid_for(cap, 256), 256, 0, st>>>(
            sim->plan, hdr, reinterpret_cast<const orca_agent_record *>(hdr + 1), (int)cap, cap_rows,
            reinterpret_cast<S4 *>(sim->pv[sim->cur]), reinterpret_cast<S4 *>(sim->goalpref[a]),
            reinterpret_cast<S2 *>(sim->radmax[a]), sim->ids[a], sim->cls[a], sim->status[a], sim->failed[a],
            sim->hint[a], sim->lrow[a], sim->a64[a]);
    k_after_append_slab<<<1, 1, 0, st>>>(sim->plan, hdr, (int)cap, cap_rows, ghost);
    CKL(sim);
    sim->launches += 2;
    return ORCA_OK;
}

extern "C" int orca_strip_append_slab(orca_sim *sim, const void *slab, int64_t cap, int ghost)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_append_slab: no resident state");
    if (!sim->strip_on) return fail(sim, ORCA_EINVAL, "orca_strip_append_slab: orca_strip_configure was not called");
    if (!slab || cap < 0 || cap > 0x7FFFFFFF || ghost < 0 || ghost > 2)
        return fail(sim, ORCA_EINVAL, "orca_strip_append_slab: bad arguments");
    if (!ghost && sim->strip_ghosts)
        return fail(sim, ORCA_EINVAL, "orca_strip_append_slab: owned rows cannot follow ghost rows");
    if (cap == 0) return ORCA_OK;
    CK(sim, cudaSetDevice(sim->device));
    int rc = sim->precision == ORCA_F64 ? strip_append_slab_impl<double>(sim, slab, cap, ghost)
                                        : strip_append_slab_impl<float>(sim, slab, cap, ghost);
    if (rc) return rc;
    // the host does not know the count and its launch bound does not move: the device clamps at
    // that bound and raises the sticky overflow flag beyond it (orca_sync -> ORCA_ECAPACITY)
    if (ghost) sim->strip_ghosts = true;
    sim->binned_frame = -1;
    sim->bbox_frame = -1; // rows appended from outside
    return ORCA_OK;
}

extern "C" int orca_strip_step(orca_sim *sim, void *migrants_left, void *migrants_right, int64_t cap)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_step: no resident state");
    if (!sim->have_params) return fail(sim, ORCA_EINVAL, "orca_strip_step: orca_set_params was not called");
    if (!sim->strip_on) return fail(sim, ORCA_EINVAL, "orca_strip_step: orca_strip_configure was not called");
    if (cap < 1 || cap > 0x7FFFFFFF) return fail(sim, ORCA_EINVAL, "orca_strip_step: slab capacity %lld", (long long)cap);
    if (sim->params.compute_metrics)
        return fail(sim, ORCA_EUNSUPPORTED, "orca_strip_step: frame metrics are per handle and would miss the "
                                            "pairs that straddle strips; set compute_metrics = 0");
    CK(sim, cudaSetDevice(sim->device));
    if (migrants_left) CK(sim, cudaMemsetAsync(migrants_left, 0, sizeof(orca_slab_header), sim->stream));
    if (migrants_right) CK(sim, cudaMemsetAsync(migrants_right, 0, sizeof(orca_slab_header), sim->stream));
    sim->mig_slab[0] = migrants_left;
    sim->mig_slab[1] = migrants_right;
    sim->mig_cap = cap;
    const int rc = step_dispatch(sim);
    sim->mig_slab[0] = sim->mig_slab[1] = nullptr;
    sim->mig_cap = 0;
    return rc;
}

// ---- the exchange through peer memory -------------------------------------------------
static inline int64_t window_slot_offset(const orca_sim *sim, int side, int64_t exchange)
{
    return 2 * ORCA_WINDOW_FLAG_BYTES + (int64_t)(side * 2 + (int)(exchange & 1)) * sim->win_stride;
}

extern "C" int orca_strip_window_close(orca_sim *sim)
{
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_strip_window_close: sim is NULL");
    if (!sim->win) return ORCA_OK;
    cudaSetDevice(sim->device);
    if (sim->stream) cudaStreamSynchronize(sim->stream);
    for (int s = 0; s < 2; ++s) {
        if (sim->win_peer[s] && sim->win_peer_ipc[s]) cudaIpcCloseMemHandle(sim->win_peer[s]);
        sim->win_peer[s] = nullptr;
        sim->win_peer_ipc[s] = false;
        sim->win_pushed[s] = sim->win_waited[s] = 0;
    }
    cudaFree(sim->win);
    cudaFree(sim->win_done);
    sim->win = nullptr;
    sim->win_done = nullptr;
    sim->win_side_bytes = sim->win_stride = 0;
    return ORCA_OK;
}

extern "C" int orca_strip_window_create(orca_sim *sim, int64_t side_bytes, void *ipc_handle_out, void **base_out)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_strip_window_create: no resident state");
    if (!sim->strip_on) return fail(sim, ORCA_EINVAL, "orca_strip_window_create: orca_strip_configure was not called");
    if (side_bytes < 2 * (int64_t)sizeof(orca_slab_header) || side_bytes % 16)
        return fail(sim, ORCA_EINVAL, "orca_strip_window_create: side_bytes = %lld", (long long)side_bytes);
    static_assert(sizeof(cudaIpcMemHandle_t) == ORCA_IPC_HANDLE_BYTES, "ORCA_IPC_HANDLE_BYTES");
    int rc = orca_strip_window_close(sim);
    if (rc) return rc;
    CK(sim, cudaSetDevice(sim->device));
    sim->win_side_bytes = side_bytes;
    sim->win_stride = (side_bytes + 255) & ~(int64_t)255;
    const size_t bytes = (size_t)(2 * ORCA_WINDOW_FLAG_BYTES + 4 * sim->win_stride);
    // (plain cudaMalloc: a pooled / virtual-memory allocation cannot be exported as an IPC handle)
    CK(sim, cudaMalloc(reinterpret_cast<void **>(&sim->win), bytes));
    CK(sim, cudaMalloc(reinterpret_cast<void **>(&sim->win_done), sizeof(unsigned)));
    CK(sim, cudaMemsetAsync(sim->win, 0, bytes, sim->stream));
    CK(sim, cudaMemsetAsync(sim->win_done, 0, sizeof(unsigned), sim->stream));
    CK(sim, cudaStreamSynchronize(sim->stream)); // a neighbour may write as soon as it has the handle
    if (const char *e = getenv("ORCA_WINDOW_TIMEOUT_MS")) {
        const long long ms = atoll(e);
        if (ms > 0) sim->win_timeout_ns = (unsigned long long)ms * 1000000ULL;
    }
    if (ipc_handle_out) {
        cudaIpcMemHandle_t h;
        CK(sim, cudaIpcGetMemHandle(&h, sim->win));
        memcpy(ipc_handle_out, &h, sizeof(h));
    }
    if (base_out) *base_out = sim->win;
    return ORCA_OK;
}

extern "C" int orca_strip_window_open(orca_sim *sim, int side, const void *ipc_handle, void *same_process_base)
{
    if (!sim || !sim->win) return fail(sim, ORCA_EINVAL, "orca_strip_window_open: orca_strip_window_create was not called");
    if (side < 0 || side > 1 || (!ipc_handle) == (!same_process_base))
        return fail(sim, ORCA_EINVAL, "orca_strip_window_open: bad arguments");
    if (sim->win_peer[side]) return fail(sim, ORCA_EINVAL, "orca_strip_window_open: side %d is already open", side);
    CK(sim, cudaSetDevice(sim->device));
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        memcpy(&h, ipc_handle, sizeof(h));
        void *p = nullptr;
        CK(sim, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        sim->win_peer[side] = static_cast<unsigned char *>(p);
        sim->win_peer_ipc[side] = true;
    } else {
        // a handle of this process on another device: its memory must be mapped here
        cudaPointerAttributes attr;
        CK(sim, cudaPointerGetAttributes(&attr, same_process_base));
        if (attr.type != cudaMemoryTypeDevice)
            return fail(sim, ORCA_EINVAL, "orca_strip_window_open: same_process_base is not device memory");
        if (attr.device != sim->device) {
            int can = 0;
            CK(sim, cudaDeviceCanAccessPeer(&can, sim->device, attr.device));
            if (!can)
                return fail(sim, ORCA_EUNSUPPORTED, "orca_strip_window_open: device %d cannot map the memory of device %d",
                            sim->device, attr.device);
            const cudaError_t e = cudaDeviceEnablePeerAccess(attr.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(sim, e);
            (void)cudaGetLastError();
        }
        sim->win_peer[side] = static_cast<unsigned char *>(same_process_base);
        sim->win_peer_ipc[side] = false;
    }
    return ORCA_OK;
}

extern "C" int orca_strip_window_push(orca_sim *sim, int side, const void *send, int64_t mig_cap, int64_t halo_cap,
                                      int64_t exchange)
{
    if (!sim || !sim->win) return fail(sim, ORCA_EINVAL, "orca_strip_window_push: no window");
    if (side < 0 || side > 1 || !sim->win_peer[side])
        return fail(sim, ORCA_EINVAL, "orca_strip_window_push: side %d is not open", side);
    if (!send || mig_cap < 0 || halo_cap < 0 || mig_cap > 0x7FFFFFFF || halo_cap > 0x7FFFFFFF)
        return fail(sim, ORCA_EINVAL, "orca_strip_window_push: bad arguments");
    const int64_t rec = orca_strip_halo_record_bytes(sim);
    const int64_t mig_bytes = (int64_t)sizeof(orca_slab_header) + mig_cap * (int64_t)sizeof(orca_agent_record);
    const int64_t halo_bytes = (int64_t)sizeof(orca_slab_header) + halo_cap * rec;
    if (mig_bytes + halo_bytes > sim->win_side_bytes)
        return fail(sim, ORCA_EINVAL, "orca_strip_window_push: slabs of %lld bytes, the windows hold %lld per side",
                    (long long)(mig_bytes + halo_bytes), (long long)sim->win_side_bytes);
    if (exchange != sim->win_pushed[side])
        return fail(sim, ORCA_EINVAL, "orca_strip_window_push: exchange %lld out of order (next is %lld)",
                    (long long)exchange, (long long)sim->win_pushed[side]);
    CK(sim, cudaSetDevice(sim->device));
    // the neighbour sees this strip on its OTHER side
    unsigned char *peer = sim->win_peer[side];
    unsigned char *dst = peer + window_slot_offset(sim, 1 - side, exchange);
    unsigned long long *flag = reinterpret_cast<unsigned long long *>(peer + (1 - side) * ORCA_WINDOW_FLAG_BYTES);
    const int64_t vec = (mig_bytes + halo_bytes) / 16;
    const int blocks = (int)std::min<int64_t>(std::max<int64_t>((vec + 1023) / 1024, 1), (int64_t)296); // (at most two blocks per SM of a B200)
    k_window_push<<<blocks, 256, 0, sim->stream>>>(static_cast<const unsigned char *>(send), dst, (long long)mig_bytes,
                                                   (int)mig_cap, (int)halo_cap, (int)rec, flag,
                                                   (unsigned long long)(exchange + 1), sim->win_done);
    CKL(sim);
    sim->launches += 1;
    sim->win_pushed[side] = exchange + 1;
    return ORCA_OK;
}

extern "C" int orca_strip_window_wait(orca_sim *sim, int side, int64_t exchange, void **slab_out)
{
    if (!sim || !sim->win) return fail(sim, ORCA_EINVAL, "orca_strip_window_wait: no window");
    if (side < 0 || side > 1 || !slab_out) return fail(sim, ORCA_EINVAL, "orca_strip_window_wait: bad arguments");
    if (exchange < sim->win_waited[side] - 1 || exchange > sim->win_waited[side])
        return fail(sim, ORCA_EINVAL, "orca_strip_window_wait: exchange %lld out of order (next is %lld)",
                    (long long)exchange, (long long)sim->win_waited[side]);
    CK(sim, cudaSetDevice(sim->device));
    const unsigned long long *flag = reinterpret_cast<const unsigned long long *>(sim->win + side * ORCA_WINDOW_FLAG_BYTES);
    if (exchange == sim->win_waited[side]) { // (a repeated wait for the last exchange just returns the address)
        k_window_wait<<<1, 1, 0, sim->stream>>>(sim->plan, flag, (unsigned long long)(exchange + 1), sim->win_timeout_ns);
        CKL(sim);
        sim->launches += 1;
        sim->win_waited[side] = exchange + 1;
    }
    *slab_out = sim->win + window_slot_offset(sim, side, exchange);
    return ORCA_OK;
}

extern "C" int orca_strip_stats(orca_sim *sim, int64_t *ghost_rows, int64_t *migrant_rows)
{
    if (!sim) return fail(nullptr, ORCA_EINVAL, "orca_strip_stats: sim is NULL");
    const int rc = fetch_plan(sim);
    if (ghost_rows) *ghost_rows = (int64_t)sim->h_plan->strip_recv[0];
    if (migrant_rows) *migrant_rows = (int64_t)sim->h_plan->strip_recv[1];
    return rc;
}

// ---------------------------------------------------------------------------
// parity taps
// ---------------------------------------------------------------------------

template <typename S, typename R>
static int debug_impl(orca_sim *sim, int64_t n, int64_t *cell_ix, int64_t *cell_iy, int64_t *nb_rows,
                      int64_t *nb_count, double *out_v, int64_t *status, int64_t *failed_at,
                      double *desired_v, bool lists_only = false)
{
    typedef typename Vec<S>::T4 S4;
    typedef typename Vec<R>::T4 R4;
    StepParams P = make_params(sim);
    const int max_n = std::max(P.max_n, 1);
    const size_t need = sizeof(double) * (size_t)n * (size_t)(2 + max_n + 1 + 2 + 2 + 2 + 2);
    if (need > sim->dbg_bytes) {
        cudaFree(sim->dbg);
        sim->dbg = nullptr;
        sim->dbg_bytes = 0;
        CK(sim, cudaMalloc(reinterpret_cast<void **>(&sim->dbg), need));
        sim->dbg_bytes = need;
    }
    cudaStream_t st = sim->stream;
    i64 *d_ix = reinterpret_cast<i64 *>(sim->dbg);
    i64 *d_iy = d_ix + n;
    i64 *d_rows = d_iy + n;
    i64 *d_cnt = d_rows + (size_t)n * max_n;
    double *d_des = reinterpret_cast<double *>(d_cnt + n);
    double *d_pos = d_des + 2 * n;
    double *d_vel = d_pos + 2 * n;
    i64 *d_st = reinterpret_cast<i64 *>(d_vel + 2 * n);
    i64 *d_fa = d_st + n;
    k_debug_rows<S, R><<<grid_for(n, 256), 256, 0, st>>>(
        (int)n, P, reinterpret_cast<const S4 *>(sim->pv[sim->pre]), sim->s_row, sim->nb, sim->nb_cnt,
        reinterpret_cast<const R4 *>(sim->s_dm), d_ix, d_iy, d_rows, d_cnt, d_des, sim->lrow[sim->acur]);
    if (!lists_only) {
        // the un-compacted post-step buffer is pv[(pre+1)%3]
        k_export_pv<S><<<grid_for(n, 256), 256, 0, st>>>(
            (int)n, reinterpret_cast<const S4 *>(sim->pv[(sim->pre + 1) % 3]), d_pos, d_vel, sim->lrow[sim->acur]);
        k_export_i8<<<grid_for(n, 256), 256, 0, st>>>((int)n, sim->status[sim->acur], d_st, sim->lrow[sim->acur]);
        k_export_i8<<<grid_for(n, 256), 256, 0, st>>>((int)n, sim->failed[sim->acur], d_fa, sim->lrow[sim->acur]);
    }
    CKL(sim);
    if (cell_ix) CK(sim, cudaMemcpyAsync(cell_ix, d_ix, sizeof(i64) * n, cudaMemcpyDeviceToHost, st));
    if (cell_iy) CK(sim, cudaMemcpyAsync(cell_iy, d_iy, sizeof(i64) * n, cudaMemcpyDeviceToHost, st));
    if (nb_rows && P.max_n > 0)
        CK(sim, cudaMemcpyAsync(nb_rows, d_rows, sizeof(i64) * n * P.max_n, cudaMemcpyDeviceToHost, st));
    if (nb_count) CK(sim, cudaMemcpyAsync(nb_count, d_cnt, sizeof(i64) * n, cudaMemcpyDeviceToHost, st));
    if (out_v) CK(sim, cudaMemcpyAsync(out_v, d_vel, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
    if (status) CK(sim, cudaMemcpyAsync(status, d_st, sizeof(i64) * n, cudaMemcpyDeviceToHost, st));
    if (failed_at) CK(sim, cudaMemcpyAsync(failed_at, d_fa, sizeof(i64) * n, cudaMemcpyDeviceToHost, st));
    if (desired_v) CK(sim, cudaMemcpyAsync(desired_v, d_des, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
    CK(sim, cudaStreamSynchronize(st));
    return ORCA_OK;
}

extern "C" int orca_debug_last_step(orca_sim *sim, int64_t n, int64_t *cell_ix, int64_t *cell_iy,
                                    int64_t *nb_rows, int64_t *nb_count, double *out_v, int64_t *status,
                                    int64_t *failed_at, double *desired_v)
{
    if (!sim || !sim->loaded) return fail(sim, ORCA_EINVAL, "orca_debug_last_step: no resident state");
    if (sim->params.remove_arrivals || sim->params.compute_metrics)
        return fail(sim, ORCA_EINVAL,
                    "orca_debug_last_step needs remove_arrivals == 0 and compute_metrics == 0");
    if (n != sim->n_pre)
        return fail(sim, ORCA_EINVAL, "orca_debug_last_step: n = %lld, last step had %lld rows", (long long)n,
                    (long long)sim->n_pre);
    CK(sim, cudaSetDevice(sim->device));
    if (n == 0) return ORCA_OK;
    switch (sim->precision) {
    case ORCA_F32:
        return debug_impl<float, float>(sim, n, cell_ix, cell_iy, nb_rows, nb_count, out_v, status, failed_at, desired_v);
    case ORCA_MIXED:
    case ORCA_CERT32:
        return debug_impl<float, double>(sim, n, cell_ix, cell_iy, nb_rows, nb_count, out_v, status, failed_at, desired_v);
    default:
        return debug_impl<double, double>(sim, n, cell_ix, cell_iy, nb_rows, nb_count, out_v, status, failed_at, desired_v);
    }
}

// ---------------------------------------------------------------------------
// batched LP
// ---------------------------------------------------------------------------

struct orca_lp_batch {
    int device = 0, precision = ORCA_F32;
    int64_t n = 0, m = 0;
    cudaStream_t stream = nullptr, own_stream = nullptr;
    i64 *coff = nullptr;
    void *cons = nullptr, *prob = nullptr, *proj = nullptr;
    u64 *seeds = nullptr;
    int *perm = nullptr;
    double *out_v = nullptr;
    i64 *out_status = nullptr, *out_failed = nullptr;
    int *fq = nullptr, *fq_count = nullptr; // problems queued for the least-penetration stage
    void *fq_state = nullptr;
};

extern "C" void orca_lp_batch_destroy(orca_lp_batch *b)
{
    if (!b) return;
    cudaSetDevice(b->device);
    if (b->stream) cudaStreamSynchronize(b->stream);
    cudaFree(b->coff);
    cudaFree(b->cons);
    cudaFree(b->prob);
    cudaFree(b->proj);
    cudaFree(b->seeds);
    cudaFree(b->perm);
    cudaFree(b->out_v);
    cudaFree(b->out_status);
    cudaFree(b->out_failed);
    cudaFree(b->fq);
    cudaFree(b->fq_count);
    cudaFree(b->fq_state);
    if (b->own_stream) cudaStreamDestroy(b->own_stream);
    delete b;
}

template <typename R>
static cudaError_t lp_pack(orca_lp_batch *b, const double *cpts, const double *cnrm, const double *tgt,
                           const double *caps)
{
    typedef typename Vec<R>::T4 R4;
    cudaError_t e;
    double *tmp = nullptr;
    const size_t m = (size_t)b->m, n = (size_t)b->n;
    const size_t words = std::max<size_t>(4 * m, 3 * n);
    if ((e = cudaMalloc(reinterpret_cast<void **>(&tmp), sizeof(double) * std::max<size_t>(words, 1))) != cudaSuccess) return e;
    cudaStream_t st = b->stream;
    if (m) {
        cudaMemcpyAsync(tmp, cpts, sizeof(double) * 2 * m, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(tmp + 2 * m, cnrm, sizeof(double) * 2 * m, cudaMemcpyHostToDevice, st);
        k_lp_pack<R><<<grid_for((int64_t)m, 256), 256, 0, st>>>((i64)m, tmp, tmp + 2 * m,
                                                               reinterpret_cast<R4 *>(b->cons));
    }
    cudaStreamSynchronize(st);
    if (n) {
        cudaMemcpyAsync(tmp, tgt, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(tmp + 2 * n, caps, sizeof(double) * n, cudaMemcpyHostToDevice, st);
        k_lp_pack_problems<R><<<grid_for((int64_t)n, 256), 256, 0, st>>>((i64)n, tmp, tmp + 2 * n,
                                                                        reinterpret_cast<R4 *>(b->prob));
    }
    e = cudaStreamSynchronize(st);
    cudaFree(tmp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

extern "C" int orca_lp_batch_create(orca_lp_batch **out, int device, int precision, int64_t n,
                                    const int64_t *coff, const double *cpts, const double *cnrm,
                                    const double *tgt, const double *caps, const uint64_t *seeds)
{
    if (!out) return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_create: out is NULL");
    *out = nullptr;
    if (n < 0 || !coff || (n > 0 && (!tgt || !caps || !seeds)))
        return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_create: bad arguments");
    if (precision != ORCA_F32 && precision != ORCA_F64)
        return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_create: precision must be ORCA_F32 or ORCA_F64, got %d", precision);
    if (coff[0] != 0) return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_create: coff[0] must be 0");
    for (int64_t i = 0; i < n; ++i)
        if (coff[i + 1] < coff[i])
            return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_create: coff is not non-decreasing at %lld", (long long)i);
    const int64_t m = coff[n];
    if (m > 0 && (!cpts || !cnrm)) return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_create: NULL constraints");
    int ndev = 0;
    CK(nullptr, cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_create: device %d not available", device);
    CK(nullptr, cudaSetDevice(device));
    orca_lp_batch *b = new (std::nothrow) orca_lp_batch();
    if (!b) return fail(nullptr, ORCA_EINVAL, "out of host memory");
    b->device = device;
    b->precision = precision;
    b->n = n;
    b->m = m;
    const size_t rs = precision == ORCA_F32 ? sizeof(float) : sizeof(double);
    const size_t nn = (size_t)std::max<int64_t>(n, 1), mm = (size_t)std::max<int64_t>(m, 1);
#define CKB(call)                                                                                 \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            int rc_ = fail(nullptr, ORCA_ECUDA, "orca_lp_batch_create: %s: %s", #call, cudaGetErrorString(e_)); \
            orca_lp_batch_destroy(b);                                                             \
            return rc_;                                                                           \
        }                                                                                         \
    } while (0)
    CKB(cudaStreamCreateWithFlags(&b->own_stream, cudaStreamNonBlocking));
    b->stream = b->own_stream;
    CKB(dalloc(&b->coff, nn + 1));
    CKB(cudaMalloc(&b->cons, mm * 4 * rs));
    CKB(cudaMalloc(&b->prob, nn * 4 * rs));
    CKB(cudaMalloc(&b->proj, mm * 4 * rs));
    CKB(dalloc(&b->seeds, nn));
    CKB(dalloc(&b->perm, mm));
    CKB(dalloc(&b->out_v, 2 * nn));
    CKB(dalloc(&b->out_status, nn));
    CKB(dalloc(&b->out_failed, nn));
    CKB(dalloc(&b->fq, nn));
    CKB(dalloc(&b->fq_count, 1));
    CKB(cudaMalloc(&b->fq_state, nn * 4 * rs));
    CKB(cudaMemcpyAsync(b->coff, coff, sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, b->stream));
    if (n) CKB(cudaMemcpyAsync(b->seeds, seeds, sizeof(u64) * n, cudaMemcpyHostToDevice, b->stream));
    CKB(precision == ORCA_F32 ? lp_pack<float>(b, cpts, cnrm, tgt, caps) : lp_pack<double>(b, cpts, cnrm, tgt, caps));
#undef CKB
    *out = b;
    return ORCA_OK;
}

extern "C" int orca_lp_batch_set_stream(orca_lp_batch *b, void *cuda_stream)
{
    if (!b) return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_set_stream: NULL batch");
    CK(nullptr, cudaSetDevice(b->device));
    CK(nullptr, cudaStreamSynchronize(b->stream));
    b->stream = cuda_stream ? reinterpret_cast<cudaStream_t>(cuda_stream) : b->own_stream;
    return ORCA_OK;
}

extern "C" int orca_lp_batch_solve(orca_lp_batch *b)
{
    if (!b) return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_solve: NULL batch");
    CK(nullptr, cudaSetDevice(b->device));
    if (b->n == 0) return ORCA_OK;
    if (b->n > 0x7FFFFFFF) return fail(nullptr, ORCA_EUNSUPPORTED, "orca_lp_batch_solve: more than 2^31-1 problems");
    CK(nullptr, cudaMemsetAsync(b->fq_count, 0, sizeof(int), b->stream));
    const int fb_ng = 128 / ORCA_LP_GL; // problems per block and pass
    const int fb_blocks = (int)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (b->n + fb_ng - 1) / fb_ng));
    if (b->precision == ORCA_F32) {
        k_lp_batch<float><<<grid_for(b->n, 128), 128, 0, b->stream>>>(
            b->n, b->coff, reinterpret_cast<const float4 *>(b->cons), reinterpret_cast<const float4 *>(b->prob),
            b->seeds, b->perm, b->out_v, b->out_status, b->out_failed, b->fq_count, b->fq,
            reinterpret_cast<float4 *>(b->fq_state));
        k_lp_batch_fallback<float><<<fb_blocks, 128, 0, b->stream>>>(
            b->fq_count, b->fq, reinterpret_cast<const float4 *>(b->fq_state), b->coff,
            reinterpret_cast<const float4 *>(b->cons), reinterpret_cast<const float4 *>(b->prob), b->perm,
            reinterpret_cast<float4 *>(b->proj), b->out_v);
    } else {
        k_lp_batch<double><<<grid_for(b->n, 128), 128, 0, b->stream>>>(
            b->n, b->coff, reinterpret_cast<const double4 *>(b->cons), reinterpret_cast<const double4 *>(b->prob),
            b->seeds, b->perm, b->out_v, b->out_status, b->out_failed, b->fq_count, b->fq,
            reinterpret_cast<double4 *>(b->fq_state));
        k_lp_batch_fallback<double><<<fb_blocks, 128, 0, b->stream>>>(
            b->fq_count, b->fq, reinterpret_cast<const double4 *>(b->fq_state), b->coff,
            reinterpret_cast<const double4 *>(b->cons), reinterpret_cast<const double4 *>(b->prob), b->perm,
            reinterpret_cast<double4 *>(b->proj), b->out_v);
    }
    CKL(nullptr);
    return ORCA_OK;
}

extern "C" int orca_lp_batch_download(orca_lp_batch *b, double *out_v, int64_t *out_status, int64_t *out_failed)
{
    if (!b) return fail(nullptr, ORCA_EINVAL, "orca_lp_batch_download: NULL batch");
    CK(nullptr, cudaSetDevice(b->device));
    const size_t n = (size_t)b->n;
    if (n) {
        if (out_v) CK(nullptr, cudaMemcpyAsync(out_v, b->out_v, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, b->stream));
        if (out_status) CK(nullptr, cudaMemcpyAsync(out_status, b->out_status, sizeof(i64) * n, cudaMemcpyDeviceToHost, b->stream));
        if (out_failed) CK(nullptr, cudaMemcpyAsync(out_failed, b->out_failed, sizeof(i64) * n, cudaMemcpyDeviceToHost, b->stream));
    }
    CK(nullptr, cudaStreamSynchronize(b->stream));
    return ORCA_OK;
}

// Scratch of the one-shot batched LP, kept between calls (grow-only, per process): allocating
// and freeing ~3 GB of device memory per call costs 10-100 ms, several times the solve itself.
// orca_lp_release_scratch() gives it back.
struct LpScratch {
    int device = -1;
    static constexpr int SLOTS = 14;
    void *ptr[SLOTS] = {};
    size_t bytes[SLOTS] = {};
    cudaStream_t st[2] = {nullptr, nullptr};
    void release()
    {
        if (device < 0) return;
        cudaSetDevice(device);
        for (int i = 0; i < SLOTS; ++i) {
            cudaFree(ptr[i]);
            ptr[i] = nullptr;
            bytes[i] = 0;
        }
        for (int i = 0; i < 2; ++i) {
            if (st[i]) cudaStreamDestroy(st[i]);
            st[i] = nullptr;
        }
        device = -1;
    }
    cudaError_t get(int slot, size_t need, void **out)
    {
        if (bytes[slot] < need) {
            cudaFree(ptr[slot]);
            ptr[slot] = nullptr;
            bytes[slot] = 0;
            const size_t grow = need + need / 8; // a little room so near-equal batches reuse it
            cudaError_t e = cudaMalloc(&ptr[slot], std::max<size_t>(grow, 256));
            if (e != cudaSuccess) return e;
            bytes[slot] = std::max<size_t>(grow, 256);
        }
        *out = ptr[slot];
        return cudaSuccess;
    }
};
static LpScratch g_lp_scratch;
static pthread_mutex_t g_lp_mutex = PTHREAD_MUTEX_INITIALIZER;

extern "C" int orca_lp_release_scratch(void)
{
    pthread_mutex_lock(&g_lp_mutex);
    g_lp_scratch.release();
    pthread_mutex_unlock(&g_lp_mutex);
    return ORCA_OK;
}

// One-shot solve of a host batch, PIPELINED: the constraints of a 1 M-problem batch are 1.2 GB of
// float64 that cross PCIe once per call (~23 ms), against 2-12 ms of solving. The batch is cut into
// chunks of problems; per chunk -- alternating between two streams, each with its own staging
// area -- the constraints and problems go up, are packed and solved (k_lp_batch + its fallback,
// with the chunk's own queue and counter), so the copies of one chunk run under the kernels of the
// other; the results (32 B per problem) come down at the end. With pinned host arrays the call is
// PCIe-bound (measured 26-32 ms for 1,048,576 problems / 37.7 M constraints).
template <typename R>
static int lp_solve_pipelined(int device, int64_t n, int64_t m, int64_t kmax, const int64_t *coff, const double *cpts,
                              const double *cnrm, const double *tgt, const double *caps, const uint64_t *seeds,
                              double *out_v, int64_t *out_status, int64_t *out_failed)
{
    typedef typename Vec<R>::T4 R4;
    const int64_t pn = std::max<int64_t>(8192, (n + 23) / 24); // problems per chunk
    const int nchunks = (int)((n + pn - 1) / pn);
    int64_t cm = 0; // most constraints in one chunk
    for (int c = 0; c < nchunks; ++c) {
        const int64_t p0 = c * pn, p1 = std::min<int64_t>(n, p0 + pn);
        cm = std::max<int64_t>(cm, coff[p1] - coff[p0]);
    }
    LpScratch &S = g_lp_scratch;
    if (S.device != device) {
        S.release();
        S.device = device;
    }
    i64 *d_coff = nullptr;
    R4 *d_cons = nullptr, *d_prob = nullptr, *d_proj = nullptr, *d_fqs = nullptr;
    u64 *d_seeds = nullptr;
    int *d_perm = nullptr, *d_fq = nullptr, *d_fqc = nullptr;
    double *d_out = nullptr, *d_stg[2] = {nullptr, nullptr};
    i64 *d_st = nullptr, *d_fa = nullptr;
    const size_t mm = (size_t)std::max<int64_t>(m, 1), nn = (size_t)n;
    const size_t stg_words = (size_t)(4 * std::max<int64_t>(cm, 1) + 3 * pn);
    cudaError_t e = cudaSuccess;
#define LPK(call)                                                                                 \
    do {                                                                                          \
        if (e == cudaSuccess) e = (call);                                                         \
    } while (0)
#define LPG(slot, p, count) LPK(S.get(slot, sizeof(*(p)) * (count), reinterpret_cast<void **>(&(p))))
    LPG(0, d_coff, nn + 1);
    LPG(1, d_cons, mm);
    LPG(2, d_prob, nn);
    LPG(3, d_seeds, nn);
    LPG(4, d_perm, mm);
    if (kmax > LP_SMEM_K) LPG(5, d_proj, mm); // only problems too large for shared memory use it
    LPG(6, d_out, 2 * nn);
    LPG(7, d_st, nn);
    LPG(8, d_fa, nn);
    LPG(9, d_fq, nn);
    LPG(10, d_fqs, nn);
    LPG(11, d_fqc, (size_t)nchunks);
    LPG(12, d_stg[0], stg_words);
    LPG(13, d_stg[1], stg_words);
#undef LPG
    for (int i = 0; i < 2; ++i)
        if (!S.st[i]) LPK(cudaStreamCreateWithFlags(&S.st[i], cudaStreamNonBlocking));
    LPK(cudaMemset(d_fqc, 0, sizeof(int) * nchunks));
    LPK(cudaMemcpy(d_coff, coff, sizeof(i64) * (nn + 1), cudaMemcpyHostToDevice));
    const int fb_ng = 128 / ORCA_LP_GL;
    for (int c = 0; c < nchunks && e == cudaSuccess; ++c) {
        cudaStream_t s = S.st[c & 1];
        double *stg = d_stg[c & 1];
        const int64_t p0 = c * pn, p1 = std::min<int64_t>(n, p0 + pn), cnt = p1 - p0;
        const int64_t lo = coff[p0], hi = coff[p1], cc = hi - lo;
        if (cc > 0) {
            LPK(cudaMemcpyAsync(stg, cpts + 2 * lo, sizeof(double) * 2 * cc, cudaMemcpyHostToDevice, s));
            LPK(cudaMemcpyAsync(stg + 2 * cc, cnrm + 2 * lo, sizeof(double) * 2 * cc, cudaMemcpyHostToDevice, s));
            k_lp_pack<R><<<grid_for(cc, 256), 256, 0, s>>>((i64)cc, stg, stg + 2 * cc, d_cons + lo);
        }
        double *sp = stg + 4 * std::max<int64_t>(cm, 1);
        LPK(cudaMemcpyAsync(sp, tgt + 2 * p0, sizeof(double) * 2 * cnt, cudaMemcpyHostToDevice, s));
        LPK(cudaMemcpyAsync(sp + 2 * cnt, caps + p0, sizeof(double) * cnt, cudaMemcpyHostToDevice, s));
        k_lp_pack_problems<R><<<grid_for(cnt, 256), 256, 0, s>>>((i64)cnt, sp, sp + 2 * cnt, d_prob + p0);
        LPK(cudaMemcpyAsync(d_seeds + p0, seeds + p0, sizeof(u64) * cnt, cudaMemcpyHostToDevice, s));
        k_lp_batch<R><<<grid_for(cnt, 128), 128, 0, s>>>(cnt, d_coff + p0, d_cons, d_prob + p0, d_seeds + p0, d_perm,
                                                        d_out + 2 * p0, d_st + p0, d_fa + p0, d_fqc + c, d_fq + p0,
                                                        d_fqs + p0);
        const int fb_blocks = (int)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (cnt + fb_ng - 1) / fb_ng));
        k_lp_batch_fallback<R><<<fb_blocks, 128, 0, s>>>(d_fqc + c, d_fq + p0, d_fqs + p0, d_coff + p0, d_cons,
                                                        d_prob + p0, d_perm, d_proj, d_out + 2 * p0);
        LPK(cudaGetLastError());
    }
    for (int i = 0; i < 2; ++i)
        if (S.st[i]) {
            const cudaError_t es = cudaStreamSynchronize(S.st[i]);
            if (e == cudaSuccess) e = es;
        }
    // the results come down in one go: a copy into PAGEABLE host memory blocks the host, and issued
    // per chunk it would serialise the pipeline
    LPK(cudaMemcpy(out_v, d_out, sizeof(double) * 2 * nn, cudaMemcpyDeviceToHost));
    LPK(cudaMemcpy(out_status, d_st, sizeof(i64) * nn, cudaMemcpyDeviceToHost));
    LPK(cudaMemcpy(out_failed, d_fa, sizeof(i64) * nn, cudaMemcpyDeviceToHost));
#undef LPK
    CK(nullptr, e);
    return ORCA_OK;
}

extern "C" int orca_lp_solve_batch(int device, int precision, int64_t n, const int64_t *coff,
                                   const double *cpts, const double *cnrm, const double *tgt,
                                   const double *caps, const uint64_t *seeds, double *out_v,
                                   int64_t *out_status, int64_t *out_failed)
{
    if (n < 0 || !coff || (n > 0 && (!tgt || !caps || !seeds || !out_v || !out_status || !out_failed)))
        return fail(nullptr, ORCA_EINVAL, "orca_lp_solve_batch: bad arguments");
    if (precision != ORCA_F32 && precision != ORCA_F64)
        return fail(nullptr, ORCA_EINVAL, "orca_lp_solve_batch: precision must be ORCA_F32 or ORCA_F64, got %d", precision);
    if (n > 0x7FFFFFFF) return fail(nullptr, ORCA_EUNSUPPORTED, "orca_lp_solve_batch: more than 2^31-1 problems");
    if (coff[0] != 0) return fail(nullptr, ORCA_EINVAL, "orca_lp_solve_batch: coff[0] must be 0");
    int64_t kmax = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (coff[i + 1] < coff[i])
            return fail(nullptr, ORCA_EINVAL, "orca_lp_solve_batch: coff is not non-decreasing at %lld", (long long)i);
        kmax = std::max(kmax, coff[i + 1] - coff[i]);
    }
    const int64_t m = coff[n];
    if (m > 0 && (!cpts || !cnrm)) return fail(nullptr, ORCA_EINVAL, "orca_lp_solve_batch: NULL constraints");
    if (n == 0) return ORCA_OK;
    int ndev = 0;
    CK(nullptr, cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(nullptr, ORCA_EINVAL, "orca_lp_solve_batch: device %d not available", device);
    CK(nullptr, cudaSetDevice(device));
    pthread_mutex_lock(&g_lp_mutex); // one scratch per process
    const int rc = precision == ORCA_F32
                       ? lp_solve_pipelined<float>(device, n, m, kmax, coff, cpts, cnrm, tgt, caps, seeds, out_v, out_status, out_failed)
                       : lp_solve_pipelined<double>(device, n, m, kmax, coff, cpts, cnrm, tgt, caps, seeds, out_v, out_status, out_failed);
    pthread_mutex_unlock(&g_lp_mutex);
    return rc;
}

// ---------------------------------------------------------------------------
// single-op taps
// ---------------------------------------------------------------------------

extern "C" int orca_vo_exit_batch(int device, int precision, int64_t count, const double *in7, double *out5)
{
    if (count < 0 || (count > 0 && (!in7 || !out5))) return fail(nullptr, ORCA_EINVAL, "orca_vo_exit_batch: bad arguments");
    if (count == 0) return ORCA_OK;
    CK(nullptr, cudaSetDevice(device));
    double *d_in = nullptr, *d_out = nullptr;
    CK(nullptr, cudaMalloc(reinterpret_cast<void **>(&d_in), sizeof(double) * 7 * count));
    CK(nullptr, cudaMalloc(reinterpret_cast<void **>(&d_out), sizeof(double) * 5 * count));
    CK(nullptr, cudaMemcpy(d_in, in7, sizeof(double) * 7 * count, cudaMemcpyHostToDevice));
    if (precision == ORCA_F32) k_vo_exit_batch<float><<<grid_for(count, 128), 128>>>(count, d_in, d_out);
    else k_vo_exit_batch<double><<<grid_for(count, 128), 128>>>(count, d_in, d_out);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out5, d_out, sizeof(double) * 5 * count, cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
    CK(nullptr, e);
    return ORCA_OK;
}

extern "C" int orca_least_penetration(int device, int precision, int64_t k, const double *cpts,
                                      const double *cnrm, double speed_cap, int64_t start_index, double wx,
                                      double wy, double *out_v)
{
    if (k < 0 || k > 0x3FFFFFFF || (k > 0 && (!cpts || !cnrm)) || !out_v || start_index < 0 || start_index > k)
        return fail(nullptr, ORCA_EINVAL, "orca_least_penetration: bad arguments");
    if (precision != ORCA_F32 && precision != ORCA_F64)
        return fail(nullptr, ORCA_EINVAL, "orca_least_penetration: precision must be ORCA_F32 or ORCA_F64");
    CK(nullptr, cudaSetDevice(device));
    const size_t kk = (size_t)std::max<int64_t>(k, 1);
    const size_t rs = precision == ORCA_F32 ? sizeof(float) : sizeof(double);
    double *d_in = nullptr, *d_out = nullptr;
    void *d_cons = nullptr, *d_proj = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&d_in), sizeof(double) * 4 * kk);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&d_out), sizeof(double) * 2);
    if (e == cudaSuccess) e = cudaMalloc(&d_cons, 4 * rs * kk);
    if (e == cudaSuccess) e = cudaMalloc(&d_proj, 4 * rs * kk);
    if (e == cudaSuccess && k > 0) e = cudaMemcpy(d_in, cpts, sizeof(double) * 2 * k, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && k > 0) e = cudaMemcpy(d_in + 2 * k, cnrm, sizeof(double) * 2 * k, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        if (precision == ORCA_F32) {
            if (k > 0) k_lp_pack<float><<<grid_for(k, 256), 256>>>((i64)k, d_in, d_in + 2 * k, reinterpret_cast<float4 *>(d_cons));
            k_least_penetration_tap<float><<<1, 1>>>((int)k, (int)start_index, reinterpret_cast<const float4 *>(d_cons),
                                                     reinterpret_cast<float4 *>(d_proj), speed_cap, wx, wy, d_out);
        } else {
            if (k > 0) k_lp_pack<double><<<grid_for(k, 256), 256>>>((i64)k, d_in, d_in + 2 * k, reinterpret_cast<double4 *>(d_cons));
            k_least_penetration_tap<double><<<1, 1>>>((int)k, (int)start_index, reinterpret_cast<const double4 *>(d_cons),
                                                      reinterpret_cast<double4 *>(d_proj), speed_cap, wx, wy, d_out);
        }
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out_v, d_out, sizeof(double) * 2, cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_cons);
    cudaFree(d_proj);
    CK(nullptr, e);
    return ORCA_OK;
}

extern "C" int orca_neighbor_query(int device, int64_t n, const int64_t *ids, const double *positions,
                                   double radius, int32_t max_count, int64_t *out_rows, int64_t *out_count)
{
    if (n < 0 || (n > 0 && (!ids || !positions || !out_count || (max_count > 0 && !out_rows))))
        return fail(nullptr, ORCA_EINVAL, "orca_neighbor_query: bad arguments");
    if (!(radius > 0.0) || !std::isfinite(radius))
        return fail(nullptr, ORCA_EINVAL, "radius must be positive, got %g", radius);
    if (max_count < 0) return fail(nullptr, ORCA_EINVAL, "max_count must be >= 0, got %d", max_count);
    if (max_count > ORCA_MAX_NEIGHBORS)
        return fail(nullptr, ORCA_EUNSUPPORTED, "max_count %d exceeds ORCA_MAX_NEIGHBORS (%d)", max_count,
                    ORCA_MAX_NEIGHBORS);
    if (n == 0) return ORCA_OK;
    orca_sim *sim = nullptr;
    int rc = orca_create(&sim, device, n, ORCA_F64);
    if (rc) return rc;
    orca_params p{};
    p.dt = 1.0;
    p.tau = 1.0;
    p.neighbor_radius = radius;
    p.max_neighbors = max_count;
    rc = orca_set_params(sim, &p);
    if (!rc) {
        // only positions and ids matter to the search; the other attributes get placeholders
        std::vector<double> zeros((size_t)2 * n, 0.0), ones((size_t)n, 1.0);
        std::vector<int64_t> cls((size_t)n, 0);
        rc = orca_upload(sim, n, 0, ids, positions, zeros.data(), ones.data(), ones.data(), ones.data(), positions,
                         ones.data(), cls.data());
        if (!rc) rc = orca_sync(sim); // the uploads read the host vectors asynchronously
    }
    if (!rc) {
        const StepParams P = make_params(sim);
        rc = bin_build<double, double>(sim, P);
        if (!rc)
            rc = max_count <= 16 ? gather_stage<double, 16>(sim, P, sim->stream, 0, (int)n, 0)
                                 : gather_stage<double, 32>(sim, P, sim->stream, 0, (int)n, 0);
        sim->pre = sim->cur;
        sim->n_pre = n;
        if (!rc) rc = debug_impl<double, double>(sim, n, nullptr, nullptr, out_rows, out_count, nullptr, nullptr,
                                                 nullptr, nullptr, /*lists_only=*/true);
        if (!rc) rc = fetch_plan(sim); // range error of a position (engine.py:152-153)
    }
    if (rc) memcpy(g_err, sim->err, sizeof(g_err));
    orca_destroy(sim);
    return rc;
}

extern "C" int orca_neighbor_query_all(int device, int64_t n, const int64_t *ids, const double *positions,
                                       double radius, int64_t cap, int64_t *out_offsets, int64_t *out_rows,
                                       int64_t *total_out)
{
    if (n < 0 || cap < 0 || !total_out || (n > 0 && (!ids || !positions || !out_offsets)) || (cap > 0 && !out_rows))
        return fail(nullptr, ORCA_EINVAL, "orca_neighbor_query_all: bad arguments");
    if (!(radius > 0.0) || !std::isfinite(radius))
        return fail(nullptr, ORCA_EINVAL, "radius must be positive, got %g", radius);
    *total_out = 0;
    if (out_offsets) out_offsets[0] = 0;
    if (n == 0) return ORCA_OK;
    orca_sim *sim = nullptr;
    int rc = orca_create(&sim, device, n, ORCA_F64);
    if (rc) return rc;
    orca_params p{};
    p.dt = 1.0;
    p.tau = 1.0;
    p.neighbor_radius = radius;
    p.max_neighbors = 1; // (sizes the search grid only; the lists of this query have no cap)
    rc = orca_set_params(sim, &p);
    if (!rc) {
        std::vector<double> zeros((size_t)2 * n, 0.0), ones((size_t)n, 1.0);
        std::vector<int64_t> cls((size_t)n, 0);
        rc = orca_upload(sim, n, 0, ids, positions, zeros.data(), ones.data(), ones.data(), ones.data(), positions,
                         ones.data(), cls.data());
        if (!rc) rc = orca_sync(sim);
    }
    double *d_keys = nullptr;
    i64 *d_rows = nullptr;
    std::vector<int> off;
    if (!rc) {
        const StepParams P = make_params(sim);
        rc = bin_build<double, double>(sim, P);
        cudaStream_t st = sim->stream;
        const dim3 blocks = grid_for(n + 1, 128);
        const double2 *xy = reinterpret_cast<const double2 *>(sim->s_xy);
        const i64 *d_ids = sim->ids[sim->acur];
        if (!rc) {
            k_neighbors_all<0><<<blocks, 128, 0, st>>>(sim->plan, P.rad2, xy, sim->cell_start, sim->s_cell, sim->s_row,
                                                       d_ids, sim->sel, nullptr, nullptr, nullptr);
            const int scan_blocks = (int)((n + 1 + SCAN_TILE - 1) / SCAN_TILE);
            k_scan_reduce<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->sel, sim->block_sums);
            k_scan_top<<<1, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->block_sums);
            k_scan_apply<<<scan_blocks, SCAN_THREADS, 0, st>>>(&sim->plan->n, 1, sim->sel, sim->block_sums, sim->sel_idx);
            off.resize((size_t)n + 1);
            cudaError_t e = cudaGetLastError();
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(off.data(), sim->sel_idx, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) rc = fail(sim, ORCA_ECUDA, "orca_neighbor_query_all: %s", cudaGetErrorString(e));
        }
        if (!rc) rc = fetch_plan(sim); // range error of a position (engine.py:152-153)
        if (!rc) {
            const int64_t total = off[(size_t)n];
            *total_out = total;
            for (int64_t i = 0; i <= n; ++i) out_offsets[i] = off[(size_t)i];
            if (total > cap)
                rc = fail(sim, ORCA_ECAPACITY, "orca_neighbor_query_all: %lld neighbour entries, the buffer holds %lld",
                          (long long)total, (long long)cap);
            else if (total > 0) {
                cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&d_keys), sizeof(double) * total);
                if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&d_rows), sizeof(i64) * total);
                if (e == cudaSuccess) {
                    k_neighbors_all<1><<<blocks, 128, 0, st>>>(sim->plan, P.rad2, xy, sim->cell_start, sim->s_cell,
                                                               sim->s_row, d_ids, nullptr, sim->sel_idx, d_keys, d_rows);
                    e = cudaGetLastError();
                }
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(out_rows, d_rows, sizeof(i64) * total, cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) rc = fail(sim, ORCA_ECUDA, "orca_neighbor_query_all: %s", cudaGetErrorString(e));
            }
        }
    }
    cudaFree(d_keys);
    cudaFree(d_rows);
    if (rc) memcpy(g_err, sim->err, sizeof(g_err));
    orca_destroy(sim);
    return rc;
}

extern "C" int orca_shuffle_order(int device, int64_t k, uint64_t seed, int64_t *perm)
{
    if (k < 0 || (k > 0 && !perm)) return fail(nullptr, ORCA_EINVAL, "orca_shuffle_order: bad arguments");
    if (k == 0) return ORCA_OK;
    CK(nullptr, cudaSetDevice(device));
    i64 *d = nullptr;
    CK(nullptr, cudaMalloc(reinterpret_cast<void **>(&d), sizeof(i64) * k));
    // k <= 32 exercises the unrolled shuffle of the step kernels, larger k the batch-LP one
    if (k <= 32) k_shuffle_tap_smem<<<1, 32>>>((int)k, seed, d);
    else k_shuffle_tap<<<1, 1>>>((int)k, seed, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(perm, d, sizeof(i64) * k, cudaMemcpyDeviceToHost);
    cudaFree(d);
    CK(nullptr, e);
    return ORCA_OK;
}

extern "C" int orca_problem_seed(int device, int64_t frame, int64_t agent_id, uint64_t *seed)
{
    if (!seed) return fail(nullptr, ORCA_EINVAL, "orca_problem_seed: seed is NULL");
    CK(nullptr, cudaSetDevice(device));
    u64 *d = nullptr;
    CK(nullptr, cudaMalloc(reinterpret_cast<void **>(&d), sizeof(u64)));
    k_seed_tap<<<1, 1>>>(frame, agent_id, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(seed, d, sizeof(u64), cudaMemcpyDeviceToHost);
    cudaFree(d);
    CK(nullptr, e);
    return ORCA_OK;
}

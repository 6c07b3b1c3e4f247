/*
 * orca_b200.h -- C ABI of the B200-native ORCA steering step (arXiv 2008.11578).
 *
 * This is the drop-in boundary for the ONE path this repository accelerates:
 * the per-frame step of the reference simulator,
 *
 *     engine._advance            pkg/src/orcasim/engine.py:194-295
 *       _grid_arrays             engine.py:149-161
 *       _desired_velocities      engine.py:133-139
 *       frame_solve_range        pkg/src/orcasim/_kernels.py:493-556
 *       new_pos = pos + v*dt     engine.py:249, arrivals engine.py:251-255
 *       min_sep_range            _kernels.py:559-589 (metrics, engine.py:270-286)
 *     solve_range                _kernels.py:306-336 (batched LP entry)
 *
 * The reference is pure Python + numba and has no FFI layer; the seam a
 * maintainer would bind is the flat-array signature of frame_solve_range /
 * solve_range and the SimState arrays of engine.py:55-74. Every entry point
 * takes plain pointers and sizes (no torch types). Host arrays use the
 * reference's own dtypes and layouts (float64 / int64, [n,2] row-major) so a
 * ctypes / cffi binding passes numpy buffers straight through; see
 * INTEGRATION.md for the stub.
 *
 * Conventions
 *   - Every function returns 0 on success and a negative ORCA_E* code on
 *     failure; orca_last_error() returns the message of the last failure on
 *     that handle (or of the last handle-less call on this thread).
 *   - A handle owns its device buffers and is bound to one CUDA device and one
 *     stream. A handle is not thread-safe; distinct handles are independent.
 *   - orca_step / orca_run are asynchronous with respect to the host; errors
 *     raised by device code (coincident centres, grid range) are sticky and
 *     surface at the next orca_sync / orca_download / orca_get_info.
 *   - Every array that crosses this boundary is in the reference's storage-row
 *     order (engine.py:56-74; compaction keeps the survivors' order,
 *     engine.py:288-294). The handle keeps its rows in cell-sorted order
 *     internally and maps them back (orca_reorder_rows).
 *   - precision (cell indices and neighbour-ordering keys are FP64 in every
 *     mode, so bins and neighbour lists are bit-exact whenever the inputs are
 *     representable in the storage type):
 *       ORCA_MIXED  FP32 device state (float4 SoA), FP64 arithmetic with no FMA
 *                   contraction for desired velocity, ORCA half-planes, LP and
 *                   integration. For float32-representable inputs the solver
 *                   takes exactly the reference's branches and the results are
 *                   the reference's, rounded once to FP32 on store.
 *       ORCA_F32    FP32 state and FP32 arithmetic: fastest; velocities agree
 *                   with the reference to ~1e-7 m/s typically, but ill-conditioned
 *                   LPs (dense crowds in the fallback stage) can differ by more
 *                   than 1e-4 m/s -- counted and reported by the parity tests.
 *       ORCA_F64    FP64 state and arithmetic: bit-identical to the reference on
 *                   any float64 input. What the reference-shaped host entry points
 *                   (engine.step / run, the CLI) use unless told otherwise.
 *       ORCA_CERT32 the results of ORCA_MIXED, faster: the half-planes and the LP run in
 *                   FP32 only to find which (at most two) half-planes decide the result;
 *                   the result itself is evaluated in FP64 on those, and accepted only
 *                   with a certificate (feasibility and optimality margins above the FP32
 *                   error bounds, csrc/orca_cert.cuh). Everything else -- infeasible LPs,
 *                   thin margins -- goes through the FP64 kernels of ORCA_MIXED, and so do
 *                   whole crowds for which the certified pass would not pay (fewer than
 *                   65,536 agents, or a quarter of the LPs infeasible at the last count).
 */
#ifndef ORCA_B200_H
#define ORCA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORCA_ABI_VERSION 2

#if defined(__GNUC__)
#define ORCA_API __attribute__((visibility("default")))
#else
#define ORCA_API
#endif

enum {
    ORCA_OK = 0,
    ORCA_EINVAL = -1,      /* bad argument */
    ORCA_ECUDA = -2,       /* CUDA runtime failure (message has the cudaError) */
    ORCA_ECOINCIDENT = -3, /* engine.py:239-245: exactly coincident centres */
    ORCA_ERANGE = -4,      /* engine.py:152-153: position outside the indexable grid */
    ORCA_ECAPACITY = -5,   /* more agents than the handle was created for */
    ORCA_EUNSUPPORTED = -6, /* e.g. max_neighbors above ORCA_MAX_NEIGHBORS */
    ORCA_ETIMEOUT = -7     /* orca_strip_window_wait: the neighbouring strip's exchange never arrived */
};

enum { ORCA_F32 = 0, ORCA_F64 = 1, ORCA_MIXED = 2, ORCA_CERT32 = 3 };

#define ORCA_MAX_NEIGHBORS 32

typedef struct orca_sim orca_sim;

/* Parameters the step reads from scenario.ScenarioConfig (scenario.py:79-99)
 * plus engine-level switches. fmat is ResponsibilityMatrix.as_array()
 * (orca.py:123-129), row-major f[self_class][other_class]. */
typedef struct orca_params {
    double dt;
    double tau;
    double neighbor_radius;
    double avoidance_margin;
    double fmat[4];
    int32_t max_neighbors;
    int32_t remove_arrivals; /* engine.py:251-255,288-294: drop agents within goal_tol */
    int32_t compute_metrics; /* engine.py:270-286: min_separation / collision_count */
    int32_t reserved;
} orca_params;

/* Counters of the most recent completed step (engine.FrameMetrics, engine.py:46-52,
 * plus SimState.frame / lp_fallbacks, engine.py:62,74). */
typedef struct orca_info {
    int64_t frame;           /* frames completed */
    int64_t active_agents;   /* rows alive after arrival removal */
    int64_t lp_fallbacks;    /* count_nonzero(out_status) of the last step (engine.py:247) */
    int64_t removed_agents;  /* arrivals removed by the last step */
    int64_t collision_count; /* last step; 0 unless compute_metrics */
    double min_separation;   /* last step; +inf unless compute_metrics */
    int32_t grid_nx, grid_ny; /* search-grid dimensions used by the last step */
    double grid_cell;         /* search-grid cell edge (m) */
    int64_t kernel_launches;  /* kernels this handle has launched since orca_create */
    int64_t gather_queue;     /* last step: agents whose neighbour list the certified fast pass could
                                 not prove exact and handed to the exact ring search */
    int64_t solve_queue;      /* last step, ORCA_CERT32 only: agents whose FP32 solve could not be
                                 certified and was redone in FP64 */
} orca_info;

/* ---- lifetime ----------------------------------------------------------- */

ORCA_API int orca_abi_version(void);

/* Create a handle for up to `capacity` agents on CUDA device `device`. */
ORCA_API int orca_create(orca_sim **out, int device, int64_t capacity, int precision);
ORCA_API void orca_destroy(orca_sim *sim);

/* Use an existing CUDA stream (cudaStream_t passed as void*; NULL = the
 * handle's own stream). Lets the caller order the step against its own work. */
ORCA_API int orca_set_stream(orca_sim *sim, void *cuda_stream);

/* Step parameters (ScenarioConfig fields consumed by engine._advance, scenario.py:80-99).
 * The first call, and a later call that raises max_neighbors from <= 16 to > 16, also allocates
 * the device scratch whose size depends on it (capacity * MAXN * 34 bytes with FP64 arithmetic,
 * 18 with FP32, MAXN = 16 or 32: insertion orders, and the half-planes handed to the least-penetration stage);
 * ORCA_ECUDA if that allocation fails. */
ORCA_API int orca_set_params(orca_sim *sim, const orca_params *params);

ORCA_API const char *orca_last_error(const orca_sim *sim);

/* ---- state in / out (engine.SimState arrays, engine.py:55-74) ------------ */

/* Host -> device. positions/velocities/goals are [n,2] row-major float64, the
 * rest [n]. `frame` is SimState.frame (frames completed so far). Pinned host
 * memory makes the copy asynchronous; pageable memory works too. */
ORCA_API int orca_upload(orca_sim *sim, int64_t n, int64_t frame, const int64_t *ids,
                const double *positions, const double *velocities, const double *radii,
                const double *pref_speeds, const double *max_speeds, const double *goals,
                const double *goal_tols, const int64_t *class_codes);

/* Device -> host; synchronises. Any pointer may be NULL to skip that array.
 * Arrays must hold orca_info.active_agents rows (query with orca_get_info).
 * status / failed_at are the out_status / out_failed of the last step for the
 * surviving rows (_kernels.py:553-556; failed_at is the neighbour rank). */
ORCA_API int orca_download(orca_sim *sim, int64_t *ids, double *positions, double *velocities,
                  double *radii, double *pref_speeds, double *max_speeds, double *goals,
                  double *goal_tols, int64_t *class_codes);

/* Only positions and velocities (the arrays a step changes). */
ORCA_API int orca_download_pv(orca_sim *sim, double *positions, double *velocities);

/* The un-compacted result of the LAST step: new positions and velocities of every row
 * that was active during that frame, arrivals included, in pre-step row order (what
 * engine._advance records in its FrameLog, engine.py:257-263). n must be the agent count
 * before that step. Synchronises. */
ORCA_API int orca_download_last_step_pv(orca_sim *sim, int64_t n, double *positions, double *velocities);

/* Which rows of the LAST step's pre-step state survived its arrival removal
 * (engine.py:251-255,288-294): kept[i] = 1 if storage row i is still resident, 0 if the
 * agent arrived and was removed. n must be the agent count before that step. A host caller
 * that keeps its own float64 copies of the per-agent attributes compacts them with this mask
 * instead of reading back the device's (possibly FP32-rounded) copies. Synchronises. */
ORCA_API int orca_download_last_step_kept(orca_sim *sim, int64_t n, uint8_t *kept);

/* Host -> device refresh of positions and velocities only (same n, same rows). */
ORCA_API int orca_upload_pv(orca_sim *sim, int64_t n, int64_t frame, const double *positions,
                   const double *velocities);

/* ---- stepping ------------------------------------------------------------ */

/* One frame of engine._advance on the resident state (asynchronous). */
ORCA_API int orca_step(orca_sim *sim);

/* `steps` consecutive frames without host round trips. */
ORCA_API int orca_run(orca_sim *sim, int64_t steps);

/* What engine.run reads after every frame (engine.py:333-346: FrameMetrics, the fallback count,
 * who arrived), recorded on the device so that a run needs no host round trip per frame. */
typedef struct orca_frame_record {
    int64_t frame;           /* frames completed after this step */
    int64_t active_agents;   /* rows alive after arrival removal */
    int64_t rows_before;     /* rows active during the frame (length of its trajectory block) */
    int64_t lp_fallbacks;
    int64_t removed_agents;
    int64_t collision_count; /* 0 unless compute_metrics */
    double min_separation;   /* +inf unless compute_metrics */
} orca_frame_record; /* 56 bytes */

/* Up to `steps` frames with NO host synchronisation in between, then one readback:
 *   records[0 .. *n_records)   one orca_frame_record per frame actually stepped. A frame
 *                              that would start with no agents left is not stepped (the
 *                              reference's loop ends there, engine.py:333), so
 *                              *n_records < steps means the crowd has fully arrived.
 *   traj (may be NULL)         float64 [rows, 4] = (x, y, vx, vy): for each frame in turn the
 *                              un-compacted result of every row active during that frame, in
 *                              storage-row order (what engine._advance logs, engine.py:257-263);
 *                              frame f's block has records[f].rows_before rows. traj_cap_rows
 *                              bounds it (steps * current agent count always suffices).
 *   arr_ids / arr_frames       the agents removed during these frames and the frame count at
 *                              which each arrived (any order); arr_cap bounds them.
 * Requires a loaded state and orca_set_params. Synchronises once, at the end. */
ORCA_API int orca_run_logged(orca_sim *sim, int64_t steps, orca_frame_record *records, int64_t *n_records,
                             double *traj, int64_t traj_cap_rows, int64_t *traj_rows, int64_t *arr_ids,
                             int64_t *arr_frames, int64_t arr_cap, int64_t *n_arrivals);

/* Wait for all queued work and report sticky device errors:
 * ORCA_ECOINCIDENT with the reference's message
 *   "frame F: agents A and B have exactly coincident centers; avoidance direction is undefined"
 * or ORCA_ERANGE with "agent position out of indexable grid range". */
ORCA_API int orca_sync(orca_sim *sim);

/* Synchronises, then fills `info`. */
ORCA_API int orca_get_info(orca_sim *sim, orca_info *info);

/* Per-stage device timing for benchmarks. While enabled, every step records CUDA
 * events on the handle's stream at the stage boundaries; orca_get_stage_ms
 * synchronises, writes the accumulated milliseconds of each stage since the last
 * call into ms[ORCA_N_STAGES] and the number of steps covered into *steps. */
#define ORCA_N_STAGES 6
enum {
    ORCA_STAGE_BINS = 0,     /* bounding box, plan, histogram, scan, scatter */
    ORCA_STAGE_GATHER = 1,   /* neighbour search */
    ORCA_STAGE_SOLVE = 2,    /* ORCA half-planes + incremental LP + integration */
    ORCA_STAGE_FALLBACK = 3, /* least-penetration stage + integration */
    ORCA_STAGE_FINISH = 4,   /* counters, arrival removal */
    ORCA_STAGE_METRICS = 5   /* post-step bin build + min separation */
};
ORCA_API int orca_profile_stages(orca_sim *sim, int enable);
ORCA_API int orca_get_stage_ms(orca_sim *sim, double *ms, int64_t *steps);

/* One whole reference step() through host buffers: upload of positions and
 * velocities, one frame, download of the new positions / velocities and the
 * per-row solver status (engine.step, engine.py:298-308, with the static agent
 * attributes already resident from orca_upload). Requires remove_arrivals == 0.
 * out_status may be NULL. */
ORCA_API int orca_step_host(orca_sim *sim, int64_t n, int64_t frame, const double *positions,
                   const double *velocities, double *new_positions, double *new_velocities,
                   int64_t *out_status);

/* engine._advance through host buffers (engine.py:194-295; what engine.step,
 * engine.py:298-308, does per call once the static agent attributes are
 * resident from orca_upload): host positions/velocities [n,2] in, the new state's
 * positions/velocities out, arrival removal and frame metrics per orca_params,
 * counters in *info (orca_get_info). The copies overlap the step: the bin build
 * and neighbour gather run on the positions while the velocities are still being
 * copied in, and the result is copied out while the metrics are computed.
 * new_positions/new_velocities must hold n rows; rows [0, info->active_agents)
 * are the new state, in storage order (engine.py:288-294). When agents were
 * removed (info->removed_agents > 0) fetch the compacted attributes with
 * orca_download. Pinned host memory makes the copies asynchronous. */
ORCA_API int orca_advance_host(orca_sim *sim, int64_t n, int64_t frame, const double *positions,
                      const double *velocities, double *new_positions, double *new_velocities,
                      orca_info *info);

/* Lay the resident rows out in the cell-sorted order of a fresh bin build (an internal
 * layout change for memory coherence; no reference counterpart -- the reference keeps
 * numpy arrays in spawn order, engine.py:179-186). orca_step does this by itself after an
 * upload and periodically; callers that keep ghost rows resident at every step
 * (parallel/strips.py) call it between migration and the next halo exchange. Every array
 * the host reads or writes stays in the reference's storage order. */
ORCA_API int orca_reorder_rows(orca_sim *sim);

/* ---- parity taps (pre-step snapshot of the LAST step; storage-row order) --- */

/* cell_ix/cell_iy: floor(pos / neighbor_radius) as int64 (engine.py:150-151).
 * nb_rows [n, max_neighbors] (-1 padded) and nb_count [n]: the ordered
 * neighbour rows of _collect_neighbors (_kernels.py:450-490).
 * out_v [n,2], status, failed_at: what frame_solve_range wrote
 * (_kernels.py:543-556). Valid only when the last step removed no agents or
 * remove_arrivals == 0; n is the agent count BEFORE that step. Any pointer may
 * be NULL. */
ORCA_API int orca_debug_last_step(orca_sim *sim, int64_t n, int64_t *cell_ix, int64_t *cell_iy,
                         int64_t *nb_rows, int64_t *nb_count, double *out_v, int64_t *status,
                         int64_t *failed_at, double *desired_v);

/* ---- batched LP (lp.solve_batch / _kernels.solve_range, CSR layout) -------- */

/* Host arrays in the layout of _kernels.py:306-312: coff int64[n+1], cpts/cnrm
 * float64[m,2], tgt float64[n,2], caps float64[n], seeds uint64[n]; outputs
 * out_v float64[n,2], out_status int64[n] (0 feasible, 1 fallback used),
 * out_failed int64[n] (original constraint index or -1). Synchronous. The batch is cut into
 * chunks of problems that are uploaded, packed and solved on two alternating streams, so with
 * pinned host arrays the call is bound by the one PCIe crossing of the constraints. */
ORCA_API int orca_lp_solve_batch(int device, int precision, int64_t n, const int64_t *coff,
                        const double *cpts, const double *cnrm, const double *tgt,
                        const double *caps, const uint64_t *seeds, double *out_v,
                        int64_t *out_status, int64_t *out_failed);

/* orca_lp_solve_batch keeps its device scratch (~3 GB for a million problems) between calls;
 * this gives it back. */
ORCA_API int orca_lp_release_scratch(void);

/* Resident variant for benchmarking: build once, solve many times on device. */
typedef struct orca_lp_batch orca_lp_batch;
ORCA_API int orca_lp_batch_create(orca_lp_batch **out, int device, int precision, int64_t n,
                         const int64_t *coff, const double *cpts, const double *cnrm,
                         const double *tgt, const double *caps, const uint64_t *seeds);
ORCA_API int orca_lp_batch_set_stream(orca_lp_batch *b, void *cuda_stream);
ORCA_API int orca_lp_batch_solve(orca_lp_batch *b);             /* asynchronous */
ORCA_API int orca_lp_batch_download(orca_lp_batch *b, double *out_v, int64_t *out_status,
                           int64_t *out_failed);        /* synchronises */
ORCA_API void orca_lp_batch_destroy(orca_lp_batch *b);

/* ---- single-op taps for known-answer tests -------------------------------- */

/* vo_exit (_kernels.py:343-419) evaluated on the device for `count` cases;
 * in7 = (rpx, rpy, rvx, rvy, comb_r, tau, dt) per case, out5 = (ux, uy, nx, ny, ok). */
ORCA_API int orca_vo_exit_batch(int device, int precision, int64_t count, const double *in7,
                       double *out5);

/* The least-penetration stage alone (lp.solve_least_penetration, lp.py:168-190 ->
 * _kernels.py:254-283 with the constraints in the given order): cpts/cnrm float64[k,2],
 * warm start (wx, wy) assumed to satisfy constraints [0, start_index); out_v[2]. */
ORCA_API int orca_least_penetration(int device, int precision, int64_t k, const double *cpts,
                                    const double *cnrm, double speed_cap, int64_t start_index,
                                    double wx, double wy, double *out_v);

/* The neighbour query alone (grid.query_neighbors, grid.py:50-83 == _kernels.py:450-490) for
 * EVERY agent at once: the up to max_count (<= ORCA_MAX_NEIGHBORS) nearest agents within
 * `radius`, ascending by (distance, id). ids int64[n], positions float64[n,2]; out_rows
 * int64[n, max_count] (row indices, -1 padded), out_count int64[n]. */
ORCA_API int orca_neighbor_query(int device, int64_t n, const int64_t *ids, const double *positions,
                                 double radius, int32_t max_count, int64_t *out_rows, int64_t *out_count);

/* grid.query_neighbors with max_count beyond ORCA_MAX_NEIGHBORS ("everyone within the radius",
 * G:50-83 called with a huge max_count): every agent's complete list, ordered by (d2, id), as
 * CSR -- out_offsets[n + 1], out_rows[cap]. *total_out = the number of entries; ORCA_ECAPACITY
 * (offsets and total valid) when they do not fit cap. An object-level operator, not the step. */
ORCA_API int orca_neighbor_query_all(int device, int64_t n, const int64_t *ids, const double *positions,
                                     double radius, int64_t cap, int64_t *out_offsets, int64_t *out_rows,
                                     int64_t *total_out);

/* Fisher-Yates order (_kernels.py:43-54) computed on the device: perm[k]. */
ORCA_API int orca_shuffle_order(int device, int64_t k, uint64_t seed, int64_t *perm);

/* _problem_seed (_kernels.py:57-61) computed on the device. */
ORCA_API int orca_problem_seed(int device, int64_t frame, int64_t agent_id, uint64_t *seed);

/* ---- multi-GPU strip decomposition (device-pointer level) ------------------
 *
 * The reference has no multi-process path; this is the B200-native
 * addition for crowds larger than one device: the plaza is cut into x-strips, one
 * handle (one process, one GPU) per strip. Every step each rank
 *   1. packs its owned agents within neighbor_radius of a strip edge
 *      (orca_strip_pack, remove = 0) and sends them to that neighbour,
 *   2. appends what it received as ghosts (orca_strip_append, ghost = 1): ghosts
 *      take part in the neighbour search of owned agents but are never solved,
 *      integrated or reported, and the step drops them again,
 *   3. steps (orca_step),
 *   4. packs-and-removes the owned agents whose new x left the strip
 *      (orca_strip_pack, remove = 1), sends them, and appends the arrivals as
 *      owned rows (ghost = 0).
 * Per-agent results depend only on the pre-step snapshot of the agents within
 * neighbor_radius, so they are bit-identical to a single-device run (keyed by id).
 * The records travel between ranks as raw bytes (NCCL send/recv). */

typedef struct orca_agent_record {
    double x, y, vx, vy;
    double radius, pref_speed, max_speed, goal_tol;
    double goal_x, goal_y;
    int64_t id;
    int64_t class_code;
} orca_agent_record; /* 96 bytes */

/* Select owned rows with x in [x_lo, x_hi), write them to `records` (DEVICE
 * pointer, room for `cap` records) and return how many were selected in
 * *count_out (HOST). If more than `cap` were selected the call fails with
 * ORCA_ECAPACITY and nothing is removed. With remove != 0 the selected rows are
 * deleted from the handle. Synchronises. */
ORCA_API int orca_strip_pack(orca_sim *sim, double x_lo, double x_hi, int remove,
                             orca_agent_record *records, int64_t cap, int64_t *count_out);

/* Append `count` records (DEVICE pointer) after the resident rows, as owned rows
 * (ghost == 0; not allowed while ghosts are resident) or as ghosts. Asynchronous. */
ORCA_API int orca_strip_append(orca_sim *sim, const orca_agent_record *records, int64_t count,
                               int ghost);

/* Forget the ghost rows without stepping. */
ORCA_API int orca_strip_drop_ghosts(orca_sim *sim);

/* ---- the same protocol without the host in the loop ----------------------------
 *
 * orca_strip_pack reports its count to the host, so every exchange costs host
 * synchronisations. The calls below keep the counts on the device: a SLAB is a
 * fixed-capacity DEVICE buffer of  sizeof(orca_slab_header) + cap * record_bytes  bytes;
 * the packing kernels count into the header, the whole slab travels (its size is
 * known to both ranks without asking), and the appending kernels read the count
 * from the header. All five calls are asynchronous; the host keeps only upper
 * bounds on the row count, refreshed whenever it does synchronise (orca_sync /
 * orca_get_info, e.g. every 16 frames). A slab, or the handle, that turns out too
 * small raises a sticky device-side flag reported by the next orca_sync as
 * ORCA_ECAPACITY; nothing is lost silently.
 *
 * Per frame and rank (parallel/strips.py), ONE exchange with each neighbour:
 *   orca_strip_append_slab(received immigrants, ghost = 0)            from the previous exchange
 *   orca_strip_append_slab(received halo, 1) + (own emigrants, 2)
 *   orca_strip_step(emigrant slabs)
 *   orca_strip_pack_halo(halo slabs)          -> exchange (emigrants + halo) with both neighbours
 * Halo slabs carry orca_halo_record_f32 (32 B; FP32 state: ORCA_MIXED, ORCA_F32) or
 * orca_halo_record_f64 (64 B; ORCA_F64): what a neighbour reads of an agent
 * (_kernels.py:525-541: position, velocity, radius, class) plus the id that orders
 * equal distances (_kernels.py:473-476). Migrant slabs carry full orca_agent_record. */

typedef struct orca_slab_header {
    int32_t count;    /* records the sender produced (may exceed the capacity: then `overflow`) */
    int32_t overflow; /* the sender could not fit a record */
    int64_t reserved[3];
} orca_slab_header; /* 32 bytes */

typedef struct orca_halo_record_f32 {
    float x, y, vx, vy;
    float radius;
    uint32_t class_code;
    int64_t id;
} orca_halo_record_f32; /* 32 bytes */

typedef struct orca_halo_record_f64 {
    double x, y, vx, vy;
    double radius;
    int64_t id;
    int64_t class_code;
    int64_t pad;
} orca_halo_record_f64; /* 64 bytes */

/* sizeof the halo record this handle's precision uses (32 or 64). */
ORCA_API int64_t orca_strip_halo_record_bytes(const orca_sim *sim);

/* After orca_upload: this handle owns x in [x_lo, x_hi) (+-inf at the ends of the domain) and
 * runs the slab protocol from here on. vmax_floor: the largest max_speed of the WHOLE crowd
 * (ghosts travel without theirs; the neighbour search's displacement bound needs it).
 * slack_rows: how many rows (ghosts + immigrants) may be appended on top of the row count the
 * host last saw before it synchronises again -- the host's launch bound is that count +
 * slack_rows and stays FIXED between synchronisations, so that one captured CUDA graph serves
 * every frame in between; appends beyond it raise the sticky overflow flag. */
ORCA_API int orca_strip_configure(orca_sim *sim, double x_lo, double x_hi, double vmax_floor,
                                  int64_t slack_rows);

/* Owned rows with x < x_lo + reach -> left slab, x >= x_hi - reach -> right slab
 * (either may be NULL: no neighbour on that side). cap = records per slab. */
ORCA_API int orca_strip_pack_halo(orca_sim *sim, double reach, void *slab_left, void *slab_right,
                                  int64_t cap);

/* Append the records of a slab: ghost == 0 -> orca_agent_record as owned rows (received
 * immigrants; not while ghosts are resident), ghost == 1 -> halo records as ghost rows (a
 * received halo), ghost == 2 -> orca_agent_record as ghost rows (this handle's OWN emigrants of
 * the last orca_strip_step: an agent that just crossed the edge is within neighbor_radius of it,
 * so it stays here as a ghost and the neighbour does not have to send it back). */
ORCA_API int orca_strip_append_slab(orca_sim *sim, const void *slab, int64_t cap, int ghost);

/* orca_step for a strip: the step, then ONE compaction that drops the ghosts, the
 * arrivals (if remove_arrivals) and the owned rows whose new x left [x_lo, x_hi) --
 * those are written to the migrant slabs (NULL = no neighbour on that side) as
 * orca_agent_record. */
ORCA_API int orca_strip_step(orca_sim *sim, void *migrants_left, void *migrants_right, int64_t cap);

/* ---- The exchange through peer memory (one node: NVLink / NVSwitch) ----------------------
 * Instead of handing the slabs to a communication library, a strip WRITES them into its
 * neighbour's memory. Each handle owns a WINDOW (one device allocation): per side a flag and two
 * receive buffers of side_bytes = [emigrant slab | halo slab], double-buffered by the parity of
 * the exchange index. orca_strip_window_push copies the used part of the sender's slabs (the
 * counts are read from the headers ON THE DEVICE) into the neighbour's window and then raises
 * the neighbour's flag to exchange + 1; orca_strip_window_wait makes the receiver's stream wait
 * for its own flag (a one-thread kernel, bounded: ORCA_WINDOW_TIMEOUT_MS, default 20,000 --
 * after that the sticky error ORCA_ETIMEOUT surfaces at the next orca_sync). Pack, copy, flag,
 * wait and append are all kernels on the handles' streams: no host call of a library, no host
 * synchronisation, nothing collective. The neighbour's window is mapped with the CUDA IPC handle
 * orca_strip_window_create returns (another process, its own or the same GPU) or, for handles
 * of the SAME process, given by its base address.
 * Exchange indices count from 0 and must be pushed / waited for in order. */
#define ORCA_IPC_HANDLE_BYTES 64
ORCA_API int orca_strip_window_create(orca_sim *sim, int64_t side_bytes, void *ipc_handle_out /* 64 bytes */,
                                      void **base_out);
/* side: 0 = the neighbour on the left, 1 = on the right. Exactly one of ipc_handle /
 * same_process_base is non-NULL. */
ORCA_API int orca_strip_window_open(orca_sim *sim, int side, const void *ipc_handle, void *same_process_base);
/* send = [emigrant slab (32 + mig_cap * 96 bytes) | halo slab (32 + halo_cap * record bytes)] */
ORCA_API int orca_strip_window_push(orca_sim *sim, int side, const void *send, int64_t mig_cap, int64_t halo_cap,
                                    int64_t exchange);
/* *slab_out: where exchange `exchange` of that side lands in THIS handle's window (valid for
 * kernels that follow on the handle's stream). */
ORCA_API int orca_strip_window_wait(orca_sim *sim, int side, int64_t exchange, void **slab_out);
/* Unmaps the neighbours' windows and frees this one (every strip must have finished its frames:
 * synchronise the ranks first). Also done by orca_destroy. */
ORCA_API int orca_strip_window_close(orca_sim *sim);

/* Rows appended from slabs since the last orca_upload: ghosts, migrants (for
 * benchmarks). Synchronises. */
ORCA_API int orca_strip_stats(orca_sim *sim, int64_t *ghost_rows, int64_t *migrant_rows);

#ifdef __cplusplus
}
#endif
#endif /* ORCA_B200_H */

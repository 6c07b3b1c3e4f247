// orca_common.cuh -- shared device structs, error plumbing and small utilities.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include "orca_b200.h"
#include "orca_math.cuh"

namespace orca {

typedef unsigned char u8;
typedef signed char i8;

// _kernels.py:426-432 / engine.py:146: |floor(pos/cell)| must stay <= 2^29 - 2
#define ORCA_CELL_LIMIT ((double)((1LL << 29) - 2))

#define ORCA_NO_ERR 0xFFFFFFFFFFFFFFFFULL

// gather + solve + fallback are issued per chunk of sorted slots, at most this many
#define ORCA_MAX_CHUNKS 4

// Device-resident per-step plan and counters. Written by k_plan / k_finish and
// read by every kernel of the step, so a step needs no host round trip.
struct GridPlan {
    // population
    int n;       // rows in the state arrays (owned + ghost)
    int n_owned; // rows [0, n_owned) are solved and integrated; the rest are halo ghosts
    int n_pre;   // n_owned at the start of the last step (rows of the un-compacted result)
    // search grid (rebuilt every step from the bounding box)
    int nx, ny, ncells, rmax, r0;
    double x0, y0, cell, inv_cell;
    // bounding-box accumulators, order-preserving u64 encodings of doubles
    u64 minx, miny, maxx, maxy;
    // bounding box of the positions the LAST bin build binned (k_count's last block folds the
    // per-block boxes into it); the next build grows it by one frame's largest displacement
    double nbox[4];
    unsigned box_done; // blocks of the running k_count that have published their box
    // sticky errors
    u64 err_pair;   // (row_i << 32 | row_j) of the first coincident pair in row order
    i64 err_frame;  // frame_new of that step
    i64 err_id_i, err_id_j;
    int err_range;  // a position left the reference's indexable grid range
    int err_capacity; // a strip-exchange slab (or the handle) overflowed: rows were dropped or kept back
    int err_window;   // k_window_wait gave up: the neighbouring strip's exchange never arrived
    // strip step: rows removed in place (orca_api.cu, strip_fill_stage)
    int strip_removed, hole_count, tail_count;
    unsigned long long strip_recv[2]; // ghost rows / migrant rows appended from slabs since the upload
    // per-step counters
    // work queues, one counter per CHUNK of sorted slots (orca_api.cu: the step issues gather, solve
    // and fallback per chunk on two streams, so that the latency-bound queue kernels of one chunk
    // overlap the throughput-bound kernels of the other)
    int fq_count[ORCA_MAX_CHUNKS]; // agents queued for the least-penetration stage; sum == lp_fallbacks
    int gq_count[ORCA_MAX_CHUNKS]; // agents the certified fast pass queued for the exact ring search (k_gather)
    int cq_count[ORCA_MAX_CHUNKS]; // ORCA_CERT32: agents whose FP32 solve was not certified (redone in FP64)
    int pack_count; // rows selected by the last orca_strip_pack
    u64 vmax_enc;  // order-preserving encoding of the largest max_speed ever uploaded
    double vmax;
    int removed;   // arrivals removed by this step
    int n_after;   // rows after arrival removal
    // metrics
    u64 min_sep_enc; // order-preserving encoding of the running minimum
    u64 sep_ub_enc;  // upper bound on it from each agent's closest candidate (k_min_sep_bound)
    u64 rmax_enc;    // largest agent radius ever uploaded
    u64 collisions;
    // frames completed
    i64 frame;
    // orca_run_logged: per-frame records / trajectories / arrivals kept on the device
    int halt_when_empty; // a frame that starts with no agents left is not a frame (engine.py:333)
    int idle;            // ... and this step is such a non-frame
    int log_count;       // frame records written since the chunk began
    i64 traj_rows;       // trajectory rows written since the chunk began
    int arr_count;       // arrivals logged since the upload
};

// The per-agent attributes a step never changes, exactly as the host uploaded them (float64):
// kept beside the FP32 state of the MIXED / F32 modes so that everything the host reads back
// after an arrival removal is the value it uploaded, not an FP32 rounding of it
// (engine.py:288-294 hands the caller's own arrays on). Unused (null) with FP64 state.
struct Attr64 {
    double radius, pref_speed, max_speed, goal_x, goal_y, goal_tol;
};

struct StepParams {
    double dt, tau, nr, rad2, half_margin;
    double fmat[4];
    int max_n;
    int stride;  // leading dimension of the slot-major neighbour table
    int max_cells;
    double occ_target;
};

__host__ __device__ __forceinline__ u64 enc_double(double x)
{
#ifdef __CUDA_ARCH__
    u64 b = (u64)__double_as_longlong(x);
#else
    u64 b;
    memcpy(&b, &x, 8);
#endif
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__host__ __device__ __forceinline__ double dec_double(u64 e)
{
    u64 b = (e >> 63) ? (e & 0x7FFFFFFFFFFFFFFFULL) : ~e;
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double x;
    memcpy(&x, &b, 8);
    return x;
#endif
}

// vector helpers
__device__ __forceinline__ float4 mk4(float a, float b, float c, float d) { return make_float4(a, b, c, d); }
__device__ __forceinline__ double4 mk4(double a, double b, double c, double d) { return make_double4(a, b, c, d); }
__device__ __forceinline__ float2 mk2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk2(double a, double b) { return make_double2(a, b); }

template <typename R> struct Fmt;
template <> struct Fmt<float> { static constexpr bool is_f32 = true; };
template <> struct Fmt<double> { static constexpr bool is_f32 = false; };

static inline int div_up(long long a, long long b) { return (int)((a + b - 1) / b); }

} // namespace orca

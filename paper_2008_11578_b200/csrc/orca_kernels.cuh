// orca_kernels.cuh -- the kernels of one steering step, sm_100a.
//
//   K0  k_bbox / k_plan      bounding box -> dense search grid for this step
//   K1  k_count              search-cell id per agent + per-cell histogram
//       k_scan_*             exclusive prefix scan of the histogram (CSR starts)
//       k_scatter            counting-sort scatter into cell-sorted SoA arrays,
//                            fused with the desired velocity (engine.py:133-139)
//   K2  k_gather             exact top-max_n neighbours by (d2, id) within
//                            neighbor_radius (_kernels.py:450-490), ring search
//   K3  k_solve              ORCA half-planes (_kernels.py:525-541) + shuffled
//                            incremental LP (_kernels.py:122-146) + integration
//       k_fallback           least-penetration stage (_kernels.py:254-283) for the
//                            agents k_solve queued, + integration
//   K4  k_finish / k_compact counters, arrival removal (engine.py:251-294)
//
// The search grid is NOT the reference's grid (cell = neighbor_radius): it is
// finer (about occ_target agents per cell) and searched in growing rings, which
// is legal because the neighbour set is defined geometrically and is invariant
// under the cell size (pkg/tests/test_grid.py:101). The reference's own cell
// index floor(pos/neighbor_radius) is still produced bit-exactly (k_ref_cells)
// and range-checked every step (engine.py:152-153).
#pragma once

#include "orca_common.cuh"
#include "orca_sortnet.inc"

#ifndef ORCA_SCAN_UNROLL
#define ORCA_SCAN_UNROLL 4
#endif
#ifndef ORCA_BUILD_UNROLL
#define ORCA_BUILD_UNROLL 1 // vo_exit chains interleaved per lane in k_solve_group's constraint build
                            // (measured at 1 M agents: 1 -> 0.498 ms, 2 -> 0.511, 4 -> 0.537: registers, not ILP)
#endif
#ifndef ORCA_GL_SHORT
#define ORCA_GL_SHORT 16         // lanes per agent in k_fallback_coop when the queue is short
#endif
#ifndef ORCA_FB_SHORT_QUEUE
#define ORCA_FB_SHORT_QUEUE 4096 // "short": every queued agent gets half a warp in one wave
#endif
#ifndef ORCA_PRESHUFFLE
#define ORCA_PRESHUFFLE 1   // k_solve_group reads the insertion order k_shuffle computed, one thread per agent
#endif
#ifndef ORCA_SCAN_SMALL_CELLS
#define ORCA_SCAN_SMALL_CELLS 65536 // search grids up to this many cells are scanned by one block (k_scan_small)
#endif
#ifndef ORCA_PRESHUFFLE_MIN_AGENTS
#define ORCA_PRESHUFFLE_MIN_AGENTS 65536
#endif
#ifndef ORCA_CHUNKS_DEFAULT
#ifndef ORCA_SMALL_SOLVE_GL
#define ORCA_SMALL_SOLVE_GL 8      // lanes per agent in the FP64 solve kernel for crowds of <= ORCA_SMALL_SOLVE_AGENTS:
#endif                             // one wave whose time is one agent's chain (1,024 agents: solve 27 -> 20 us; 4 lanes: 23)
#ifndef ORCA_SMALL_SOLVE_AGENTS
#define ORCA_SMALL_SOLVE_AGENTS 8192
#endif
#ifndef ORCA_QUEUE_GL
#define ORCA_QUEUE_GL 4 // lanes per agent in the FP64 pass over the agents ORCA_CERT32 could not certify: a few
                        // percent of the crowd, i.e. one wave whose time is ONE agent's chain of sixteen FP64
                        // half-planes -- four lanes build four each (2 lanes: solve stage 0.422 ms, 4: 0.394, 8: 0.403)
#endif
#define ORCA_CHUNKS_DEFAULT 2          // gather + solve + fallback pipelined over this many chunks of sorted slots ...
#endif
#ifndef ORCA_CHUNK_MIN_AGENTS
#define ORCA_CHUNK_MIN_AGENTS 262144   // ... for crowds of at least this many agents (below: one chunk)
#endif
#ifndef ORCA_SG_BLOCKS
#define ORCA_SG_BLOCKS 6    // resident blocks per SM k_solve_group is compiled for (register cap)
#endif

namespace orca {

// ---------------------------------------------------------------------------
// K0: bounding box + grid plan
// ---------------------------------------------------------------------------

// per-step counters (start of every step)
__global__ void k_begin_step(GridPlan *plan)
{
    for (int c = 0; c < ORCA_MAX_CHUNKS; ++c) plan->fq_count[c] = plan->cq_count[c] = plan->gq_count[c] = 0;
    plan->n_pre = plan->n_owned;
    plan->idle = plan->halt_when_empty && plan->n_owned == 0;
    plan->strip_removed = plan->hole_count = plan->tail_count = 0;
    plan->removed = 0;
    plan->min_sep_enc = enc_double(__longlong_as_double(0x7FF0000000000000LL));
    plan->sep_ub_enc = plan->min_sep_enc;
    plan->collisions = 0;
}

// bounding-box accumulators (start of every bin build)
__global__ void k_begin_bins(GridPlan *plan)
{
    plan->minx = plan->miny = 0xFFFFFFFFFFFFFFFFULL;
    plan->maxx = plan->maxy = 0ULL;
}

template <typename R>
__global__ void __launch_bounds__(256) k_bbox(GridPlan *plan, const typename Vec<R>::T4 *__restrict__ pv)
{
    const int n = plan->n;
    double lox = 1e300, loy = 1e300, hix = -1e300, hiy = -1e300;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const typename Vec<R>::T4 a = pv[i];
        const double x = (double)a.x, y = (double)a.y;
        lox = fmin(lox, x);
        hix = fmax(hix, x);
        loy = fmin(loy, y);
        hiy = fmax(hiy, y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lox = fmin(lox, __shfl_xor_sync(0xFFFFFFFFu, lox, o));
        loy = fmin(loy, __shfl_xor_sync(0xFFFFFFFFu, loy, o));
        hix = fmax(hix, __shfl_xor_sync(0xFFFFFFFFu, hix, o));
        hiy = fmax(hiy, __shfl_xor_sync(0xFFFFFFFFu, hiy, o));
    }
    if ((threadIdx.x & 31) == 0 && lox <= hix) {
        atomicMin(&plan->minx, enc_double(lox));
        atomicMin(&plan->miny, enc_double(loy));
        atomicMax(&plan->maxx, enc_double(hix));
        atomicMax(&plan->maxy, enc_double(hiy));
    }
}

// One thread: choose the search-cell edge from the mean density, snap it so an
// integer number of rings covers neighbor_radius, and make the dense grid fit.
// grow >= 0: no k_bbox ran; take the box k_count accumulated at the previous build, grown by
// `grow` frames of the largest possible displacement (|v| <= max_speed after every LP, K:127-135).
// A position that still ends up outside is clamped into an edge cell by search_cell, which
// only makes it look closer to the grid than it is -- the ring-search bound stays valid.
__global__ void k_plan(GridPlan *plan, StepParams P, double grow)
{
    const int n = plan->n;
    plan->vmax = fmax(dec_double(plan->vmax_enc), 0.0);
    double x0 = 0.0, y0 = 0.0, w = 0.0, h = 0.0;
    if (n > 0) {
        if (grow >= 0.0) {
            const double m = grow * plan->vmax * P.dt * (1.0 + 1e-6) + 1e-9;
            x0 = plan->nbox[0] - m;
            y0 = plan->nbox[1] - m;
            w = plan->nbox[2] + m - x0;
            h = plan->nbox[3] + m - y0;
        } else {
            x0 = dec_double(plan->minx);
            y0 = dec_double(plan->miny);
            w = dec_double(plan->maxx) - x0;
            h = dec_double(plan->maxy) - y0;
        }
    }
    const double nr = P.nr;
    const double area = fmax(w, 1e-3 * nr) * fmax(h, 1e-3 * nr);
    double c = sqrt(P.occ_target * area / fmax((double)n, 1.0));
    c = fmin(fmax(c, nr / 16.0), nr);
    // snap: rings * c covers nr with a 1e-6 relative margin, so rmax == rings
    const double rings = ceil(nr / c);
    c = nr / rings * (1.0 + 1e-6);
    while ((floor(w / c) + 2.0) * (floor(h / c) + 2.0) > (double)P.max_cells) c *= 1.25;
    // Anchor the grid to multiples of the cell edge: the cells then stay where they are from
    // step to step (c only takes the values nr / rings), so the cell-sorted order -- and with
    // it the row order chosen at the last reordering -- stays coherent while the box breathes.
    {
        const double ax = floor(x0 / c) * c, ay = floor(y0 / c) * c;
        if (isfinite(ax) && isfinite(ay) && x0 - ax <= c && y0 - ay <= c) {
            w += x0 - ax;
            h += y0 - ay;
            x0 = ax;
            y0 = ay;
        }
    }
    const int nx = (int)floor(w / c) + 1, ny = (int)floor(h / c) + 1;
    plan->x0 = x0;
    plan->y0 = y0;
    plan->cell = c;
    plan->inv_cell = 1.0 / c;
    plan->nx = nx;
    plan->ny = ny;
    plan->ncells = nx * ny;
    plan->rmax = (int)ceil(nr / c * (1.0 + 1e-9));
    // first ring radius: the smallest block of cells expected to hold ~1.3 * max_n agents
    // at the mean density (the search still grows ring by ring where that is not enough)
    const double occ = fmax((double)n, 1.0) * c * c / area;
    int r0 = (int)ceil((sqrt(1.3 * (double)max(P.max_n, 1) / fmax(occ, 1e-9)) - 1.0) * 0.5);
    plan->r0 = min(max(r0, 1), plan->rmax);
}

__device__ __forceinline__ void search_cell(const GridPlan *plan, double x, double y, int &cx, int &cy)
{
    // monotone in x and y; the ring-termination bound in k_gather relies on that
    const double fx = (x - plan->x0) * plan->inv_cell;
    const double fy = (y - plan->y0) * plan->inv_cell;
    cx = min(max((int)floor(fx), 0), plan->nx - 1);
    cy = min(max((int)floor(fy), 0), plan->ny - 1);
}

// ---------------------------------------------------------------------------
// K1: count, scan, scatter
// ---------------------------------------------------------------------------

template <typename R>
__global__ void __launch_bounds__(256)
k_count(GridPlan *plan, const typename Vec<R>::T4 *__restrict__ pv, int *__restrict__ cell_of,
        int *__restrict__ rank_of, int *__restrict__ cell_count, double nr, double4 *box_part)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < plan->n;
    const typename Vec<R>::T4 a = pv[live ? i : 0];
    const double x = (double)a.x, y = (double)a.y;
    {   // bounding box of what is binned now, for the next build's plan (see k_plan)
        double lox = live ? x : 1e300, hix = live ? x : -1e300, loy = live ? y : 1e300, hiy = live ? y : -1e300;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lox = fmin(lox, __shfl_xor_sync(0xFFFFFFFFu, lox, o));
            loy = fmin(loy, __shfl_xor_sync(0xFFFFFFFFu, loy, o));
            hix = fmax(hix, __shfl_xor_sync(0xFFFFFFFFu, hix, o));
            hiy = fmax(hiy, __shfl_xor_sync(0xFFFFFFFFu, hiy, o));
        }
        // one partial box per block, folded by the block that finishes last: same-address atomics
        // (or even same-address loads) from every warp of the grid serialise in one L2 slice and
        // cost more than the k_bbox pass this replaces
        __shared__ double4 sm_box[8];
        if ((threadIdx.x & 31) == 0) sm_box[threadIdx.x >> 5] = make_double4(lox, loy, hix, hiy);
        __syncthreads();
        __shared__ bool sm_last;
        if (threadIdx.x == 0) {
            double4 b = sm_box[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                b.x = fmin(b.x, sm_box[w].x);
                b.y = fmin(b.y, sm_box[w].y);
                b.z = fmax(b.z, sm_box[w].z);
                b.w = fmax(b.w, sm_box[w].w);
            }
            box_part[blockIdx.x] = b;
            __threadfence();
            sm_last = atomicAdd(&plan->box_done, 1u) == gridDim.x - 1u;
        }
        __syncthreads();
        if (sm_last) { // the block that finishes last folds the partial boxes into the plan
            double4 b = make_double4(1e300, 1e300, -1e300, -1e300);
            for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
                // (written by other blocks of this launch: read through L2, not the L1 of this SM)
                const double2 lo2 = __ldcg(reinterpret_cast<const double2 *>(&box_part[i]));
                const double2 hi2 = __ldcg(reinterpret_cast<const double2 *>(&box_part[i]) + 1);
                const double4 p = make_double4(lo2.x, lo2.y, hi2.x, hi2.y);
                b.x = fmin(b.x, p.x);
                b.y = fmin(b.y, p.y);
                b.z = fmax(b.z, p.z);
                b.w = fmax(b.w, p.w);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                b.x = fmin(b.x, __shfl_xor_sync(0xFFFFFFFFu, b.x, o));
                b.y = fmin(b.y, __shfl_xor_sync(0xFFFFFFFFu, b.y, o));
                b.z = fmax(b.z, __shfl_xor_sync(0xFFFFFFFFu, b.z, o));
                b.w = fmax(b.w, __shfl_xor_sync(0xFFFFFFFFu, b.w, o));
            }
            __syncthreads(); // sm_box is reused
            if ((threadIdx.x & 31) == 0) sm_box[threadIdx.x >> 5] = b;
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                    b.x = fmin(b.x, sm_box[w].x);
                    b.y = fmin(b.y, sm_box[w].y);
                    b.z = fmax(b.z, sm_box[w].z);
                    b.w = fmax(b.w, sm_box[w].w);
                }
                plan->nbox[0] = b.x;
                plan->nbox[1] = b.y;
                plan->nbox[2] = b.z;
                plan->nbox[3] = b.w;
                plan->box_done = 0u;
            }
        }
    }
    if (!live) return;
    // engine.py:150-153: the reference's own bin index must stay indexable
    const double rix = floor(__ddiv_rn(x, nr)), riy = floor(__ddiv_rn(y, nr));
    if (!(fabs(rix) <= ORCA_CELL_LIMIT) || !(fabs(riy) <= ORCA_CELL_LIMIT)) plan->err_range = 1;
    int cx, cy;
    search_cell(plan, x, y, cx, cy);
    const int c = cx * plan->ny + cy; // column-major: a column's rows are contiguous
    cell_of[i] = c;
    rank_of[i] = atomicAdd(&cell_count[c], 1);
}

// Exclusive scan of `in[0 .. len)` where len = *len_ptr + len_extra (device
// value). Three phases; tiles of SCAN_TILE elements per block.
#define SCAN_THREADS 256
#define SCAN_ITEMS 8
#define SCAN_TILE (SCAN_THREADS * SCAN_ITEMS)

__device__ __forceinline__ int block_exclusive_scan(int v, int *smem_warp, int &block_total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) smem_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int w = lane < (SCAN_THREADS / 32) ? smem_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, w, o);
            if (lane >= o) w += t;
        }
        smem_warp[32 + lane] = w; // inclusive over warps
    }
    __syncthreads();
    const int warp_off = wid == 0 ? 0 : smem_warp[32 + wid - 1];
    block_total = smem_warp[32 + SCAN_THREADS / 32 - 1];
    __syncthreads();
    return warp_off + inc - v;
}

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_reduce(const int *__restrict__ len_ptr, int len_extra, const int *__restrict__ in,
              int *__restrict__ block_sums)
{
    const int len = *len_ptr + len_extra;
    const int base = blockIdx.x * SCAN_TILE;
    if (base >= len) return;
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        const int i = base + k * SCAN_THREADS + threadIdx.x;
        if (i < len) s += in[i];
    }
    __shared__ int sm[64];
    int total;
    block_exclusive_scan(s, sm, total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_top(const int *__restrict__ len_ptr, int len_extra, int *__restrict__ block_sums)
{
    const int len = *len_ptr + len_extra;
    const int nb = (len + SCAN_TILE - 1) / SCAN_TILE;
    __shared__ int sm[64];
    int carry = 0;
    for (int base = 0; base < nb; base += SCAN_THREADS) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? block_sums[i] : 0;
        int total;
        const int ex = block_exclusive_scan(v, sm, total);
        if (i < nb) block_sums[i] = carry + ex;
        carry += total;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_apply(const int *__restrict__ len_ptr, int len_extra, const int *__restrict__ in,
             const int *__restrict__ block_sums, int *__restrict__ out)
{
    const int len = *len_ptr + len_extra;
    const int base = blockIdx.x * SCAN_TILE;
    if (base >= len) return;
    // thread t owns SCAN_ITEMS consecutive elements
    const int first = base + threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        v[k] = (first + k) < len ? in[first + k] : 0;
        s += v[k];
    }
    __shared__ int sm[64];
    int total;
    int run = block_sums[blockIdx.x] + block_exclusive_scan(s, sm, total);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if ((first + k) < len) out[first + k] = run;
        run += v[k];
    }
}

// The same exclusive scan by ONE block, tile after tile with a running carry: for the search
// grids of small crowds (a few tiles) one launch instead of three -- those steps are bound by
// launch latency, not by work (1,024 agents: 13 dependent kernels in ~0.09 ms).
__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_small(const int *__restrict__ len_ptr, int len_extra, const int *__restrict__ in, int *__restrict__ out)
{
    const int len = *len_ptr + len_extra;
    __shared__ int sm[64];
    int carry = 0;
    for (int base = 0; base < len; base += SCAN_TILE) {
        const int first = base + threadIdx.x * SCAN_ITEMS;
        int v[SCAN_ITEMS];
        int s = 0;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            v[k] = (first + k) < len ? in[first + k] : 0;
            s += v[k];
        }
        int total;
        int run = carry + block_exclusive_scan(s, sm, total);
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            if ((first + k) < len) out[first + k] = run;
            run += v[k];
        }
        carry += total;
    }
}

// Everything the removal of arrivals needs before the rows move, for a SMALL crowd, by one block
// (k_keep_flags + scan, k_keep_by_logical + scan: eight launches of a few microseconds each --
// a 2,500-agent frame is a chain of ~26 dependent launches and nothing else).
#ifndef ORCA_SMALL_ROWS
#define ORCA_SMALL_ROWS 16384
#endif
__device__ __forceinline__ void block_scan_tiles(int len, const int *in, int *out, int *sm)
{
    int carry = 0;
    for (int base = 0; base < len; base += SCAN_TILE) {
        const int first = base + threadIdx.x * SCAN_ITEMS;
        int v[SCAN_ITEMS];
        int s = 0;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            v[k] = (first + k) < len ? in[first + k] : 0;
            s += v[k];
        }
        int total;
        int run = carry + block_exclusive_scan(s, sm, total);
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            if ((first + k) < len) out[first + k] = run;
            run += v[k];
        }
        carry += total;
        __syncthreads(); // sm is reused by the next tile
    }
}

__global__ void __launch_bounds__(SCAN_THREADS)
k_removal_scans_small(const GridPlan *__restrict__ plan, const u8 *__restrict__ arrived, int remove_arrivals,
                      int *keep, int *dst_idx, const int *__restrict__ lrow, int *lkeep, int *lscan)
{
    __shared__ int sm[64];
    const int n = plan->n, n_owned = plan->n_owned;
    for (int i = threadIdx.x; i <= n; i += SCAN_THREADS)
        keep[i] = (i < n_owned && !(remove_arrivals && arrived[i])) ? 1 : 0; // (k_keep_flags)
    __syncthreads();
    block_scan_tiles(n + 1, keep, dst_idx, sm);
    if (!lrow) return;
    for (int i = threadIdx.x; i <= n; i += SCAN_THREADS) { // (k_keep_by_logical)
        if (i == n) lkeep[n] = 0;
        else lkeep[lrow[i]] = keep[i];
    }
    __syncthreads();
    block_scan_tiles(n + 1, lkeep, lscan, sm);
}

// Scatter into cell-sorted order. Writes, per sorted slot s:
//   s_xy  (x, y)                         candidate stream of the neighbour search
//   s_nr  (x, y, vx, vy | radius, class code | pad)   pre-step snapshot, one 32 B record (NbRec):
//                                                      what neighbours read of an agent
//   s_dm  (des_vx, des_vy, max_speed, avoid_radius)   own LP inputs, arithmetic type
//   s_row storage row, s_cell search cell
template <typename S, typename R>
__global__ void __launch_bounds__(256)
k_scatter(const GridPlan *__restrict__ plan, StepParams P,
          const typename Vec<S>::T4 *__restrict__ pv, const typename Vec<S>::T4 *__restrict__ goalpref,
          const typename Vec<S>::T2 *__restrict__ radmax, const u8 *__restrict__ cls,
          const int *__restrict__ cell_of, const int *__restrict__ rank_of,
          const int *__restrict__ cell_start, typename Vec<S>::T2 *__restrict__ s_xy,
          NbRec<S> *__restrict__ s_nr, typename Vec<R>::T4 *__restrict__ s_dm,
          int *__restrict__ s_row, int *__restrict__ s_cell)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= plan->n) return;
    const int c = cell_of[i];
    const int s = cell_start[c] + rank_of[i];
    const typename Vec<S>::T4 a = pv[i];
    const typename Vec<S>::T4 g = goalpref[i]; // gx, gy, pref_speed, goal_tol
    const typename Vec<S>::T2 rm = radmax[i];  // radius, max_speed
    // engine.py:133-139
    const R dx = (R)g.x - (R)a.x, dy = (R)g.y - (R)a.y;
    const R dist = sqrt_rn<R>(dx * dx + dy * dy);
    R speed = div_rn<R>(dist, (R)P.dt);
    if ((R)g.z < speed) speed = (R)g.z;
    const R scale = dist > R(0) ? div_rn<R>(speed, dist) : R(0);
    // engine.py:227 (evaluated in FP64, then rounded to R)
    const R avoid = (R)((double)rm.x + P.half_margin);
    s_xy[s] = mk2(a.x, a.y);
    NbRec<S> rec;
    rec.pv = a;
    rec.rc = mk2(rm.x, (S)cls[i]); // radius and class: what a neighbour needs besides pv
    rec.pad = mk2(S(0), S(0));
    s_nr[s] = rec;
    s_dm[s] = mk4(dx * scale, dy * scale, (R)rm.y, avoid);
    s_row[s] = i;
    s_cell[s] = c;
}

// ---------------------------------------------------------------------------
// K2: neighbour gather
// ---------------------------------------------------------------------------

#define ORCA_INF __longlong_as_double(0x7FF0000000000000LL)

// The kept list of one agent, in registers, ascending by (d2, id). Slots
// [0, MAXN-max_n) hold -1 sentinels so the admission threshold is always the last
// register. Keys are FP64 d2 = dx*dx + dy*dy evaluated exactly like
// _kernels.py:467-469 (no FMA), so the list is bit-identical to the reference's
// whenever the positions are representable in the storage type.
template <int MAXN> struct TopK {
    double key[MAXN];
    int idx[MAXN];
    int cnt;

    __device__ __forceinline__ void init(int max_n)
    {
        const int off = MAXN - max_n;
#pragma unroll
        for (int t = 0; t < MAXN; ++t) {
            key[t] = t < off ? -1.0 : ORCA_INF;
            idx[t] = -1;
        }
        cnt = 0;
    }

    // _kernels.py:473-489: admit (d2, id) if it precedes the current last entry, then
    // shift it into place. Returns true if the list changed.
    __device__ __forceinline__ bool insert(double d2, int s2, int max_n, const int *__restrict__ s_row,
                                           const i64 *__restrict__ ids)
    {
        const double last = key[MAXN - 1];
        if (d2 > last) return false;
        i64 my_id = 0;
        bool have_id = false;
        if (d2 == last) {
            my_id = ids[s_row[s2]];
            have_id = true;
            if (my_id >= ids[s_row[idx[MAXN - 1]]]) return false;
        }
        bool c_next = true;
#pragma unroll
        for (int p = MAXN - 1; p >= 1; --p) {
            bool cp = d2 < key[p - 1];
            if (d2 == key[p - 1]) {
                if (!have_id) {
                    my_id = ids[s_row[s2]];
                    have_id = true;
                }
                cp = my_id < ids[s_row[idx[p - 1]]];
            }
            if (cp) {
                key[p] = key[p - 1];
                idx[p] = idx[p - 1];
            } else if (c_next) {
                key[p] = d2;
                idx[p] = s2;
            }
            c_next = cp;
        }
        if (c_next) {
            key[0] = d2;
            idx[0] = s2;
        }
        cnt = min(cnt + 1, max_n);
        return true;
    }

    // slot-major neighbour table + count + next step's radius hint
    __device__ __forceinline__ void store(int s, int row, int max_n, int stride, int *__restrict__ nb,
                                          u8 *__restrict__ nb_cnt, float *__restrict__ hint) const
    {
        const int off = MAXN - max_n;
        nb_cnt[s] = (u8)cnt;
#pragma unroll
        for (int t = 0; t < MAXN; ++t) {
            const int slot = t - off;
            if (slot >= 0 && slot < cnt) nb[(size_t)slot * stride + s] = idx[t];
        }
        // radius that held the whole list this step (rounded up); +inf when fewer than
        // max_n agents are in range, so the next fast pass scans the full radius
        hint[row] = cnt == max_n ? __double2float_ru(__dsqrt_ru(key[MAXN - 1])) : __int_as_float(0x7F800000);
    }
};

// Fast pass, one thread per agent in cell-sorted order. It relies on temporal coherence but
// never on it for correctness: last step every kept neighbour was within `hint`, and nobody
// moves faster than its max_speed, so this step at least max_n agents are within
//   b = hint + (my max_speed + fastest max_speed) * dt.
// The thread scans the cells covering b once and appends every candidate passing an FP32
// distance test to a small shared-memory buffer. The result is accepted only if it is
// provably the exact list (see below); otherwise the agent goes to the queue of the exact
// ring search (k_gather): no hint yet, a removed neighbour, a teleported agent, an exact tie,
// or more than CAP candidates. The buffered candidates are ranked by ONE 32-bit integer each,
//     key = (bits of the FP32 squared distance with the low 6 mantissa bits cleared) | slot
// where slot < 64 is the candidate's position in the shared-memory buffer. Positive
// floats order like their bit patterns, so the sorting network and the insertion of the
// candidates beyond max_n are plain integer min / max pairs (2 instructions per
// compare-exchange, 16 registers for the list, against an FP64 compare + 6 selects and 48
// registers). The order is the exact (d2, id) order whenever neighbouring keys differ by
// at least 2 units of the kept 17 mantissa bits (2^-17 relative; FP32 evaluation error is
// below 2^-21), which is checked on the final list and against the closest rejected
// candidate; otherwise -- about 0.4 % of agents, and every exact tie -- the agent is
// queued for k_gather. Nothing here decides a result that FP64 would decide differently.
template <typename R, int MAXN, int CAP>
__global__ void __launch_bounds__(128)
k_gather_fast32(GridPlan *__restrict__ plan, StepParams P, const typename Vec<R>::T2 *__restrict__ s_xy,
                const int *__restrict__ cell_start, const int *__restrict__ s_cell,
                const int *__restrict__ s_row, const typename Vec<R>::T2 *__restrict__ radmax,
                float *__restrict__ hint, int *__restrict__ nb, u8 *__restrict__ nb_cnt,
                int *__restrict__ gq, int *__restrict__ gq_cnt, int s0, int s1)
{
    static_assert(CAP <= 64, "slot must fit the 6 cleared mantissa bits");
    __shared__ int buf[CAP * 128];
    const int s = s0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= min(s1, plan->n)) return;
    const int row = s_row[s];
    if (row >= plan->n_owned || P.max_n == 0) {
        nb_cnt[s] = 0;
        return;
    }
    const float h = hint[row];
    const double rad2 = P.rad2;
    const int max_n = P.max_n;
    const typename Vec<R>::T2 me = s_xy[s];
    const double mx = (double)me.x, my = (double)me.y;
    double b = (double)h + ((double)radmax[row].y + plan->vmax) * P.dt * (1.0 + 1e-6) + 1e-3;
    const double T = fmin(b * b, rad2);
    const float T_f = __double2float_ru(T * (1.0 + 1e-6));
    // FP32 band around rad2 that the FP32 squared distance cannot resolve (its error is
    // below 2^-22 relative; the band is 1e-6 on either side)
    const float cut_lo = __double2float_rd(rad2 * (1.0 - 1e-6)), cut_hi = __double2float_ru(rad2 * (1.0 + 1e-6));

    const int nx = plan->nx, ny = plan->ny;
    const int c0 = s_cell[s];
    const int cx = c0 / ny, cy = c0 - cx * ny;
    const int r = min(plan->rmax, (int)(sqrt(T) * plan->inv_cell * (1.0 + 1e-9)) + 1);
    const int gx_lo = max(cx - r, 0), gx_hi = min(cx + r, nx - 1);
    const int y_lo = max(cy - r, 0), y_hi = min(cy + r, ny - 1);
    int *my_buf = buf + threadIdx.x;

    auto d2_f32 = [&](const typename Vec<R>::T2 &q) -> float {
        float dxf, dyf;
        if (Fmt<R>::is_f32) {
            dxf = (float)q.x - (float)me.x;
            dyf = (float)q.y - (float)me.y;
        } else {
            dxf = (float)((double)q.x - mx);
            dyf = (float)((double)q.y - my);
        }
        return __fmaf_rn(dxf, dxf, dyf * dyf); // one rounding fewer than mul+add: inside the same error bound
    };

    int nbuf = 0;
    const float cell_f = (float)plan->cell * (1.0f - 1e-6f), inv_cell_f = (float)plan->inv_cell * (1.0f + 1e-6f);
    // Clip each column's rows to the circle: everything in column gx is at least
    // (|gx - cx| - 1) cells away in x (cell indices are monotone in x), so only rows within
    // sqrt(T - that^2) of mine, rounded up by a cell, can hold a candidate. The candidate
    // range of the NEXT column is requested while this column is scanned.
    auto column_range = [&](int gx, int &first, int &end) {
        const float dxc = (float)max(abs(gx - cx) - 1, 0) * cell_f;
        const int ry = (int)(sqrtf(fmaxf(T_f - dxc * dxc, 0.0f)) * inv_cell_f) + 1;
        const int *cs = cell_start + gx * ny;
        first = cs[max(cy - ry, y_lo)];
        end = cs[min(cy + ry, y_hi) + 1];
    };
    int a_next, e_next;
    column_range(gx_lo, a_next, e_next);
    for (int gx = gx_lo; gx <= gx_hi; ++gx) {
        const int a0 = a_next, e = e_next;
        if (gx < gx_hi) column_range(gx + 1, a_next, e_next);
        constexpr int kScanUnroll = ORCA_SCAN_UNROLL;
#pragma unroll kScanUnroll
        for (int s2 = a0; s2 < e; ++s2) {
            // (one predicated store, no branch: past CAP the last slot is overwritten, and the
            //  count alone sends the agent to the exact search)
            const bool pass = d2_f32(s_xy[s2]) <= T_f && s2 != s;
            if (pass) my_buf[min(nbuf, CAP - 1) * 128] = s2;
            nbuf += pass ? 1 : 0;
        }
    }
    bool ok = nbuf <= CAP;
    if (ok) {
        // The d2 <= rad2 cut (K:470) in FP32: candidates clearly outside are dropped, a
        // candidate within the rounding band around rad2 sends the agent to the exact
        // search. Both tests are vacuous unless the scan reaches the whole radius.
        bool near_cut = false;
        auto make_key = [&](int e) -> unsigned {
            const float d2f = d2_f32(s_xy[my_buf[e * 128]]);
            near_cut = near_cut || (d2f >= cut_lo && d2f <= cut_hi);
            return d2f > cut_hi ? 0xFFFFFFFFu : ((__float_as_uint(d2f) & ~63u) | (unsigned)e);
        };
        // sentinels 0 in front so the list proper is the last max_n registers
        const int off = MAXN - max_n;
        unsigned key[MAXN];
#pragma unroll
        for (int t = 0; t < MAXN; ++t) {
            const int e = t - off;
            key[t] = e < 0 ? 0u : 0xFFFFFFFFu;
            if (e >= 0 && e < nbuf) key[t] = make_key(e);
        }
#define CEX(a, b)                                                                                  \
    {                                                                                              \
        const unsigned lo_ = min(key[a], key[b]), hi_ = max(key[a], key[b]);                       \
        key[a] = lo_;                                                                              \
        key[b] = hi_;                                                                              \
    }
        if constexpr (MAXN == 16) {
            ORCA_SORTNET_16
        } else {
            ORCA_SORTNET_32
        }
#undef CEX
        // the candidates beyond max_n: min/max chain through the sorted list; what falls
        // off the end is rejected, and the closest rejected key is remembered
        unsigned rej = 0xFFFFFFFFu;
        for (int e = max_n; e < nbuf; ++e) {
            unsigned x = make_key(e);
#pragma unroll
            for (int t = 0; t < MAXN; ++t) {
                const unsigned lo_ = min(key[t], x);
                x = max(key[t], x);
                key[t] = lo_;
            }
            rej = min(rej, x);
        }
        // separated by >= 2 units of the kept mantissa bits => same order as exact (d2, id)
        int cnt = 0;
        unsigned prev = 0u; // sentinel / nothing
#pragma unroll
        for (int t = 0; t < MAXN; ++t) {
            const bool real = t >= off && key[t] != 0xFFFFFFFFu;
            if (real) {
                ok = ok && ((key[t] >> 6) >= (prev >> 6) + 2u);
                prev = key[t];
                ++cnt;
            }
        }
        if (rej != 0xFFFFFFFFu) ok = ok && ((rej >> 6) >= (prev >> 6) + 2u);
        ok = ok && !near_cut;
        // exact squared distance of the last kept entry: the acceptance test and the hint
        double d2_last = 0.0;
        if (cnt > 0) {
            const typename Vec<R>::T2 q = s_xy[my_buf[(int)(prev & 63u) * 128]]; // prev = last real key
            const double dx = (double)q.x - mx, dy = (double)q.y - my;
            d2_last = dx * dx + dy * dy;
        }
        ok = ok && (T >= rad2 || (cnt == max_n && d2_last <= T));
        if (ok) {
            nb_cnt[s] = (u8)cnt;
#pragma unroll
            for (int t = 0; t < MAXN; ++t) {
                const int slot = t - off;
                if (slot >= 0 && slot < cnt) nb[(size_t)slot * P.stride + s] = my_buf[(int)(key[t] & 63u) * 128];
            }
            hint[row] = cnt == max_n ? __double2float_ru(__dsqrt_ru(d2_last)) : __int_as_float(0x7F800000);
            return;
        }
    }
    gq[atomicAdd(gq_cnt, 1)] = s;
}

// grid.query_neighbors without a cap on the count (orca_neighbor_query_all): EVERY agent within the
// radius, ordered by (d2, id) (G:60-83). Thread per sorted slot over the search grid of the bin
// build; pass 0 counts (cnt[row]), pass 1 -- after a scan of the counts -- writes the rows at
// off[row] and orders its own segment by insertion (the segments of an object-level query are
// short; the step itself never comes here). Same FP64 operations as the reference: d2 = dx*dx +
// dy*dy, kept unless d2 > radius*radius.
template <int PASS>
__global__ void __launch_bounds__(128)
k_neighbors_all(const GridPlan *__restrict__ plan, double rad2, const double2 *__restrict__ s_xy,
                const int *__restrict__ cell_start, const int *__restrict__ s_cell, const int *__restrict__ s_row,
                const i64 *__restrict__ ids, int *__restrict__ cnt, const int *__restrict__ off,
                double *__restrict__ keys, i64 *__restrict__ rows)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = plan->n;
    if (PASS == 0 && s == n) cnt[n] = 0; // (the scan runs over n + 1 entries: off[n] = total)
    if (s >= n) return;
    const int nx = plan->nx, ny = plan->ny, r = plan->rmax;
    const double2 me = s_xy[s];
    const int row = s_row[s];
    const int c0 = s_cell[s];
    const int cx = c0 / ny, cy = c0 - cx * ny;
    const int y_lo = max(cy - r, 0), y_hi = min(cy + r, ny - 1);
    const int base = PASS ? off[row] : 0;
    int m = 0;
    for (int gx = max(cx - r, 0); gx <= min(cx + r, nx - 1); ++gx) {
        const int a = cell_start[gx * ny + y_lo], e = cell_start[gx * ny + y_hi + 1];
        for (int s2 = a; s2 < e; ++s2) {
            if (s2 == s) continue;
            const double2 q = s_xy[s2];
            const double dx = q.x - me.x, dy = q.y - me.y;
            const double d2 = dx * dx + dy * dy;
            if (d2 > rad2) continue;
            if (PASS) {
                const i64 row2 = (i64)s_row[s2];
                const i64 id2 = ids[row2];
                int at = m; // insertion into the ordered prefix [base, base + m)
                while (at > 0) {
                    const double kp = keys[base + at - 1];
                    if (kp < d2 || (kp == d2 && ids[rows[base + at - 1]] < id2)) break;
                    keys[base + at] = kp;
                    rows[base + at] = rows[base + at - 1];
                    --at;
                }
                keys[base + at] = d2;
                rows[base + at] = row2;
            }
            ++m;
        }
    }
    if (!PASS) cnt[row] = m;
}

// Exact ring search for the agents the fast pass queued (all of them on the first step
// after an upload). The search grid is walked in growing square rings around the
// agent's cell; it stops as soon as the list is full and every unscanned cell is
// provably farther than its last entry. The FP32 build pre-filters with an FP32
// distance against a slightly inflated threshold before touching FP64.
template <typename R, int MAXN>
__global__ void __launch_bounds__(128)
k_gather(const GridPlan *__restrict__ plan, StepParams P,
         const typename Vec<R>::T2 *__restrict__ s_xy, const int *__restrict__ cell_start,
         const int *__restrict__ s_cell, const int *__restrict__ s_row,
         const i64 *__restrict__ ids, float *__restrict__ hint, int *__restrict__ nb,
         u8 *__restrict__ nb_cnt, const int *__restrict__ gq, const int *__restrict__ gq_cnt)
{
    const int nq = *gq_cnt;
    const int nx = plan->nx, ny = plan->ny, rmax = plan->rmax;
    const double cell = plan->cell;
    const double rad2 = P.rad2;
    const int max_n = P.max_n;
    // A short queue (the steady state: the few agents the fast pass could not certify) is
    // spread over the warps of the grid, L entries per warp: with 32 unrelated searches in
    // one warp every insertion of any lane stalls the other 31, and the kernel's time is the
    // latency of its slowest warp. L reaches 32 (the plain thread-per-agent mapping, which
    // keeps neighbouring agents in neighbouring lanes) when everyone is queued.
    const int total_warps = gridDim.x * (blockDim.x >> 5);
    const int L = min(32, max(1, (nq + total_warps - 1) / total_warps));
    const int lane = threadIdx.x & 31;
    const int warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    // One entry per warp at most: the whole warp searches for it. The lanes stride over the
    // candidate ranges (coalesced), the in-range candidates are compacted into shared memory
    // with their exact FP64 keys, and max_n + 1 rounds of a warp-wide arg-min pick the list in
    // order. A single thread needs ~40 us for this (~90 candidates, ~50 register insertions of
    // 115 instructions, every load exposed); the warp ~6. Exactly equal keys -- the order is
    // then decided by id (K:473-476) -- or more than WCAP candidates send the entry to the
    // single-lane search below, which handles everything.
    constexpr int WCAP = 256;
    __shared__ double w_key[4][WCAP];
    __shared__ int w_idx[4][WCAP];
    bool warp_done = false;
    if (L == 1 && warp < nq && max_n <= 31) { // (uniform per warp; grid >= nq warps when L == 1)
        double *wk = w_key[threadIdx.x >> 5];
        int *wi = w_idx[threadIdx.x >> 5];
        const int s = gq[warp];
        const typename Vec<R>::T2 me = s_xy[s];
        const double mx = (double)me.x, my = (double)me.y;
        const int c0 = s_cell[s];
        const int cx = c0 / ny, cy = c0 - cx * ny;
        const unsigned lt = (1u << lane) - 1u;
        // start at the ring that held last step's list, when there was one (an entry of a
        // short queue normally has a finite hint: the fast pass only failed to certify it)
        int r = plan->r0;
        const float h = hint[s_row[s]];
        if (h < 1e30f) r = max(r, min(rmax, (int)((double)h * plan->inv_cell) + 1));
        bool bail = false;
        while (true) {
            const int gx_lo = max(cx - r, 0), gx_hi = min(cx + r, nx - 1);
            const int y_lo = max(cy - r, 0), y_hi = min(cy + r, ny - 1);
            if (gx_hi - gx_lo >= 32) { // (never with rmax <= 15; keeps the lane-per-column load valid)
                bail = true;
                break;
            }
            // lane c fetches the candidate range of column gx_lo + c: all columns at once
            int col_a = 0, col_e = 0;
            if (gx_lo + lane <= gx_hi) {
                const int *cs = cell_start + (gx_lo + lane) * ny;
                col_a = cs[y_lo];
                col_e = cs[y_hi + 1];
            }
            int count = 0;
            for (int gx = gx_lo; gx <= gx_hi; ++gx) {
                const int a = __shfl_sync(0xFFFFFFFFu, col_a, gx - gx_lo);
                const int e = __shfl_sync(0xFFFFFFFFu, col_e, gx - gx_lo);
                for (int base = a; base < e; base += 32) {
                    const int s2 = base + lane;
                    bool pass = false;
                    double d2 = 0.0;
                    if (s2 < e && s2 != s) {
                        const typename Vec<R>::T2 q = s_xy[s2];
                        const double dx = (double)q.x - mx, dy = (double)q.y - my;
                        d2 = dx * dx + dy * dy;
                        pass = !(d2 > rad2);
                    }
                    const unsigned m = __ballot_sync(0xFFFFFFFFu, pass);
                    const int at = count + __popc(m & lt);
                    if (pass && at < WCAP) {
                        wk[at] = d2;
                        wi[at] = s2;
                    }
                    count += __popc(m);
                }
            }
            if (count > WCAP) {
                bail = true;
                break;
            }
            __syncwarp();
            // max_n + 1 smallest keys in ascending order; lane t keeps the t-th
            double my_key = ORCA_INF, prev = -1.0;
            int my_s2 = -1, found = 0;
            bool tie = false;
            for (int t = 0; t <= max_n && t < count; ++t) {
                double best = ORCA_INF;
                int best_at = -1;
                for (int e = lane; e < count; e += 32) {
                    const double k = wk[e];
                    if (k < best) {
                        best = k;
                        best_at = e;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ok_ = __shfl_xor_sync(0xFFFFFFFFu, best, o);
                    const int oa = __shfl_xor_sync(0xFFFFFFFFu, best_at, o);
                    if (ok_ < best || (ok_ == best && oa >= 0 && (best_at < 0 || oa < best_at))) {
                        best = ok_;
                        best_at = oa;
                    }
                }
                // (all lanes agree on best / best_at now)
                tie = tie || best == prev;
                prev = best;
                if (t < max_n) {
                    if (lane == t) {
                        my_key = best;
                        my_s2 = wi[best_at];
                    }
                    found = t + 1;
                }
                __syncwarp(); // every lane has read the keys of this round
                if (lane == 0) wk[best_at] = ORCA_INF; // taken
                __syncwarp();
            }
            if (tie) {
                bail = true;
                break;
            }
            // ring termination, as in the single-lane search
            if (r >= rmax) {
                bail = false;
            } else if (found == max_n) {
                const double d_last = __shfl_sync(0xFFFFFFFFu, my_key, max_n - 1);
                const double reach = (double)r * cell;
                if (!(d_last < reach * reach * (1.0 - 1e-9))) {
                    const int need = (int)(sqrt(d_last) / cell * (1.0 + 1e-9)) + 1;
                    r = min(rmax, max(r + 1, need));
                    __syncwarp();
                    continue;
                }
            } else {
                r = min(rmax, r + 1);
                __syncwarp();
                continue;
            }
            // store: slot-major table, count, next step's radius hint
            const int row = s_row[s];
            if (lane < found) nb[(size_t)lane * P.stride + s] = my_s2;
            const double d_last = __shfl_sync(0xFFFFFFFFu, my_key, max(found - 1, 0));
            if (lane == 0) {
                nb_cnt[s] = (u8)found;
                hint[row] = found == max_n ? __double2float_ru(__dsqrt_ru(d_last)) : __int_as_float(0x7F800000);
            }
            break;
        }
        warp_done = !bail;
    }
    if (L == 1 && warp_done) return;
    if (lane >= L) return;
    for (int qi = warp * L + lane; qi < nq; qi += total_warps * L) {
        const int s = gq[qi];
        const int row = s_row[s];
        const typename Vec<R>::T2 me = s_xy[s];
        const double mx = (double)me.x, my = (double)me.y;
        const int c0 = s_cell[s];
        const int cx = c0 / ny, cy = c0 - cx * ny;

        TopK<MAXN> top;
        top.init(max_n);
        float thr_f = __double2float_ru(rad2 * (1.0 + 1e-6));

        auto scan_range = [&](int a, int b) {
            for (int s2 = a; s2 < b; ++s2) {
                const typename Vec<R>::T2 q = s_xy[s2];
                if (Fmt<R>::is_f32) {
                    const float dxf = (float)q.x - (float)me.x, dyf = (float)q.y - (float)me.y;
                    if (dxf * dxf + dyf * dyf > thr_f) continue;
                }
                const double dx = (double)q.x - mx, dy = (double)q.y - my;
                const double d2 = dx * dx + dy * dy;
                if (s2 == s || d2 > rad2) continue;
                if (top.insert(d2, s2, max_n, s_row, ids) && Fmt<R>::is_f32)
                    thr_f = __double2float_ru(fmin(top.key[MAXN - 1], rad2) * (1.0 + 1e-6));
            }
        };

        int r_done = -1;
        int r_next = plan->r0;
        while (true) {
            const int gx_lo = max(cx - r_next, 0), gx_hi = min(cx + r_next, nx - 1);
            const int y_lo = max(cy - r_next, 0), y_hi = min(cy + r_next, ny - 1);
            for (int gx = gx_lo; gx <= gx_hi; ++gx) {
                const int *cs = cell_start + gx * ny;
                if (abs(gx - cx) > r_done) {
                    scan_range(cs[y_lo], cs[y_hi + 1]);
                } else {
                    const int b_hi = cy - r_done - 1;
                    if (b_hi >= y_lo) scan_range(cs[y_lo], cs[b_hi + 1]);
                    const int t_lo = cy + r_done + 1;
                    if (t_lo <= y_hi) scan_range(cs[t_lo], cs[y_hi + 1]);
                }
            }
            r_done = r_next;
            if (r_done >= rmax) break;
            if (top.cnt == max_n) {
                // Every unscanned agent is farther than r_done*cell (1e-9 margin for the
                // rounding of the cell index); stop once the kept list is closer than that.
                const double d_last = top.key[MAXN - 1];
                const double reach = (double)r_done * cell;
                if (d_last < reach * reach * (1.0 - 1e-9)) break;
                const int need = (int)(sqrt(d_last) / cell * (1.0 + 1e-9)) + 1;
                r_next = min(rmax, max(r_done + 1, need));
            } else {
                r_next = min(rmax, r_done + 1);
            }
        }
        top.store(s, row, max_n, P.stride, nb, nb_cnt, hint);
    }
}

// ---------------------------------------------------------------------------
// K3: constraints + LP
// ---------------------------------------------------------------------------

template <typename R> struct SmemCons {
    typename Vec<R>::T4 *base; // already offset by the thread index
    int stride;
    __device__ __forceinline__ void get(int pos, R &px, R &py, R &nx, R &ny) const
    {
        const typename Vec<R>::T4 c = base[pos * stride];
        px = c.x;
        py = c.y;
        nx = c.z;
        ny = c.w;
    }
    __device__ __forceinline__ void set(int pos, R px, R py, R nx, R ny)
    {
        base[pos * stride] = mk4(px, py, nx, ny);
    }
};

// identity-order view: original constraint t sits at shuffled position inv[t]
template <typename R> struct SmemConsIdent {
    const typename Vec<R>::T4 *base;
    const u8 *inv;
    int stride;
    __device__ __forceinline__ void get(int t, R &px, R &py, R &nx, R &ny) const
    {
        const typename Vec<R>::T4 c = base[(int)inv[t * stride] * stride];
        px = c.x;
        py = c.y;
        nx = c.z;
        ny = c.w;
    }
};

// Fisher-Yates order of _kernels.py:43-54 into perm[pos*stride]; MAXN <= 32.
template <int MAXN>
__device__ __forceinline__ void shuffle_smem(u8 *perm, int stride, int k, u64 seed)
{
    for (int t = 0; t < k; ++t) perm[t * stride] = (u8)t;
    u64 state = seed;
#pragma unroll
    for (int i = MAXN - 1; i > 0; --i) {
        if (i < k) {
            state += ORCA_GOLDEN;
            const int j = (int)(mix64(state) % (u64)(i + 1)); // constant divisor after unrolling
            const u8 tmp = perm[i * stride];
            perm[i * stride] = perm[j * stride];
            perm[j * stride] = tmp;
        }
    }
}

// An agent queued for the least-penetration stage takes its half-planes (in shuffled order,
// as they sit in shared memory) and its insertion order along: k_fallback_coop used to redo
// the Fisher-Yates shuffle (one lane, ~630 instructions) and the whole constraint build
// (16 vo_exit chains + 16 neighbour gathers) for every queued agent -- a quarter of its
// instructions. MAXN * (sizeof(R4) + 1) bytes per queued agent go through L2/HBM instead.
template <typename R, int MAXN>
__device__ __forceinline__ void spill_constraints(typename Vec<R>::T4 *__restrict__ fq_cons,
                                                  u8 *__restrict__ fq_perm, int q, int cnt,
                                                  const typename Vec<R>::T4 *cons_base, const u8 *perm,
                                                  int stride, int first, int step)
{
    typename Vec<R>::T4 *dst = fq_cons + (size_t)q * MAXN;
    u8 *dp = fq_perm + (size_t)q * MAXN;
    for (int pos = first; pos < cnt; pos += step) {
        dst[pos] = cons_base[pos * stride];
        dp[pos] = perm[pos * stride];
    }
}

// Build the ORCA half-planes of agent s into `cons` in SHUFFLED order
// (_kernels.py:525-541). Returns false on exactly coincident centres. (Walking the
// neighbour ranks and scattering to the inverse permutation instead was measured 6 %
// slower, profiles/r01_notes.md.)
template <typename S, typename R>
__device__ __forceinline__ bool build_constraints(
    int s, int cnt, const StepParams &P, const NbRec<S> *__restrict__ s_nr,
    const int *__restrict__ nb, const u8 *perm,
    int stride, SmemCons<R> &cons, int &bad_j)
{
    const typename Vec<S>::T4 me_s = s_nr[s].pv;
    const R mex = (R)me_s.x, mey = (R)me_s.y, mevx = (R)me_s.z, mevy = (R)me_s.w;
    const typename Vec<S>::T2 rc_i = s_nr[s].rc;
    const R ri = (R)((double)rc_i.x + P.half_margin); // engine.py:227, as in k_scatter
    const int ci = (int)rc_i.y;
    const R inv_tau = div_rn<R>(R(1), (R)P.tau), inv_dt = div_rn<R>(R(1), (R)P.dt); // K:358 / K:378, once
    const R f0 = (R)(ci ? P.fmat[2] : P.fmat[0]), f1 = (R)(ci ? P.fmat[3] : P.fmat[1]); // no dynamic index: keeps P out of local memory
    bool ok_all = true;
    // software pipeline, as in k_solve_group: next neighbour's record requested one iteration ahead
    typename Vec<S>::T4 q_next = me_s;
    typename Vec<S>::T2 rc_next = rc_i;
    if (cnt > 0) {
        const int jn = nb[(size_t)perm[0] * P.stride + s];
        const NbRec<S> rn = s_nr[jn];
        q_next = rn.pv;
        rc_next = rn.rc;
    }
    for (int pos = 0; pos < cnt; ++pos) {
        const typename Vec<S>::T4 q = q_next;
        const typename Vec<S>::T2 rc_j = rc_next;
        if (pos + 1 < cnt) {
            const int jn = nb[(size_t)perm[(pos + 1) * stride] * P.stride + s];
            const NbRec<S> rn = s_nr[jn];
            q_next = rn.pv;
            rc_next = rn.rc;
        }
        const R rj = (R)((double)rc_j.x + P.half_margin);
        R ux, uy, nx, ny;
        ok_all &= vo_exit_inv<R>((R)q.x - mex, (R)q.y - mey, mevx - (R)q.z, mevy - (R)q.w, ri + rj, inv_tau,
                                 inv_dt, ux, uy, nx, ny);
        const R f = rc_j.y != S(0) ? f1 : f0; // fmat[cls_i, cls_j], _kernels.py:537
        cons.set(pos, mevx + f * ux, mevy + f * uy, nx, ny);
    }
    if (!ok_all) {
        // coincident neighbours have d2 == 0 and therefore lead the list; the reference
        // reports the first one in rank order (_kernels.py:533-536)
        bad_j = nb[s];
        return false;
    }
    return true;
}

// Integration + arrival test (engine.py:249-253) for storage row `row`.
template <typename S, typename R>
__device__ __forceinline__ void integrate_row(int row, const typename Vec<S>::T4 &me, R vx, R vy,
                                              const StepParams &P,
                                              const typename Vec<S>::T4 *__restrict__ goalpref,
                                              typename Vec<S>::T4 *__restrict__ pv_out,
                                              u8 *__restrict__ arrived)
{
    const R dt = (R)P.dt;
    const R nxp = (R)me.x + vx * dt, nyp = (R)me.y + vy * dt;
    pv_out[row] = mk4((S)nxp, (S)nyp, (S)vx, (S)vy);
    const typename Vec<S>::T4 g = goalpref[row];
    const R gx = (R)g.x - nxp, gy = (R)g.y - nyp;
    arrived[row] = sqrt_rn<R>(gx * gx + gy * gy) <= (R)g.w ? 1 : 0;
}

template <typename S, typename R, int MAXN, int THREADS>
__global__ void __launch_bounds__(THREADS)
k_solve(GridPlan *__restrict__ plan, StepParams P, const NbRec<S> *__restrict__ s_nr,
        const typename Vec<R>::T4 *__restrict__ s_dm,
        const int *__restrict__ s_row, const i64 *__restrict__ ids, const int *__restrict__ nb,
        const u8 *__restrict__ nb_cnt, const typename Vec<S>::T4 *__restrict__ goalpref,
        typename Vec<S>::T4 *__restrict__ pv_out, i8 *__restrict__ status,
        i8 *__restrict__ failed_at, u8 *__restrict__ arrived, int *__restrict__ fq,
        typename Vec<R>::T4 *__restrict__ fq_state, int s0, int s1, const int *__restrict__ lrow,
        typename Vec<R>::T4 *__restrict__ fq_cons, u8 *__restrict__ fq_perm, int *__restrict__ fq_cnt)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typename Vec<R>::T4 *sm_cons = reinterpret_cast<typename Vec<R>::T4 *>(smem_raw);
    u8 *sm_perm = smem_raw + sizeof(typename Vec<R>::T4) * MAXN * THREADS;

    const int s = s0 + blockIdx.x * THREADS + threadIdx.x; // sorted slots [s0, s1)
    const bool in_range = s < min(s1, plan->n);
    const int row = in_range ? s_row[s] : 0;
    const bool active = in_range && row < plan->n_owned; // halo ghosts are searched, never solved
    const unsigned live = __ballot_sync(0xFFFFFFFFu, active);
    if (!active) return;

    const int cnt = nb_cnt[s];
    const typename Vec<S>::T4 me = s_nr[s].pv;
    const typename Vec<R>::T4 dm = s_dm[s];
    u8 *perm = sm_perm + threadIdx.x;
    SmemCons<R> cons{sm_cons + threadIdx.x, THREADS};

    shuffle_smem<MAXN>(perm, THREADS, cnt, problem_seed(plan->frame, ids[row]));
    int bad_j = -1;
    const bool built = build_constraints<S, R>(s, cnt, P, s_nr, nb, perm, THREADS, cons, bad_j);
    int fail_pos;
    R vx, vy;
    const bool feasible =
        lp2_target_runahead<R, SmemCons<R>>(cons, cnt, dm.z, dm.x, dm.y, fail_pos, vx, vy, live, built);
    if (!built) {
        // _kernels.py:542-547 + engine.py:239-245
        if (plan->err_frame < 0) // sticky: only the first failing frame is reported
            atomicMin(&plan->err_pair, ((u64)(unsigned)lrow[row] << 32) | (u64)(unsigned)lrow[s_row[bad_j]]);
        status[row] = 0;
        failed_at[row] = -1;
        integrate_row<S, R>(row, me, (R)me.z, (R)me.w, P, goalpref, pv_out, arrived);
        return;
    }
    if (feasible) {
        status[row] = 0;
        failed_at[row] = -1;
        integrate_row<S, R>(row, me, vx, vy, P, goalpref, pv_out, arrived);
        return;
    }
    // queue for the least-penetration stage (warp-aggregated by the compiler)
    status[row] = 1;
    failed_at[row] = (i8)perm[fail_pos * THREADS];
    const int q = atomicAdd(fq_cnt, 1);
    fq[q] = s;
    fq_state[q] = mk4(vx, vy, (R)fail_pos, R(0));
    spill_constraints<R, MAXN>(fq_cons, fq_perm, q, cnt, sm_cons + threadIdx.x, perm, THREADS, 0, 1);
}

// The seeded Fisher-Yates order of every agent (K:43-61), one THREAD per agent. Inside
// k_solve_group one lane of each pair drew it while its partner idled (12 % of that kernel's
// warp instructions at half the lanes); here all 32 lanes of a warp draw. MAXN bytes per agent
// go through L2 to the solve kernel.
template <int MAXN>
__global__ void __launch_bounds__(128)
k_shuffle(const GridPlan *__restrict__ plan, const int *__restrict__ s_row, const i64 *__restrict__ ids,
          const u8 *__restrict__ nb_cnt, uint4 *__restrict__ s_perm, int s0, int s1)
{
    __shared__ __align__(16) u8 sm[MAXN * 128];
    const int s = s0 + blockIdx.x * 128 + threadIdx.x;
    if (s >= min(s1, plan->n)) return;
    const int row = s_row[s];
    if (row >= plan->n_owned) return;
    u8 *perm = sm + threadIdx.x;
    const int cnt = nb_cnt[s];
    shuffle_smem<MAXN>(perm, 128, cnt, problem_seed(plan->frame, ids[row]));
    uint32_t w[MAXN / 4];
#pragma unroll
    for (int t = 0; t < MAXN / 4; ++t)
        w[t] = (uint32_t)perm[(4 * t) * 128] | ((uint32_t)perm[(4 * t + 1) * 128] << 8) |
               ((uint32_t)perm[(4 * t + 2) * 128] << 16) | ((uint32_t)perm[(4 * t + 3) * 128] << 24);
#pragma unroll
    for (int t = 0; t < MAXN / 16; ++t)
        s_perm[(size_t)s * (MAXN / 16) + t] = make_uint4(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3]);
}

// k_solve with GL (2 or 4) adjacent lanes per agent. k_solve is bound by the latency of
// dependent FP64 chains at the 12 warps/SM its shared memory allows (512 B of constraints
// per thread). A group shares ONE agent's constraints, so the same shared memory holds GL
// times more threads, each with a 1/GL share of the serial work: lane gl builds the
// half-planes at positions gl, gl+GL, ..., the run-ahead scan is executed redundantly and
// the j loops of the 1-D solves are split over the group (max / min / any combinations:
// exact and order-independent, so results are unchanged).
template <typename S, typename R, int MAXN, int THREADS, int GL, bool PRESH>
__device__ __forceinline__ void
solve_group_body(int idx, bool in_range, int s,
              GridPlan *__restrict__ plan, StepParams P, const NbRec<S> *__restrict__ s_nr,
              const typename Vec<R>::T4 *__restrict__ s_dm,
              const int *__restrict__ s_row, const i64 *__restrict__ ids, const int *__restrict__ nb,
              const u8 *__restrict__ nb_cnt, const typename Vec<S>::T4 *__restrict__ goalpref,
              typename Vec<S>::T4 *__restrict__ pv_out, i8 *__restrict__ status,
              i8 *__restrict__ failed_at, u8 *__restrict__ arrived, int *__restrict__ fq,
              typename Vec<R>::T4 *__restrict__ fq_state, int s0, int s1, const int *__restrict__ lrow,
              typename Vec<R>::T4 *__restrict__ fq_cons, u8 *__restrict__ fq_perm,
              const uint32_t *__restrict__ s_perm, int *__restrict__ fq_cnt)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int NG = THREADS / GL; // agents per block
    typename Vec<R>::T4 *sm_cons = reinterpret_cast<typename Vec<R>::T4 *>(smem_raw);
    u8 *sm_perm = smem_raw + sizeof(typename Vec<R>::T4) * MAXN * NG;

    const int g = threadIdx.x / GL, gl = threadIdx.x % GL;
    const int gshift = (threadIdx.x & 31) - gl;
    const unsigned gmask = ((1u << GL) - 1u) << gshift;
    (void)idx;
    (void)s0;
    (void)s1;
    const int row = in_range ? s_row[s] : 0;
    const bool active = in_range && row < plan->n_owned;
    const unsigned live = __ballot_sync(0xFFFFFFFFu, active);
    if (!active) return; // uniform over the group

    const int cnt = nb_cnt[s];
    const typename Vec<S>::T4 me = s_nr[s].pv;
    const typename Vec<R>::T4 dm = s_dm[s];
    u8 *perm = sm_perm + g;
    SmemCons<R> cons{sm_cons + g, NG};

    if constexpr (PRESH) { // the order k_shuffle drew: lane gl copies words gl, gl + GL, ... (4 positions each)
        const uint32_t *src = s_perm + (size_t)s * (MAXN / 4);
        for (int t = gl; 4 * t < cnt; t += GL) {
            const uint32_t w = src[t];
            perm[(4 * t) * NG] = (u8)(w & 0xFFu);
            perm[(4 * t + 1) * NG] = (u8)((w >> 8) & 0xFFu);
            perm[(4 * t + 2) * NG] = (u8)((w >> 16) & 0xFFu);
            perm[(4 * t + 3) * NG] = (u8)(w >> 24);
        }
    } else { // small crowds: one launch fewer beats the idle lanes (separate instance: with both
             // paths in one kernel the register cap spills and the gain is gone)
        if (gl == 0) shuffle_smem<MAXN>(perm, NG, cnt, problem_seed(plan->frame, ids[row]));
    }
    __syncwarp(gmask);
    bool ok_mine = true;
    {   // constraints in shuffled order, one vo_exit per lane and round (K:525-541)
        const R mex = (R)me.x, mey = (R)me.y, mevx = (R)me.z, mevy = (R)me.w;
        const typename Vec<S>::T2 rc_i = s_nr[s].rc;
        const R ri = (R)((double)rc_i.x + P.half_margin);
        const int ci = (int)rc_i.y;
        const R f0 = (R)(ci ? P.fmat[2] : P.fmat[0]), f1 = (R)(ci ? P.fmat[3] : P.fmat[1]); // no dynamic index: keeps P out of local memory
        const R inv_tau = div_rn<R>(R(1), (R)P.tau), inv_dt = div_rn<R>(R(1), (R)P.dt); // K:358 / K:378, once
        constexpr int kBuildUnroll = ORCA_BUILD_UNROLL;
        // software pipeline: the next neighbour's index and record are requested before this
        // neighbour's ~130-instruction FP64 chain starts, so their (L2) latency hides behind it
        typename Vec<S>::T4 q_next = me;
        typename Vec<S>::T2 rc_next = rc_i;
        if (gl < cnt) {
            const int jn = nb[(size_t)perm[gl * NG] * P.stride + s];
            const NbRec<S> rn = s_nr[jn];
            q_next = rn.pv;
            rc_next = rn.rc;
        }
#pragma unroll kBuildUnroll
        for (int pos = gl; pos < cnt; pos += GL) {
            const typename Vec<S>::T4 qv = q_next;
            const typename Vec<S>::T2 rc_j = rc_next;
            if (pos + GL < cnt) {
                const int jn = nb[(size_t)perm[(pos + GL) * NG] * P.stride + s];
                const NbRec<S> rn = s_nr[jn];
                q_next = rn.pv;
                rc_next = rn.rc;
            }
            const R rj = (R)((double)rc_j.x + P.half_margin);
            R ux, uy, nx, ny;
            ok_mine &= vo_exit_inv<R>((R)qv.x - mex, (R)qv.y - mey, mevx - (R)qv.z, mevy - (R)qv.w, ri + rj,
                                      inv_tau, inv_dt, ux, uy, nx, ny);
            const R f = rc_j.y != S(0) ? f1 : f0;
            cons.set(pos, mevx + f * ux, mevy + f * uy, nx, ny);
        }
    }
    __syncwarp(gmask); // the partner's half-planes are read from here on (a vote alone orders no memory)
    const bool built = (__ballot_sync(gmask, !ok_mine) & gmask) == 0u;
    int fail_pos;
    R vx, vy;
    const bool feasible = g_lp2_target_runahead<R, GL, false, SmemCons<R>>(
        cons, cnt, R(0), dm.z, dm.x, dm.y, fail_pos, vx, vy, live, built, gl, gmask);
    int q = 0;
    if (built && !feasible) { // uniform over the group: queue for the least-penetration stage
        if (gl == 0) q = atomicAdd(fq_cnt, 1);
        q = __shfl_sync(gmask, q, gshift);
        spill_constraints<R, MAXN>(fq_cons, fq_perm, q, cnt, sm_cons + g, perm, NG, gl, GL);
    }
    if (gl != 0) return;
    if (!built) {
        // _kernels.py:542-547 + engine.py:239-245; coincident neighbours lead the list
        if (plan->err_frame < 0)
            atomicMin(&plan->err_pair, ((u64)(unsigned)lrow[row] << 32) | (u64)(unsigned)lrow[s_row[nb[s]]]);
        status[row] = 0;
        failed_at[row] = -1;
        integrate_row<S, R>(row, me, (R)me.z, (R)me.w, P, goalpref, pv_out, arrived);
        return;
    }
    if (feasible) {
        status[row] = 0;
        failed_at[row] = -1;
        integrate_row<S, R>(row, me, vx, vy, P, goalpref, pv_out, arrived);
        return;
    }
    status[row] = 1;
    failed_at[row] = (i8)perm[fail_pos * NG];
    fq[q] = s;
    fq_state[q] = mk4(vx, vy, (R)fail_pos, R(0));
}

template <typename S, typename R, int MAXN, int THREADS, int GL, bool PRESH>
__global__ void __launch_bounds__(THREADS, (GL == 2 ? ORCA_SG_BLOCKS : 8))
k_solve_group(GridPlan *__restrict__ plan, StepParams P, const NbRec<S> *__restrict__ s_nr,
              const typename Vec<R>::T4 *__restrict__ s_dm,
              const int *__restrict__ s_row, const i64 *__restrict__ ids, const int *__restrict__ nb,
              const u8 *__restrict__ nb_cnt, const typename Vec<S>::T4 *__restrict__ goalpref,
              typename Vec<S>::T4 *__restrict__ pv_out, i8 *__restrict__ status,
              i8 *__restrict__ failed_at, u8 *__restrict__ arrived, int *__restrict__ fq,
              typename Vec<R>::T4 *__restrict__ fq_state, int s0, int s1, const int *__restrict__ lrow,
              typename Vec<R>::T4 *__restrict__ fq_cons, u8 *__restrict__ fq_perm,
              const uint32_t *__restrict__ s_perm, int *__restrict__ fq_cnt)
{
    const int idx = s0 + blockIdx.x * (THREADS / GL) + threadIdx.x / GL;
    solve_group_body<S, R, MAXN, THREADS, GL, PRESH>(idx, idx < min(s1, plan->n), idx, plan, P, s_nr, s_dm, s_row, ids, nb,
                                                     nb_cnt, goalpref, pv_out, status, failed_at, arrived, fq, fq_state,
                                                     s0, s1, lrow, fq_cons, fq_perm, s_perm, fq_cnt);
}

// The same for a QUEUE of sorted slots (ORCA_CERT32: the agents k_solve_cert could not certify,
// cq[0 .. plan->cq_count)): a fixed grid walks the queue, so the launch does not depend on a
// count only the device knows.
template <typename S, typename R, int MAXN, int THREADS, int GL, bool PRESH>
__global__ void __launch_bounds__(THREADS, (GL == 2 ? ORCA_SG_BLOCKS : 8))
k_solve_group_queue(GridPlan *__restrict__ plan, StepParams P, const NbRec<S> *__restrict__ s_nr,
                    const typename Vec<R>::T4 *__restrict__ s_dm,
                    const int *__restrict__ s_row, const i64 *__restrict__ ids, const int *__restrict__ nb,
                    const u8 *__restrict__ nb_cnt, const typename Vec<S>::T4 *__restrict__ goalpref,
                    typename Vec<S>::T4 *__restrict__ pv_out, i8 *__restrict__ status,
                    i8 *__restrict__ failed_at, u8 *__restrict__ arrived, int *__restrict__ fq,
                    typename Vec<R>::T4 *__restrict__ fq_state, int s0, int s1, const int *__restrict__ lrow,
                    typename Vec<R>::T4 *__restrict__ fq_cons, u8 *__restrict__ fq_perm,
                    const uint32_t *__restrict__ s_perm, int *__restrict__ fq_cnt,
                    const int *__restrict__ queue, const int *__restrict__ cq_cnt)
{
    constexpr int NG = THREADS / GL;
    const int nq = *cq_cnt;
    for (int base = blockIdx.x * NG; base < nq; base += gridDim.x * NG) { // uniform trip count per block
        const int idx = base + threadIdx.x / GL;
        const bool in_range = idx < nq;
        solve_group_body<S, R, MAXN, THREADS, GL, PRESH>(idx, in_range, in_range ? queue[idx] : 0, plan, P, s_nr, s_dm,
                                                         s_row, ids, nb, nb_cnt, goalpref, pv_out, status, failed_at,
                                                         arrived, fq, fq_state, s0, s1, lrow, fq_cons, fq_perm, s_perm,
                                                         fq_cnt);
        __syncthreads(); // the block's shared memory is reused by the next queue chunk
    }
}

// Least-penetration stage for the agents the solve kernels queued, GL adjacent lanes per
// queued agent. The stage is a long chain of dependent operations whose control flow differs
// from agent to agent; the lanes of a group share the agent's constraints (handed over by the
// solve kernel, spill_constraints) through shared memory and split every inner loop of the
// stage (orca_math.cuh, g_* functions): ~3x fewer warp instructions per agent in dense crowds
// than one thread per agent, where the stage dominates the step.
// Two instances are launched back to back and the queue length picks the one that works:
// GL = ORCA_GL (4) when the queue is long (throughput: 8 agents per warp), GL = ORCA_GL_SHORT
// (16) when every queued agent can have half a warp to itself (a short queue's time is the
// latency of one agent's dependent chain: 54 -> 31 us at 1,024 agents, 64 -> 38 us at 16,640).
template <typename S, typename R, int MAXN, int THREADS, int GL>
__global__ void __launch_bounds__(THREADS)
k_fallback_coop(const GridPlan *__restrict__ plan, StepParams P,
                const NbRec<S> *__restrict__ s_nr, const typename Vec<R>::T4 *__restrict__ s_dm,
        const int *__restrict__ s_row,
                const i64 *__restrict__ ids, const int *__restrict__ nb, const u8 *__restrict__ nb_cnt,
                const typename Vec<S>::T4 *__restrict__ goalpref, typename Vec<S>::T4 *__restrict__ pv_out,
                u8 *__restrict__ arrived, const int *__restrict__ fq,
                const typename Vec<R>::T4 *__restrict__ fq_state,
                const typename Vec<R>::T4 *__restrict__ fq_cons, const u8 *__restrict__ fq_perm,
                const int *__restrict__ fq_cnt)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typedef typename Vec<R>::T4 R4;
    {   // which instance serves this queue length (both see the same count, exactly one runs)
        const bool is_short = *fq_cnt <= ORCA_FB_SHORT_QUEUE;
        if (ORCA_GL_SHORT != ORCA_GL && is_short != (GL == ORCA_GL_SHORT)) return;
    }
    constexpr int NG = THREADS / GL;                  // agents (groups) per block and pass
    const int g = threadIdx.x / GL;                   // group within the block
    const int gl = threadIdx.x % GL;                  // lane within the group
    const int gshift = (threadIdx.x & 31) - gl;       // first lane of the group within its warp
    const unsigned gmask = ((1u << GL) - 1u) << gshift;
    R4 *sm_cons = reinterpret_cast<R4 *>(smem_raw);
    R4 *sm_proj = sm_cons + MAXN * NG;
    u8 *sm_perm = reinterpret_cast<u8 *>(sm_proj + MAXN * NG);
    u8 *sm_inv = sm_perm + MAXN * NG;

    const int nq = *fq_cnt;
    // every lane makes the same number of passes (a group without an agent rides along
    // disabled), so the run-ahead stage can vote over the whole warp
    for (int base = blockIdx.x * NG; base < nq; base += gridDim.x * NG) {
        const int q = base + g;
        const bool enabled = q < nq;
        const int s = enabled ? fq[q] : 0;
        const R4 st = enabled ? fq_state[q] : mk4(R(0), R(0), R(0), R(0));
        const int row = enabled ? s_row[s] : 0;
        const int cnt = enabled ? (int)nb_cnt[s] : 0;
        typename Vec<S>::T4 me = mk4(S(0), S(0), S(0), S(0));
        R4 dm = mk4(R(0), R(0), R(0), R(0));
        if (enabled) {
            me = s_nr[s].pv;
            dm = s_dm[s];
        }
        u8 *perm = sm_perm + g;
        u8 *inv = sm_inv + g;
        SmemCons<R> cons{sm_cons + g, NG};
        SmemCons<R> proj{sm_proj + g, NG};
        (void)perm;

        if (enabled) { // the half-planes and their order as the solve kernel left them
            const R4 *src = fq_cons + (size_t)q * MAXN;
            const u8 *sp = fq_perm + (size_t)q * MAXN;
            for (int pos = gl; pos < cnt; pos += GL) {
                sm_cons[g + pos * NG] = src[pos];
                inv[(int)sp[pos] * NG] = (u8)pos;
            }
        }
        __syncwarp(gmask);

        SmemConsIdent<R> ident{sm_cons + g, inv, NG};
        R rx, ry;
        g_least_penetration_ra<R, GL, SmemCons<R>, SmemConsIdent<R>, SmemCons<R>>(
            cons, ident, proj, cnt, (int)st.z, dm.z, st.x, st.y, rx, ry, gl, gmask, gshift, 0xFFFFFFFFu, enabled);
        if (gl == 0 && enabled) integrate_row<S, R>(row, me, rx, ry, P, goalpref, pv_out, arrived);
        __syncwarp(gmask); // the group's shared memory is reused by the next queue entry
    }
}

// ---------------------------------------------------------------------------
// K4: finish, arrival removal
// ---------------------------------------------------------------------------

// frames completed += 1 (the frame index lives on the device so that a captured CUDA
// graph of the step can be replayed without patching kernel arguments)
// ids != nullptr: also resolve a pending coincident-centre error. err_pair holds LOGICAL rows
// (the reference reports the first bad row in its storage order); the ids are looked up by a
// linear search -- this runs once, on the way to an error.
__global__ void k_finish(GridPlan *plan, int remove_arrivals, const i64 *__restrict__ ids,
                         const int *__restrict__ lrow)
{
    if (ids && plan->err_pair != ORCA_NO_ERR && plan->err_frame < 0) {
        plan->err_frame = plan->frame + 1; // the reference names the frame being computed
        const int li = (int)(unsigned)(plan->err_pair >> 32), lj = (int)(unsigned)(plan->err_pair & 0xFFFFFFFFu);
        for (int p = 0; p < plan->n; ++p) {
            if (lrow[p] == li) plan->err_id_i = ids[p];
            if (lrow[p] == lj) plan->err_id_j = ids[p];
        }
    }
    if (!plan->idle) plan->frame = plan->frame + 1;
    if (!remove_arrivals) {
        plan->removed = 0;
        plan->n_after = plan->n_owned;
    }
}

// keep[i] = 1 for owned rows that have not arrived; ghosts are always dropped.
__global__ void __launch_bounds__(256)
k_keep_flags(const GridPlan *__restrict__ plan, const u8 *__restrict__ arrived,
             int *__restrict__ keep, int remove_arrivals)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = plan->n;
    if (i > n) return;
    keep[i] = (i < plan->n_owned && !(remove_arrivals && arrived[i])) ? 1 : 0;
}

template <typename R>
__global__ void __launch_bounds__(256)
k_compact(GridPlan *__restrict__ plan, const int *__restrict__ keep, const int *__restrict__ dst_idx,
          const typename Vec<R>::T4 *__restrict__ pv, typename Vec<R>::T4 *__restrict__ pv2,
          const typename Vec<R>::T4 *__restrict__ gp, typename Vec<R>::T4 *__restrict__ gp2,
          const typename Vec<R>::T2 *__restrict__ rm, typename Vec<R>::T2 *__restrict__ rm2,
          const i64 *__restrict__ ids, i64 *__restrict__ ids2, const u8 *__restrict__ cls,
          u8 *__restrict__ cls2, const i8 *__restrict__ st, i8 *__restrict__ st2,
          const i8 *__restrict__ fa, i8 *__restrict__ fa2, const float *__restrict__ hint,
          float *__restrict__ hint2, const int *__restrict__ lrow, int *__restrict__ lrow2,
          const int *__restrict__ lscan, const Attr64 *__restrict__ a64, Attr64 *__restrict__ a64_2,
          i64 *__restrict__ arr_ids, i64 *__restrict__ arr_frames, int arr_cap)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = plan->n;
    if (i >= n) return;
    if (arr_ids && !keep[i] && i < plan->n_owned) {
        // an owned row that is dropped arrived in the frame just completed (engine.py:251-255):
        // who and when, for the run loop's travel times (orca_run_logged)
        const int slot = atomicAdd(&plan->arr_count, 1);
        if (slot < arr_cap) {
            arr_ids[slot] = ids[i];
            arr_frames[slot] = plan->frame;
        }
    }
    if (keep[i]) {
        const int d = dst_idx[i];
        if (a64) a64_2[d] = a64[i];
        // logical row of the survivor: its rank among the surviving logical rows (lscan), or,
        // while storage order still is logical order, simply its new position
        lrow2[d] = lscan ? lscan[lrow[i]] : d;
        pv2[d] = pv[i];
        gp2[d] = gp[i];
        rm2[d] = rm[i];
        ids2[d] = ids[i];
        cls2[d] = cls[i];
        st2[d] = st[i];
        fa2[d] = fa[i];
        hint2[d] = hint[i];
    }
}

// lkeep[logical row] = keep[physical row] (and 0 one past the end, closing the scan): the
// exclusive scan of lkeep is each survivor's new logical row
__global__ void __launch_bounds__(256)
k_keep_by_logical(const GridPlan *__restrict__ plan, const int *__restrict__ keep,
                  const int *__restrict__ lrow, int *__restrict__ lkeep)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = plan->n;
    if (i > n) return;
    if (i == n) lkeep[n] = 0;
    else lkeep[lrow[i]] = keep[i];
}

// Row reordering: physical row s of the new arrays := physical row s_row[s] of the old ones,
// i.e. the state is laid out in the cell-sorted order of the bin build just done. Agents
// move a small fraction of a cell per frame, so for many frames afterwards the counting
// sort's scatter, the per-row reads of the gather / LP kernels and their result writes are
// nearly sequential instead of random (measured with presorted input: step -8 % at 1 M
// agents, -23 % at 8.5 M). lrow carries each row's logical (reference) index so that
// everything the host sees keeps the reference's storage order.
template <typename R>
__global__ void __launch_bounds__(256)
k_permute_rows(const GridPlan *__restrict__ plan, const int *__restrict__ s_row,
               const typename Vec<R>::T4 *__restrict__ pv, typename Vec<R>::T4 *__restrict__ pv2,
               const typename Vec<R>::T4 *__restrict__ gp, typename Vec<R>::T4 *__restrict__ gp2,
               const typename Vec<R>::T2 *__restrict__ rm, typename Vec<R>::T2 *__restrict__ rm2,
               const i64 *__restrict__ ids, i64 *__restrict__ ids2, const u8 *__restrict__ cls,
               u8 *__restrict__ cls2, const i8 *__restrict__ st, i8 *__restrict__ st2,
               const i8 *__restrict__ fa, i8 *__restrict__ fa2, const float *__restrict__ hint,
               float *__restrict__ hint2, const int *__restrict__ lrow, int *__restrict__ lrow2,
               const Attr64 *__restrict__ a64, Attr64 *__restrict__ a64_2)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= plan->n) return;
    const int i = s_row[s];
    if (a64) a64_2[s] = a64[i];
    pv2[s] = pv[i];
    gp2[s] = gp[i];
    rm2[s] = rm[i];
    ids2[s] = ids[i];
    cls2[s] = cls[i];
    st2[s] = st[i];
    fa2[s] = fa[i];
    hint2[s] = hint[i];
    lrow2[s] = lrow[i];
}

__global__ void k_after_compact(GridPlan *plan, const int *__restrict__ dst_idx)
{
    const int kept = dst_idx[plan->n]; // exclusive scan evaluated one past the end
    plan->removed = plan->n_owned - kept;
    plan->n_after = kept;
    plan->n = kept;
    plan->n_owned = kept;
}

// ---------------------------------------------------------------------------
// strip decomposition: select / pack / append agent records (multi-GPU halo
// exchange and migration; the records travel over NCCL, see parallel/strips.py)
// ---------------------------------------------------------------------------

// sel[i] = 1 for owned rows with x in [x_lo, x_hi); sel[n] = 0 closes the scan
template <typename S>
__global__ void __launch_bounds__(256)
k_strip_flags(const GridPlan *__restrict__ plan, const typename Vec<S>::T4 *__restrict__ pv,
              double x_lo, double x_hi, int *__restrict__ sel)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > plan->n) return;
    int f = 0;
    if (i < plan->n_owned) {
        const double x = (double)pv[i].x;
        f = (x >= x_lo && x < x_hi) ? 1 : 0;
    }
    sel[i] = f;
}

template <typename S>
__global__ void __launch_bounds__(256)
k_strip_pack(GridPlan *__restrict__ plan, const int *__restrict__ sel, const int *__restrict__ sel_idx,
             const typename Vec<S>::T4 *__restrict__ pv, const typename Vec<S>::T4 *__restrict__ goalpref,
             const typename Vec<S>::T2 *__restrict__ radmax, const i64 *__restrict__ ids,
             const u8 *__restrict__ cls, orca_agent_record *__restrict__ rec, i64 cap,
             const Attr64 *__restrict__ a64)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = plan->n;
    if (i == 0) plan->pack_count = sel_idx[n];
    if (i >= n || !sel[i]) return;
    const int d = sel_idx[i];
    if (d >= cap) return;
    const typename Vec<S>::T4 a = pv[i];
    const typename Vec<S>::T4 g = goalpref[i];
    const typename Vec<S>::T2 rm = radmax[i];
    orca_agent_record r;
    r.x = (double)a.x;
    r.y = (double)a.y;
    r.vx = (double)a.z;
    r.vy = (double)a.w;
    r.radius = (double)rm.x;
    r.pref_speed = (double)g.z;
    r.max_speed = (double)rm.y;
    r.goal_tol = (double)g.w;
    r.goal_x = (double)g.x;
    r.goal_y = (double)g.y;
    r.id = ids[i];
    r.class_code = (i64)cls[i];
    if (a64) { // migrants keep the float64 attributes their first owner uploaded
        const Attr64 a = a64[i];
        r.radius = a.radius;
        r.pref_speed = a.pref_speed;
        r.max_speed = a.max_speed;
        r.goal_tol = a.goal_tol;
        r.goal_x = a.goal_x;
        r.goal_y = a.goal_y;
    }
    rec[d] = r;
}

// keep everything owned that was NOT selected (migration removes the packed rows)
__global__ void __launch_bounds__(256)
k_keep_unselected(const GridPlan *__restrict__ plan, const int *__restrict__ sel, int *__restrict__ keep)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > plan->n) return;
    keep[i] = (i < plan->n_owned && !sel[i]) ? 1 : 0;
}

template <typename S>
__global__ void __launch_bounds__(256)
k_strip_append(GridPlan *__restrict__ plan, const orca_agent_record *__restrict__ rec, int count,
               typename Vec<S>::T4 *__restrict__ pv, typename Vec<S>::T4 *__restrict__ goalpref,
               typename Vec<S>::T2 *__restrict__ radmax, i64 *__restrict__ ids, u8 *__restrict__ cls,
               i8 *__restrict__ status, i8 *__restrict__ failed, float *__restrict__ hint,
               int *__restrict__ lrow, Attr64 *__restrict__ a64)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int row = plan->n + i;
    lrow[row] = row; // logical rows are dense, so the next logical row is the next physical one
    const orca_agent_record r = rec[i];
    if (a64) a64[row] = Attr64{r.radius, r.pref_speed, r.max_speed, r.goal_x, r.goal_y, r.goal_tol};
    pv[row] = mk4((S)r.x, (S)r.y, (S)r.vx, (S)r.vy);
    goalpref[row] = mk4((S)r.goal_x, (S)r.goal_y, (S)r.pref_speed, (S)r.goal_tol);
    radmax[row] = mk2((S)r.radius, (S)r.max_speed);
    ids[row] = r.id;
    cls[row] = (u8)r.class_code;
    status[row] = 0;
    failed[row] = -1;
    hint[row] = __int_as_float(0x7F800000);
    atomicMax(&plan->vmax_enc, enc_double(r.max_speed));
    atomicMax(&plan->rmax_enc, enc_double(r.radius));
}

__global__ void k_after_append(GridPlan *plan, int count, int ghost)
{
    plan->n += count;
    if (!ghost) plan->n_owned += count;
    plan->n_after = plan->n_owned;
}

__global__ void k_drop_ghosts(GridPlan *plan) { plan->n = plan->n_owned; }

// ---- device-side frame log (orca_run_logged): what engine.run reads per frame, kept in HBM ----

__global__ void k_log_reset(GridPlan *plan, int halt_when_empty)
{
    plan->halt_when_empty = halt_when_empty;
    plan->log_count = 0;
    plan->traj_rows = 0;
}

// the frame's un-compacted result (every row active during the frame, arrivals included,
// engine.py:257-263) appended to the trajectory buffer in storage-row order
template <typename S>
__global__ void __launch_bounds__(256)
k_log_traj(const GridPlan *__restrict__ plan, const typename Vec<S>::T4 *__restrict__ pv_out,
           const int *__restrict__ lrow, double4 *__restrict__ traj, i64 cap_rows)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (plan->idle || i >= plan->n_pre) return;
    const i64 dst = plan->traj_rows + lrow[i];
    if (dst >= cap_rows) return;
    const typename Vec<S>::T4 a = pv_out[i];
    traj[dst] = make_double4((double)a.x, (double)a.y, (double)a.z, (double)a.w);
}

// one record per frame (engine.FrameMetrics + SimState.lp_fallbacks, engine.py:46-52,247,270-286)
__global__ void k_log_frame(GridPlan *plan, orca_frame_record *__restrict__ rec, int cap, int with_traj)
{
    if (plan->idle) return;
    if (plan->log_count < cap) {
        orca_frame_record r;
        r.frame = plan->frame;
        r.active_agents = plan->n_owned;
        r.rows_before = plan->n_pre;
        r.lp_fallbacks = 0;
        for (int c = 0; c < ORCA_MAX_CHUNKS; ++c) r.lp_fallbacks += plan->fq_count[c];
        r.removed_agents = plan->removed;
        r.collision_count = (i64)plan->collisions;
        r.min_separation = dec_double(plan->min_sep_enc);
        rec[plan->log_count] = r;
    }
    plan->log_count += 1;
    if (with_traj) plan->traj_rows += plan->n_pre;
}

// ---- device-side exchange protocol (no host round trip per frame) -------------------
//
// A slab is a fixed-capacity device buffer: an orca_slab_header (32 B) followed by `cap`
// records. The sender's kernels count into the header with atomics, the whole slab travels
// (NCCL send/recv of a size both sides know without asking), and the receiver's append
// kernel reads the count from the header. The host only keeps upper bounds (orca_api.cu).

// What a ghost needs: the pre-step snapshot a neighbour reads (NbRec) plus the id that
// breaks distance ties (K:473-476). 32 B with FP32 state, 64 B with FP64 state.
template <typename S> struct HaloRec;
template <> struct __align__(16) HaloRec<float> {
    float x, y, vx, vy;
    float radius;
    unsigned cls;
    i64 id;
};
template <> struct __align__(16) HaloRec<double> {
    double x, y, vx, vy;
    double radius;
    i64 id;
    i64 cls;
    i64 pad;
};
static_assert(sizeof(HaloRec<float>) == 32 && sizeof(HaloRec<double>) == 64, "halo record layout");

__global__ void k_strip_configure(GridPlan *plan, double vmax_floor)
{
    // ghosts travel without their max_speed: the fast gather's displacement bound
    // (hint + (own + fastest max_speed) * dt) must cover the fastest agent of ANY strip
    atomicMax(&plan->vmax_enc, enc_double(vmax_floor));
}

// Owned agents within `reach` of a strip edge -> that side's halo slab (either may be null).
template <typename S>
__global__ void __launch_bounds__(256)
k_strip_pack_halo(const GridPlan *__restrict__ plan, const typename Vec<S>::T4 *__restrict__ pv,
                  const typename Vec<S>::T2 *__restrict__ radmax, const i64 *__restrict__ ids,
                  const u8 *__restrict__ cls, double left_edge, double right_edge,
                  orca_slab_header *hdr_l, HaloRec<S> *__restrict__ rec_l, orca_slab_header *hdr_r,
                  HaloRec<S> *__restrict__ rec_r, int cap)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= plan->n_owned) return;
    const typename Vec<S>::T4 a = pv[i];
    const double x = (double)a.x;
    const bool to_l = hdr_l && x < left_edge, to_r = hdr_r && x >= right_edge;
    if (!to_l && !to_r) return;
    HaloRec<S> r;
    r.x = a.x;
    r.y = a.y;
    r.vx = a.z;
    r.vy = a.w;
    r.radius = radmax[i].x;
    r.cls = cls[i];
    r.id = ids[i];
    if (to_l) {
        const int slot = atomicAdd(&hdr_l->count, 1);
        if (slot < cap) rec_l[slot] = r;
    }
    if (to_r) {
        const int slot = atomicAdd(&hdr_r->count, 1);
        if (slot < cap) rec_r[slot] = r;
    }
}

// Ghost rows from a halo slab, appended after the resident rows. cap_rows = handle capacity.
template <typename S>
__global__ void __launch_bounds__(256)
k_strip_append_halo(GridPlan *__restrict__ plan, const orca_slab_header *__restrict__ hdr,
                    const HaloRec<S> *__restrict__ rec, int cap, int cap_rows,
                    typename Vec<S>::T4 *__restrict__ pv, typename Vec<S>::T4 *__restrict__ goalpref,
                    typename Vec<S>::T2 *__restrict__ radmax, i64 *__restrict__ ids, u8 *__restrict__ cls,
                    i8 *__restrict__ status, i8 *__restrict__ failed, float *__restrict__ hint,
                    int *__restrict__ lrow, Attr64 *__restrict__ a64)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int count = min(min(hdr->count, cap), cap_rows - plan->n);
    if (i >= count) return;
    const int row = plan->n + i;
    const HaloRec<S> r = rec[i];
    lrow[row] = row;
    if (a64) a64[row] = Attr64{(double)r.radius, 0.0, 0.0, (double)r.x, (double)r.y, 0.0};
    pv[row] = mk4(r.x, r.y, r.vx, r.vy);
    goalpref[row] = mk4(r.x, r.y, S(0), S(0)); // a ghost is never steered: goal = where it stands
    radmax[row] = mk2(r.radius, S(0));         // (its max_speed is covered by the strip-wide vmax floor)
    ids[row] = r.id;
    cls[row] = (u8)r.cls;
    status[row] = 0;
    failed[row] = -1;
    hint[row] = __int_as_float(0x7F800000);
    atomicMax(&plan->rmax_enc, enc_double((double)r.radius));
}

// Owned rows from a migrant slab (orca_agent_record), count taken from the slab header.
template <typename S>
__global__ void __launch_bounds__(256)
k_strip_append_slab(GridPlan *__restrict__ plan, const orca_slab_header *__restrict__ hdr,
                    const orca_agent_record *__restrict__ rec, int cap, int cap_rows,
                    typename Vec<S>::T4 *__restrict__ pv, typename Vec<S>::T4 *__restrict__ goalpref,
                    typename Vec<S>::T2 *__restrict__ radmax, i64 *__restrict__ ids, u8 *__restrict__ cls,
                    i8 *__restrict__ status, i8 *__restrict__ failed, float *__restrict__ hint,
                    int *__restrict__ lrow, Attr64 *__restrict__ a64)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int count = min(min(hdr->count, cap), cap_rows - plan->n);
    if (i >= count) return;
    const int row = plan->n + i;
    lrow[row] = row;
    const orca_agent_record r = rec[i];
    if (a64) a64[row] = Attr64{r.radius, r.pref_speed, r.max_speed, r.goal_x, r.goal_y, r.goal_tol};
    pv[row] = mk4((S)r.x, (S)r.y, (S)r.vx, (S)r.vy);
    goalpref[row] = mk4((S)r.goal_x, (S)r.goal_y, (S)r.pref_speed, (S)r.goal_tol);
    radmax[row] = mk2((S)r.radius, (S)r.max_speed);
    ids[row] = r.id;
    cls[row] = (u8)r.class_code;
    status[row] = 0;
    failed[row] = -1;
    hint[row] = __int_as_float(0x7F800000);
    atomicMax(&plan->vmax_enc, enc_double(r.max_speed));
    atomicMax(&plan->rmax_enc, enc_double(r.radius));
}

// after either append: the row counts, and the sticky overflow flag when the sender produced
// more records than the slab (or this handle) holds
__global__ void k_after_append_slab(GridPlan *plan, const orca_slab_header *__restrict__ hdr, int cap,
                                    int cap_rows, int ghost)
{
    const int want = hdr->count;
    const int count = min(min(want, cap), cap_rows - plan->n);
    if (count < want || hdr->overflow) plan->err_capacity = 1;
    plan->n += count;
    if (!ghost) plan->n_owned += count;
    plan->n_after = plan->n_owned;
    if (ghost != 2) plan->strip_recv[ghost ? 0 : 1] += (unsigned long long)count; // (2: own emigrants kept as ghosts)
}

// ---- peer-memory window (orca_strip_window_*): the exchange without a communication library ----
// A strip's window is one device allocation: a flag line per side, then per side two receive
// buffers ([emigrant slab | halo slab], double-buffered by the parity of the exchange index).
// The SENDER writes its slabs straight into the neighbour's window (peer mapping: NVLink) and
// then raises that window's flag to `exchange + 1`; the RECEIVER's stream waits on its own
// flag. Double buffering is enough without an acknowledgement: exchange e + 2 (same parity as
// e) is only pushed after this rank has waited for the neighbour's exchange e + 1, which the
// neighbour pushed -- in stream order -- after appending what exchange e brought.
#define ORCA_WINDOW_FLAG_BYTES 128

// copy the USED part of [emigrant slab | halo slab] (the counts are in the headers) to `dst`,
// then -- once every block's stores are fenced system-wide -- publish the flag
__global__ void __launch_bounds__(256)
k_window_push(const unsigned char *__restrict__ send, unsigned char *__restrict__ dst, long long mig_bytes,
              int mig_cap, int halo_cap, int halo_rec_bytes, unsigned long long *flag, unsigned long long value,
              unsigned *done)
{
    const orca_slab_header *hm = reinterpret_cast<const orca_slab_header *>(send);
    const orca_slab_header *hh = reinterpret_cast<const orca_slab_header *>(send + mig_bytes);
    const long long used_m = (long long)sizeof(orca_slab_header) +
                             (long long)min(max(hm->count, 0), mig_cap) * (long long)sizeof(orca_agent_record);
    const long long used_h = (long long)sizeof(orca_slab_header) +
                             (long long)min(max(hh->count, 0), halo_cap) * (long long)halo_rec_bytes;
    const long long vm = used_m / 16, vh = used_h / 16; // (every size above is a multiple of 16)
    const uint4 *sm = reinterpret_cast<const uint4 *>(send), *sh = reinterpret_cast<const uint4 *>(send + mig_bytes);
    uint4 *dm = reinterpret_cast<uint4 *>(dst), *dh = reinterpret_cast<uint4 *>(dst + mig_bytes);
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < vm + vh; i += stride) {
        if (i < vm) dm[i] = sm[i];
        else dh[i - vm] = sh[i - vm];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned ticket = atomicAdd(done, 1u);
        if (ticket == gridDim.x - 1) { // the last block: every other block's stores are fenced
            *done = 0;
            __threadfence_system();
            *reinterpret_cast<volatile unsigned long long *>(flag) = value;
            __threadfence_system();
        }
    }
}

// the receiving stream stalls here until the neighbour's exchange has landed; bounded, so a
// neighbour that died surfaces as ORCA_ETIMEOUT at the next synchronisation instead of a hang
__global__ void k_window_wait(GridPlan *plan, const unsigned long long *flag, unsigned long long want,
                              unsigned long long timeout_ns)
{
    if (plan->err_window) return;
    const volatile unsigned long long *f = flag;
    unsigned long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*f < want) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > timeout_ns) {
            plan->err_window = 1;
            break;
        }
        __nanosleep(256);
    }
    __threadfence_system();
}

// keep flags of the strip step: owned rows that have not arrived AND whose new x is still
// inside [lo, hi); the ones that left go into the migrant slab of that side as full records
// and are removed by the compaction that follows (ghosts are always dropped). A row that does
// not fit its slab stays (and raises the sticky overflow flag on both sides of the exchange).
template <typename S>
__global__ void __launch_bounds__(256)
k_strip_keep_flags(GridPlan *__restrict__ plan, const u8 *__restrict__ arrived, int *__restrict__ keep,
                   int remove_arrivals, const typename Vec<S>::T4 *__restrict__ pv_new,
                   const typename Vec<S>::T4 *__restrict__ goalpref,
                   const typename Vec<S>::T2 *__restrict__ radmax, const i64 *__restrict__ ids,
                   const u8 *__restrict__ cls, double lo, double hi, orca_slab_header *hdr_l,
                   orca_agent_record *__restrict__ rec_l, orca_slab_header *hdr_r,
                   orca_agent_record *__restrict__ rec_r, int cap, const Attr64 *__restrict__ a64)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = plan->n;
    if (i > n) return;
    int k = 0;
    if (i < plan->n_owned && !(remove_arrivals && arrived[i])) {
        const typename Vec<S>::T4 a = pv_new[i];
        const double x = (double)a.x;
        orca_slab_header *hdr = x < lo ? hdr_l : (x >= hi ? hdr_r : nullptr);
        k = 1;
        if (hdr) {
            const int slot = atomicAdd(&hdr->count, 1);
            if (slot < cap) {
                const typename Vec<S>::T4 g = goalpref[i];
                const typename Vec<S>::T2 rm = radmax[i];
                orca_agent_record r;
                r.x = (double)a.x;
                r.y = (double)a.y;
                r.vx = (double)a.z;
                r.vy = (double)a.w;
                r.radius = (double)rm.x;
                r.pref_speed = (double)g.z;
                r.max_speed = (double)rm.y;
                r.goal_tol = (double)g.w;
                r.goal_x = (double)g.x;
                r.goal_y = (double)g.y;
                r.id = ids[i];
                r.class_code = (i64)cls[i];
                if (a64) {
                    const Attr64 e = a64[i];
                    r.radius = e.radius;
                    r.pref_speed = e.pref_speed;
                    r.max_speed = e.max_speed;
                    r.goal_tol = e.goal_tol;
                    r.goal_x = e.goal_x;
                    r.goal_y = e.goal_y;
                }
                (x < lo ? rec_l : rec_r)[slot] = r;
                k = 0;
            } else {
                hdr->overflow = 1;
                plan->err_capacity = 1;
            }
        }
    }
    keep[i] = k;
    // owned rows that go (emigrants, arrivals): counted for the in-place removal that follows
    const unsigned gone = __ballot_sync(__activemask(), i < plan->n_owned && !k);
    if (gone && (threadIdx.x & 31) == (unsigned)(__ffs((int)gone) - 1)) atomicAdd(&plan->strip_removed, __popc(gone));
}

// In-place removal for a strip. The step's result sits in rows [0, n_owned) followed by the ghosts;
// the rows that go (keep == 0: emigrants, arrivals) are few. Instead of compacting every array into
// its twin (214 B per agent of traffic, ~60 us per million agents), the survivors of the TAIL
// [n', n_owned) -- n' = n_owned - removed -- move into the HOLES below n', and the ghosts are
// dropped by the new row count. The order of a strip's rows means nothing (agents come and go
// with every exchange): the logical row of a row IS its physical row there.
__global__ void __launch_bounds__(256)
k_strip_holes(GridPlan *__restrict__ plan, const int *__restrict__ keep, int *__restrict__ holes,
              int *__restrict__ tail)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_o = plan->n_owned;
    if (i >= n_o) return;
    const int n_new = n_o - plan->strip_removed;
    if (i < n_new) {
        if (!keep[i]) holes[atomicAdd(&plan->hole_count, 1)] = i;
    } else if (keep[i]) {
        tail[atomicAdd(&plan->tail_count, 1)] = i;
    }
}

template <typename R>
__global__ void __launch_bounds__(256)
k_strip_fill(const GridPlan *__restrict__ plan, const int *__restrict__ holes, const int *__restrict__ tail,
             typename Vec<R>::T4 *__restrict__ pv, typename Vec<R>::T4 *__restrict__ gp,
             typename Vec<R>::T2 *__restrict__ rm, i64 *__restrict__ ids, u8 *__restrict__ cls,
             i8 *__restrict__ st, i8 *__restrict__ fa, float *__restrict__ hint, int *__restrict__ lrow,
             Attr64 *__restrict__ a64)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= plan->hole_count) return; // == tail_count
    const int d = holes[r], i = tail[r];
    pv[d] = pv[i];
    gp[d] = gp[i];
    rm[d] = rm[i];
    ids[d] = ids[i];
    cls[d] = cls[i];
    st[d] = st[i];
    fa[d] = fa[i];
    hint[d] = hint[i];
    lrow[d] = d;
    if (a64) a64[d] = a64[i];
}

__global__ void k_after_strip_fill(GridPlan *plan)
{
    const int kept = plan->n_owned - plan->strip_removed;
    plan->removed = plan->strip_removed;
    plan->n_after = kept;
    plan->n = kept;
    plan->n_owned = kept;
}

__global__ void k_set_frame(GridPlan *plan, i64 frame) { plan->frame = frame; }

// ---------------------------------------------------------------------------
// metrics: min separation / collision count (_kernels.py:559-589) on the
// post-step positions, using the grid of the NEXT bin build (same positions).
// ---------------------------------------------------------------------------

// Pass 1: an upper bound on the minimum separation -- the separation of each agent's
// closest candidate in the 3x3 block of search cells (one square root per agent).
template <typename R>
__global__ void __launch_bounds__(128)
k_min_sep_bound(GridPlan *__restrict__ plan, StepParams P, const typename Vec<R>::T2 *__restrict__ s_xy,
                const int *__restrict__ cell_start, const int *__restrict__ s_cell,
                const int *__restrict__ s_row, const typename Vec<R>::T2 *__restrict__ radmax)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    double ub = ORCA_INF;
    if (s < plan->n) {
        const int nx = plan->nx, ny = plan->ny, r = min(1, plan->rmax);
        const typename Vec<R>::T2 me = s_xy[s];
        const int c0 = s_cell[s];
        const int cx = c0 / ny, cy = c0 - cx * ny;
        const int y_lo = max(cy - r, 0), y_hi = min(cy + r, ny - 1);
        double best_d2 = ORCA_INF;
        int best_s = -1;
        for (int gx = max(cx - r, 0); gx <= min(cx + r, nx - 1); ++gx) {
            const int *cs = cell_start + gx * ny;
            for (int s2 = cs[y_lo]; s2 < cs[y_hi + 1]; ++s2) {
                const typename Vec<R>::T2 q = s_xy[s2];
                const double dx = (double)q.x - (double)me.x, dy = (double)q.y - (double)me.y;
                const double d2 = dx * dx + dy * dy;
                if (s2 != s && d2 < best_d2) {
                    best_d2 = d2;
                    best_s = s2;
                }
            }
        }
        if (best_s >= 0 && best_d2 <= P.rad2)
            ub = __dsqrt_rn(best_d2) - ((double)radmax[s_row[s]].x + (double)radmax[s_row[best_s]].x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ub = fmin(ub, __shfl_xor_sync(0xFFFFFFFFu, ub, o));
    if ((threadIdx.x & 31) == 0 && ub < ORCA_INF) atomicMin(&plan->sep_ub_enc, enc_double(ub));
}

// Pass 2: exact minimum separation and collision count (K:559-589), each pair counted
// from its lower-id side. Only pairs closer than  max(bound, 0) + 2 * (largest radius)
// can attain the minimum or collide, so the scan covers that distance instead of the
// whole neighbor_radius (about 50x fewer candidates in a typical crowd).
template <typename R>
__global__ void __launch_bounds__(128)
k_min_sep(GridPlan *__restrict__ plan, StepParams P, const typename Vec<R>::T2 *__restrict__ s_xy,
          const int *__restrict__ cell_start, const int *__restrict__ s_cell,
          const int *__restrict__ s_row, const i64 *__restrict__ ids,
          const typename Vec<R>::T2 *__restrict__ radmax, double coll_tol)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    double best = ORCA_INF;
    unsigned cnt = 0;
    if (s < plan->n) {
        const double ub = dec_double(plan->sep_ub_enc);
        const double rr = fmax(dec_double(plan->rmax_enc), 0.0);
        double reach = ub < ORCA_INF ? (fmax(ub, 0.0) + 2.0 * rr) * (1.0 + 1e-9) + 1e-9 : P.nr;
        const double T2 = fmin(reach * reach, P.rad2);
        const int nx = plan->nx, ny = plan->ny;
        const int r = min(plan->rmax, (int)(sqrt(T2) * plan->inv_cell * (1.0 + 1e-9)) + 1);
        const typename Vec<R>::T2 me = s_xy[s];
        const int row = s_row[s];
        const i64 my_id = ids[row];
        const double my_r = (double)radmax[row].x;
        const int c0 = s_cell[s];
        const int cx = c0 / ny, cy = c0 - cx * ny;
        const int y_lo = max(cy - r, 0), y_hi = min(cy + r, ny - 1);
        for (int gx = max(cx - r, 0); gx <= min(cx + r, nx - 1); ++gx) {
            const int *cs = cell_start + gx * ny;
            for (int s2 = cs[y_lo]; s2 < cs[y_hi + 1]; ++s2) {
                const typename Vec<R>::T2 q = s_xy[s2];
                const double dx = (double)q.x - (double)me.x, dy = (double)q.y - (double)me.y;
                const double d2 = dx * dx + dy * dy;
                if (d2 > T2) continue;
                const int row2 = s_row[s2];
                if (ids[row2] <= my_id) continue;
                const double sep = __dsqrt_rn(d2) - (my_r + (double)radmax[row2].x);
                if (sep < best) best = sep;
                if (sep < -coll_tol) ++cnt;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        best = fmin(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
        cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&plan->min_sep_enc, enc_double(best));
        if (cnt) atomicAdd(&plan->collisions, (u64)cnt);
    }
}

// ---------------------------------------------------------------------------
// conversions between the reference's float64 / int64 host layout and the
// device state
// ---------------------------------------------------------------------------

template <typename R>
__global__ void __launch_bounds__(256)
k_import_pv(int n, const double *__restrict__ pos, const double *__restrict__ vel,
            typename Vec<R>::T4 *__restrict__ pv, const int *__restrict__ lrow)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int l = lrow[i]; // host arrays are in logical (reference) row order
    pv[i] = mk4((R)pos[2 * l], (R)pos[2 * l + 1], (R)vel[2 * l], (R)vel[2 * l + 1]);
}

// positions only (orca_advance_host): the velocity half of pv keeps its old content until
// k_patch_vel replaces it
template <typename R>
__global__ void __launch_bounds__(256)
k_import_pos(int n, const double *__restrict__ pos, typename Vec<R>::T4 *__restrict__ pv,
             const int *__restrict__ lrow)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int l = lrow[i];
    typename Vec<R>::T4 a = pv[i];
    a.x = (R)pos[2 * l];
    a.y = (R)pos[2 * l + 1];
    pv[i] = a;
}

// velocities that arrived after the bin build: into the row-ordered state and into the
// cell-sorted snapshot k_scatter already wrote (slot = cell_start[cell] + rank)
template <typename R>
__global__ void __launch_bounds__(256)
k_patch_vel(const GridPlan *__restrict__ plan, const double *__restrict__ vel,
            typename Vec<R>::T4 *__restrict__ pv, NbRec<R> *__restrict__ s_nr,
            const int *__restrict__ cell_of, const int *__restrict__ rank_of,
            const int *__restrict__ cell_start, const int *__restrict__ lrow)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= plan->n) return;
    const int l = lrow[i];
    typename Vec<R>::T4 a = pv[i];
    a.z = (R)vel[2 * l];
    a.w = (R)vel[2 * l + 1];
    pv[i] = a;
    s_nr[cell_start[cell_of[i]] + rank_of[i]].pv = a;
}

template <typename R>
__global__ void __launch_bounds__(256)
k_import_attrs(int n, const double *__restrict__ radii, const double *__restrict__ pref,
               const double *__restrict__ maxs, const double *__restrict__ goals,
               const double *__restrict__ gtol, const i64 *__restrict__ cls_in,
               typename Vec<R>::T4 *__restrict__ goalpref, typename Vec<R>::T2 *__restrict__ radmax,
               u8 *__restrict__ cls, float *__restrict__ hint, GridPlan *__restrict__ plan,
               Attr64 *__restrict__ a64)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    // largest max_speed / radius of the crowd: one atomic per warp (a million same-address
    // atomics took 1.4 ms)
    double vm = i < n ? maxs[i] : -1e300, rm_ = i < n ? radii[i] : -1e300;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vm = fmax(vm, __shfl_xor_sync(0xFFFFFFFFu, vm, o));
        rm_ = fmax(rm_, __shfl_xor_sync(0xFFFFFFFFu, rm_, o));
    }
    if ((threadIdx.x & 31) == 0 && vm > -1e300) {
        atomicMax(&plan->vmax_enc, enc_double(vm));
        atomicMax(&plan->rmax_enc, enc_double(rm_));
    }
    if (i >= n) return;
    hint[i] = __int_as_float(0x7F800000); // no neighbour list yet
    goalpref[i] = mk4((R)goals[2 * i], (R)goals[2 * i + 1], (R)pref[i], (R)gtol[i]);
    radmax[i] = mk2((R)radii[i], (R)maxs[i]);
    cls[i] = (u8)cls_in[i];
    if (a64) a64[i] = Attr64{radii[i], pref[i], maxs[i], goals[2 * i], goals[2 * i + 1], gtol[i]};
}

template <typename R>
__global__ void __launch_bounds__(256)
k_export_pv(int n, const typename Vec<R>::T4 *__restrict__ pv, double *__restrict__ pos,
            double *__restrict__ vel, const int *__restrict__ lrow, const int *__restrict__ n_dev = nullptr)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (n_dev && i >= *n_dev)) return; // n_dev: row count known only on the device
    const int l = lrow[i];
    const typename Vec<R>::T4 a = pv[i];
    pos[2 * l] = (double)a.x;
    pos[2 * l + 1] = (double)a.y;
    vel[2 * l] = (double)a.z;
    vel[2 * l + 1] = (double)a.w;
}

template <typename R>
__global__ void __launch_bounds__(256)
k_export_attrs(int n, const typename Vec<R>::T4 *__restrict__ goalpref,
               const typename Vec<R>::T2 *__restrict__ radmax, const u8 *__restrict__ cls,
               double *__restrict__ radii, double *__restrict__ pref, double *__restrict__ maxs,
               double *__restrict__ goals, double *__restrict__ gtol, i64 *__restrict__ cls_out,
               const int *__restrict__ lrow, const Attr64 *__restrict__ a64)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int l = lrow[i];
    cls_out[l] = (i64)cls[i];
    if (a64) { // the float64 values the host uploaded
        const Attr64 a = a64[i];
        goals[2 * l] = a.goal_x;
        goals[2 * l + 1] = a.goal_y;
        pref[l] = a.pref_speed;
        gtol[l] = a.goal_tol;
        radii[l] = a.radius;
        maxs[l] = a.max_speed;
        return;
    }
    const typename Vec<R>::T4 g = goalpref[i];
    const typename Vec<R>::T2 rm = radmax[i];
    goals[2 * l] = (double)g.x;
    goals[2 * l + 1] = (double)g.y;
    pref[l] = (double)g.z;
    gtol[l] = (double)g.w;
    radii[l] = (double)rm.x;
    maxs[l] = (double)rm.y;
}

__global__ void __launch_bounds__(256)
k_export_i8(int n, const i8 *__restrict__ in, i64 *__restrict__ out, const int *__restrict__ lrow)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[lrow[i]] = (i64)in[i];
}

__global__ void __launch_bounds__(256)
k_export_i64(int n, const i64 *__restrict__ in, i64 *__restrict__ out, const int *__restrict__ lrow)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[lrow[i]] = in[i];
}

// kept[logical row] = keep flag of that row in the last compaction (orca_download_last_step_kept)
__global__ void __launch_bounds__(256)
k_export_keep(int n, const int *__restrict__ keep, const int *__restrict__ lrow, u8 *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[lrow[i]] = keep[i] ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_iota(int n, int *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

// parity taps, storage-row order (see orca_debug_last_step)
template <typename S, typename R>
__global__ void __launch_bounds__(256)
k_debug_rows(int n, StepParams P, const typename Vec<S>::T4 *__restrict__ pv_pre,
             const int *__restrict__ s_row, const int *__restrict__ nb,
             const u8 *__restrict__ nb_cnt, const typename Vec<R>::T4 *__restrict__ s_dm,
             i64 *__restrict__ cell_ix, i64 *__restrict__ cell_iy, i64 *__restrict__ nb_rows,
             i64 *__restrict__ nb_count, double *__restrict__ des, const int *__restrict__ lrow)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const typename Vec<S>::T4 a = pv_pre[s_row[s]];
    const int row = lrow[s_row[s]]; // outputs are in logical (reference) row order
    cell_ix[row] = (i64)floor(__ddiv_rn((double)a.x, P.nr));
    cell_iy[row] = (i64)floor(__ddiv_rn((double)a.y, P.nr));
    const int cnt = nb_cnt[s];
    nb_count[row] = cnt;
    for (int t = 0; t < P.max_n; ++t)
        nb_rows[(size_t)row * P.max_n + t] = t < cnt ? (i64)lrow[s_row[nb[(size_t)t * P.stride + s]]] : -1;
    des[2 * row] = (double)s_dm[s].x;
    des[2 * row + 1] = (double)s_dm[s].y;
}

} // namespace orca

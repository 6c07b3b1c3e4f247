// orca_math.cuh -- scalar building blocks of the steering step, templated on the
// arithmetic type R (float: the FP32 product path; double: bit-exact twin of the
// float64 reference). Device-only, header-only.
//
// Reference behaviour restated here ("K" = pkg/src/orcasim/_kernels.py):
//   mix64 / problem_seed / Fisher-Yates   K:36-61
//   vo_exit                                K:343-419
//   closest-point LP                       K:74-146
//   direction LP + least penetration       K:153-283
//
// The translation unit is compiled with -fmad=false: the reference never fuses a
// multiply-add (numba/LLVM without fastmath), and the FP64 instantiation relies
// on that to be bit-identical. Expression trees follow the reference's
// evaluation order (Python binary operators associate left to right).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace orca {

typedef unsigned long long u64;
typedef long long i64;

template <typename R> struct Vec;
template <> struct Vec<float> { typedef float2 T2; typedef float4 T4; };
template <> struct Vec<double> { typedef double2 T2; typedef double4 T4; };

// What a neighbour reads of an agent, in ONE aligned record of the cell-sorted snapshot:
// (x, y, vx, vy) and (radius, class code). FP32 state: 32 B = one DRAM/L2 sector, fetched by a
// single 256-bit load (LDG.E.ENL2.256); as two arrays (16 B + 8 B) every neighbour cost two sectors.
template <typename S> struct __align__(8 * sizeof(S)) NbRec {
    typename Vec<S>::T4 pv;
    typename Vec<S>::T2 rc;
    typename Vec<S>::T2 pad;
};

template <typename R> __device__ __forceinline__ R rsqrt_exact(R x);
template <> __device__ __forceinline__ float rsqrt_exact<float>(float x) { return __fsqrt_rn(x); }
template <> __device__ __forceinline__ double rsqrt_exact<double>(double x) { return __dsqrt_rn(x); }
// correctly rounded square root (np.sqrt)
template <typename R> __device__ __forceinline__ R sqrt_rn(R x) { return rsqrt_exact<R>(x); }

template <typename R> __device__ __forceinline__ R div_rn(R a, R b);
template <> __device__ __forceinline__ float div_rn<float>(float a, float b) { return __fdiv_rn(a, b); }
template <> __device__ __forceinline__ double div_rn<double>(double a, double b) { return __ddiv_rn(a, b); }

// ---------------------------------------------------------------------------
// splitmix64, per-problem seed, shuffle                                K:36-61
// ---------------------------------------------------------------------------

__host__ __device__ __forceinline__ u64 mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// K:57-61 (frame is the PRE-step frame index, engine.py:233)
__host__ __device__ __forceinline__ u64 problem_seed(i64 frame, i64 agent_id)
{
    return mix64(((u64)frame << 32) | ((u64)agent_id & 0xFFFFFFFFULL));
}

#define ORCA_GOLDEN 0x9E3779B97F4A7C15ULL

// x mod m for 1 <= m <= 2^16 without a 64-bit division
__device__ __forceinline__ uint32_t mod_small(u64 x, uint32_t m)
{
    uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
    uint32_t two32 = (uint32_t)(0xFFFFFFFFu % m) + 1u; // 2^32 mod m, possibly == m
    if (two32 == m) two32 = 0;
    uint32_t r = (hi % m) * two32 + (lo % m); // < m*m + m <= 2^32 for m <= 2^16 - 1
    return r % m;
}

// ---------------------------------------------------------------------------
// velocity-obstacle exit                                              K:343-419
// ---------------------------------------------------------------------------

// Returns false only for exactly coincident centres. (ux,uy) is the shortest
// displacement of the relative velocity to the VO boundary, (nx,ny) the outward
// unit normal there.
//
// The reference branches per case (overlap K:357-376, cut-off arc K:395-401, tangent leg
// K:403-419). Here the three cases are merged into ONE straight-line sequence (one square
// root, two divisions, selects): in a warp of 32 agent-neighbour pairs ~28 lanes take the arc
// and ~3 a leg, and a branchy form runs both paths back to back (profiles/r01_notes.md). Every
// value that reaches an output is produced by the same operations on the same operands as in
// the reference, so FP64 stays bit-identical (tests/test_gpu_kat.py: 4,004 reference exits).
// Only the two measure-zero cases (coincident centres, |w|^2 < 1e-24) still branch.
// vo_exit_inv takes 1/tau and 1/dt (K:358, K:378: `inv = 1.0 / tau`) so that callers with a
// loop over neighbours divide once per kernel, not per neighbour; vo_exit computes them.
template <typename R>
__device__ __forceinline__ bool vo_exit_inv(R rpx, R rpy, R rvx, R rvy, R comb_r, R inv_tau, R inv_dt,
                                            R &ux, R &uy, R &nx, R &ny);

template <typename R>
__device__ __forceinline__ bool vo_exit(R rpx, R rpy, R rvx, R rvy, R comb_r, R tau, R dt,
                                        R &ux, R &uy, R &nx, R &ny)
{
    return vo_exit_inv<R>(rpx, rpy, rvx, rvy, comb_r, div_rn<R>(R(1), tau), div_rn<R>(R(1), dt), ux, uy, nx, ny);
}

template <typename R>
__device__ __forceinline__ bool vo_exit_inv(R rpx, R rpy, R rvx, R rvy, R comb_r, R inv_tau, R inv_dt,
                                            R &ux, R &uy, R &nx, R &ny)
{
    const R d2 = rpx * rpx + rpy * rpy;
    const R r2 = comb_r * comb_r;
    const bool overlap = d2 < r2;                                   // K:357
    const R inv = overlap ? inv_dt : inv_tau;                       // K:358 / K:378
    const R cx = rpx * inv, cy = rpy * inv;
    const R rr = comb_r * inv;
    const R wx = rvx - cx, wy = rvy - cy;
    const R wl2 = wx * wx + wy * wy;
    const R dot_wp = wx * rpx + wy * rpy;
    if ((rpx == R(0) && rpy == R(0)) || wl2 < R(1e-24)) {           // measure-zero cases
        if (rpx == R(0) && rpy == R(0)) {
            ux = uy = nx = ny = R(0);
            return false;
        }
        // relative velocity at the centre of the (dt or tau) disc, K:364-368 / K:387-393
        const R d = sqrt_rn<R>(d2);
        const R hx = div_rn<R>(-rpx, d), hy = div_rn<R>(-rpy, d);
        ux = rr * hx; // overlap: (rr - 0) * h == rr * h exactly
        uy = rr * hy;
        nx = hx;
        ny = hy;
        return true;
    }
    const bool arc = overlap || (dot_wp < R(0) && dot_wp * dot_wp > r2 * wl2); // K:395
    const R sq = sqrt_rn<R>(arc ? wl2 : d2 - r2);                   // |w|  or  leg
    const bool side = rpx * wy - rpy * wx > R(0);                   // K:404
    const R a1 = rpx * sq, a2 = rpy * comb_r, b1 = rpx * comb_r, b2 = rpy * sq;
    const R lx = side ? a1 - a2 : -(a1 + a2);                       // K:405-410 numerators
    const R ly = side ? b1 + b2 : b1 - b2;
    const R den = arc ? sq : d2;
    const R qx = div_rn<R>(arc ? wx : lx, den);                     // w/|w|  or  leg direction
    const R qy = div_rn<R>(arc ? wy : ly, den);
    // arc: K:397-401
    const R s = rr - sq;
    // leg: K:411-419
    const R t = rvx * qx + rvy * qy;
    R mx = -qy, my = qx;
    if (mx * rpx + my * rpy > R(0)) {
        mx = -mx;
        my = -my;
    }
    ux = arc ? s * qx : t * qx - rvx;
    uy = arc ? s * qy : t * qy - rvy;
    nx = arc ? qx : mx;
    ny = arc ? qy : my;
    return true;
}

// ---------------------------------------------------------------------------
// LP core, written against a constraint "view" V:
//     V::get(pos, px, py, nx, ny)   constraint at position `pos` of the order
//                                   this view walks (shuffled or identity)
// and a projected-constraint scratch P with get(m, ...)/set(m, ...).
// ---------------------------------------------------------------------------

#define ORCA_PARALLEL_EPS 1e-12

// experiment switches (see profiles/): defaults are the measured-best variants
#ifndef ORCA_RA_SCAN_UNROLL
#define ORCA_RA_SCAN_UNROLL 1 // positions per iteration of the run-ahead scan loops (1, 2, 4 measured: no difference)
#endif

// K:74-119. `zz` shifts every constraint point by -zz*normal (the z-relaxed set
// of K:276-278); SHIFT=false compiles the shift out.
template <typename R, bool SHIFT, typename V>
__device__ __forceinline__ bool lp1_target(const V &view, int i_pos, R zz, R cap, R tx, R ty,
                                           R &ox, R &oy)
{
    R px, py, nx, ny;
    view.get(i_pos, px, py, nx, ny);
    if (SHIFT) {
        px = px - zz * nx;
        py = py - zz * ny;
    }
    const R dx = -ny, dy = nx;
    const R pd = px * dx + py * dy;
    const R disc = pd * pd + cap * cap - (px * px + py * py);
    if (disc < R(0)) return false;
    const R sq = sqrt_rn<R>(disc);
    R t_left = -pd - sq;
    R t_right = -pd + sq;

    if (!SHIFT) {
        // Main LP (k_solve, all 32 lanes busy): no early exit inside the loop. The outcome
        // does not depend on where the interval first becomes empty (t_left only grows,
        // t_right only shrinks), and without exits the division chains of successive
        // iterations overlap.
        bool bad = false;
#pragma unroll 4
        for (int j_pos = 0; j_pos < i_pos; ++j_pos) {
            R qx, qy, mx, my;
            view.get(j_pos, qx, qy, mx, my);
            const R a = dx * mx + dy * my;
            const R b = (qx - px) * mx + (qy - py) * my;
            const bool par = R(-ORCA_PARALLEL_EPS) <= a && a <= R(ORCA_PARALLEL_EPS);
            bad = bad || (par && b > R(0));
            const R t = div_rn<R>(b, a); // unused when par
            if (!par && a > R(0) && t > t_left) t_left = t;
            if (!par && !(a > R(0)) && t < t_right) t_right = t;
        }
        if (bad || t_left > t_right) return false;
    } else {
        // Re-solve on the z-relaxed set (k_fallback, few lanes per warp): infeasibility is
        // common here, so leaving at the first empty interval saves more than overlap gains.
        for (int j_pos = 0; j_pos < i_pos; ++j_pos) {
            R qx, qy, mx, my;
            view.get(j_pos, qx, qy, mx, my);
            qx = qx - zz * mx;
            qy = qy - zz * my;
            const R a = dx * mx + dy * my;
            const R b = (qx - px) * mx + (qy - py) * my;
            if (R(-ORCA_PARALLEL_EPS) <= a && a <= R(ORCA_PARALLEL_EPS)) {
                if (b > R(0)) return false;
                continue;
            }
            const R t = div_rn<R>(b, a);
            if (a > R(0)) {
                if (t > t_left) t_left = t;
            } else {
                if (t < t_right) t_right = t;
            }
            if (t_left > t_right) return false;
        }
    }
    R t = (tx - px) * dx + (ty - py) * dy;
    if (t < t_left) t = t_left;
    else if (t > t_right) t = t_right;
    ox = px + t * dx;
    oy = py + t * dy;
    return true;
}

// K:122-146. Returns true if feasible; otherwise fail_pos is set and (vx,vy) is
// the last point that satisfied positions [0, fail_pos).
template <typename R, bool SHIFT, typename V>
__device__ __forceinline__ bool lp2_target(const V &view, int k, R zz, R cap, R tx, R ty,
                                           int &fail_pos, R &vx, R &vy)
{
    const R t2 = tx * tx + ty * ty;
    if (t2 > cap * cap) {
        const R s = div_rn<R>(cap, sqrt_rn<R>(t2));
        vx = tx * s;
        vy = ty * s;
    } else {
        vx = tx;
        vy = ty;
    }
    for (int i_pos = 0; i_pos < k; ++i_pos) {
        R px, py, nx, ny;
        view.get(i_pos, px, py, nx, ny);
        if (SHIFT) {
            px = px - zz * nx;
            py = py - zz * ny;
        }
        if ((vx - px) * nx + (vy - py) * ny < R(0)) {
            R nvx, nvy;
            if (!lp1_target<R, SHIFT, V>(view, i_pos, zz, cap, tx, ty, nvx, nvy)) {
                fail_pos = i_pos;
                return false;
            }
            vx = nvx;
            vy = nvy;
        }
    }
    fail_pos = -1;
    return true;
}

// K:122-146 again, same arithmetic, different loop nest for a warp of 32 independent LPs.
// lp2_target walks the positions in lock step: at every position the ~2 lanes whose
// constraint is violated run lp1_target while 30 wait (measured: 55 % of k_solve's warp
// instructions at 2 of 32 lanes, profiles/r02_notes.md). Here every lane first runs ahead
// to ITS next violated position (a cheap scan), then all lanes that found one solve their
// 1-D problems together: the warp pays max-over-lanes(#violations) rounds (~4) instead of
// k (16). The vote between the two phases is what keeps them apart -- without it the
// control-flow graph is the lock-step one and the compiler emits the same code.
// `live` = the lanes of this warp that call the function (all of them must);
// `enabled` = false lets a lane ride along without a problem of its own.
template <typename R, typename V>
__device__ __forceinline__ bool lp2_target_runahead(const V &view, int k, R cap, R tx, R ty,
                                                    int &fail_pos, R &vx, R &vy, unsigned live,
                                                    bool enabled)
{
    const R t2 = tx * tx + ty * ty;
    if (t2 > cap * cap) {
        const R s = div_rn<R>(cap, sqrt_rn<R>(t2));
        vx = tx * s;
        vy = ty * s;
    } else {
        vx = tx;
        vy = ty;
    }
    int i_pos = 0;
    bool done = !enabled, ok = true;
    fail_pos = -1;
    while (true) {
        bool found = false;
        if (!done) {
            constexpr int kRaScanUnroll = ORCA_RA_SCAN_UNROLL;
#pragma unroll kRaScanUnroll
            for (; i_pos < k; ++i_pos) {
                R px, py, nx, ny;
                view.get(i_pos, px, py, nx, ny);
                if ((vx - px) * nx + (vy - py) * ny < R(0)) {
                    found = true;
                    break;
                }
            }
            done = !found;
        }
        if (!__any_sync(live, found)) break;
        if (found) {
            R nvx, nvy;
            if (lp1_target<R, false, V>(view, i_pos, R(0), cap, tx, ty, nvx, nvy)) {
                vx = nvx;
                vy = nvy;
                ++i_pos;
            } else {
                fail_pos = i_pos;
                ok = false;
                done = true;
            }
        }
    }
    return ok;
}

// K:153-190, identity order over the projected constraints
template <typename R, typename P>
__device__ __forceinline__ bool lp1_dir(const P &proj, int upto, R cap, R ox, R oy, R &rx, R &ry)
{
    R px, py, nx, ny;
    proj.get(upto, px, py, nx, ny);
    const R dx = -ny, dy = nx;
    const R pd = px * dx + py * dy;
    const R disc = pd * pd + cap * cap - (px * px + py * py);
    if (disc < R(0)) return false;
    const R sq = sqrt_rn<R>(disc);
    R t_left = -pd - sq;
    R t_right = -pd + sq;
    for (int j = 0; j < upto; ++j) {
        R qx, qy, mx, my;
        proj.get(j, qx, qy, mx, my);
        const R a = dx * mx + dy * my;
        const R b = (qx - px) * mx + (qy - py) * my;
        if (R(-ORCA_PARALLEL_EPS) <= a && a <= R(ORCA_PARALLEL_EPS)) {
            if (b > R(0)) return false;
            continue;
        }
        const R t = div_rn<R>(b, a);
        if (a > R(0)) {
            if (t > t_left) t_left = t;
        } else {
            if (t < t_right) t_right = t;
        }
        if (t_left > t_right) return false;
    }
    const R t = (dx * ox + dy * oy) > R(0) ? t_right : t_left;
    rx = px + t * dx;
    ry = py + t * dy;
    return true;
}

// K:193-205
template <typename R, typename P>
__device__ __forceinline__ bool lp2_dir(const P &proj, int m, R cap, R ox, R oy, R &rx, R &ry)
{
    R vx = cap * ox, vy = cap * oy;
    for (int i = 0; i < m; ++i) {
        R px, py, nx, ny;
        proj.get(i, px, py, nx, ny);
        if ((vx - px) * nx + (vy - py) * ny < R(0)) {
            R nvx, nvy;
            if (!lp1_dir<R, P>(proj, i, cap, ox, oy, nvx, nvy)) {
                rx = vx;
                ry = vy;
                return false;
            }
            vx = nvx;
            vy = nvy;
        }
    }
    rx = vx;
    ry = vy;
    return true;
}

// K:212-251: minimise the maximum (clamped) violation over the shuffled order,
// starting at position `begin` from (vx,vy).
template <typename R, typename V, typename P>
__device__ __forceinline__ void lp3_minmax(const V &view, P &proj, int k, int begin, R cap, R &vx,
                                           R &vy, R &z)
{
    R dist = R(0);
    for (int i_pos = begin; i_pos < k; ++i_pos) {
        R cpx, cpy, cnx, cny;
        view.get(i_pos, cpx, cpy, cnx, cny);
        const R viol = (cpx - vx) * cnx + (cpy - vy) * cny;
        if (viol > dist) {
            int m = 0;
#pragma unroll 2
            for (int j_pos = 0; j_pos < i_pos; ++j_pos) {
                R jpx, jpy, jnx, jny;
                view.get(j_pos, jpx, jpy, jnx, jny);
                const R mx = jnx - cnx;
                const R my = jny - cny;
                const R ml2 = mx * mx + my * my;
                const R rhs = jpx * jnx + jpy * jny - cpx * cnx - cpy * cny;
                const R ml = sqrt_rn<R>(ml2);
                const R ppx = div_rn<R>(mx * rhs, ml2), ppy = div_rn<R>(my * rhs, ml2);
                const R pnx = div_rn<R>(mx, ml), pny = div_rn<R>(my, ml);
                if (!(ml2 < R(1e-24))) { // same normal: no half-plane induced (K:231-235)
                    proj.set(m, ppx, ppy, pnx, pny);
                    ++m;
                }
            }
            R nvx, nvy;
            if (lp2_dir<R, P>(proj, m, cap, cnx, cny, nvx, nvy)) {
                vx = nvx;
                vy = nvy;
            }
            dist = (cpx - vx) * cnx + (cpy - vy) * cny;
            if (dist < R(0)) dist = R(0);
        }
    }
    z = dist;
}

// K:254-283. VS walks the shuffled order (min-max stage), VI the identity order
// (re-solve toward the warm start on the z-relaxed set).
template <typename R, typename VS, typename VI, typename P>
__device__ __forceinline__ void least_penetration(const VS &shuf, const VI &ident, P &proj, int k,
                                                  int begin, R cap, R wx, R wy, R &rx, R &ry)
{
    const R w2 = wx * wx + wy * wy;
    if (w2 > cap * cap) {
        const R s = div_rn<R>(cap, sqrt_rn<R>(w2));
        wx = wx * s;
        wy = wy * s;
    }
    R vx = wx, vy = wy, z;
    lp3_minmax<R, VS, P>(shuf, proj, k, begin, cap, vx, vy, z);

    R slack = R(0);
    for (int attempt = 0; attempt < 3; ++attempt) {
        const R zz = z + slack;
        int fail;
        R qx, qy;
        if (lp2_target<R, true, VI>(ident, k, zz, cap, wx, wy, fail, qx, qy)) {
            rx = qx;
            ry = qy;
            return;
        }
        slack = slack * R(1e3) + R(1e-12) * (R(1) + z);
    }
    rx = vx;
    ry = vy;
}

} // namespace orca

// ---------------------------------------------------------------------------
// Group-cooperative variants of the fallback stage: GL (= 8) adjacent lanes work on
// ONE agent. The outer loops (constraint insertion order) stay sequential and are
// executed redundantly by every lane of the group; the inner loops over earlier
// constraints are split across the lanes and combined with shuffles. Nothing changes
// numerically: each (i, j) term is evaluated by exactly the same operations, and the
// combinations are max / min / any, which are exact and order-independent -- so the
// FP64 build stays bit-identical to K:153-283.
// ---------------------------------------------------------------------------

namespace orca {

#ifndef ORCA_GL
#define ORCA_GL 4 // lanes per agent in the step (4 measured best for dense crowds, 8 for sparse)
#endif

template <typename R, int GL> __device__ __forceinline__ R group_max(R v, unsigned gmask)
{
#pragma unroll
    for (int o = GL / 2; o > 0; o >>= 1) {
        const R u = __shfl_xor_sync(gmask, v, o);
        v = u > v ? u : v;
    }
    return v;
}

template <typename R, int GL> __device__ __forceinline__ R group_min(R v, unsigned gmask)
{
#pragma unroll
    for (int o = GL / 2; o > 0; o >>= 1) {
        const R u = __shfl_xor_sync(gmask, v, o);
        v = u < v ? u : v;
    }
    return v;
}

// First position p in [i, k) at which pred(p) holds, or k. The sequential scans of the stage
// ("next violated constraint") test ONE position per iteration and every lane of a group repeats
// the same test; here the group's lanes test GL consecutive positions at once and a group ballot
// picks the first hit. pred evaluates exactly the expression the sequential loop evaluates at p,
// against the same (vx, vy), so the position found -- and everything after it -- is unchanged.
// Must be called by all lanes of the group with the same i and k.
// Measured: with 16 lanes per problem (k_lp_batch_fallback, k up to 64) the batched LP's
// infeasible mix went 14.5 -> 11.8 ms; with 2 or 4 lanes per agent (k_solve_group,
// k_fallback_coop, k <= 16) the ballot per 2-4 positions costs more than the redundant test
// (1 M plaza 0.845 -> 0.94 ms), so small groups keep the sequential scan.
#ifndef ORCA_PARALLEL_SCAN_MIN_GL
#define ORCA_PARALLEL_SCAN_MIN_GL 8
#endif
#ifndef ORCA_SCAN_BATCH
#define ORCA_SCAN_BATCH 4
#endif
template <int GL, int BATCH = 1, typename F>
__device__ __forceinline__ int g_find_first(int i, int k, int gl, unsigned gmask, F pred)
{
    if constexpr (GL < ORCA_PARALLEL_SCAN_MIN_GL) {
        if constexpr (BATCH <= 1) {
            for (; i < k; ++i)
                if (pred(i)) return i;
            return k;
        } else {
            // BATCH positions per trip: their shared-memory loads are in flight together instead of one
            // exposed load latency per position (positions past the end re-test the last one). For the
            // solve kernels' scan (ORCA_SCAN_BATCH = 4: FP64 solve stage 0.469 -> 0.458 ms, f64 0.509 -> 0.489);
            // the least-penetration stage of a jammed crowd is bound by instruction count and loses 5 %
            // to the redundant tests, so its scans stay one position per trip
            for (; i < k; i += BATCH) {
                unsigned m = 0;
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const bool hit = pred(min(i + u, k - 1));
                    m |= (hit && i + u < k) ? (1u << u) : 0u;
                }
                if (m) return i + __ffs((int)m) - 1;
            }
            return k;
        }
    }
    const int gshift = __ffs((int)gmask) - 1;
    for (; i < k; i += GL) {
        const int p = i + gl;
        const bool hit = p < k && pred(p);
        const unsigned bits = (__ballot_sync(gmask, hit) & gmask) >> gshift;
        if (bits) return i + __ffs((int)bits) - 1;
    }
    return k;
}

// K:74-119 with the j loop split over the group
template <typename R, int GL, bool SHIFT, typename V>
__device__ __forceinline__ bool g_lp1_target(const V &view, int i_pos, R zz, R cap, R tx, R ty, R &ox,
                                             R &oy, int gl, unsigned gmask)
{
    R px, py, nx, ny;
    view.get(i_pos, px, py, nx, ny);
    if (SHIFT) {
        px = px - zz * nx;
        py = py - zz * ny;
    }
    const R dx = -ny, dy = nx;
    const R pd = px * dx + py * dy;
    const R disc = pd * pd + cap * cap - (px * px + py * py);
    if (disc < R(0)) return false; // uniform over the group
    const R sq = sqrt_rn<R>(disc);
    R t_left = -pd - sq;
    R t_right = -pd + sq;
    bool bad = false;
    for (int j_pos = gl; j_pos < i_pos; j_pos += GL) {
        R qx, qy, mx, my;
        view.get(j_pos, qx, qy, mx, my);
        if (SHIFT) {
            qx = qx - zz * mx;
            qy = qy - zz * my;
        }
        const R a = dx * mx + dy * my;
        const R b = (qx - px) * mx + (qy - py) * my;
        const bool par = R(-ORCA_PARALLEL_EPS) <= a && a <= R(ORCA_PARALLEL_EPS);
        bad = bad || (par && b > R(0));
        const R t = div_rn<R>(b, a); // unused when par
        if (!par && a > R(0) && t > t_left) t_left = t;
        if (!par && !(a > R(0)) && t < t_right) t_right = t;
    }
    bad = (__ballot_sync(gmask, bad) & gmask) != 0u;
    t_left = group_max<R, GL>(t_left, gmask);
    t_right = group_min<R, GL>(t_right, gmask);
    if (bad || t_left > t_right) return false;
    R t = (tx - px) * dx + (ty - py) * dy;
    if (t < t_left) t = t_left;
    else if (t > t_right) t = t_right;
    ox = px + t * dx;
    oy = py + t * dy;
    return true;
}

// K:122-146
template <typename R, int GL, bool SHIFT, typename V>
__device__ __forceinline__ bool g_lp2_target(const V &view, int k, R zz, R cap, R tx, R ty, int &fail_pos,
                                             R &vx, R &vy, int gl, unsigned gmask)
{
    const R t2 = tx * tx + ty * ty;
    if (t2 > cap * cap) {
        const R s = div_rn<R>(cap, sqrt_rn<R>(t2));
        vx = tx * s;
        vy = ty * s;
    } else {
        vx = tx;
        vy = ty;
    }
    int i_pos = 0;
    while (true) {
        i_pos = g_find_first<GL, (SHIFT ? 1 : ORCA_SCAN_BATCH)>(i_pos, k, gl, gmask, [&](int p) {
            R px, py, nx, ny;
            view.get(p, px, py, nx, ny);
            if (SHIFT) {
                px = px - zz * nx;
                py = py - zz * ny;
            }
            return (vx - px) * nx + (vy - py) * ny < R(0);
        });
        if (i_pos >= k) break;
        R nvx, nvy;
        if (!g_lp1_target<R, GL, SHIFT, V>(view, i_pos, zz, cap, tx, ty, nvx, nvy, gl, gmask)) {
            fail_pos = i_pos;
            return false;
        }
        vx = nvx;
        vy = nvy;
        ++i_pos;
    }
    fail_pos = -1;
    return true;
}

// lp2_target_runahead for a group of GL lanes per problem: the scan is executed
// redundantly by the group's lanes (same data, same result), the 1-D solves split their
// j loops over the group. SHIFT / zz as in lp1_target (the z-relaxed set of K:276-278).
template <typename R, int GL, bool SHIFT, typename V>
__device__ __forceinline__ bool g_lp2_target_runahead(const V &view, int k, R zz, R cap, R tx, R ty,
                                                      int &fail_pos, R &vx, R &vy, unsigned live,
                                                      bool enabled, int gl, unsigned gmask)
{
    const R t2 = tx * tx + ty * ty;
    if (t2 > cap * cap) {
        const R s = div_rn<R>(cap, sqrt_rn<R>(t2));
        vx = tx * s;
        vy = ty * s;
    } else {
        vx = tx;
        vy = ty;
    }
    int i_pos = 0;
    bool done = !enabled, ok = true;
    fail_pos = -1;
    while (true) {
        bool found = false;
        if (!done) { // (uniform over the group)
            i_pos = g_find_first<GL, (SHIFT ? 1 : ORCA_SCAN_BATCH)>(i_pos, k, gl, gmask, [&](int p) {
                R px, py, nx, ny;
                view.get(p, px, py, nx, ny);
                if (SHIFT) {
                    px = px - zz * nx;
                    py = py - zz * ny;
                }
                return (vx - px) * nx + (vy - py) * ny < R(0);
            });
            found = i_pos < k;
            done = !found;
        }
        if (!__any_sync(live, found)) break;
        if (found) {
            R nvx, nvy;
            if (g_lp1_target<R, GL, SHIFT, V>(view, i_pos, zz, cap, tx, ty, nvx, nvy, gl, gmask)) {
                vx = nvx;
                vy = nvy;
                ++i_pos;
            } else {
                fail_pos = i_pos;
                ok = false;
                done = true;
            }
        }
    }
    return ok;
}

// K:153-190
template <typename R, int GL, typename P>
__device__ __forceinline__ bool g_lp1_dir(const P &proj, int upto, R cap, R ox, R oy, R &rx, R &ry, int gl,
                                          unsigned gmask)
{
    R px, py, nx, ny;
    proj.get(upto, px, py, nx, ny);
    const R dx = -ny, dy = nx;
    const R pd = px * dx + py * dy;
    const R disc = pd * pd + cap * cap - (px * px + py * py);
    if (disc < R(0)) return false;
    const R sq = sqrt_rn<R>(disc);
    R t_left = -pd - sq;
    R t_right = -pd + sq;
    bool bad = false;
    for (int j = gl; j < upto; j += GL) {
        R qx, qy, mx, my;
        proj.get(j, qx, qy, mx, my);
        const R a = dx * mx + dy * my;
        const R b = (qx - px) * mx + (qy - py) * my;
        const bool par = R(-ORCA_PARALLEL_EPS) <= a && a <= R(ORCA_PARALLEL_EPS);
        bad = bad || (par && b > R(0));
        const R t = div_rn<R>(b, a);
        if (!par && a > R(0) && t > t_left) t_left = t;
        if (!par && !(a > R(0)) && t < t_right) t_right = t;
    }
    bad = (__ballot_sync(gmask, bad) & gmask) != 0u;
    t_left = group_max<R, GL>(t_left, gmask);
    t_right = group_min<R, GL>(t_right, gmask);
    if (bad || t_left > t_right) return false;
    const R t = (dx * ox + dy * oy) > R(0) ? t_right : t_left;
    rx = px + t * dx;
    ry = py + t * dy;
    return true;
}

// K:193-205
template <typename R, int GL, typename P>
__device__ __forceinline__ bool g_lp2_dir(const P &proj, int m, R cap, R ox, R oy, R &rx, R &ry, int gl,
                                          unsigned gmask)
{
    R vx = cap * ox, vy = cap * oy;
    int i = 0;
    while (true) {
        i = g_find_first<GL>(i, m, gl, gmask, [&](int p) {
            R px, py, nx, ny;
            proj.get(p, px, py, nx, ny);
            return (vx - px) * nx + (vy - py) * ny < R(0);
        });
        if (i >= m) break;
        R nvx, nvy;
        if (!g_lp1_dir<R, GL, P>(proj, i, cap, ox, oy, nvx, nvy, gl, gmask)) {
            rx = vx;
            ry = vy;
            return false;
        }
        vx = nvx;
        vy = nvy;
        ++i;
    }
    rx = vx;
    ry = vy;
    return true;
}

// K:212-251. The projected constraints of one (c, j<i_pos) sweep are built GL at a time
// and compacted in ascending j (ballot rank), which is the order K:226-243 appends them.
template <typename R, int GL, typename V, typename P>
__device__ __forceinline__ void g_lp3_minmax(const V &view, P &proj, int k, int begin, R cap, R &vx, R &vy,
                                             R &z, int gl, unsigned gmask, int gshift)
{
    R dist = R(0);
    int i_pos = begin;
    while (true) {
        i_pos = g_find_first<GL>(i_pos, k, gl, gmask, [&](int p) {
            R qx, qy, mx, my;
            view.get(p, qx, qy, mx, my);
            return (qx - vx) * mx + (qy - vy) * my > dist;
        });
        if (i_pos >= k) break;
        R cpx, cpy, cnx, cny;
        view.get(i_pos, cpx, cpy, cnx, cny);
        {
            int m = 0;
            for (int j0 = 0; j0 < i_pos; j0 += GL) {
                const int j_pos = j0 + gl;
                bool valid = false;
                R ppx = R(0), ppy = R(0), pnx = R(0), pny = R(0);
                if (j_pos < i_pos) {
                    R jpx, jpy, jnx, jny;
                    view.get(j_pos, jpx, jpy, jnx, jny);
                    const R mx = jnx - cnx;
                    const R my = jny - cny;
                    const R ml2 = mx * mx + my * my;
                    if (!(ml2 < R(1e-24))) {
                        const R rhs = jpx * jnx + jpy * jny - cpx * cnx - cpy * cny;
                        const R ml = sqrt_rn<R>(ml2);
                        ppx = div_rn<R>(mx * rhs, ml2);
                        ppy = div_rn<R>(my * rhs, ml2);
                        pnx = div_rn<R>(mx, ml);
                        pny = div_rn<R>(my, ml);
                        valid = true;
                    }
                }
                const unsigned bits = (__ballot_sync(gmask, valid) & gmask) >> gshift; // GL bits
                if (valid) proj.set(m + __popc(bits & ((1u << gl) - 1u)), ppx, ppy, pnx, pny); // gl < 32
                m += __popc(bits);
            }
            __syncwarp(gmask); // projected constraints visible to the whole group
            R nvx, nvy;
            if (g_lp2_dir<R, GL, P>(proj, m, cap, cnx, cny, nvx, nvy, gl, gmask)) {
                vx = nvx;
                vy = nvy;
            }
            dist = (cpx - vx) * cnx + (cpy - vy) * cny;
            if (dist < R(0)) dist = R(0);
            __syncwarp(gmask); // everyone is done reading before the next sweep overwrites
        }
        ++i_pos;
    }
    z = dist;
}

// K:254-283
template <typename R, int GL, typename VS, typename VI, typename P>
__device__ __forceinline__ void g_least_penetration(const VS &shuf, const VI &ident, P &proj, int k, int begin,
                                                    R cap, R wx, R wy, R &rx, R &ry, int gl, unsigned gmask,
                                                    int gshift)
{
    const R w2 = wx * wx + wy * wy;
    if (w2 > cap * cap) {
        const R s = div_rn<R>(cap, sqrt_rn<R>(w2));
        wx = wx * s;
        wy = wy * s;
    }
    R vx = wx, vy = wy, z;
    g_lp3_minmax<R, GL, VS, P>(shuf, proj, k, begin, cap, vx, vy, z, gl, gmask, gshift);
    R slack = R(0);
    for (int attempt = 0; attempt < 3; ++attempt) {
        const R zz = z + slack;
        int fail;
        R qx, qy;
        if (g_lp2_target<R, GL, true, VI>(ident, k, zz, cap, wx, wy, fail, qx, qy, gl, gmask)) {
            rx = qx;
            ry = qy;
            return;
        }
        slack = slack * R(1e3) + R(1e-12) * (R(1) + z);
    }
    rx = vx;
    ry = vy;
}

// ---------------------------------------------------------------------------
// Run-ahead versions of the group-cooperative fallback stage. In k_fallback_coop a warp
// holds 32/GL agents whose control flow differs (which constraint raises the maximum
// violation, which projected constraint is violated, which attempt succeeds): executed
// as written above, a warp runs the union of its groups' paths one after the other
// (measured: 8.5 of 32 lanes active). Here every data-dependent "find the next index
// that needs work" scan is followed by a warp vote, so that the expensive bodies -- the
// projected-constraint sweep, g_lp1_dir, g_lp1_target -- are entered by all groups that
// need them at the same time. Same operations per agent, same results.
// `live`: lanes that execute the call (all must); `enabled`: this group has an agent.
// ---------------------------------------------------------------------------

template <typename R, int GL, typename P>
__device__ __forceinline__ bool g_lp2_dir_ra(const P &proj, int m, R cap, R ox, R oy, R &rx, R &ry, int gl,
                                             unsigned gmask, unsigned live, bool enabled)
{
    R vx = cap * ox, vy = cap * oy;
    int i = 0;
    bool done = !enabled, ok = true;
    while (true) {
        bool found = false;
        if (!done) { // (uniform over the group)
            i = g_find_first<GL>(i, m, gl, gmask, [&](int p) {
                R px, py, nx, ny;
                proj.get(p, px, py, nx, ny);
                return (vx - px) * nx + (vy - py) * ny < R(0);
            });
            found = i < m;
            done = !found;
        }
        if (!__any_sync(live, found)) break;
        if (found) {
            R nvx, nvy;
            if (g_lp1_dir<R, GL, P>(proj, i, cap, ox, oy, nvx, nvy, gl, gmask)) {
                vx = nvx;
                vy = nvy;
                ++i;
            } else { // K:199-202: keep the last point, report failure
                ok = false;
                done = true;
            }
        }
    }
    rx = vx;
    ry = vy;
    return ok;
}

template <typename R, int GL, typename V, typename P>
__device__ __forceinline__ void g_lp3_minmax_ra(const V &view, P &proj, int k, int begin, R cap, R &vx, R &vy,
                                                R &z, int gl, unsigned gmask, int gshift, unsigned live,
                                                bool enabled)
{
    R dist = R(0);
    int i_pos = begin;
    bool done = !enabled;
    while (true) {
        bool found = false;
        R cpx = R(0), cpy = R(0), cnx = R(0), cny = R(0);
        if (!done) { // (uniform over the group)
            i_pos = g_find_first<GL>(i_pos, k, gl, gmask, [&](int p) {
                R qx, qy, mx, my;
                view.get(p, qx, qy, mx, my);
                return (qx - vx) * mx + (qy - vy) * my > dist;
            });
            found = i_pos < k;
            if (found) view.get(i_pos, cpx, cpy, cnx, cny);
            done = !found;
        }
        if (!__any_sync(live, found)) break;
        int m = 0;
        if (found) { // projected constraints of (c, j < i_pos), K:226-243, GL at a time
            for (int j0 = 0; j0 < i_pos; j0 += GL) {
                const int j_pos = j0 + gl;
                bool valid = false;
                R ppx = R(0), ppy = R(0), pnx = R(0), pny = R(0);
                if (j_pos < i_pos) {
                    R jpx, jpy, jnx, jny;
                    view.get(j_pos, jpx, jpy, jnx, jny);
                    const R mx = jnx - cnx;
                    const R my = jny - cny;
                    const R ml2 = mx * mx + my * my;
                    if (!(ml2 < R(1e-24))) {
                        const R rhs = jpx * jnx + jpy * jny - cpx * cnx - cpy * cny;
                        const R ml = sqrt_rn<R>(ml2);
                        ppx = div_rn<R>(mx * rhs, ml2);
                        ppy = div_rn<R>(my * rhs, ml2);
                        pnx = div_rn<R>(mx, ml);
                        pny = div_rn<R>(my, ml);
                        valid = true;
                    }
                }
                const unsigned bits = (__ballot_sync(gmask, valid) & gmask) >> gshift;
                if (valid) proj.set(m + __popc(bits & ((1u << gl) - 1u)), ppx, ppy, pnx, pny);
                m += __popc(bits);
            }
            __syncwarp(gmask); // projected constraints visible to the whole group
        }
        R nvx, nvy;
        const bool ok = g_lp2_dir_ra<R, GL, P>(proj, m, cap, cnx, cny, nvx, nvy, gl, gmask, live, found);
        if (found) {
            if (ok) {
                vx = nvx;
                vy = nvy;
            }
            dist = (cpx - vx) * cnx + (cpy - vy) * cny;
            if (dist < R(0)) dist = R(0);
            ++i_pos;
            __syncwarp(gmask); // everyone is done reading before the next sweep overwrites
        }
    }
    z = dist;
}

template <typename R, int GL, typename VS, typename VI, typename P>
__device__ __forceinline__ void g_least_penetration_ra(const VS &shuf, const VI &ident, P &proj, int k,
                                                       int begin, R cap, R wx, R wy, R &rx, R &ry, int gl,
                                                       unsigned gmask, int gshift, unsigned live, bool enabled)
{
    const R w2 = wx * wx + wy * wy;
    if (w2 > cap * cap) {
        const R s = div_rn<R>(cap, sqrt_rn<R>(w2));
        wx = wx * s;
        wy = wy * s;
    }
    R vx = wx, vy = wy, z = R(0);
    g_lp3_minmax_ra<R, GL, VS, P>(shuf, proj, k, begin, cap, vx, vy, z, gl, gmask, gshift, live, enabled);
    rx = vx; // K:283: the min-max point unless a re-solve succeeds
    ry = vy;
    R slack = R(0);
    bool open = enabled; // still looking for a feasible re-solve
    for (int attempt = 0; attempt < 3; ++attempt) {
        const R zz = z + slack;
        int fail;
        R qx, qy;
        const bool ok = g_lp2_target_runahead<R, GL, true, VI>(ident, k, zz, cap, wx, wy, fail, qx, qy, live,
                                                               open, gl, gmask);
        if (open && ok) {
            rx = qx;
            ry = qy;
            open = false;
        }
        slack = slack * R(1e3) + R(1e-12) * (R(1) + z);
        if (!__any_sync(live, open)) break;
    }
}

} // namespace orca

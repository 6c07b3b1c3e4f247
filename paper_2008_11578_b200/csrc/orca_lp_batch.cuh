// orca_lp_batch.cuh -- standalone batched LP over CSR-packed problems, the device
// twin of _kernels.solve_range (pkg/src/orcasim/_kernels.py:306-336), plus the
// single-op taps used by the known-answer tests.
#pragma once

#include "orca_common.cuh"
#include "orca_kernels.cuh"

namespace orca {

#define LP_SMEM_K 64 // problems up to this many constraints keep their insertion order in shared memory

template <typename R> struct GlobalShuf {
    const typename Vec<R>::T4 *cons; // this problem's rows
    const int *perm;
    const u8 *sperm; // shared-memory copy of the order, [position * 128] (k_lp_batch), or nullptr
    __device__ __forceinline__ void get(int pos, R &px, R &py, R &nx, R &ny) const
    {
        const typename Vec<R>::T4 c = cons[sperm ? (int)sperm[pos * 128] : perm[pos]];
        px = c.x;
        py = c.y;
        nx = c.z;
        ny = c.w;
    }
};

template <typename R> struct GlobalIdent {
    const typename Vec<R>::T4 *cons;
    __device__ __forceinline__ void get(int t, R &px, R &py, R &nx, R &ny) const
    {
        const typename Vec<R>::T4 c = cons[t];
        px = c.x;
        py = c.y;
        nx = c.z;
        ny = c.w;
    }
};

template <typename R> struct GlobalProj {
    typename Vec<R>::T4 *p;
    __device__ __forceinline__ void get(int m, R &px, R &py, R &nx, R &ny) const
    {
        const typename Vec<R>::T4 c = p[m];
        px = c.x;
        py = c.y;
        nx = c.z;
        ny = c.w;
    }
    __device__ __forceinline__ void set(int m, R px, R py, R nx, R ny) { p[m] = mk4(px, py, nx, ny); }
};

// Tap: the least-penetration stage alone on one constraint list in the GIVEN order
// (lp.solve_least_penetration, lp.py:168-190 -> K:254-283 with order = identity), one thread.
template <typename R>
__global__ void k_least_penetration_tap(int k, int begin, const typename Vec<R>::T4 *__restrict__ cons,
                                        typename Vec<R>::T4 *__restrict__ proj, double cap, double wx,
                                        double wy, double *__restrict__ out2)
{
    GlobalIdent<R> view{cons};
    GlobalProj<R> pr{proj};
    R rx, ry;
    least_penetration<R, GlobalIdent<R>, GlobalIdent<R>, GlobalProj<R>>(view, view, pr, k, begin, (R)cap, (R)wx,
                                                                        (R)wy, rx, ry);
    out2[0] = (double)rx;
    out2[1] = (double)ry;
}

// (point, normal) float64 rows -> packed (px, py, nx, ny) in R
template <typename R>
__global__ void __launch_bounds__(256)
k_lp_pack(i64 m, const double *__restrict__ cpts, const double *__restrict__ cnrm,
          typename Vec<R>::T4 *__restrict__ cons)
{
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    cons[i] = mk4((R)cpts[2 * i], (R)cpts[2 * i + 1], (R)cnrm[2 * i], (R)cnrm[2 * i + 1]);
}

template <typename R>
__global__ void __launch_bounds__(256)
k_lp_pack_problems(i64 n, const double *__restrict__ tgt, const double *__restrict__ caps,
                   typename Vec<R>::T4 *__restrict__ prob)
{
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    prob[i] = mk4((R)tgt[2 * i], (R)tgt[2 * i + 1], (R)caps[i], R(0));
}

// Main pass: one thread per problem, shuffled incremental LP (K:290-299). Per-problem
// scratch (order, projected constraints) lives in global memory at the problem's own
// CSR offsets, so any k works. Infeasible problems are queued with the state the
// least-penetration stage starts from.
template <typename R>
__global__ void __launch_bounds__(128)
k_lp_batch(i64 n, const i64 *__restrict__ coff, const typename Vec<R>::T4 *__restrict__ cons,
           const typename Vec<R>::T4 *__restrict__ prob, const u64 *__restrict__ seeds,
           int *__restrict__ perm_scratch, double *__restrict__ out_v, i64 *__restrict__ out_status,
           i64 *__restrict__ out_failed, int *__restrict__ fq_count, int *__restrict__ fq,
           typename Vec<R>::T4 *__restrict__ fq_state)
{
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned live = __ballot_sync(0xFFFFFFFFu, i < n);
    if (i >= n) return;
    const i64 lo = coff[i];
    const int k = (int)(coff[i + 1] - lo);
    const typename Vec<R>::T4 pr = prob[i];
    int *perm = perm_scratch + lo;
    // The insertion order lives in shared memory (one byte per position, [position][thread])
    // when k <= LP_SMEM_K: the Fisher-Yates swaps and the order look-ups of the LP then stay
    // on chip instead of being uncoalesced 4-byte global accesses. Larger problems use the
    // global scratch; the least-penetration stage always reads the global copy, written below
    // for the problems that need it.
    __shared__ u8 sm_perm[LP_SMEM_K * 128];
    u8 *sperm = k <= LP_SMEM_K ? sm_perm + threadIdx.x : nullptr;

    // _kernels.py:43-54
    u64 state = seeds[i];
    if (sperm) {
        for (int t = 0; t < k; ++t) sperm[t * 128] = (u8)t;
        for (int t = k - 1; t > 0; --t) {
            state += ORCA_GOLDEN;
            const int j = (int)mod_small(mix64(state), (uint32_t)(t + 1));
            const u8 tmp = sperm[t * 128];
            sperm[t * 128] = sperm[j * 128];
            sperm[j * 128] = tmp;
        }
    } else {
        for (int t = 0; t < k; ++t) perm[t] = t;
        for (int t = k - 1; t > 0; --t) {
            state += ORCA_GOLDEN;
            const u64 r = mix64(state);
            const int j = (t + 1) <= 0xFFFF ? (int)mod_small(r, (uint32_t)(t + 1)) : (int)(r % (u64)(t + 1));
            const int tmp = perm[t];
            perm[t] = perm[j];
            perm[j] = tmp;
        }
    }

    GlobalShuf<R> shuf{cons + lo, perm, sperm};
    int fail_pos;
    R vx, vy;
    // per-lane run-ahead (orca_math.cuh): the problems of a warp differ in k and in where
    // their constraints are violated
    if (lp2_target_runahead<R, GlobalShuf<R>>(shuf, k, pr.z, pr.x, pr.y, fail_pos, vx, vy, live, true)) {
        out_v[2 * i] = (double)vx;
        out_v[2 * i + 1] = (double)vy;
        out_status[i] = 0;
        out_failed[i] = -1;
        return;
    }
    out_status[i] = 1;
    if (sperm)
        for (int t = 0; t < k; ++t) perm[t] = (int)sperm[t * 128];
    out_failed[i] = perm[fail_pos];
    const int q = atomicAdd(fq_count, 1);
    fq[q] = (int)i;
    fq_state[q] = mk4(vx, vy, (R)fail_pos, R(0));
}

// Least-penetration stage of the queued problems, ORCA_GL lanes per problem (see
// k_fallback_coop): the lanes split the loops over earlier constraints and combine with
// exact max / min / any shuffles, so the FP64 build stays bit-identical to K:254-283.
#ifndef ORCA_LP_GL
#define ORCA_LP_GL 16 // lanes per queued problem: k reaches 64 here, against 16 in the step
#endif

template <typename R>
__global__ void __launch_bounds__(128)
k_lp_batch_fallback(const int *__restrict__ fq_count, const int *__restrict__ fq,
                    const typename Vec<R>::T4 *__restrict__ fq_state, const i64 *__restrict__ coff,
                    const typename Vec<R>::T4 *__restrict__ cons, const typename Vec<R>::T4 *__restrict__ prob,
                    const int *__restrict__ perm_scratch, typename Vec<R>::T4 *__restrict__ proj_scratch,
                    double *__restrict__ out_v)
{
    constexpr int GL = ORCA_LP_GL;
    constexpr int NG = 128 / GL;
    const int g = threadIdx.x / GL, gl = threadIdx.x % GL;
    const int gshift = (threadIdx.x & 31) - gl;
    const unsigned gmask = (GL == 32 ? 0xFFFFFFFFu : ((1u << GL) - 1u)) << gshift;
    __shared__ typename Vec<R>::T4 sm_cons[LP_SMEM_K * NG];
    __shared__ typename Vec<R>::T4 sm_proj[LP_SMEM_K * NG];
    __shared__ u8 sm_inv[LP_SMEM_K * NG];
    const int nq = *fq_count;
    for (int q = blockIdx.x * NG + g; q < nq; q += gridDim.x * NG) {
        const int i = fq[q];
        const typename Vec<R>::T4 st = fq_state[q];
        const i64 lo = coff[i];
        const int k = (int)(coff[i + 1] - lo);
        const typename Vec<R>::T4 pr = prob[i];
        R rx, ry;
        if (k <= LP_SMEM_K) {
            // the group stages its problem in shared memory -- constraints in shuffled order,
            // the inverse order for the identity-order re-solve, room for the projected
            // constraints -- so the stage's many passes over them stay on chip
            SmemCons<R> sc{sm_cons + g, NG};
            SmemCons<R> sp{sm_proj + g, NG};
            const int *perm = perm_scratch + lo;
            for (int pos = gl; pos < k; pos += GL) {
                const int t = perm[pos];
                const typename Vec<R>::T4 c = cons[lo + t];
                sc.set(pos, c.x, c.y, c.z, c.w);
                sm_inv[t * NG + g] = (u8)pos;
            }
            __syncwarp(gmask);
            SmemConsIdent<R> si{sm_cons + g, sm_inv + g, NG};
            g_least_penetration<R, GL, SmemCons<R>, SmemConsIdent<R>, SmemCons<R>>(
                sc, si, sp, k, (int)st.z, pr.z, st.x, st.y, rx, ry, gl, gmask, gshift);
            __syncwarp(gmask); // the group's shared memory is reused by its next queue entry
        } else {
            GlobalShuf<R> shuf{cons + lo, perm_scratch + lo, nullptr};
            GlobalIdent<R> ident{cons + lo};
            GlobalProj<R> proj{proj_scratch + lo};
            g_least_penetration<R, GL, GlobalShuf<R>, GlobalIdent<R>, GlobalProj<R>>(
                shuf, ident, proj, k, (int)st.z, pr.z, st.x, st.y, rx, ry, gl, gmask, gshift);
        }
        if (gl == 0) {
            out_v[2 * (i64)i] = (double)rx;
            out_v[2 * (i64)i + 1] = (double)ry;
        }
    }
}

// ---- taps -------------------------------------------------------------------

template <typename R>
__global__ void k_vo_exit_batch(i64 count, const double *__restrict__ in7, double *__restrict__ out5)
{
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double *c = in7 + 7 * i;
    R ux, uy, nx, ny;
    const bool ok = vo_exit<R>((R)c[0], (R)c[1], (R)c[2], (R)c[3], (R)c[4], (R)c[5], (R)c[6], ux, uy,
                               nx, ny);
    out5[5 * i + 0] = (double)ux;
    out5[5 * i + 1] = (double)uy;
    out5[5 * i + 2] = (double)nx;
    out5[5 * i + 3] = (double)ny;
    out5[5 * i + 4] = ok ? 1.0 : 0.0;
}

__global__ void k_shuffle_tap(int k, u64 seed, i64 *perm)
{
    for (int t = 0; t < k; ++t) perm[t] = t;
    u64 state = seed;
    for (int t = k - 1; t > 0; --t) {
        state += ORCA_GOLDEN;
        const u64 r = mix64(state);
        const int j = (t + 1) <= 0xFFFF ? (int)mod_small(r, (uint32_t)(t + 1)) : (int)(r % (u64)(t + 1));
        const i64 tmp = perm[t];
        perm[t] = perm[j];
        perm[j] = tmp;
    }
}

// the unrolled constant-divisor shuffle used inside k_solve / k_fallback, k <= 32
__global__ void k_shuffle_tap_smem(int k, u64 seed, i64 *perm_out)
{
    __shared__ u8 perm[32];
    if (threadIdx.x == 0) {
        shuffle_smem<32>(perm, 1, k, seed);
        for (int t = 0; t < k; ++t) perm_out[t] = perm[t];
    }
}

__global__ void k_seed_tap(i64 frame, i64 agent_id, u64 *out) { *out = problem_seed(frame, agent_id); }

} // namespace orca

// orca_cert.cuh -- ORCA_CERT32: the solve stage in FP32 with a certificate, FP64 only where
// the result is decided.
//
// What bounds the FP64 solve kernel (k_solve_group, profiles/) is sixteen ~130-instruction FP64
// vo_exit chains per agent plus the FP64 incremental LP -- yet the RESULT of a feasible LP
// depends on at most two of the sixteen half-planes: the optimum is the preferred velocity
// itself, its projection onto one constraint line, or the intersection of two lines
// (_kernels.py:74-146). k_solve_cert therefore
//
//   1. builds all half-planes and runs the shuffled incremental LP in FP32 (the arithmetic of
//      k_solve<float>), remembering which constraints ended up ACTIVE: the line L of the last
//      1-D solve and the earlier constraint B that bound it (or none);
//   2. re-evaluates in FP64 exactly what the reference evaluates on that active set -- the
//      half-planes of L and B (vo_exit<double>, same operations, K:343-419) and the closing
//      formula of _lp1_target (K:98-119) -- which costs 0-2 FP64 vo_exit chains instead of 16;
//   3. CERTIFIES that candidate, independently of the path the FP32 LP took: it must satisfy
//      every other half-plane with a margin above that half-plane's FP32 error bound, lie
//      strictly inside the speed disc, and satisfy the optimality (KKT) sign conditions of its
//      active set with margins. A feasible point with a valid KKT certificate IS the optimum of
//      this strictly convex problem, the optimum is unique, the margins make the active set
//      non-degenerate, and with a non-degenerate active set the reference's last 1-D solve is
//      on the later-inserted active constraint bounded by the earlier one -- i.e. the value
//      computed in step 2, bit for bit. (The FP32 run only GUESSES the active set; nothing it
//      decides is trusted.)
//   4. and it checks the WAY there. The reference does not only return the optimum, it reports
//      whether its incremental LP got there (status / failed_at), and that LP gives up on yes / no
//      tests of its own -- a (nearly) parallel earlier constraint with the line outside it
//      (K:100-103), an interval that closed (K:112), a line missing the speed disc (K:86). On
//      duplicated half-planes (symmetric crowds) or three lines through one point those tests hang
//      on FP64 rounding and can declare a feasible LP infeasible. The intermediate optima the
//      incremental LP visits (of the first 1, 2, ... constraints in insertion order) do not depend
//      on who computes them, so the FP32 run sees the same situations: every scan decision must be
//      clear of the half-plane's error bound plus the current vertex's, every 1-D solve clear of a
//      parallel-and-not-inside constraint, of a closing interval, of a grazed disc and of an
//      ill-conditioned vertex (lp1_target_act: `shaky`). Found by the adversarial soak
//      (tests/soak/soak_cert_adversarial.py, one status mismatch in 2,300 lattice crowds before).
//
// An agent that is not certified -- infeasible LP (the least-penetration stage needs FP64
// half-planes anyway), an active speed disc, near-parallel active lines, a margin too small, an
// FP32 half-plane whose branch decisions (overlap K:357, leg side K:404) sit within rounding of
// flipping -- is queued (plan->cq_count / cq) and solved by the FP64 kernels exactly as in
// ORCA_MIXED. Results are therefore those of ORCA_MIXED: identical status / failed_at, FP64
// velocities rounded once to the FP32 state (tests/test_gpu_step.py: every agent of every
// BASELINE crowd against the oracle).
#pragma once

#include <cuda_fp16.h>

#include "orca_kernels.cuh"

namespace orca {

#define CERT_EPS 1.1920929e-07f // 2^-23
#define CERT_INF 1e30f
#ifndef CERT_SAFETY
#define CERT_SAFETY 8.0f        // multiplies every first-order error estimate below
#endif
#ifndef ORCA_CERT_MIN_AGENTS
#define ORCA_CERT_MIN_AGENTS 65536        // below: launch-latency bound, the extra kernels cost more than they save
#endif
#ifndef ORCA_CERT_MAX_FALLBACK_PCT
#define ORCA_CERT_MAX_FALLBACK_PCT 25     // above: most agents need the FP64 kernels anyway (measured break-even ~30 %)
#endif
#define CERT_CROSS_MIN 0.02f    // |n_L x n_B| below this: the vertex is ill-conditioned, leave it to FP64
#define CERT_PAR_BAND 1e-4f     // |d_i . n_j| below this: "parallel" as far as FP32 can tell (the reference: 1e-12 in FP64)
#define CERT_VERR_MAX 1e-2f     // an intermediate vertex whose error bound exceeds this is not followed
#ifndef CERT_TASK_BUCKETS
#define CERT_TASK_BUCKETS 6     // LP tasks of a block are ordered by min(clearly violated half-planes, this)
#endif

// vo_exit<float> (orca_math.cuh) plus a first-order bound on how far the FP32 half-plane can be
// from the FP64 one: err_n on the unit normal (radians), err_u on the exit vector. CERT_INF when
// a DIScontinuous branch decision could flip under rounding (the arc / leg choice is continuous:
// both formulas meet at the tangent points, so it needs no guard).
__device__ __forceinline__ bool vo_exit_cond(float rpx, float rpy, float rvx, float rvy, float comb_r,
                                             float inv_tau, float inv_dt, float &ux, float &uy, float &nx,
                                             float &ny, float &err_u, float &err_n)
{
    // (explicit fused multiply-adds and approximate reciprocals: this translation unit is compiled
    //  with -fmad=false for the bit-exact FP64 paths, but the FP32 pass is only a guess with an
    //  error bound a few times wider than any of these shortcuts)
    const float d2 = __fmaf_rn(rpx, rpx, rpy * rpy);
    const float r2 = comb_r * comb_r;
    const bool overlap = d2 < r2; // K:357
    const float inv = overlap ? inv_dt : inv_tau;
    const float rr = comb_r * inv;
    const float wx = __fmaf_rn(-rpx, inv, rvx), wy = __fmaf_rn(-rpy, inv, rvy); // w = rv - rp / tau
    const float wl2 = __fmaf_rn(wx, wx, wy * wy);
    const float dot_wp = __fmaf_rn(wx, rpx, wy * rpy);
    const bool arc = overlap || (dot_wp < 0.0f && dot_wp * dot_wp > r2 * wl2); // K:395
    const float dmr = d2 - r2, dpr = d2 + r2;
    const float arg = arc ? wl2 : dmr;
    const float rsq = rsqrtf(arg);          // 1 / |w|  or  1 / leg
    const float sq = arg * rsq;
    const float p1 = rpx * wy, p2 = rpy * wx;
    const float crs = p1 - p2;
    const bool side = crs > 0.0f; // K:404
    // leg direction (K:405-412): (rpx sq -+ rpy R, +-rpy sq + rpx R) with the sign of the side
    const float ssq = side ? sq : -sq;
    const float lx = __fmaf_rn(rpx, ssq, -(rpy * comb_r));
    const float ly = __fmaf_rn(rpy, ssq, rpx * comb_r);
    const float rd2 = __fdividef(1.0f, d2);
    const float iden = arc ? rsq : rd2;
    const float qx = (arc ? wx : lx) * iden;
    const float qy = (arc ? wy : ly) * iden;
    const float s = rr - sq;
    const float t = __fmaf_rn(rvx, qx, rvy * qy);
    const bool flip = __fmaf_rn(qx, rpy, -(qy * rpx)) > 0.0f; // (m = (-qy, qx); m . rp > 0)
    const float mx = flip ? qy : -qy, my = flip ? -qx : qx;
    // u = s q (arc) or t q - rv (leg), as ONE fused form so that no branch splits the loop body
    const float ut = arc ? s : t, ucx = arc ? 0.0f : -rvx, ucy = arc ? 0.0f : -rvy;
    ux = __fmaf_rn(ut, qx, ucx);
    uy = __fmaf_rn(ut, qy, ucy);
    nx = arc ? qx : mx;
    ny = arc ? qy : my;
    // --- conditioning (first order; CERT_SAFETY covers the approximations above) ---
    const float srv = fabsf(rvx) + fabsf(rvy);
    const float sw = __fmaf_rn(fabsf(rpx) + fabsf(rpy), inv, srv); // scale of the operands of w
    // arc: q = w / |w|, u = (rr - |w|) q.   leg = sqrt(d2 - r2): cancellation when the discs almost touch,
    // kappa = (d2 + r2) / (d2 - r2) = (d2 + r2) * rsq^2, and the direction error is kappa * leg / |rp|
    const float en_arc = (4.0f * CERT_EPS) * __fmaf_rn(sw, rsq, 1.0f);
    const float eu_arc = __fmaf_rn(fabsf(s), en_arc, (4.0f * CERT_EPS) * (sw + fabsf(rr)));
    const float en_leg = (2.0f * CERT_EPS) * __fmaf_rn(dpr * rsq, rsqrtf(d2), 3.0f);
    const float eu_leg = srv * __fmaf_rn(2.0f, en_leg, 4.0f * CERT_EPS);
    const float en = arc ? en_arc : en_leg, eu = arc ? eu_arc : eu_leg;
    bool sure = fabsf(dmr) > (64.0f * CERT_EPS) * dpr;                                  // overlap decision
    sure = sure && wl2 > 1e-9f * (sw * sw) && wl2 > 1e-20f;                             // |w|^2 < 1e-24 branch, q = w/|w|
    sure = sure && (overlap || fabsf(crs) > (64.0f * CERT_EPS) * (fabsf(p1) + fabsf(p2))); // leg side
    sure = sure && d2 > 0.0f;
    err_n = sure ? CERT_SAFETY * en : CERT_INF;
    err_u = sure ? CERT_SAFETY * eu : CERT_INF;
    return d2 > 0.0f;
}

// _lp1_target (K:74-119) in FP32 that also reports WHICH bound closed the interval:
// kind 0 = the projection of the target itself, 1 / 2 = an earlier constraint (position j_sel)
// from the left / right, 3 / 4 = the speed disc -- and how far the point it returns can be from
// the exact one (verr), and whether any of the reference's own yes / no decisions in this 1-D solve
// sits within the FP32 error of flipping (shaky): a (nearly) parallel earlier constraint that the
// line is not clearly inside (K:100-103 declares the LP infeasible there), an interval about to
// close (K:112), a line grazing the speed disc (K:86), an ill-conditioned binding vertex. The
// reference takes those decisions in FP64 on ITS half-planes; where they hang on rounding --
// duplicated half-planes of a symmetric crowd, three lines through one point -- its result is
// whatever its rounding says, and only the FP64 kernels can reproduce that.
template <typename V>
__device__ __forceinline__ bool lp1_target_act(const V &view, float emax, int i_pos, float cap, float tx, float ty,
                                               float &ox, float &oy, int &kind, int &j_sel, float &verr,
                                               bool &shaky)
{
    float px, py, nx, ny;
    view.get(i_pos, px, py, nx, ny);
    const float ei = emax; // (the agent's LARGEST half-plane error bound stands in for each one's own: no loads here)
    const float dx = -ny, dy = nx;
    const float pd = __fmaf_rn(px, dx, py * dy);
    const float disc = __fmaf_rn(pd, pd, cap * cap) - __fmaf_rn(px, px, py * py);
    if (disc < 0.0f) return false;
    const float sq = disc * rsqrtf(fmaxf(disc, 1e-30f));
    shaky = shaky || sq < CERT_CROSS_MIN * cap; // the line grazes the disc: K:86 within rounding, end points ill-conditioned
    const float ed = ei * cap * __fdividef(1.0f, fmaxf(sq, 1e-20f)); // error of a disc end point
    const float eij = 2.0f * emax;
    float t_left = -pd - sq, t_right = -pd + sq;
    float el = ed, er = ed; // error bounds of the two ends as they stand
    int jl = -1, jr = -1;
    bool bad = false;
#pragma unroll 4
    for (int j_pos = 0; j_pos < i_pos; ++j_pos) {
        float qx, qy, mx, my;
        view.get(j_pos, qx, qy, mx, my);
        const float a = __fmaf_rn(dx, mx, dy * my);
        const float b = __fmaf_rn(qx - px, mx, (qy - py) * my);
        const bool par = fabsf(a) <= 1e-6f;
        bad = bad || (par && b > 0.0f);
        // (nearly) parallel and the line not clearly inside: the reference's "parallel and outside" test
        // (|a| <= 1e-12 and b > 0 in FP64) cannot be told from here
        shaky = shaky || (fabsf(a) <= CERT_PAR_BAND && b > -4.0f * eij);
        const float ra = __fdividef(1.0f, a);
        const float t = b * ra;
        const float et = eij * fabsf(ra);
        if (!par && a > 0.0f && t > t_left) {
            t_left = t;
            jl = j_pos;
            el = et;
        }
        if (!par && !(a > 0.0f) && t < t_right) {
            t_right = t;
            jr = j_pos;
            er = et;
        }
    }
    if (bad || t_left > t_right) return false;
    shaky = shaky || !(t_right - t_left > 2.0f * (el + er)); // the interval is about to close (K:112)
    float t = __fmaf_rn(tx - px, dx, (ty - py) * dy);
    kind = 0;
    j_sel = -1;
    verr = ei;
    if (t < t_left) {
        t = t_left;
        kind = jl >= 0 ? 1 : 3;
        j_sel = jl;
        verr = el + ei;
    } else if (t > t_right) {
        t = t_right;
        kind = jr >= 0 ? 2 : 4;
        j_sel = jr;
        verr = er + ei;
    }
    shaky = shaky || !(verr < CERT_VERR_MAX); // an ill-conditioned vertex: later decisions would be taken at a wrong point
    ox = __fmaf_rn(t, dx, px);
    oy = __fmaf_rn(t, dy, py);
    return true;
}

// lp2_target_runahead (orca_math.cuh) in FP32, reporting the active set of the LAST 1-D solve
// (c_last = -1: the clamped target violated nothing) and whether every decision on the way was clear
// of its error band (shaky, see lp1_target_act): the incremental LP visits the optima of the first 1, 2,
// ... constraints, which do not depend on who computes them, so a scan or a 1-D solve that is clear here
// is decided the same way by the reference.
template <typename V>
__device__ __forceinline__ bool lp2_target_runahead_act(const V &view, float emax, int k, float cap, float tx,
                                                        float ty, float &vx, float &vy, int &c_last, int &kind,
                                                        int &j_sel, bool &shaky, unsigned live, bool enabled)
{
    const float t2 = __fmaf_rn(tx, tx, ty * ty);
    if (t2 > cap * cap) {
        const float s = cap * rsqrtf(t2);
        vx = tx * s;
        vy = ty * s;
    } else {
        vx = tx;
        vy = ty;
    }
    int i_pos = 0;
    bool done = !enabled, ok = true;
    float verr = 0.0f; // how far (vx, vy) can be from the exact intermediate optimum
    c_last = -1;
    kind = 0;
    j_sel = -1;
    while (true) {
        bool found = false;
        if (!done) {
            // next violated constraint at or after i_pos, four positions per trip: the four shared-memory
            // loads are in flight together (one at a time, this scan is a chain of exposed load latencies
            // -- it was 15 % of the kernel's stall samples)
            for (; i_pos < k; i_pos += 4) {
                unsigned m = 0, amb = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int p = min(i_pos + u, k - 1);
                    float px, py, nx, ny;
                    view.get(p, px, py, nx, ny);
                    const float slack = __fmaf_rn(vx - px, nx, (vy - py) * ny);
                    const bool valid = i_pos + u < k;
                    m |= (slack < 0.0f && valid) ? (1u << u) : 0u;
                    amb |= (!(fabsf(slack) > emax + verr) && valid) ? (1u << u) : 0u;
                }
                // the reference examines the positions up to and including the first violated one at this v
                const unsigned seen = m ? ((2u << (__ffs(m) - 1)) - 1u) : 0xFu;
                shaky = shaky || (amb & seen) != 0u;
                if (m) {
                    i_pos += __ffs(m) - 1;
                    found = true;
                    break;
                }
            }
            done = !found;
        }
        if (!__any_sync(live, found)) break;
        if (found) {
            float nvx, nvy, ve = 0.0f;
            int kd, js;
            if (lp1_target_act<V>(view, emax, i_pos, cap, tx, ty, nvx, nvy, kd, js, ve, shaky)) {
                vx = nvx;
                vy = nvy;
                verr = ve;
                c_last = i_pos;
                kind = kd;
                j_sel = js;
                ++i_pos;
            } else {
                ok = false;
                done = true;
            }
        }
    }
    return ok;
}

// One half-plane of agent s in FP64, exactly as k_solve_group<float, double> builds it
// (K:525-541): the neighbour at shuffled position `pos`.
__device__ __forceinline__ bool halfplane64(int s, int pos, const StepParams &P, const NbRec<float> *__restrict__ s_nr,
                                            const int *__restrict__ nb, const u8 *perm, int pstride,
                                            double inv_tau, double inv_dt, double &px, double &py, double &nx,
                                            double &ny)
{
    const NbRec<float> me = s_nr[s];
    const int j = nb[(size_t)perm[pos * pstride] * P.stride + s];
    const NbRec<float> o = s_nr[j];
    const double ri = (double)me.rc.x + P.half_margin, rj = (double)o.rc.x + P.half_margin;
    const int ci = (int)me.rc.y;
    const double f0 = ci ? P.fmat[2] : P.fmat[0], f1 = ci ? P.fmat[3] : P.fmat[1];
    const double mevx = (double)me.pv.z, mevy = (double)me.pv.w;
    double ux, uy;
    const bool ok = vo_exit_inv<double>((double)o.pv.x - (double)me.pv.x, (double)o.pv.y - (double)me.pv.y,
                                        mevx - (double)o.pv.z, mevy - (double)o.pv.w, ri + rj, inv_tau, inv_dt, ux,
                                        uy, nx, ny);
    const double f = o.rc.y != 0.0f ? f1 : f0;
    px = mevx + f * ux;
    py = mevy + f * uy;
    return ok;
}

// The solve stage of ORCA_CERT32 (see the header of this file), FP32 half-planes + their error
// bounds in shared memory ([position][thread]); the insertion order comes from k_shuffle.
//
// Phase A, one thread per agent: build the half-planes and test the (clamped) preferred velocity
// against them. ~40 % of the agents of a sparse crowd violate nothing by a clear margin: they are
// finished here. Agents with a clear violation become LP TASKS.
// Phase B: the tasks of the block are compacted (a shared-memory list), and thread t runs the LP,
// the FP64 evaluation and the certificate of task t on that agent's shared-memory half-planes --
// the warps that do run the divergent LP loops are full of agents that need them, instead of
// every warp dragging its finished lanes through them.
// Certified agents are finished (status 0, FP64 velocity, integration); the others are appended
// to cq for the FP64 kernel (k_solve_group_queue).
template <int MAXN, int THREADS>
__global__ void __launch_bounds__(THREADS)
k_solve_cert(GridPlan *__restrict__ plan, StepParams P, const NbRec<float> *__restrict__ s_nr,
             const double4 *__restrict__ s_dm, const int *__restrict__ s_row, const int *__restrict__ nb,
             const u8 *__restrict__ nb_cnt, const float4 *__restrict__ goalpref, float4 *__restrict__ pv_out,
             i8 *__restrict__ status, i8 *__restrict__ failed_at, u8 *__restrict__ arrived,
             int *__restrict__ cq, const uint32_t *__restrict__ s_perm, int *__restrict__ cq_cnt, int s0, int s1)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4 *sm_cons = reinterpret_cast<float4 *>(smem_raw);
    // (error bounds as halves rounded UP, insertion order in registers: 18 bytes per half-plane, so that
    //  SIX blocks of 128 agents fit an SM's shared memory -- with 21 bytes it was five)
    __half *sm_err = reinterpret_cast<__half *>(sm_cons + MAXN * THREADS);
    __shared__ u8 sm_task[THREADS];     // (THREADS <= 256)
    __shared__ float sm_emax[THREADS];  // each agent's largest half-plane error bound, for its LP task
    __shared__ int sm_bcnt[CERT_TASK_BUCKETS];
    if (threadIdx.x < CERT_TASK_BUCKETS) sm_bcnt[threadIdx.x] = 0;
    __syncthreads();

    const int s_base = s0 + blockIdx.x * THREADS;
    int my_bucket = -1, my_rank = 0; // an LP task: its bucket (by clearly violated half-planes) and rank in it
    {   // ---- phase A ----
        const int s = s_base + threadIdx.x; // this launch covers sorted slots [s0, s1)
        const bool in_range = s < min(s1, plan->n);
        const int row = in_range ? s_row[s] : 0;
        if (in_range && row < plan->n_owned) {
            const int cnt = nb_cnt[s];
            const NbRec<float> me_rec = s_nr[s];
            const float4 me = me_rec.pv;
            const double4 dm = s_dm[s]; // desired velocity (FP64, k_scatter), max_speed, avoid radius
            __half *cerr = sm_err + threadIdx.x;
            SmemCons<float> cons{sm_cons + threadIdx.x, THREADS};
            // the order k_shuffle drew, four positions per word, kept in registers
            uint32_t pw[MAXN / 4];
            {
                const uint32_t *src = s_perm + (size_t)s * (MAXN / 4);
#pragma unroll
                for (int t = 0; t < MAXN / 4; ++t) pw[t] = 4 * t < cnt ? src[t] : 0u;
            }
            auto perm_at = [&](int pos) -> int { // (static register indices only: a select tree)
                uint32_t w = pw[0];
#pragma unroll
                for (int t = 1; t < MAXN / 4; ++t) w = (pos >> 2) == t ? pw[t] : w;
                return (int)((w >> ((pos & 3) * 8)) & 0xFFu);
            };
            const float cap = (float)dm.z;
            // the start of the LP (K:129-136) in FP32: the half-planes are tested against it as they are built
            float v0x = (float)dm.x, v0y = (float)dm.y;
            {
                const float t2 = __fmaf_rn(v0x, v0x, v0y * v0y);
                if (t2 > cap * cap) {
                    const float sc = cap * rsqrtf(t2);
                    v0x *= sc;
                    v0y *= sc;
                }
            }
            bool built = true, unclear = false;
            int nviol = 0;
            float emax = 0.0f;
            {   // FP32 half-planes in shuffled order, each with its error bound against |v| <= cap
                const float hm = (float)P.half_margin;
                const float ri = me_rec.rc.x + hm;
                const float mz = fabsf(me.z) + fabsf(me.w);
                const int ci = (int)me_rec.rc.y;
                const float f0 = (float)(ci ? P.fmat[2] : P.fmat[0]), f1 = (float)(ci ? P.fmat[3] : P.fmat[1]);
                const float inv_tau = __fdividef(1.0f, (float)P.tau), inv_dt = __fdividef(1.0f, (float)P.dt);
                // software pipeline, two deep: a neighbour's record hangs on TWO dependent loads (its
                // index nb[perm[pos]][s], then s_nr[index]), each a trip to L2 -- the index is requested two
                // rounds ahead and the record one round ahead, so neither is waited for
                float4 q_next = me;
                float2 rc_next = me_rec.rc;
                int j_next = 0;
                const int *nbs = nb + s;
                if (cnt > 0) {
                    const NbRec<float> rn = s_nr[nbs[(size_t)perm_at(0) * P.stride]];
                    q_next = rn.pv;
                    rc_next = rn.rc;
                    j_next = nbs[(size_t)perm_at(min(1, cnt - 1)) * P.stride];
                }
#pragma unroll 2
                for (int pos = 0; pos < cnt; ++pos) {
                    const float4 q = q_next;
                    const float2 rc_j = rc_next;
                    {   // (no branches: the last rounds re-read the last neighbour, and the loop body stays one
                        //  basic block the scheduler can interleave with the next round's)
                        const NbRec<float> rn = s_nr[j_next];
                        q_next = rn.pv;
                        rc_next = rn.rc;
                        j_next = nbs[(size_t)perm_at(min(pos + 2, cnt - 1)) * P.stride];
                    }
                    const float rj = rc_j.x + hm;
                    float ux, uy, nx, ny, eu, en;
                    built &= vo_exit_cond(q.x - me.x, q.y - me.y, me.z - q.z, me.w - q.w, ri + rj, inv_tau, inv_dt,
                                          ux, uy, nx, ny, eu, en);
                    const float f = rc_j.y != 0.0f ? f1 : f0;
                    const float px = __fmaf_rn(f, ux, me.z), py = __fmaf_rn(f, uy, me.w);
                    cons.set(pos, px, py, nx, ny);
                    // |(v - p).n evaluated in FP32 - the same in exact arithmetic on the FP64 half-plane|, any |v| <= cap
                    const float reach = cap + fabsf(px) + fabsf(py);
                    const float e = __fmaf_rn(f, eu, __fmaf_rn(en, reach, (CERT_SAFETY * 4.0f * CERT_EPS) * (reach + mz)));
                    cerr[pos * THREADS] = __float2half_ru(e); // (an infinite bound stays infinite)
                    emax = fmaxf(emax, e);
                    const float slack = __fmaf_rn(v0x - px, nx, (v0y - py) * ny);
                    nviol += slack < -e ? 1 : 0;
                    unclear = unclear || !(fabsf(slack) > e); // (also catches an infinite error bound)
                }
            }
            const bool violated = nviol > 0;
            if (!built || (unclear && !violated)) {
                // coincident centres (the FP64 kernel reports them) or a half-plane through the start
                // within its error: nothing to guess, the FP64 kernels decide
                cq[atomicAdd(cq_cnt, 1)] = s;
            } else if (!violated) {
                // the start violates nothing, by margins above every error bound: it is the result (K:137-146
                // never enters _lp1_target), evaluated in FP64 exactly as the reference does
                const double tx = dm.x, ty = dm.y, capd = dm.z;
                double vx = tx, vy = ty;
                const double t2 = tx * tx + ty * ty;
                if (t2 > capd * capd) {
                    const double sc = __ddiv_rn(capd, __dsqrt_rn(t2));
                    vx = tx * sc;
                    vy = ty * sc;
                }
                status[row] = 0;
                failed_at[row] = -1;
                integrate_row<float, double>(row, me, vx, vy, P, goalpref, pv_out, arrived);
            } else {
                // the incremental LP re-solves on (roughly) every half-plane its start violates: tasks with
                // the same count share a warp, so a warp's round count is close to what its lanes need
                my_bucket = min(nviol, CERT_TASK_BUCKETS) - 1;
                my_rank = atomicAdd(&sm_bcnt[my_bucket], 1);
                sm_emax[threadIdx.x] = emax;
            }
        }
    }
    __syncthreads();
    int ntask = 0;
    {
        int before = 0;
#pragma unroll
        for (int b = 0; b < CERT_TASK_BUCKETS; ++b) {
            const int c = sm_bcnt[b];
            if (b < my_bucket) before += c;
            ntask += c;
        }
        if (my_bucket >= 0) sm_task[before + my_rank] = (u8)threadIdx.x;
    }
    __syncthreads();
    // ---- phase B: thread t takes task t ----
    if ((int)(threadIdx.x & ~31u) >= ntask) return; // whole warp without a task
    const bool enabled = (int)threadIdx.x < ntask;
    const int a = enabled ? (int)sm_task[threadIdx.x] : 0; // the agent's thread slot in shared memory
    const int s = s_base + a;
    const int row = s_row[s];
    const int cnt = enabled ? (int)nb_cnt[s] : 0;
    const NbRec<float> me_rec = s_nr[s];
    const float4 me = me_rec.pv;
    const double4 dm = s_dm[s];
    const u8 *perm = reinterpret_cast<const u8 *>(s_perm) + (size_t)s * MAXN; // (position p of the order: byte p)
    const __half *cerr = sm_err + a;
    SmemCons<float> cons{sm_cons + a, THREADS};
    const float cap = (float)dm.z;
    float vxf, vyf;
    int c_last, kind, j_sel;
    bool shaky = false;
    const bool feasible = lp2_target_runahead_act<SmemCons<float>>(cons, sm_emax[a], cnt, cap, (float)dm.x, (float)dm.y,
                                                                  vxf, vyf, c_last, kind, j_sel, shaky, 0xFFFFFFFFu,
                                                                  enabled);
    if (!enabled) return;
    bool certified = feasible && !shaky && kind <= 2 && c_last >= 0;
    double vx = 0.0, vy = 0.0;
    if (certified) {
        const double tx = dm.x, ty = dm.y;
        {   // the closing formula of _lp1_target on line L = c_last, bound B = j_sel (K:98-119)
            const double inv_tau = __ddiv_rn(1.0, P.tau), inv_dt = __ddiv_rn(1.0, P.dt);
            double px, py, nx, ny;
            halfplane64(s, c_last, P, s_nr, nb, perm, 1, inv_tau, inv_dt, px, py, nx, ny);
            const double dx = -ny, dy = nx;
            double t;
            if (kind == 0) {
                t = (tx - px) * dx + (ty - py) * dy;
            } else {
                double qx, qy, mx, my;
                halfplane64(s, j_sel, P, s_nr, nb, perm, 1, inv_tau, inv_dt, qx, qy, mx, my);
                const double a_ = dx * mx + dy * my;
                const double b_ = (qx - px) * mx + (qy - py) * my;
                t = __ddiv_rn(b_, a_);
            }
            vx = px + t * dx;
            vy = py + t * dy;
        }
        // ---- the certificate, at the FP64 candidate ----
        const float cvx = (float)vx, cvy = (float)vy;
        const float txf = (float)tx, tyf = (float)ty;
        // strictly inside the speed disc (an active disc is left to FP64)
        certified = cvx * cvx + cvy * cvy < cap * cap * (1.0f - 1e-4f);
        float e_act = 0.0f;
        for (int pos = 0; pos < cnt; ++pos) { // every inactive half-plane holds with a margin above its error
            float px, py, nx, ny;
            cons.get(pos, px, py, nx, ny);
            const float e = __half2float(cerr[pos * THREADS]);
            const bool act = pos == c_last || (kind != 0 && pos == j_sel);
            const float slack = __fmaf_rn(cvx - px, nx, (cvy - py) * ny);
            if (act) e_act += e;
            certified = certified && (act ? e < 1.0f : slack > e);
        }
        if (certified) { // optimality: target - v = alpha n_L + beta n_B with alpha, beta < 0
            float lx, ly, lnx, lny;
            cons.get(c_last, lx, ly, lnx, lny);
            const float gx = txf - cvx, gy = tyf - cvy;
            const float gl = fabsf(gx) + fabsf(gy);
            if (kind == 0) { // the target violates L: its projection is the optimum
                const float viol = (txf - lx) * lnx + (tyf - ly) * lny;
                certified = viol < -(e_act + CERT_SAFETY * 8.0f * CERT_EPS * (gl + 1.0f));
            } else {
                float bx, by, bnx, bny;
                cons.get(j_sel, bx, by, bnx, bny);
                const float D = lnx * bny - lny * bnx;
                const float alpha = __fdiv_rn(gx * bny - gy * bnx, D);
                const float beta = __fdiv_rn(lnx * gy - lny * gx, D);
                const float m = __fdiv_rn((e_act + CERT_SAFETY * 8.0f * CERT_EPS) * (gl + fabsf(alpha) + fabsf(beta) + 1.0f),
                                          fabsf(D));
                certified = fabsf(D) > CERT_CROSS_MIN && alpha < -m && beta < -m;
            }
        }
    }
    if (!certified) {
        cq[atomicAdd(cq_cnt, 1)] = s;
        return;
    }
    status[row] = 0;
    failed_at[row] = -1;
    integrate_row<float, double>(row, me, vx, vy, P, goalpref, pv_out, arrived);
}

} // namespace orca

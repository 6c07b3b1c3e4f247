/*
 * orca_oracle.c -- CPU restatement (IEEE float64, plain C) of the reference's
 * per-timestep ORCA steering step.
 *
 * THIS IS TEST INFRASTRUCTURE, NOT THE PRODUCT.  Only tests/, the smoke check
 * in __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs may
 * build, link, import or execute anything under oracle/.  The product path
 * (paper_2008_11578_b200/) never calls into this file.
 *
 * Parity status: PINNED.  oracle/gen_golden.py runs the reference itself
 * (numba kernels under /root/reference/pkg/src/orcasim) in the build container
 * and tests/test_oracle_golden.py checks this file against those outputs
 * bit for bit (tests/golden/ npz files), plus the known-answer vectors of the
 * reference's own tests (pkg/tests/test_lp.py, test_orca.py, test_grid.py,
 * test_engine.py).
 *
 * Every function cites the reference lines it restates; "K" is
 * pkg/src/orcasim/_kernels.py and "E" is pkg/src/orcasim/engine.py.
 *
 * Build: see oracle/Makefile.  Must be compiled with -ffp-contract=off and
 * without -ffast-math: the reference (numba/LLVM without fastmath, numpy)
 * never fuses a multiply-add, and bitwise agreement depends on that.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_API __attribute__((visibility("default")))

typedef int64_t i64;
typedef uint64_t u64;

/* K:24-25 */
static const double PARALLEL_EPS = 1e-12;

/* ------------------------------------------------------------------------ */
/* splitmix64 and the seeded shuffle                                         */
/* ------------------------------------------------------------------------ */

/* K:36-40 */
static inline u64 mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* K:43-54 */
static void fisher_yates(i64 *perm, i64 k, u64 seed)
{
    for (i64 i = 0; i < k; ++i) perm[i] = i;
    u64 state = seed;
    for (i64 i = k - 1; i > 0; --i) {
        state += 0x9E3779B97F4A7C15ULL;
        i64 j = (i64)(mix64(state) % (u64)(i + 1));
        i64 tmp = perm[i];
        perm[i] = perm[j];
        perm[j] = tmp;
    }
}

/* K:57-61 */
static inline u64 problem_seed(i64 frame, i64 agent_id)
{
    u64 z = ((u64)frame << 32) | ((u64)agent_id & 0xFFFFFFFFULL);
    return mix64(z);
}

ORACLE_API u64 oracle_mix64(u64 z) { return mix64(z); }
ORACLE_API u64 oracle_problem_seed(i64 frame, i64 agent_id) { return problem_seed(frame, agent_id); }
/* K:64-67 */
ORACLE_API void oracle_shuffle_into(i64 *perm, i64 k, u64 seed) { fisher_yates(perm, k, seed); }

/* ------------------------------------------------------------------------ */
/* closest-point LP                                                          */
/* ------------------------------------------------------------------------ */

/* Constraint rows are stored [k][2] row-major like the reference arrays. */
#define PX(a, r) ((a)[2 * (r)])
#define PY(a, r) ((a)[2 * (r) + 1])

/* K:74-119.  Returns 1 when a point exists on the line, 0 otherwise. */
static int lp1_target(const double *pts, const double *nrm, const i64 *order, i64 i_pos,
                      double cap, double tx, double ty, double *ox, double *oy)
{
    i64 c = order[i_pos];
    double px = PX(pts, c), py = PY(pts, c);
    double nx = PX(nrm, c), ny = PY(nrm, c);
    double dx = -ny, dy = nx;

    double pd = px * dx + py * dy;
    double disc = pd * pd + cap * cap - (px * px + py * py);
    if (disc < 0.0) return 0;
    double sq = sqrt(disc);
    double t_left = -pd - sq;
    double t_right = -pd + sq;

    for (i64 j_pos = 0; j_pos < i_pos; ++j_pos) {
        i64 j = order[j_pos];
        double a = dx * PX(nrm, j) + dy * PY(nrm, j);
        double b = (PX(pts, j) - px) * PX(nrm, j) + (PY(pts, j) - py) * PY(nrm, j);
        if (-PARALLEL_EPS <= a && a <= PARALLEL_EPS) {
            if (b > 0.0) return 0;
            continue;
        }
        double t = b / a;
        if (a > 0.0) {
            if (t > t_left) t_left = t;
        } else {
            if (t < t_right) t_right = t;
        }
        if (t_left > t_right) return 0;
    }

    double t = (tx - px) * dx + (ty - py) * dy;
    if (t < t_left) t = t_left;
    else if (t > t_right) t = t_right;
    *ox = px + t * dx;
    *oy = py + t * dy;
    return 1;
}

/* K:122-146.  Returns 1 if feasible; else 0 with *fail_pos set and (vx,vy) the
 * last point that satisfied order[:fail_pos]. */
static int lp2_target(const double *pts, const double *nrm, const i64 *order, i64 k,
                      double cap, double tx, double ty, i64 *fail_pos, double *ovx, double *ovy)
{
    double vx, vy;
    double t2 = tx * tx + ty * ty;
    if (t2 > cap * cap) {
        double s = cap / sqrt(t2);
        vx = tx * s;
        vy = ty * s;
    } else {
        vx = tx;
        vy = ty;
    }
    for (i64 i_pos = 0; i_pos < k; ++i_pos) {
        i64 c = order[i_pos];
        if ((vx - PX(pts, c)) * PX(nrm, c) + (vy - PY(pts, c)) * PY(nrm, c) < 0.0) {
            double nvx, nvy;
            if (!lp1_target(pts, nrm, order, i_pos, cap, tx, ty, &nvx, &nvy)) {
                *fail_pos = i_pos;
                *ovx = vx;
                *ovy = vy;
                return 0;
            }
            vx = nvx;
            vy = nvy;
        }
    }
    *fail_pos = -1;
    *ovx = vx;
    *ovy = vy;
    return 1;
}

/* K:153-190 */
static int lp1_dir(const double *pts, const double *nrm, i64 upto, double cap,
                   double ox, double oy, double *rx, double *ry)
{
    double px = PX(pts, upto), py = PY(pts, upto);
    double nx = PX(nrm, upto), ny = PY(nrm, upto);
    double dx = -ny, dy = nx;

    double pd = px * dx + py * dy;
    double disc = pd * pd + cap * cap - (px * px + py * py);
    if (disc < 0.0) return 0;
    double sq = sqrt(disc);
    double t_left = -pd - sq;
    double t_right = -pd + sq;

    for (i64 j = 0; j < upto; ++j) {
        double a = dx * PX(nrm, j) + dy * PY(nrm, j);
        double b = (PX(pts, j) - px) * PX(nrm, j) + (PY(pts, j) - py) * PY(nrm, j);
        if (-PARALLEL_EPS <= a && a <= PARALLEL_EPS) {
            if (b > 0.0) return 0;
            continue;
        }
        double t = b / a;
        if (a > 0.0) {
            if (t > t_left) t_left = t;
        } else {
            if (t < t_right) t_right = t;
        }
        if (t_left > t_right) return 0;
    }
    double t = (dx * ox + dy * oy) > 0.0 ? t_right : t_left;
    *rx = px + t * dx;
    *ry = py + t * dy;
    return 1;
}

/* K:193-205 */
static int lp2_dir(const double *pts, const double *nrm, i64 m, double cap,
                   double ox, double oy, double *rx, double *ry)
{
    double vx = cap * ox, vy = cap * oy;
    for (i64 i = 0; i < m; ++i) {
        if ((vx - PX(pts, i)) * PX(nrm, i) + (vy - PY(pts, i)) * PY(nrm, i) < 0.0) {
            double nvx, nvy;
            if (!lp1_dir(pts, nrm, i, cap, ox, oy, &nvx, &nvy)) {
                *rx = vx;
                *ry = vy;
                return 0;
            }
            vx = nvx;
            vy = nvy;
        }
    }
    *rx = vx;
    *ry = vy;
    return 1;
}

/* K:212-251 */
static void lp3_minmax(const double *pts, const double *nrm, const i64 *order, i64 k, i64 begin,
                       double cap, double vx, double vy, double *ppts, double *pnrm,
                       double *rx, double *ry, double *rz)
{
    double dist = 0.0;
    for (i64 i_pos = begin; i_pos < k; ++i_pos) {
        i64 c = order[i_pos];
        double viol = (PX(pts, c) - vx) * PX(nrm, c) + (PY(pts, c) - vy) * PY(nrm, c);
        if (viol > dist) {
            i64 m = 0;
            for (i64 j_pos = 0; j_pos < i_pos; ++j_pos) {
                i64 j = order[j_pos];
                double mx = PX(nrm, j) - PX(nrm, c);
                double my = PY(nrm, j) - PY(nrm, c);
                double ml2 = mx * mx + my * my;
                if (ml2 < 1e-24) continue;
                double rhs = (PX(pts, j) * PX(nrm, j) + PY(pts, j) * PY(nrm, j)
                              - PX(pts, c) * PX(nrm, c) - PY(pts, c) * PY(nrm, c));
                double ml = sqrt(ml2);
                PX(pnrm, m) = mx / ml;
                PY(pnrm, m) = my / ml;
                PX(ppts, m) = mx * rhs / ml2;
                PY(ppts, m) = my * rhs / ml2;
                ++m;
            }
            double nvx, nvy;
            if (lp2_dir(ppts, pnrm, m, cap, PX(nrm, c), PY(nrm, c), &nvx, &nvy)) {
                vx = nvx;
                vy = nvy;
            }
            dist = (PX(pts, c) - vx) * PX(nrm, c) + (PY(pts, c) - vy) * PY(nrm, c);
            if (dist < 0.0) dist = 0.0;
        }
    }
    *rx = vx;
    *ry = vy;
    *rz = dist;
}

/* K:254-283 */
static void least_penetration(const double *pts, const double *nrm, const i64 *order, i64 k,
                              i64 begin, double cap, double wx, double wy, double *ppts,
                              double *pnrm, double *spts, i64 *ident, double *rx, double *ry)
{
    double w2 = wx * wx + wy * wy;
    if (w2 > cap * cap) {
        double s = cap / sqrt(w2);
        wx = wx * s;
        wy = wy * s;
    }
    double vx, vy, z;
    lp3_minmax(pts, nrm, order, k, begin, cap, wx, wy, ppts, pnrm, &vx, &vy, &z);

    for (i64 i = 0; i < k; ++i) ident[i] = i;
    double slack = 0.0;
    for (int attempt = 0; attempt < 3; ++attempt) {
        double zz = z + slack;
        for (i64 j = 0; j < k; ++j) {
            PX(spts, j) = PX(pts, j) - zz * PX(nrm, j);
            PY(spts, j) = PY(pts, j) - zz * PY(nrm, j);
        }
        i64 fail;
        double qx, qy;
        if (lp2_target(spts, nrm, ident, k, cap, wx, wy, &fail, &qx, &qy)) {
            *rx = qx;
            *ry = qy;
            return;
        }
        slack = slack * 1e3 + 1e-12 * (1.0 + z);
    }
    *rx = vx;
    *ry = vy;
}

/* K:290-303.  status: 0 feasible, 1 fallback used. */
static void solve_one(const double *pts, const double *nrm, i64 k, double cap, double tx, double ty,
                      u64 seed, i64 *perm, double *ppts, double *pnrm, double *spts, i64 *ident,
                      double *rx, double *ry, i64 *status, i64 *failed_at)
{
    fisher_yates(perm, k, seed);
    i64 fail_pos;
    double vx, vy;
    if (lp2_target(pts, nrm, perm, k, cap, tx, ty, &fail_pos, &vx, &vy)) {
        *rx = vx;
        *ry = vy;
        *status = 0;
        *failed_at = -1;
        return;
    }
    *failed_at = perm[fail_pos];
    least_penetration(pts, nrm, perm, k, fail_pos, cap, vx, vy, ppts, pnrm, spts, ident, rx, ry);
    *status = 1;
}

typedef struct {
    i64 cap_k;
    i64 *perm, *ident;
    double *ppts, *pnrm, *spts;
} lp_scratch;

static int scratch_init(lp_scratch *s, i64 k)
{
    if (k < 1) k = 1;
    s->cap_k = k;
    s->perm = (i64 *)malloc(sizeof(i64) * (size_t)k);
    s->ident = (i64 *)malloc(sizeof(i64) * (size_t)k);
    s->ppts = (double *)malloc(sizeof(double) * 2 * (size_t)k);
    s->pnrm = (double *)malloc(sizeof(double) * 2 * (size_t)k);
    s->spts = (double *)malloc(sizeof(double) * 2 * (size_t)k);
    return s->perm && s->ident && s->ppts && s->pnrm && s->spts;
}

static void scratch_free(lp_scratch *s)
{
    free(s->perm);
    free(s->ident);
    free(s->ppts);
    free(s->pnrm);
    free(s->spts);
}

/* Object-level entry: lp.solve_closest_point (pkg/src/orcasim/lp.py:152-165). */
ORACLE_API int oracle_solve_one(const double *pts, const double *nrm, i64 k, double cap, double tx,
                                double ty, u64 seed, double *out_xy, i64 *status, i64 *failed_at)
{
    lp_scratch s;
    if (!scratch_init(&s, k)) return -1;
    solve_one(pts, nrm, k, cap, tx, ty, seed, s.perm, s.ppts, s.pnrm, s.spts, s.ident,
              &out_xy[0], &out_xy[1], status, failed_at);
    scratch_free(&s);
    return 0;
}

/* Object-level entry: lp.solve_least_penetration (lp.py:168-190), identity order. */
ORACLE_API int oracle_least_penetration(const double *pts, const double *nrm, i64 k, i64 begin,
                                        double cap, double wx, double wy, double *out_xy)
{
    lp_scratch s;
    if (!scratch_init(&s, k)) return -1;
    i64 *order = (i64 *)malloc(sizeof(i64) * (size_t)(k < 1 ? 1 : k));
    for (i64 i = 0; i < k; ++i) order[i] = i;
    least_penetration(pts, nrm, order, k, begin, cap, wx, wy, s.ppts, s.pnrm, s.spts, s.ident,
                      &out_xy[0], &out_xy[1]);
    free(order);
    scratch_free(&s);
    return 0;
}

/* K:306-336 */
ORACLE_API int oracle_solve_range(const i64 *coff, const double *cpts, const double *cnrm,
                                  const double *tgt, const double *caps, const u64 *seeds,
                                  double *out_v, i64 *out_status, i64 *out_failed, i64 start,
                                  i64 stop)
{
    i64 max_k = 0;
    for (i64 i = start; i < stop; ++i) {
        i64 k = coff[i + 1] - coff[i];
        if (k > max_k) max_k = k;
    }
    lp_scratch s;
    if (!scratch_init(&s, max_k)) return -1;
    for (i64 i = start; i < stop; ++i) {
        i64 lo = coff[i];
        i64 k = coff[i + 1] - lo;
        solve_one(cpts + 2 * lo, cnrm + 2 * lo, k, caps[i], tgt[2 * i], tgt[2 * i + 1], seeds[i],
                  s.perm, s.ppts, s.pnrm, s.spts, s.ident, &out_v[2 * i], &out_v[2 * i + 1],
                  &out_status[i], &out_failed[i]);
    }
    scratch_free(&s);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* velocity-obstacle exit                                                     */
/* ------------------------------------------------------------------------ */

/* K:343-419.  out = (ux, uy, nx, ny); returns 0 only for coincident centres. */
static int vo_exit(double rpx, double rpy, double rvx, double rvy, double comb_r, double tau,
                   double dt, double *out)
{
    if (rpx == 0.0 && rpy == 0.0) {
        out[0] = out[1] = out[2] = out[3] = 0.0;
        return 0;
    }
    double d2 = rpx * rpx + rpy * rpy;
    double r2 = comb_r * comb_r;

    if (d2 < r2) {
        double inv = 1.0 / dt;
        double cx = rpx * inv, cy = rpy * inv;
        double rr = comb_r * inv;
        double wx = rvx - cx, wy = rvy - cy;
        double wl2 = wx * wx + wy * wy;
        double uxh, uyh, wl;
        if (wl2 < 1e-24) {
            double d = sqrt(d2);
            uxh = -rpx / d;
            uyh = -rpy / d;
            wl = 0.0;
        } else {
            wl = sqrt(wl2);
            uxh = wx / wl;
            uyh = wy / wl;
        }
        double s = rr - wl;
        out[0] = s * uxh;
        out[1] = s * uyh;
        out[2] = uxh;
        out[3] = uyh;
        return 1;
    }

    double inv = 1.0 / tau;
    double cx = rpx * inv, cy = rpy * inv;
    double rr = comb_r * inv;
    double wx = rvx - cx, wy = rvy - cy;
    double wl2 = wx * wx + wy * wy;
    double dot_wp = wx * rpx + wy * rpy;

    if (wl2 < 1e-24) {
        double d = sqrt(d2);
        double uxh = -rpx / d, uyh = -rpy / d;
        out[0] = rr * uxh;
        out[1] = rr * uyh;
        out[2] = uxh;
        out[3] = uyh;
        return 1;
    }

    if (dot_wp < 0.0 && dot_wp * dot_wp > r2 * wl2) {
        double wl = sqrt(wl2);
        double uxh = wx / wl, uyh = wy / wl;
        double s = rr - wl;
        out[0] = s * uxh;
        out[1] = s * uyh;
        out[2] = uxh;
        out[3] = uyh;
        return 1;
    }

    double leg = sqrt(d2 - r2);
    double dx, dy;
    if (rpx * wy - rpy * wx > 0.0) {
        dx = (rpx * leg - rpy * comb_r) / d2;
        dy = (rpx * comb_r + rpy * leg) / d2;
    } else {
        dx = -(rpx * leg + rpy * comb_r) / d2;
        dy = (rpx * comb_r - rpy * leg) / d2;
    }
    double t = rvx * dx + rvy * dy;
    double ux = t * dx - rvx;
    double uy = t * dy - rvy;
    double nx = -dy, ny = dx;
    if (nx * rpx + ny * rpy > 0.0) {
        nx = -nx;
        ny = -ny;
    }
    out[0] = ux;
    out[1] = uy;
    out[2] = nx;
    out[3] = ny;
    return 1;
}

ORACLE_API int oracle_vo_exit(double rpx, double rpy, double rvx, double rvy, double comb_r,
                              double tau, double dt, double *out4)
{
    return vo_exit(rpx, rpy, rvx, rvy, comb_r, tau, dt, out4);
}

/* ------------------------------------------------------------------------ */
/* uniform grid: CSR over sorted cell keys                                   */
/* ------------------------------------------------------------------------ */

/* K:426-432 */
#define CELL_OFFSET ((i64)1 << 29)
#define CELL_STRIDE ((i64)1 << 30)
#define CELL_LIMIT (CELL_OFFSET - 2) /* E:146 */

static inline i64 cell_key(i64 ix, i64 iy)
{
    return (ix + CELL_OFFSET) * CELL_STRIDE + (iy + CELL_OFFSET);
}

typedef struct {
    i64 key, row;
} keyrow;

static int keyrow_cmp(const void *a, const void *b)
{
    const keyrow *x = (const keyrow *)a, *y = (const keyrow *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    /* row as secondary key == numpy's stable argsort (E:155) */
    return x->row < y->row ? -1 : (x->row > y->row);
}

/* E:149-161.  cell_ix/cell_iy (may be NULL) receive floor(pos/cell) per agent.
 * Returns the number of occupied cells, -2 when a position is outside the
 * indexable range (E:152-153), -1 on allocation failure.
 * order[n], ukeys[n], starts[n+1] are caller-allocated at worst-case size. */
ORACLE_API i64 oracle_grid_arrays(const double *pos, i64 n, double cell_size, i64 *order,
                                  i64 *ukeys, i64 *starts, i64 *cell_ix, i64 *cell_iy)
{
    keyrow *kr = (keyrow *)malloc(sizeof(keyrow) * (size_t)(n < 1 ? 1 : n));
    if (!kr) return -1;
    for (i64 i = 0; i < n; ++i) {
        i64 ix = (i64)floor(pos[2 * i] / cell_size);
        i64 iy = (i64)floor(pos[2 * i + 1] / cell_size);
        if (cell_ix) cell_ix[i] = ix;
        if (cell_iy) cell_iy[i] = iy;
        if (llabs(ix) > CELL_LIMIT || llabs(iy) > CELL_LIMIT) {
            free(kr);
            return -2;
        }
        kr[i].key = cell_key(ix, iy);
        kr[i].row = i;
    }
    qsort(kr, (size_t)n, sizeof(keyrow), keyrow_cmp);
    i64 nc = 0;
    for (i64 s = 0; s < n; ++s) {
        order[s] = kr[s].row;
        if (s == 0 || kr[s].key != kr[s - 1].key) {
            ukeys[nc] = kr[s].key;
            starts[nc] = s;
            ++nc;
        }
    }
    starts[nc] = n;
    free(kr);
    return nc;
}

/* K:435-447 */
static i64 find_cell(const i64 *ukeys, i64 nkeys, i64 key)
{
    i64 lo = 0, hi = nkeys;
    while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        if (ukeys[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    if (lo < nkeys && ukeys[lo] == key) return lo;
    return -1;
}

/* K:450-490 */
static i64 collect_neighbors(i64 i, const double *pos, const i64 *ids, const i64 *sorted_idx,
                             const i64 *ukeys, i64 nkeys, const i64 *starts, double cell_size,
                             i64 reach, double rad2, i64 max_n, double *nb_d2, i64 *nb_id,
                             i64 *nb_ix)
{
    i64 count = 0;
    i64 cxi = (i64)floor(pos[2 * i] / cell_size);
    i64 cyi = (i64)floor(pos[2 * i + 1] / cell_size);
    for (i64 gx = cxi - reach; gx <= cxi + reach; ++gx) {
        for (i64 gy = cyi - reach; gy <= cyi + reach; ++gy) {
            i64 t = find_cell(ukeys, nkeys, cell_key(gx, gy));
            if (t < 0) continue;
            for (i64 s = starts[t]; s < starts[t + 1]; ++s) {
                i64 j = sorted_idx[s];
                if (j == i) continue;
                double dx = pos[2 * j] - pos[2 * i];
                double dy = pos[2 * j + 1] - pos[2 * i + 1];
                double d2 = dx * dx + dy * dy;
                if (d2 > rad2) continue;
                i64 jid = ids[j];
                i64 p;
                if (count == max_n) {
                    i64 last = count - 1;
                    if (d2 > nb_d2[last] || (d2 == nb_d2[last] && jid >= nb_id[last])) continue;
                    p = last;
                } else {
                    p = count;
                    ++count;
                }
                while (p > 0 && (nb_d2[p - 1] > d2 || (nb_d2[p - 1] == d2 && nb_id[p - 1] > jid))) {
                    nb_d2[p] = nb_d2[p - 1];
                    nb_id[p] = nb_id[p - 1];
                    nb_ix[p] = nb_ix[p - 1];
                    --p;
                }
                nb_d2[p] = d2;
                nb_id[p] = jid;
                nb_ix[p] = j;
            }
        }
    }
    return count;
}

/* Test entry for the neighbour query alone (rows of the ordered list). */
ORACLE_API i64 oracle_collect_neighbors(i64 i, const double *pos, const i64 *ids,
                                        const i64 *sorted_idx, const i64 *ukeys, i64 nkeys,
                                        const i64 *starts, double cell_size, i64 reach, double rad2,
                                        i64 max_n, double *nb_d2, i64 *nb_id, i64 *nb_ix)
{
    return collect_neighbors(i, pos, ids, sorted_idx, ukeys, nkeys, starts, cell_size, reach, rad2,
                             max_n, nb_d2, nb_id, nb_ix);
}

/* ------------------------------------------------------------------------ */
/* fused per-agent frame kernel                                              */
/* ------------------------------------------------------------------------ */

typedef struct {
    const double *pos, *vel, *radius, *max_speed;
    const i64 *cls_code, *ids;
    const double *fmat; /* [2][2] row-major, O:123-129 */
    const double *des;
    const i64 *sorted_idx, *ukeys;
    i64 nkeys;
    const i64 *starts;
    double cell_size;
    i64 reach;
    double rad2;
    i64 max_n;
    double tau, dt;
    i64 frame;
    double *out_v;
    i64 *out_status, *out_failed, *out_err;
    /* optional debug taps (NULL to skip): neighbour rows / count, constraints */
    i64 *dbg_nb_rows;  /* [n][max_n], -1 padded */
    i64 *dbg_nb_count; /* [n] */
    double *dbg_cons;  /* [n][max_n][4] = point.x, point.y, normal.x, normal.y */
} frame_args;

/* K:493-556 */
static int frame_solve_range(const frame_args *A, i64 start, i64 stop)
{
    i64 max_n = A->max_n;
    i64 cap_n = max_n > 0 ? max_n : 1;
    double *nb_d2 = (double *)malloc(sizeof(double) * (size_t)cap_n);
    i64 *nb_id = (i64 *)malloc(sizeof(i64) * (size_t)cap_n);
    i64 *nb_ix = (i64 *)malloc(sizeof(i64) * (size_t)cap_n);
    double *cpts = (double *)malloc(sizeof(double) * 2 * (size_t)cap_n);
    double *cnrm = (double *)malloc(sizeof(double) * 2 * (size_t)cap_n);
    lp_scratch s;
    int ok_alloc = scratch_init(&s, cap_n);
    if (!nb_d2 || !nb_id || !nb_ix || !cpts || !cnrm || !ok_alloc) return -1;

    const double *pos = A->pos, *vel = A->vel;
    for (i64 i = start; i < stop; ++i) {
        A->out_err[i] = -1;
        i64 count = 0;
        if (max_n > 0)
            count = collect_neighbors(i, pos, A->ids, A->sorted_idx, A->ukeys, A->nkeys, A->starts,
                                      A->cell_size, A->reach, A->rad2, max_n, nb_d2, nb_id, nb_ix);
        if (A->dbg_nb_count) A->dbg_nb_count[i] = count;
        if (A->dbg_nb_rows) {
            for (i64 t = 0; t < max_n; ++t)
                A->dbg_nb_rows[i * max_n + t] = t < count ? nb_ix[t] : -1;
        }

        int bad = 0;
        for (i64 t = 0; t < count; ++t) {
            i64 j = nb_ix[t];
            double rpx = pos[2 * j] - pos[2 * i];
            double rpy = pos[2 * j + 1] - pos[2 * i + 1];
            double rvx = vel[2 * i] - vel[2 * j];
            double rvy = vel[2 * i + 1] - vel[2 * j + 1];
            double e[4];
            if (!vo_exit(rpx, rpy, rvx, rvy, A->radius[i] + A->radius[j], A->tau, A->dt, e)) {
                A->out_err[i] = j;
                bad = 1;
                break;
            }
            double f = A->fmat[2 * A->cls_code[i] + A->cls_code[j]];
            cpts[2 * t] = vel[2 * i] + f * e[0];
            cpts[2 * t + 1] = vel[2 * i + 1] + f * e[1];
            cnrm[2 * t] = e[2];
            cnrm[2 * t + 1] = e[3];
        }
        if (bad) {
            A->out_v[2 * i] = vel[2 * i];
            A->out_v[2 * i + 1] = vel[2 * i + 1];
            A->out_status[i] = 0;
            A->out_failed[i] = -1;
            continue;
        }
        if (A->dbg_cons) {
            double *row = A->dbg_cons + 4 * max_n * i;
            for (i64 t = 0; t < max_n; ++t) {
                row[4 * t + 0] = t < count ? cpts[2 * t] : 0.0;
                row[4 * t + 1] = t < count ? cpts[2 * t + 1] : 0.0;
                row[4 * t + 2] = t < count ? cnrm[2 * t] : 0.0;
                row[4 * t + 3] = t < count ? cnrm[2 * t + 1] : 0.0;
            }
        }

        u64 seed = problem_seed(A->frame, A->ids[i]);
        solve_one(cpts, cnrm, count, A->max_speed[i], A->des[2 * i], A->des[2 * i + 1], seed,
                  s.perm, s.ppts, s.pnrm, s.spts, s.ident, &A->out_v[2 * i], &A->out_v[2 * i + 1],
                  &A->out_status[i], &A->out_failed[i]);
    }
    free(nb_d2);
    free(nb_id);
    free(nb_ix);
    free(cpts);
    free(cnrm);
    scratch_free(&s);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* worker pool: the reference's run_units (lp.py:236-260) -- work units are   */
/* popped from a shared queue by up to worker_count threads                  */
/* ------------------------------------------------------------------------ */

typedef struct {
    const frame_args *A;
    i64 n, per_unit;
    i64 next; /* atomically advanced unit index */
    int rc;
} pool_job;

static void *frame_worker(void *p)
{
    pool_job *J = (pool_job *)p;
    for (;;) {
        i64 u = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        i64 a = u * J->per_unit;
        if (a >= J->n) break;
        i64 b = a + J->per_unit;
        if (b > J->n) b = J->n;
        if (frame_solve_range(J->A, a, b) != 0) J->rc = -1;
    }
    return NULL;
}

/* E:164-166 + E:229-237: ranges of work_unit_steps // max_neighbors agents. */
ORACLE_API int oracle_frame_solve(
    const double *pos, const double *vel, const double *radius, const double *max_speed,
    const i64 *cls_code, const i64 *ids, const double *fmat, const double *des,
    const i64 *sorted_idx, const i64 *ukeys, i64 nkeys, const i64 *starts, double cell_size,
    i64 reach, double rad2, i64 max_n, double tau, double dt, i64 frame, double *out_v,
    i64 *out_status, i64 *out_failed, i64 *out_err, i64 n, i64 worker_count, i64 work_unit_steps,
    i64 *dbg_nb_rows, i64 *dbg_nb_count, double *dbg_cons)
{
    frame_args A = {pos, vel, radius, max_speed, cls_code, ids, fmat, des, sorted_idx, ukeys, nkeys,
                    starts, cell_size, reach, rad2, max_n, tau, dt, frame, out_v, out_status,
                    out_failed, out_err, dbg_nb_rows, dbg_nb_count, dbg_cons};
    i64 per_unit = work_unit_steps / (max_n > 1 ? max_n : 1);
    if (per_unit < 1) per_unit = 1;
    pool_job J = {&A, n, per_unit, 0, 0};
    i64 units = (n + per_unit - 1) / per_unit;
    if (worker_count <= 1 || units <= 1) {
        frame_worker(&J);
        return J.rc;
    }
    i64 nt = worker_count < units ? worker_count : units;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nt);
    if (!th) return -1;
    for (i64 t = 0; t < nt; ++t) pthread_create(&th[t], NULL, frame_worker, &J);
    for (i64 t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(th);
    return J.rc;
}

/* ------------------------------------------------------------------------ */
/* batched LP with the same worker pool (lp.solve_batch, lp.py:263-291)      */
/* ------------------------------------------------------------------------ */

typedef struct {
    const i64 *coff;
    const double *cpts, *cnrm, *tgt, *caps;
    const u64 *seeds;
    double *out_v;
    i64 *out_status, *out_failed;
    i64 n, per_unit, next;
    int rc;
} lp_job;

static void *lp_worker(void *p)
{
    lp_job *J = (lp_job *)p;
    for (;;) {
        i64 u = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        i64 a = u * J->per_unit;
        if (a >= J->n) break;
        i64 b = a + J->per_unit;
        if (b > J->n) b = J->n;
        if (oracle_solve_range(J->coff, J->cpts, J->cnrm, J->tgt, J->caps, J->seeds, J->out_v,
                               J->out_status, J->out_failed, a, b) != 0)
            J->rc = -1;
    }
    return NULL;
}

/* Results do not depend on how problems are cut into units (each problem is a
 * pure function of its inputs), so fixed-size units replace lp._unit_ranges. */
ORACLE_API int oracle_solve_batch(const i64 *coff, const double *cpts, const double *cnrm,
                                  const double *tgt, const double *caps, const u64 *seeds,
                                  double *out_v, i64 *out_status, i64 *out_failed, i64 n,
                                  i64 worker_count)
{
    lp_job J = {coff, cpts, cnrm, tgt, caps, seeds, out_v, out_status, out_failed, n, 256, 0, 0};
    if (worker_count <= 1) {
        lp_worker(&J);
        return J.rc;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)worker_count);
    if (!th) return -1;
    for (i64 t = 0; t < worker_count; ++t) pthread_create(&th[t], NULL, lp_worker, &J);
    for (i64 t = 0; t < worker_count; ++t) pthread_join(th[t], NULL);
    free(th);
    return J.rc;
}

/* ------------------------------------------------------------------------ */
/* numpy-side pieces of engine._advance                                      */
/* ------------------------------------------------------------------------ */

/* E:133-139 */
ORACLE_API void oracle_desired_velocities(const double *pos, const double *goals,
                                          const double *pref, double dt, i64 n, double *des)
{
    for (i64 i = 0; i < n; ++i) {
        double dx = goals[2 * i] - pos[2 * i];
        double dy = goals[2 * i + 1] - pos[2 * i + 1];
        double dist = sqrt(dx * dx + dy * dy);
        double speed = dist / dt;
        if (pref[i] < speed) speed = pref[i]; /* np.minimum; inputs are finite */
        double scale = dist > 0.0 ? speed / dist : 0.0;
        des[2 * i] = dx * scale;
        des[2 * i + 1] = dy * scale;
    }
}

/* E:249 and E:251-253: new_pos = pos + out_v*dt; arrived = |goal-new_pos| <= tol */
ORACLE_API void oracle_integrate(const double *pos, const double *out_v, double dt,
                                 const double *goals, const double *goal_tols, i64 n,
                                 double *new_pos, uint8_t *arrived)
{
    for (i64 i = 0; i < n; ++i) {
        double nx = pos[2 * i] + out_v[2 * i] * dt;
        double ny = pos[2 * i + 1] + out_v[2 * i + 1] * dt;
        new_pos[2 * i] = nx;
        new_pos[2 * i + 1] = ny;
        double gx = goals[2 * i] - nx, gy = goals[2 * i + 1] - ny;
        arrived[i] = sqrt(gx * gx + gy * gy) <= goal_tols[i];
    }
}

/* K:559-589 over the whole population (E:270-286 takes min / sum of the parts,
 * which is order independent). best = +inf when no pair is in range. */
ORACLE_API void oracle_min_sep(const double *pos, const double *radius, const i64 *ids,
                               const i64 *sorted_idx, const i64 *ukeys, i64 nkeys,
                               const i64 *starts, double cell_size, i64 reach, double rad2,
                               double coll_tol, i64 n, double *best_out, i64 *count_out)
{
    double best = INFINITY;
    i64 count = 0;
    for (i64 i = 0; i < n; ++i) {
        i64 cxi = (i64)floor(pos[2 * i] / cell_size);
        i64 cyi = (i64)floor(pos[2 * i + 1] / cell_size);
        for (i64 gx = cxi - reach; gx <= cxi + reach; ++gx)
            for (i64 gy = cyi - reach; gy <= cyi + reach; ++gy) {
                i64 t = find_cell(ukeys, nkeys, cell_key(gx, gy));
                if (t < 0) continue;
                for (i64 s = starts[t]; s < starts[t + 1]; ++s) {
                    i64 j = sorted_idx[s];
                    if (ids[j] <= ids[i]) continue;
                    double dx = pos[2 * j] - pos[2 * i];
                    double dy = pos[2 * j + 1] - pos[2 * i + 1];
                    double d2 = dx * dx + dy * dy;
                    if (d2 > rad2) continue;
                    double sep = sqrt(d2) - (radius[i] + radius[j]);
                    if (sep < best) best = sep;
                    if (sep < -coll_tol) ++count;
                }
            }
    }
    *best_out = best;
    *count_out = count;
}

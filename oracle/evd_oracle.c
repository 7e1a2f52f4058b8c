/*
 * evd_oracle.c -- CPU restatement of the reference bound-evaluation path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker for the CUDA product path and
 * the CPU baseline timed by bench.py; nothing in paper_2209_13168_b200/ links
 * or calls it.  It restates, operation for operation, the reference's
 * numpy/numba arithmetic:
 *
 *   warp            pkg/src/eventdiv/geometry.py:70-87   (warp_scale, radial_warp)
 *   point image     pkg/src/eventdiv/contrast.py:48-58   (accumulate_image)
 *   _mark_point     pkg/src/eventdiv/contrast.py:73-91   (closed-square rule, stamp dedup)
 *   _rasterize_into pkg/src/eventdiv/contrast.py:94-182  (Liang-Barsky clip, crossings, sort)
 *   _bound_image_kernel pkg/src/eventdiv/contrast.py:185-203 (half-open fully-inside count)
 *
 * The reference's dedup device (a per-pixel stamp grid tagged with the event
 * index) and its per-event sort of the crossing parameters are kept as-is,
 * deliberately unlike the device design, so the two are independent.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; no FMA contraction, IEEE
 * binary64 round-to-nearest, exactly like numpy ufuncs and numba's output).
 * Counts are held as uint32 (the reference's float64 counts are small exact
 * integers, so the two are value-identical).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* geometry.py:70-87: s = (1 + nu*t) / (1 + nu*tau); x' = cx + (x - cx) * s */
void orc_warp(const double *x, const double *y, const double *t, int64_t n,
              double nu, double tau, int32_t width, int32_t height,
              double *xo, double *yo)
{
    const double denom = 1.0 + nu * tau;
    const double cx = width / 2.0, cy = height / 2.0;
    for (int64_t i = 0; i < n; i++) {
        const double s = (1.0 + nu * t[i]) / denom;
        xo[i] = cx + (x[i] - cx) * s;
        yo[i] = cy + (y[i] - cy) * s;
    }
}

/* contrast.py:48-58: floor-bin, half-open frame test, bincount. */
static int64_t point_image_range(const double *x, const double *y, const double *t,
                                 int64_t i0, int64_t i1, double nu, double tau,
                                 int32_t width, int32_t height, uint32_t *counts)
{
    const double denom = 1.0 + nu * tau;
    const double cx = width / 2.0, cy = height / 2.0;
    int64_t inside = 0;
    for (int64_t i = i0; i < i1; i++) {
        const double s = (1.0 + nu * t[i]) / denom;
        const double wx = cx + (x[i] - cx) * s;
        const double wy = cy + (y[i] - cy) * s;
        const int64_t ix = (int64_t)floor(wx), iy = (int64_t)floor(wy);
        if (ix >= 0 && ix < width && iy >= 0 && iy < height) {
            counts[iy * (int64_t)width + ix] += 1;
            inside++;
        }
    }
    return inside;
}

int64_t orc_point_image(const double *x, const double *y, const double *t, int64_t n,
                        double nu, double tau, int32_t width, int32_t height,
                        uint32_t *counts)
{
    memset(counts, 0, sizeof(uint32_t) * (size_t)width * (size_t)height);
    return point_image_range(x, y, t, 0, n, nu, tau, width, height, counts);
}

/* contrast.py:73-91 */
static inline void mark_point(uint32_t *counts, int64_t *stamp, int64_t tag,
                              double px, double py, int32_t width, int32_t height)
{
    const double fx = floor(px), fy = floor(py);
    const int64_t ix0 = (int64_t)fx, iy0 = (int64_t)fy;
    const int64_t x_lo = (px == fx) ? ix0 - 1 : ix0;
    const int64_t y_lo = (py == fy) ? iy0 - 1 : iy0;
    for (int64_t ix = x_lo; ix <= ix0; ix++) {
        if (ix < 0 || ix >= width) continue;
        for (int64_t iy = y_lo; iy <= iy0; iy++) {
            if (iy < 0 || iy >= height) continue;
            const int64_t p = iy * (int64_t)width + ix;
            if (stamp[p] != tag) {
                stamp[p] = tag;
                counts[p] += 1;
            }
        }
    }
}

static int cmp_double(const void *a, const void *b)
{
    const double da = *(const double *)a, db = *(const double *)b;
    return (da > db) - (da < db);
}

/* contrast.py:94-182 */
static void rasterize_into(uint32_t *counts, int64_t *stamp, int64_t tag,
                           double ax, double ay, double bx, double by,
                           int32_t width, int32_t height, double *ts)
{
    if (ax == bx && ay == by) {
        const int64_t ix = (int64_t)floor(ax), iy = (int64_t)floor(ay);
        if (ix >= 0 && ix < width && iy >= 0 && iy < height) {
            const int64_t p = iy * (int64_t)width + ix;
            if (stamp[p] != tag) { stamp[p] = tag; counts[p] += 1; }
        }
        return;
    }
    const double dx = bx - ax, dy = by - ay;
    double t0 = 0.0, t1 = 1.0;
    if (dx == 0.0) {
        if (ax < 0.0 || ax > width) return;
    } else {
        double ta = (0.0 - ax) / dx, tb = (width - ax) / dx;
        if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
    }
    if (dy == 0.0) {
        if (ay < 0.0 || ay > height) return;
    } else {
        double ta = (0.0 - ay) / dy, tb = (height - ay) / dy;
        if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
    }
    if (t0 > t1) return;
    const double cx0 = ax + t0 * dx, cy0 = ay + t0 * dy;
    const double cx1 = ax + t1 * dx, cy1 = ay + t1 * dy;
    const double ddx = cx1 - cx0, ddy = cy1 - cy0;
    int64_t n_ts = 0;
    ts[n_ts++] = 0.0;
    ts[n_ts++] = 1.0;
    if (ddx != 0.0) {
        const double xmin = cx0 < cx1 ? cx0 : cx1, xmax = cx0 < cx1 ? cx1 : cx0;
        for (int64_t k = (int64_t)ceil(xmin); (double)k <= xmax; k++) {
            double s = ((double)k - cx0) / ddx;
            if (s < 0.0) s = 0.0; else if (s > 1.0) s = 1.0;
            ts[n_ts++] = s;
        }
    }
    if (ddy != 0.0) {
        const double ymin = cy0 < cy1 ? cy0 : cy1, ymax = cy0 < cy1 ? cy1 : cy0;
        for (int64_t k = (int64_t)ceil(ymin); (double)k <= ymax; k++) {
            double s = ((double)k - cy0) / ddy;
            if (s < 0.0) s = 0.0; else if (s > 1.0) s = 1.0;
            ts[n_ts++] = s;
        }
    }
    qsort(ts, (size_t)n_ts, sizeof(double), cmp_double);
    for (int64_t j = 0; j < n_ts; j++) {
        const double s = ts[j];
        mark_point(counts, stamp, tag, cx0 + s * ddx, cy0 + s * ddy, width, height);
        if (j + 1 < n_ts) {
            const double sm = 0.5 * (s + ts[j + 1]);
            mark_point(counts, stamp, tag, cx0 + sm * ddx, cy0 + sm * ddy, width, height);
        }
    }
}

/* contrast.py:185-203 over events [i0, i1); returns the fully-inside count. */
static int64_t bound_image_range(const double *x0, const double *y0,
                                 const double *x1, const double *y1,
                                 int64_t i0, int64_t i1, int32_t width, int32_t height,
                                 uint32_t *counts, int64_t *stamp, double *ts)
{
    int64_t fully_inside = 0;
    for (int64_t i = i0; i < i1; i++) {
        const double ax = x0[i], ay = y0[i], bx = x1[i], by = y1[i];
        if (0.0 <= ax && ax < width && 0.0 <= ay && ay < height &&
            0.0 <= bx && bx < width && 0.0 <= by && by < height)
            fully_inside++;
        rasterize_into(counts, stamp, i, ax, ay, bx, by, width, height, ts);
    }
    return fully_inside;
}

/* _bound_image_kernel on pre-warped endpoints; counts must be zeroed by caller. */
int64_t orc_bound_image_endpoints(const double *x0, const double *y0,
                                  const double *x1, const double *y1, int64_t n,
                                  int32_t width, int32_t height, uint32_t *counts)
{
    const size_t m = (size_t)width * (size_t)height;
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * m);
    double *ts = (double *)malloc(sizeof(double) * ((size_t)width + height + 6));
    for (size_t p = 0; p < m; p++) stamp[p] = -1;
    const int64_t fi = bound_image_range(x0, y0, x1, y1, 0, n, width, height, counts, stamp, ts);
    free(stamp);
    free(ts);
    return fi;
}

/* rasterize_segment (contrast.py:206-222): marks into a zeroed counts grid. */
void orc_rasterize_segment(double ax, double ay, double bx, double by,
                           int32_t width, int32_t height, uint32_t *counts)
{
    const size_t m = (size_t)width * (size_t)height;
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * m);
    double *ts = (double *)malloc(sizeof(double) * ((size_t)width + height + 6));
    for (size_t p = 0; p < m; p++) stamp[p] = -1;
    memset(counts, 0, sizeof(uint32_t) * m);
    rasterize_into(counts, stamp, 0, ax, ay, bx, by, width, height, ts);
    free(stamp);
    free(ts);
}

/* ---- multi-threaded drivers (CPU baseline): private images, integer merge ---- */

typedef struct {
    const double *x, *y, *t;
    int64_t i0, i1;
    double lo, hi, tau;
    int32_t width, height;
    int mode; /* 0 = point image at lo, 1 = bound image over [lo, hi] */
    uint32_t *counts;
    int64_t result;
} job_t;

static void *run_job(void *arg)
{
    job_t *j = (job_t *)arg;
    const int64_t n = j->i1 - j->i0;
    const size_t m = (size_t)j->width * (size_t)j->height;
    if (j->mode == 0) {
        j->result = point_image_range(j->x, j->y, j->t, j->i0, j->i1, j->lo, j->tau,
                                      j->width, j->height, j->counts);
        return NULL;
    }
    /* _segment_endpoints (contrast.py:225-228): warp at both endpoints */
    double *w = (double *)malloc(sizeof(double) * 4 * (size_t)(n > 0 ? n : 1));
    orc_warp(j->x + j->i0, j->y + j->i0, j->t + j->i0, n, j->lo, j->tau, j->width, j->height,
             w, w + n);
    orc_warp(j->x + j->i0, j->y + j->i0, j->t + j->i0, n, j->hi, j->tau, j->width, j->height,
             w + 2 * n, w + 3 * n);
    int64_t *stamp = (int64_t *)malloc(sizeof(int64_t) * m);
    double *ts = (double *)malloc(sizeof(double) * ((size_t)j->width + j->height + 6));
    for (size_t p = 0; p < m; p++) stamp[p] = -1;
    j->result = bound_image_range(w, w + n, w + 2 * n, w + 3 * n, 0, n, j->width, j->height,
                                  j->counts, stamp, ts);
    free(stamp);
    free(ts);
    free(w);
    return NULL;
}

static int64_t run_split(const double *x, const double *y, const double *t, int64_t n,
                         double lo, double hi, double tau, int32_t width, int32_t height,
                         int mode, uint32_t *counts, int nthreads)
{
    const size_t m = (size_t)width * (size_t)height;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
    pthread_t th[256];
    job_t jobs[256];
    memset(counts, 0, sizeof(uint32_t) * m);
    for (int k = 0; k < nthreads; k++) {
        job_t *j = &jobs[k];
        j->x = x; j->y = y; j->t = t;
        j->i0 = n * k / nthreads;
        j->i1 = n * (k + 1) / nthreads;
        j->lo = lo; j->hi = hi; j->tau = tau;
        j->width = width; j->height = height;
        j->mode = mode;
        j->counts = k == 0 ? counts : (uint32_t *)calloc(m, sizeof(uint32_t));
        j->result = 0;
        if (nthreads == 1) run_job(j);
        else pthread_create(&th[k], NULL, run_job, j);
    }
    int64_t total = 0;
    for (int k = 0; k < nthreads; k++) {
        if (nthreads > 1) pthread_join(th[k], NULL);
        total += jobs[k].result;
        if (k > 0) {
            for (size_t p = 0; p < m; p++) counts[p] += jobs[k].counts[p];
            free(jobs[k].counts);
        }
    }
    return total;
}

/* accumulate_image over all events, split across nthreads; returns in_image. */
int64_t orc_point_image_mt(const double *x, const double *y, const double *t, int64_t n,
                           double nu, double tau, int32_t width, int32_t height,
                           uint32_t *counts, int nthreads)
{
    return run_split(x, y, t, n, nu, 0.0, tau, width, height, 0, counts, nthreads);
}

/* upper_bound_image / bound_terms image over all events; returns fully_inside. */
int64_t orc_bound_image_mt(const double *x, const double *y, const double *t, int64_t n,
                           double lo, double hi, double tau, int32_t width, int32_t height,
                           uint32_t *counts, int nthreads)
{
    return run_split(x, y, t, n, lo, hi, tau, width, height, 1, counts, nthreads);
}

/* exact integer reductions used by the assembly (contrast.py:238,249) */
void orc_image_sums(const uint32_t *counts, int64_t m, uint64_t *sum, uint64_t *sum_sq)
{
    uint64_t s = 0, q = 0;
    for (int64_t p = 0; p < m; p++) {
        s += counts[p];
        q += (uint64_t)counts[p] * counts[p];
    }
    *sum = s;
    *sum_sq = q;
}

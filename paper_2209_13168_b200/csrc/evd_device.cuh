// evd_device.cuh -- device building blocks of the bound-evaluation hot path (sm_100a).
//
// Every floating-point operation that feeds a reference-visible value is an
// explicit round-to-nearest binary64 intrinsic (no FMA contraction anywhere;
// the library is also compiled with --fmad=false), reproducing the numpy /
// numba arithmetic of the reference bit for bit.
//
//   warp            pkg/src/eventdiv/geometry.py:70-87
//   point binning   pkg/src/eventdiv/contrast.py:48-58
//   supercover      pkg/src/eventdiv/contrast.py:73-182 (_mark_point, _rasterize_into)
//   fully-inside    pkg/src/eventdiv/contrast.py:195-201
//   pairwise sum    numpy float64 pairwise summation behind np.sum (contrast.py:64)
#pragma once
#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

namespace evd {

// Device-side bounds checks, compiled into libevd_checked.so only
// (-DEVD_CHECKED; tests/test_gpu_checked.py runs the GPU suite on it): every
// mark lands inside the frame with p == y * W + x, queue slots stay inside
// their arrays.  A failed check traps the kernel (cudaErrorAssert).
#ifdef EVD_CHECKED
#define EVD_CHECK(cond) assert(cond)
#else
#define EVD_CHECK(cond) ((void)0)
#endif
__device__ __forceinline__ void check_mark(long long p, int x, int y, int W, int H)
{
    EVD_CHECK(x >= 0 && x < W && y >= 0 && y < H && p == (long long)y * W + x);
}

// ---------------------------------------------------------------- exact fp64
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Radial warp of one event with centred coordinates (xc, yc) = (x - cx, y - cy):
// s = (1 + nu*t) / denom, x' = cx + xc*s   (geometry.py:75, :87)
struct Warped { double x, y; };
__device__ __forceinline__ Warped warp_event(double xc, double yc, double t, double nu,
                                            double denom, double cx, double cy)
{
    const double s = ddiv(dadd(1.0, dmul(nu, t)), denom);
    return {dadd(cx, dmul(xc, s)), dadd(cy, dmul(yc, s))};
}

// contrast.py:52-54: int64 floor bin + half-open frame test; returns -1 if outside
__device__ __forceinline__ long long floor_bin(double x, double y, int W, int H)
{
    const long long ix = (long long)floor(x), iy = (long long)floor(y);
    if (ix >= 0 && ix < W && iy >= 0 && iy < H) return iy * (long long)W + ix;
    return -1;
}

// contrast.py:195-201 (half-open rectangle on both endpoints)
__device__ __forceinline__ int fully_inside(double ax, double ay, double bx, double by,
                                            int W, int H)
{
    return (0.0 <= ax && ax < W && 0.0 <= ay && ay < H &&
            0.0 <= bx && bx < W && 0.0 <= by && by < H) ? 1 : 0;
}

// Root-bound certificate (k_solve_spec, kModeRootCert).  A lower bound on the
// number of in-frame pixels the reference marks for the closed segment
// a -> b (contrast.py:94-182): clip it to the frame (approximately), shrink
// its extent by a margin far above any rounding of the reference's own clip
// and samples, and count the integers x = k strictly inside the shrunk
// x-extent (nx; likewise ny).  Each such line is crossed by the segment, so
// the reference's midpoint samples visit nx + 1 distinct columns, all inside
// the frame (ceil(lo) >= 1, floor(hi) <= W - 1), and mark a pixel of each
// (a sample on y = H also marks its row H - 1 square): >= max(nx, ny) + 1
// pixels when that maximum is positive.  Summed over events this bounds
// sum(counts) from below, and sum(counts^2) >= sum(counts)^2 / M.
__device__ __forceinline__ unsigned int root_cells_lb(double ax, double ay, double bx, double by,
                                                      int W, int H)
{
    const double dx = bx - ax, dy = by - ay;
    double t0 = 0.0, t1 = 1.0;
    if (dx == 0.0) {
        if (ax < 0.0 || ax > W) return 0;
    } else {
        double ta = -ax / dx, tb = (W - ax) / dx;
        if (ta > tb) { const double u = ta; ta = tb; tb = u; }
        t0 = fmax(t0, ta);
        t1 = fmin(t1, tb);
    }
    if (dy == 0.0) {
        if (ay < 0.0 || ay > H) return 0;
    } else {
        double ta = -ay / dy, tb = (H - ay) / dy;
        if (ta > tb) { const double u = ta; ta = tb; tb = u; }
        t0 = fmax(t0, ta);
        t1 = fmin(t1, tb);
    }
    if (!(t0 < t1)) return 0;
    const double x0 = ax + t0 * dx, x1 = ax + t1 * dx, y0 = ay + t0 * dy, y1 = ay + t1 * dy;
    constexpr double m = 1e-6;
    const double xl = fmax(fmin(x0, x1), 0.0) + m, xh = fmin(fmax(x0, x1), (double)W) - m;
    const double yl = fmax(fmin(y0, y1), 0.0) + m, yh = fmin(fmax(y0, y1), (double)H) - m;
    const double nx = xh > xl ? floor(xh) - ceil(xl) + 1.0 : 0.0;
    const double ny = yh > yl ? floor(yh) - ceil(yl) + 1.0 : 0.0;
    const double k = fmax(nx, ny);
    return k > 0.0 ? (unsigned int)k + 1u : 0u;
}

// ---------------------------------------------------------------- filtered path
// Approximate warp with r = RN(1/denom) (correctly rounded, computed once per
// velocity): s~ = RN(num * r) is within 3 ulp-relative of the exact
// RN(num / denom) (r and both products carry <= 2^-53 relative error each), so
// the approximate coordinate is within (|x'| + |xc s| + cx) * 1e-15 of the
// exact one.  kSure(v) below is a margin ~100x that bound; a geometry decided
// with it is the geometry of the exact values.
__device__ __forceinline__ Warped warp_approx(double xc, double yc, double t, double nu,
                                             double rden, double cx, double cy)
{
    const double s = dmul(dadd(1.0, dmul(nu, t)), rden);
    return {dadd(cx, dmul(xc, s)), dadd(cy, dmul(yc, s))};
}

__device__ __forceinline__ double sure_margin(const Warped &p, double cx, double cy)
{
    return 1e-13 * (1.0 + fabs(p.x) + fabs(p.y) + cx + cy);
}

// true if the exact coordinate lies strictly inside (f, f + 1)
__device__ __forceinline__ bool sure_cell(double v, double m, double &f)
{
    f = floor(v);
    return v - m > f && v + m < f + 1.0;
}

// Certified outcome of the point binning (contrast.py:52-55) from an
// approximate position: returns false if uncertain, else sets pix (-1 when
// the exact point bins outside the frame).
__device__ __forceinline__ bool sure_point(const Warped &p, double m, int W, int H, long long &pix)
{
    double fx, fy;
    if (!sure_cell(p.x, m, fx) || !sure_cell(p.y, m, fy)) return false;
    pix = (fx >= 0.0 && fx < W && fy >= 0.0 && fy < H) ? (long long)fy * W + (long long)fx : -1;
    return true;
}

// Certified outcome of one segment a -> b (contrast.py:94-203) from
// approximate endpoints: false if uncertain; else pix (-1: marks nothing)
// and inside (the fully-inside indicator).  Two certain cases:
//  * both endpoints strictly inside the same pixel: every sample of the
//    reference (p(0) = a, p(1) = a + ddx within 2 ulp of b, p(0.5) between)
//    is strictly inside it, so the reference marks exactly that pixel if it is
//    in the frame (else the clip rejects the segment), and the segment is
//    fully inside iff the pixel is in the frame;
//  * both endpoints strictly beyond the same frame edge (by the approximation
//    margin plus the reference's own rounding slack, (|a|+|b|) 2^-50): every
//    sample is then strictly beyond that edge, and a closed pixel square that
//    contains a point left of x = 0 (right of x = W, ...) is out of the frame.
__device__ __forceinline__ bool sure_segment(const Warped &a, const Warped &b, double ma,
                                             double mb, int W, int H, long long &pix, int &inside)
{
    const double sx = ma + mb + 1e-12 * (1.0 + fabs(a.x) + fabs(b.x));
    const double sy = ma + mb + 1e-12 * (1.0 + fabs(a.y) + fabs(b.y));
    if ((a.x < -sx && b.x < -sx) || (a.x > W + sx && b.x > W + sx) ||
        (a.y < -sy && b.y < -sy) || (a.y > H + sy && b.y > H + sy)) {
        pix = -1;
        inside = 0;
        return true;
    }
    double fax, fay, fbx, fby;
    if (!sure_cell(a.x, ma, fax) || !sure_cell(a.y, ma, fay) || !sure_cell(b.x, mb, fbx) ||
        !sure_cell(b.y, mb, fby) || fax != fbx || fay != fby)
        return false;
    inside = (fax >= 0.0 && fax < W && fay >= 0.0 && fay < H) ? 1 : 0;
    pix = inside ? (long long)fay * W + (long long)fax : -1;
    return true;
}

// sure_segment, also certifying edge-adjacent end cells: both exact end
// samples surely strictly inside cells that are equal or share an edge mark
// exactly those cells (build_segment's short-segment rule; the end sample
// p(1) = a + (b - a) is within a few ulps of b, far inside the margin).
// pix_b is -1 when the cells are equal.
__device__ __forceinline__ bool sure_segment_adj(const Warped &a, const Warped &b, double ma,
                                                 double mb, int W, int H, long long &pix_a,
                                                 long long &pix_b, int &inside)
{
    const double sx = ma + mb + 1e-12 * (1.0 + fabs(a.x) + fabs(b.x));
    const double sy = ma + mb + 1e-12 * (1.0 + fabs(a.y) + fabs(b.y));
    pix_b = -1;
    if ((a.x < -sx && b.x < -sx) || (a.x > W + sx && b.x > W + sx) ||
        (a.y < -sy && b.y < -sy) || (a.y > H + sy && b.y > H + sy)) {
        pix_a = -1;
        inside = 0;
        return true;
    }
    double fax, fay, fbx, fby;
    if (!sure_cell(a.x, ma, fax) || !sure_cell(a.y, ma, fay) || !sure_cell(b.x, mb, fbx) ||
        !sure_cell(b.y, mb, fby) || fabs(fax - fbx) + fabs(fay - fby) > 1.0)
        return false;
    const bool ia = fax >= 0.0 && fax < W && fay >= 0.0 && fay < H;
    const bool ib = fbx >= 0.0 && fbx < W && fby >= 0.0 && fby < H;
    inside = (ia && ib) ? 1 : 0;
    pix_a = ia ? (long long)fay * W + (long long)fax : -1;
    if (ib && (fax != fbx || fay != fby)) pix_b = (long long)fby * W + (long long)fbx;
    return true;
}

// ---------------------------------------------------------------- supercover
// Per-event dedup.  The reference marks each pixel at most once per event with
// a stamp grid (contrast.py:89-91).  The device compares against the previous
// _mark_point call only, which is exact: the sample parameters are visited in
// sorted order, x(s) = cx0 + s*ddx and y(s) = cy0 + s*ddy are monotone in s
// under round-to-nearest, and a pixel's closed square is an axis-aligned box,
// so the calls that mark a given pixel form one contiguous run -- a pixel
// already marked by this event was marked by the immediately preceding call.
// (DESIGN.md "Exact dedup" has the full argument.)
struct Prev {
    int x0, x1, y0, y1;  // previous call's closed-square pixel range (inclusive)
};

// Sinks take a pixel as (row-major index p, column, row); sinks that index a
// full image use p, the tiled frontier (evd_frontier_tiles.cu) uses (x, y).
//
// Pixel range [x0, x1] x [y0, y1] of the closed unit squares containing (px, py)
// (contrast.py:73-91).  Points reaching here come from a segment clipped to
// the frame, so the ranges fit in int.
__device__ __forceinline__ Prev point_range(double px, double py)
{
    const double fx = floor(px), fy = floor(py);
    const int ix1 = (int)fx, iy1 = (int)fy;
    return {(px == fx) ? ix1 - 1 : ix1, ix1, (py == fy) ? iy1 - 1 : iy1, iy1};
}

template <class Sink>
__device__ __forceinline__ int mark_point(double px, double py, int W, int H, Prev &prev,
                                          Sink &sink)
{
    // the (up to) 2 x 2 candidate pixels as four predicates built from row /
    // column tests shared between them, so lanes do not diverge
    const Prev r = point_range(px, py);
    const bool sx = r.x1 != r.x0, sy = r.y1 != r.y0;
    const bool px0 = r.x0 >= prev.x0 && r.x0 <= prev.x1, px1 = r.x1 >= prev.x0 && r.x1 <= prev.x1;
    const bool py0 = r.y0 >= prev.y0 && r.y0 <= prev.y1, py1 = r.y1 >= prev.y0 && r.y1 <= prev.y1;
    const bool fx0 = (unsigned)r.x0 < (unsigned)W, fx1 = sx && (unsigned)r.x1 < (unsigned)W;
    const bool fy0 = (unsigned)r.y0 < (unsigned)H, fy1 = sy && (unsigned)r.y1 < (unsigned)H;
    const int base = r.y0 * W + r.x0;  // the frame has < 2^31 pixels
    int marks = 0;
    if (fx0 && fy0 && !(px0 && py0)) { check_mark(base, r.x0, r.y0, W, H); sink(base, r.x0, r.y0); marks++; }
    if (fx1 && fy0 && !(px1 && py0)) { check_mark(base + 1, r.x1, r.y0, W, H); sink(base + 1, r.x1, r.y0); marks++; }
    if (fx0 && fy1 && !(px0 && py1)) { check_mark(base + W, r.x0, r.y1, W, H); sink(base + W, r.x0, r.y1); marks++; }
    if (fx1 && fy1 && !(px1 && py1)) { check_mark(base + W + 1, r.x1, r.y1, W, H); sink(base + W + 1, r.x1, r.y1); marks++; }
    prev = r;
    return marks;
}

// the segment end samples' calls (cursor_head / cursor_tail): the general
// closed-square call, or mark_interior (same marks: its single-cell fast path
// is mark_point's result for a point off the grid lines)
#ifndef EVD_END_INTERIOR
#define EVD_END_INTERIOR 1
#endif
#if EVD_END_INTERIOR
#define EVD_END_MARK mark_interior
#else
#define EVD_END_MARK mark_point
#endif
// mark_point for a point that is usually inside one pixel (a midpoint
// between consecutive crossings): the single-cell case tests one pixel;
// points on a grid line take the general path.
template <class Sink>
__device__ __forceinline__ int mark_interior(double px, double py, int W, int H, Prev &prev,
                                             Sink &sink)
{
    const double fx = floor(px), fy = floor(py);
    if (px != fx && py != fy) {
        const int ix = (int)fx, iy = (int)fy;
        const bool seen = ix >= prev.x0 && ix <= prev.x1 && iy >= prev.y0 && iy <= prev.y1;
        prev = Prev{ix, ix, iy, iy};
        if (!seen && (unsigned)ix < (unsigned)W && (unsigned)iy < (unsigned)H) {
            check_mark(iy * W + ix, ix, iy, W, H);
            sink(iy * W + ix, ix, iy);
            return 1;
        }
        return 0;
    }
    return mark_point(px, py, W, H, prev, sink);
}

// One monotone list of grid-line crossing parameters along the clipped segment
// (contrast.py:150-175): item i is s = clamp01((k_i - c0) / dd) for the
// integers k in [ceil(min), floor(max)], enumerated in increasing-s order
// (k ascending when dd > 0, descending when dd < 0).
struct CrossList {
    double c0, dd;
    long long k0;
    int n, step;

    __device__ __forceinline__ void init(double a0, double a1)
    {
        c0 = a0;
        dd = dsub(a1, a0);
        n = 0;
        step = 1;
        k0 = 0;
        if (dd == 0.0) return;
        const double lo = a0 < a1 ? a0 : a1, hi = a0 < a1 ? a1 : a0;
        const long long kmin = (long long)ceil(lo), kmax = (long long)floor(hi);
        if (kmin > kmax) return;
        n = (int)(kmax - kmin + 1);
        if (dd > 0.0) { k0 = kmin; step = 1; }
        else          { k0 = kmax; step = -1; }
    }
    __device__ __forceinline__ double at(int i) const
    {
        double s = ddiv(dsub((double)(k0 + (long long)step * i), c0), dd);
        if (s < 0.0) s = 0.0;
        else if (s > 1.0) s = 1.0;
        return s;
    }
};

// Skipping the calls of plain crossings (cursor_step).  Take an X item P at
// x ~ k (ddx > 0; ddx < 0 is the mirror image) whose y lies farther than
// delta = 2^-30 (1 + |y|) from every integer.  Positions are monotone in s
// and a crossing item lies within a few ulps (eps << delta) of its grid line,
// so:
//  * rows: a row line between P and the midpoint M1 before it (or M2 after
//    it) would put that line's Y item strictly between the two samples
//    around P, which are consecutive -- so M1, M2 and P share P's row, and
//    M1, M2 are not on a row line;
//  * columns: x is linear in s up to eps and the neighbouring samples lie in
//    [k-1-eps, k+1+eps], so M1.x is in [k-1/2-eps, x_P] and M2.x in
//    [x_P, k+1/2+eps].  P's closed squares are (floor(x_P), row), plus
//    (k-1, row) when x_P == k exactly: x_P < k is M1's cell, x_P > k is M2's,
//    and x_P == k gives M1 in column k-1 and M2 in column k (or a midpoint on
//    the line, whose own call marks both).
// So P's pixels are among those its neighbouring midpoints mark (their calls,
// or an earlier call of the same event -- the dedup only drops repeats), and
// skipping P's call leaves the pixel set, the image and the mark count
// unchanged.  The leading / trailing samples and near-corner crossings take
// the reference's closed-square call.
#ifndef EVD_SKIP_PLAIN
#define EVD_SKIP_PLAIN 1
#endif
__device__ __forceinline__ bool plain_crossing(double o)
{
    const double f = floor(o), slack = 0x1p-30 * (1.0 + fabs(o));
    return o - f > slack && (f + 1.0) - o > slack;
}

// A clipped segment ready for sampling.  Its sample sequence is
// S = [0, merge(X, Y), 1] (np.sort of the reference's ts array: both lists are
// monotone and clamped into [0, 1], so a two-way merge reproduces the sorted
// multiset).  Long sequences are cut by position into chunks of `csize`
// items: chunk j marks items [j*csize, (j+1)*csize) and the midpoint after
// each of them.  A chunk finds its first item with a merge-path search (an
// arithmetic estimate fixed up with exact item values) and recomputes its
// predecessor and the midpoint call before it for dedup, so the marks equal one
// sequential pass for any chunk size, and every chunk but a segment's last
// holds exactly csize items (lanes of a warp sampling chunks stay in step).
struct SegDesc {
    CrossList X, Y;  // X.c0 = cx0, X.dd = ddx, Y.c0 = cy0, Y.dd = ddy
    int chunks, csize;
};

// Clip the closed segment a -> b (contrast.py:94-146).  Returns the number of
// chunks to sample (0 if nothing is left to mark: off-frame, or degenerate /
// single-pixel segments, which are marked here directly).
template <class Sink>
__device__ __forceinline__ int build_segment(double ax, double ay, double bx, double by, int W,
                                             int H, int C, SegDesc &d, Sink &sink, int &marks)
{
    if (ax == bx && ay == by) {  // degenerate: floor rule, not the closed-square rule
        const long long p = floor_bin(ax, ay, W, H);
        if (p >= 0) {
            check_mark(p, (int)(p % W), (int)(p / W), W, H);
            sink(p, (int)(p % W), (int)(p / W));
            marks++;
        }
        return 0;
    }
    // Division-free rejection, exact: every sample the reference would mark
    // lies within (|ax|+|bx|)*2^-50 of the x-extent [min(ax,bx), max(ax,bx)]
    // (monotone rounding of t*dx, s*ddx), so a segment entirely left of -1
    // (right of W+1, ...) by that slack marks nothing in any rounding.
    {
        const double sx = 1.0 + 1e-12 * (fabs(ax) + fabs(bx));
        const double sy = 1.0 + 1e-12 * (fabs(ay) + fabs(by));
        if ((ax < -sx && bx < -sx) || (ax > W + sx && bx > W + sx) ||
            (ay < -sy && by < -sy) || (ay > H + sy && by > H + sy))
            return 0;
    }
    const double dx = dsub(bx, ax), dy = dsub(by, ay);
    double t0 = 0.0, t1 = 1.0;
    const bool in_closed = ax >= 0.0 && ax <= W && bx >= 0.0 && bx <= W &&
                           ay >= 0.0 && ay <= H && by >= 0.0 && by <= H;
    // Liang-Barsky (contrast.py:109-138).  When both endpoints lie in the
    // closed frame the reference's quotients provably leave t0 = 0, t1 = 1
    // (monotone rounding), so the four divisions are skipped.
    if (!in_closed) {
        if (dx == 0.0) {
            if (ax < 0.0 || ax > W) return 0;
        } else {
            double ta = ddiv(dsub(0.0, ax), dx), tb = ddiv(dsub((double)W, ax), dx);
            if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
        if (dy == 0.0) {
            if (ay < 0.0 || ay > H) return 0;
        } else {
            double ta = ddiv(dsub(0.0, ay), dy), tb = ddiv(dsub((double)H, ay), dy);
            if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
        if (t0 > t1) return 0;
    }
    // contrast.py:139-144
    const double xs = dadd(ax, dmul(t0, dx)), xe = dadd(ax, dmul(t1, dx));
    const double ys = dadd(ay, dmul(t0, dy)), ye = dadd(ay, dmul(t1, dy));
    {
        // Short segments.  The samples p(s) = (cx0 + s ddx, cy0 + s ddy),
        // s in [0, 1], are monotone in s, so every sample -- crossings and
        // midpoints included -- lies in the box spanned by p(0) = (cx0, cy0)
        // and p(1) = (cx0 + ddx, cy0 + ddy).  With both strictly inside their
        // pixels and those pixels equal or edge-adjacent, every closed square
        // containing a sample is one of the two, and the calls at p(0) and
        // p(1) mark both: the segment marks exactly them (in the frame).
        const double x0 = xs, y0 = ys;
        const double x1 = dadd(xs, dsub(xe, xs)), y1 = dadd(ys, dsub(ye, ys));
        const double fx0 = floor(x0), fy0 = floor(y0), fx1 = floor(x1), fy1 = floor(y1);
        if (fx0 != x0 && fy0 != y0 && fx1 != x1 && fy1 != y1 &&
            fabs(fx1 - fx0) + fabs(fy1 - fy0) <= 1.0) {
            if (fx0 >= 0.0 && fx0 < W && fy0 >= 0.0 && fy0 < H) {
                check_mark((long long)fy0 * W + (long long)fx0, (int)fx0, (int)fy0, W, H);
                sink((long long)fy0 * W + (long long)fx0, (int)fx0, (int)fy0);
                marks++;
            }
            if ((fx1 != fx0 || fy1 != fy0) && fx1 >= 0.0 && fx1 < W && fy1 >= 0.0 && fy1 < H) {
                check_mark((long long)fy1 * W + (long long)fx1, (int)fx1, (int)fy1, W, H);
                sink((long long)fy1 * W + (long long)fx1, (int)fx1, (int)fy1);
                marks++;
            }
            return 0;
        }
    }
    d.X.init(xs, xe);
    d.Y.init(ys, ye);
    const int items = 2 + d.X.n + d.Y.n;
    d.chunks = (items + C - 1) / C;
    d.csize = C;
    return d.chunks;
}

// Resumable walk over one chunk's items: mark every item, then the midpoint
// to its successor (contrast.py:176-182).  Each list keeps its next two item
// values, so the division that refills a list is off the critical path.
struct Cursor {
    int iX, iY;           // next unconsumed item of each list
    int left;             // items of the chunk still to mark, cur included
    int fin;              // cur is the trailing ts = 1
    double sX, sX2;       // values of X items iX, iX+1 (2 = none)
    double sY, sY2;
    double kX, kY;        // grid coordinate of the item that enters each lookahead next
    double cur;           // item to mark next
    int kind;             // origin of cur: 0 = the leading 0 / trailing 1, 1 = X list, 2 = Y list
    Prev prev;
};

__device__ __forceinline__ double item_or_none(const CrossList &L, int i)
{
    return i < L.n ? L.at(i) : 2.0;
}

// Number of X items among the first p items of merge(X, Y) (X first on
// equal values, as the walk takes them).  i is right iff X[i] does not come
// before Y[p-i-1] and X[i-1] comes before Y[p-i]; the estimate from the
// lists' arithmetic spacing is usually exact or one off.
__device__ __forceinline__ int merge_split(const SegDesc &d, int p)
{
    const CrossList &X = d.X, &Y = d.Y;
    const int lo = p - Y.n > 0 ? p - Y.n : 0, hi = p < X.n ? p : X.n;
    const double ax = fabs(X.dd), ay = fabs(Y.dd);
    const double ox = (X.c0 - (double)X.k0) * X.step, oy = (Y.c0 - (double)Y.k0) * Y.step;
    const double v = (ax + ay > 0.0) ? ((double)p - ox - oy) / (ax + ay) : 0.0;
    const double est = ceil(ox + v * ax);
    int i = est < (double)lo ? lo : (est > (double)hi ? hi : (int)est);
    // X[i] before Y[p-i-1]: then X[i] is among the first p (i too small)
    auto too_small = [&](int k) { return k < X.n && p - k > 0 && X.at(k) <= Y.at(p - k - 1); };
    while (i < hi && too_small(i)) i++;
    while (i > lo && !too_small(i - 1)) i--;
    return i;
}

// Position the cursor at chunk j (items [j*csize, (j+1)*csize) of S).
__device__ __forceinline__ bool cursor_init(const SegDesc &d, int j, Cursor &c)
{
    const CrossList &X = d.X, &Y = d.Y;
    const int T = X.n + Y.n, N = T + 2, m0 = j * d.csize;
    if (m0 >= N) return false;
    c.left = N - m0 < d.csize ? N - m0 : d.csize;
    c.fin = 0;
    if (m0 == 0) {  // the leading ts = 0 starts the first chunk
        c.iX = 0;
        c.iY = 0;
        c.cur = 0.0;
        c.kind = 0;
        c.prev = Prev{1, 0, 1, 0};
        c.sX = item_or_none(X, 0);
        c.sX2 = item_or_none(X, 1);
        c.sY = item_or_none(Y, 0);
        c.sY2 = item_or_none(Y, 1);
    } else {
        const int p = m0 - 1;  // S[m0] = merged[p], or the trailing 1 when p == T
        const int i = p < T ? merge_split(d, p) : X.n, jy = p - i;
        const double xp = i > 0 ? X.at(i - 1) : -1.0, yp = jy > 0 ? Y.at(jy - 1) : -1.0;
        double first;
        if (p >= T) {
            first = 1.0;
            c.kind = 0;
            c.fin = 1;
            c.iX = X.n;
            c.iY = Y.n;
            c.sX = c.sX2 = c.sY = c.sY2 = 2.0;
        } else {
            const double xi = item_or_none(X, i), yj = item_or_none(Y, jy);
            if (xi <= yj) {  // X first on equal values
                first = xi;
                c.kind = 1;
                c.iX = i + 1;
                c.iY = jy;
                c.sX = item_or_none(X, i + 1);
                c.sX2 = item_or_none(X, i + 2);
                c.sY = yj;
                c.sY2 = item_or_none(Y, jy + 1);
            } else {
                first = yj;
                c.kind = 2;
                c.iX = i;
                c.iY = jy + 1;
                c.sX = xi;
                c.sX2 = item_or_none(X, i + 1);
                c.sY = item_or_none(Y, jy + 1);
                c.sY2 = item_or_none(Y, jy + 2);
            }
        }
        // predecessor: the largest earlier item, or the leading ts = 0
        double pr = xp > yp ? xp : yp;
        if (pr < 0.0) pr = 0.0;
        const double sm = dmul(0.5, dadd(pr, first));
        c.prev = point_range(dadd(X.c0, dmul(sm, X.dd)), dadd(Y.c0, dmul(sm, Y.dd)));
        c.cur = first;
    }
    // integers below 2^53, so the running k stays exact in binary64
    c.kX = (double)(X.k0 + (long long)X.step * (c.iX + 2));
    c.kY = (double)(Y.k0 + (long long)Y.step * (c.iY + 2));
    return true;
}

// One item: mark it, find its successor (the list it comes from shifts its
// lookahead and refills it with one division on selected operands, so lanes
// stay converged), mark the midpoint.  Returns false once the chunk is done.
//
// The segment's end samples ts = 0 and ts = 1 (closed-square calls, the
// costliest marks) are not marked here but by cursor_head / cursor_tail,
// once per chunk outside the step loop: inside it a warp paid for them on
// ~60% of its steps (some lane is almost always at an end sample), outside
// it pays once per round.  The calls happen in the same order with the same
// dedup state, so the marks are unchanged.  c.fin on return: the chunk ends
// with the trailing sample, still to be marked by cursor_tail.
#ifdef EVD_OUTLINE_STEP
#define EVD_STEP_INLINE __noinline__
#else
#define EVD_STEP_INLINE __forceinline__
#endif
template <class Sink>
__device__ EVD_STEP_INLINE bool cursor_step(const SegDesc &d, Cursor &c, int W, int H, Sink &sink,
                                            int &marks)
{
    const double cx0 = d.X.c0, ddx = d.X.dd, cy0 = d.Y.c0, ddy = d.Y.dd;
    // A grid-line crossing whose other coordinate is not near a grid line
    // marks only pixels of the cells of the midpoints on either side of it,
    // which mark them anyway (plain_crossing), so its call adds no pixel and
    // is skipped; near-corner crossings take the reference's closed-square
    // call.  (kind 0: the leading sample, already marked by cursor_head.)
    if (c.kind != 0) {
        const double o = c.kind == 1 ? dadd(cy0, dmul(c.cur, ddy)) : dadd(cx0, dmul(c.cur, ddx));
        if (!(EVD_SKIP_PLAIN && plain_crossing(o)))
            marks += mark_point(dadd(cx0, dmul(c.cur, ddx)), dadd(cy0, dmul(c.cur, ddy)), W, H,
                                c.prev, sink);
    }
    const bool tX = c.sX < 2.0 && c.sX <= c.sY;
    const bool tY = !tX && c.sY < 2.0;
    double nxt = 1.0;  // the trailing ts = 1 when both lists are spent
    if (tX || tY) {
        nxt = tX ? c.sX : c.sY;
        const int idx = (tX ? c.iX : c.iY) + 2;  // the item that enters the lookahead
        const int lim = tX ? d.X.n : d.Y.n;
        const double k = tX ? c.kX : c.kY;
        double v = ddiv(dsub(k, tX ? cx0 : cy0), tX ? ddx : ddy);
        v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        if (idx >= lim) v = 2.0;
        c.kind = tX ? 1 : 2;
        if (tX) {
            c.iX++;
            c.sX = c.sX2;
            c.sX2 = v;
            c.kX = dadd(c.kX, (double)d.X.step);
        } else {
            c.iY++;
            c.sY = c.sY2;
            c.sY2 = v;
            c.kY = dadd(c.kY, (double)d.Y.step);
        }
    } else {
        c.kind = 0;
    }
    const double sm = dmul(0.5, dadd(c.cur, nxt));
    marks += mark_interior(dadd(cx0, dmul(sm, ddx)), dadd(cy0, dmul(sm, ddy)), W, H, c.prev, sink);
    c.cur = nxt;
    if (--c.left == 0) return false;  // the next item (trailing or not) starts the next chunk
    c.fin = (tX || tY) ? 0 : 1;       // the trailing sample is this chunk's last item
    return !c.fin;
}

// Before a chunk's steps: the leading sample ts = 0 of a segment's first chunk
// (the reference's closed-square call).  Returns whether the chunk has steps
// (a chunk holding only the trailing sample has none: c.fin).
template <class Sink>
__device__ __forceinline__ bool cursor_head(const SegDesc &d, Cursor &c, int W, int H, Sink &sink,
                                            int &marks)
{
    if (c.fin) return false;
    if (c.kind == 0)
        marks += EVD_END_MARK(dadd(d.X.c0, dmul(0.0, d.X.dd)), dadd(d.Y.c0, dmul(0.0, d.Y.dd)), W,
                            H, c.prev, sink);  // p(0), the reference's expression
    return true;
}

// After a chunk's steps: the trailing sample ts = 1 when it is in this chunk.
template <class Sink>
__device__ __forceinline__ void cursor_tail(const SegDesc &d, const Cursor &c, int W, int H,
                                            Sink &sink, int &marks)
{
    if (c.fin) {
        Prev prev = c.prev;
        marks += EVD_END_MARK(dadd(d.X.c0, dmul(1.0, d.X.dd)), dadd(d.Y.c0, dmul(1.0, d.Y.dd)), W, H,
                            prev, sink);
    }
}

// Sample chunk j of a built segment to the end.
template <class Sink>
__device__ __forceinline__ int sample_chunk(const SegDesc &d, int j, int W, int H, Sink &sink)
{
    Cursor c;
    int marks = 0;
    if (cursor_init(d, j, c)) {
        if (cursor_head(d, c, W, H, sink, marks))
            while (cursor_step(d, c, W, H, sink, marks)) {
            }
        cursor_tail(d, c, W, H, sink, marks);
    }
    return marks;
}

// _rasterize_into (contrast.py:94-182) for one segment by one thread, chunk
// by chunk (chunk size C only moves the seams).  Returns the sink calls.
template <class Sink>
__device__ int raster_segment(double ax, double ay, double bx, double by, int W, int H, int C,
                              Sink &sink)
{
    SegDesc d;
    int marks = 0;
    const int chunks = build_segment(ax, ay, bx, by, W, H, C, d, sink, marks);
    for (int j = 0; j < chunks; j++) marks += sample_chunk(d, j, W, H, sink);
    return marks;
}


// ---------------------------------------------------------------- reductions
template <class T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum of up to 4 u64 counters, then one global atomicAdd each.
// Requires blockDim.x a multiple of 32 and <= 1024.
template <int K>
__device__ __forceinline__ void block_add_u64(unsigned long long (&v)[K],
                                              unsigned long long *dst)
{
    __shared__ unsigned long long red[32][K];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; k++) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) red[wid][k] = v[k];
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
#pragma unroll
        for (int k = 0; k < K; k++) {
            unsigned long long s = lane < nw ? red[lane][k] : 0ull;
            s = warp_sum(s);
            if (lane == 0 && s) atomicAdd(dst + k, s);
        }
    }
    __syncthreads();
}

// One pairwise-sum leaf (numpy's n <= 128 block, loops_utils.h.src) computed by
// an aligned group of 8 lanes: lane j owns accumulator r[j], the fixed combine
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) is three xor-shuffle steps (IEEE
// addition is commutative, only association matters), and lane 0 adds the
// n % 8 tail sequentially.  n < 8 (only when M < 8) is the sequential branch.
// All loads of the leaf are issued before the first add (one memory round
// trip).  Q provides load(i) -> raw, term(raw) -> summand, clear(i).
template <class Q>
__device__ __forceinline__ double pairwise_leaf8(int off, int n, int j, const Q &q)
{
    const unsigned gmask = 0xffu << (threadIdx.x & 24);
    if (n < 8) {
        double r = 0.0;
        if (j == 0) {
            for (int i = 0; i < n; i++) r = dadd(r, q.term(q.load(off + i)));
            for (int i = 0; i < n; i++) q.clear(off + i);
        }
        return r;
    }
    const int body = n - (n % 8), rows = body / 8;  // rows in [1, 16]
    typename Q::raw v[16], tail[7];
#pragma unroll
    for (int k = 0; k < 16; k++)
        if (k < rows) v[k] = q.load(off + 8 * k + j);
#pragma unroll
    for (int k = 0; k < 7; k++)
        if (j == 0 && body + k < n) tail[k] = q.load(off + body + k);
#pragma unroll
    for (int k = 0; k < 16; k++)
        if (k < rows) q.clear(off + 8 * k + j);
    if (j == 0)
        for (int k = body; k < n; k++) q.clear(off + k);
    double r = q.term(v[0]);
#pragma unroll
    for (int k = 1; k < 16; k++)
        if (k < rows) r = dadd(r, q.term(v[k]));
    r = dadd(r, __shfl_xor_sync(gmask, r, 1, 8));
    r = dadd(r, __shfl_xor_sync(gmask, r, 2, 8));
    r = dadd(r, __shfl_xor_sync(gmask, r, 4, 8));
    if (j == 0) {
#pragma unroll
        for (int k = 0; k < 7; k++)
            if (body + k < n) r = dadd(r, q.term(tail[k]));
    }
    return r;
}

// ---------------------------------------------------------------- grid barrier
// Counting barrier for a cooperative (co-resident) grid; the last block to
// arrive optionally runs `leader` before releasing the others.
struct GridBar {
    unsigned int count;
    unsigned int gen;
};

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <class Leader>
__device__ __forceinline__ void grid_barrier(GridBar *b, Leader &&leader)
{
    __shared__ unsigned int s_gen;
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        s_gen = ld_acquire(&b->gen);
        __threadfence();
        s_last = atomicAdd(&b->count, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        leader();
        __syncthreads();
        if (threadIdx.x == 0) {
            b->count = 0;
            __threadfence();
            atomicExch(&b->gen, s_gen + 1);
        }
    } else if (threadIdx.x == 0) {
        while (ld_acquire(&b->gen) == s_gen) __nanosleep(20);
    }
    if (threadIdx.x == 0) __threadfence();
    __syncthreads();
}

}  // namespace evd

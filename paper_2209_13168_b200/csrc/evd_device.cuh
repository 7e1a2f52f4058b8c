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
#include <cstdint>
#include <cuda_runtime.h>

namespace evd {

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

// ---------------------------------------------------------------- supercover
// Per-event dedup.  The reference marks each pixel at most once per event with
// a stamp grid (contrast.py:89-91).  The device replaces it with a comparison
// against the previous _mark_point call only, which is exact: the sample
// parameters are visited in sorted order, x(s) = cx0 + s*ddx and y(s) are
// monotone in s under round-to-nearest, and a pixel's closed square is an
// axis-aligned box, so the calls that mark a given pixel form one contiguous
// run.  A pixel already marked by this event was therefore marked by the
// immediately preceding call.  (DESIGN.md "Exact dedup" has the full argument.)
struct Prev {
    long long x0, x1, y0, y1;  // previous call's closed-square pixel range (inclusive)
};

template <class Sink>
__device__ __forceinline__ void mark_point(double px, double py, int W, int H, Prev &prev,
                                           Sink &sink)
{
    // contrast.py:73-91: every pixel whose closed unit square contains (px, py)
    const double fx = floor(px), fy = floor(py);
    const long long ix1 = (long long)fx, iy1 = (long long)fy;
    const long long ix0 = (px == fx) ? ix1 - 1 : ix1;
    const long long iy0 = (py == fy) ? iy1 - 1 : iy1;
    for (long long ix = ix0; ix <= ix1; ix++) {
        if (ix < 0 || ix >= W) continue;
        const bool px_in = ix >= prev.x0 && ix <= prev.x1;
        for (long long iy = iy0; iy <= iy1; iy++) {
            if (iy < 0 || iy >= H) continue;
            if (px_in && iy >= prev.y0 && iy <= prev.y1) continue;
            sink(iy * (long long)W + ix);
        }
    }
    prev.x0 = ix0; prev.x1 = ix1; prev.y0 = iy0; prev.y1 = iy1;
}

// One monotone list of grid-line crossing parameters along the clipped segment
// (contrast.py:150-175): s_k = clamp01((k - c0) / dd) for integer k in
// [ceil(min), floor(max)], enumerated in increasing-s order (k ascending when
// dd > 0, descending when dd < 0).
struct Crossings {
    double c0, dd;
    long long k, k_end;  // current and last k (inclusive)
    int step;            // +1 / -1
    bool live;
    __device__ __forceinline__ void init(double a0, double a1)
    {
        c0 = a0;
        dd = dsub(a1, a0);
        if (dd == 0.0) { live = false; return; }
        const double lo = a0 < a1 ? a0 : a1, hi = a0 < a1 ? a1 : a0;
        const long long kmin = (long long)ceil(lo), kmax = (long long)floor(hi);
        if (kmin > kmax) { live = false; return; }
        live = true;
        if (dd > 0.0) { k = kmin; k_end = kmax; step = 1; }
        else          { k = kmax; k_end = kmin; step = -1; }
    }
    __device__ __forceinline__ double value() const
    {
        double s = ddiv(dsub((double)k, c0), dd);
        if (s < 0.0) s = 0.0;
        else if (s > 1.0) s = 1.0;
        return s;
    }
    __device__ __forceinline__ void advance()
    {
        if (k == k_end) live = false;
        else k += step;
    }
};

// _rasterize_into (contrast.py:94-182) for the closed segment a -> b, calling
// sink(pixel) once for every in-image pixel whose closed square it touches.
// Returns the number of sink calls.
template <class Sink>
__device__ __noinline__ int raster_segment(double ax, double ay, double bx, double by,
                                           int W, int H, Sink &sink)
{
    int marks = 0;
    auto counted = [&](long long p) { marks++; sink(p); };
    if (ax == bx && ay == by) {  // degenerate: floor rule, not the closed-square rule
        const long long p = floor_bin(ax, ay, W, H);
        if (p >= 0) counted(p);
        return marks;
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
    const double cx0 = dadd(ax, dmul(t0, dx)), cy0 = dadd(ay, dmul(t0, dy));
    const double cx1 = dadd(ax, dmul(t1, dx)), cy1 = dadd(ay, dmul(t1, dy));
    Crossings X, Y;
    X.init(cx0, cx1);
    Y.init(cy0, cy1);
    const double ddx = X.dd, ddy = Y.dd;
    // np.sort(ts) == [0, merge(X, Y), 1]: both crossing lists are monotone and
    // clamped into [0, 1], so a two-way merge reproduces the sorted multiset.
    double sx = X.live ? X.value() : 2.0;
    double sy = Y.live ? Y.value() : 2.0;
    Prev prev{1, 0, 1, 0};
    double cur = 0.0;
    while (true) {
        mark_point(dadd(cx0, dmul(cur, ddx)), dadd(cy0, dmul(cur, ddy)), W, H, prev, counted);
        double nxt;
        bool last = false;
        if (X.live && (!Y.live || sx <= sy)) {
            nxt = sx;
            X.advance();
            sx = X.live ? X.value() : 2.0;
        } else if (Y.live) {
            nxt = sy;
            Y.advance();
            sy = Y.live ? Y.value() : 2.0;
        } else {
            nxt = 1.0;
            last = true;
        }
        const double sm = dmul(0.5, dadd(cur, nxt));
        mark_point(dadd(cx0, dmul(sm, ddx)), dadd(cy0, dmul(sm, ddy)), W, H, prev, counted);
        cur = nxt;
        if (last) {
            mark_point(dadd(cx0, dmul(cur, ddx)), dadd(cy0, dmul(cur, ddy)), W, H, prev, counted);
            break;
        }
    }
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
// q(i) yields the i-th summand.  Result valid in lane (j == 0) of the group.
template <class Q>
__device__ __forceinline__ double pairwise_leaf8(int off, int n, int j, const Q &q)
{
    const unsigned gmask = 0xffu << (threadIdx.x & 24);
    if (n < 8) {
        double r = 0.0;
        if (j == 0)
            for (int i = 0; i < n; i++) r = dadd(r, q(off + i));
        return r;
    }
    double r = q(off + j);
    const int body = n - (n % 8);
    for (int i = 8; i < body; i += 8) r = dadd(r, q(off + i + j));
    r = dadd(r, __shfl_xor_sync(gmask, r, 1, 8));
    r = dadd(r, __shfl_xor_sync(gmask, r, 2, 8));
    r = dadd(r, __shfl_xor_sync(gmask, r, 4, 8));
    if (j == 0)
        for (int i = body; i < n; i++) r = dadd(r, q(off + i));
    return r;
}

// ---------------------------------------------------------------- grid barrier
// Sense-counting barrier for a cooperative (co-resident) grid; the last block
// to arrive optionally runs `leader` before releasing the others.
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

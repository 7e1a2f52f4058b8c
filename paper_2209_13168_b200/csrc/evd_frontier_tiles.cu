// evd_frontier_tiles.cu -- the batched frontier (bound_terms for K intervals,
// contrast.py:241-251) with every bound image kept in shared memory.
//
// The radial warp x' = c + (x - c) s, s = (1 + nu t) / (1 + nu tau)
// (geometry.py:70-87), moves an event along the ray from the FOE c through
// it, and for nu <= 0, t in [0, tau] the scale is s >= 1 (also in binary64:
// RN(1 + nu t) >= RN(1 + nu tau) > 0 and RN(a / b) >= 1 for a >= b).  Every
// point the supercover samples (contrast.py:94-182) lies on that ray, beyond
// the event, up to rounding (~1e-8 px even for the 1e8 px warps of the root
// interval), and every pixel it marks has its centre within sqrt(2)/2 of a
// sample.  So a partition of the pixels into angular tiles around the FOE is
// valid for every velocity at once:
//
//  * tile 0 is a disc of pixel centres |q| < R0 around the FOE, the others
//    are wedges of equal pixel count (pixel centres sorted by angle);
//  * an event is listed in every tile owning a pixel centre within
//    delta = 0.75 px of its ray {c + rho (x - c)/|x - c| : rho >= |x - c|}:
//    the disc if |x - c| <= Rc + delta (Rc: the disc's largest centre
//    radius), a wedge if its angular range comes within
//    asin(delta / max(Rw, |x - c| - delta)) of the event's angle (a centre q
//    at angle phi from the ray is at distance >= |q| sin(phi) from it, and
//    >= |x - c| - |q| when it lies before the ray's start; Rw <= |q| for every
//    wedge pixel);
//  * a CTA takes one (tile, group of 32 intervals) work item at a time: lane j
//    of every warp evaluates interval j on the same event (k_frontier_f's
//    certified filtered warp, exact path for the uncertain pairs), marks land
//    in the tile's 32 images in shared memory -- only pixels the tile owns --
//    and the item ends by reducing sum(H), sum(H^2) of each image in shared
//    memory straight into the per-interval u64 results.
//
// Each pixel is owned by one tile and an event marks a pixel at most once per
// interval (the reference's stamp dedup, kept exactly by the sampler), so
// every image of the reference is the disjoint union of the tiles' images:
// S_bar = sum(H^2) and marks = sum(H) add up over tiles.  fully_inside is
// counted by the event's first ("home") tile only.  Counters are u16 pairs:
// a pixel's count never exceeds the number of events listed in its tile, and
// the tiled path is taken only when every tile lists fewer than 65,536.
// Windows with non-finite coordinates, frames the plan cannot tile and
// intervals reaching nu > 0 take the global-image path (k_frontier_f).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "evd_device.cuh"
#include "evd_internal.h"

namespace evd {

constexpr double kTileDelta = 0.75;  // > sqrt(2)/2 + rounding of the sampled positions
#ifndef EVD_TILE_THREADS
#define EVD_TILE_THREADS 512
#endif
constexpr int kTileThreads = EVD_TILE_THREADS;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kTileMaxEvents = 65535;  // u16 counters
constexpr int kTileMaxWords = 32768;   // bound on a tile image's words (checked builds)

// ---------------------------------------------------------------- host plan
namespace {

template <class T>
cudaError_t ensure(T *&p, size_t &cap, size_t n)
{
    if (n <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) cap = std::max<size_t>(n, 1);
    return e;
}

}  // namespace

struct FrontierTiles {
    // plan (per frame size and tile capacity)
    int W = 0, H = 0, P = 0;        // P: largest tile, pixels
    int S = 0;                      // wedges (tiles 1..S); tile 0 is the disc
    int max_rows = 0;
    double Rc = -1.0, Rw = 0.0;
    bool plan_ok = false;
    int4 *meta = nullptr;           // per tile: y0, nrows, row_off, npix
    size_t meta_cap = 0;
    int4 *rows = nullptr;           // per tile row: two runs (x_lo | x_hi << 16, base)
    size_t rows_cap = 0;
    double2 *ang = nullptr;         // per wedge: angular range of its pixel centres
    size_t ang_cap = 0;
    std::vector<int4> h_meta;
    // binned window
    unsigned long long gen = ~0ull;
    bool bin_ok = false;
    long long total = 0;            // sum of list lengths
    long long *start = nullptr;     // per tile: first listed event
    size_t start_cap = 0;
    int2 *cnt = nullptr;            // per tile: (home, all)
    size_t cnt_cap = 0;
    unsigned long long *cursor = nullptr;  // fill cursors (home, foreign) per tile
    size_t cursor_cap = 0;
    unsigned int *flag = nullptr;   // non-finite event seen
    size_t flag_cap = 0;
    double *xs = nullptr, *ys = nullptr, *ts = nullptr;
    size_t xs_cap = 0, ys_cap = 0, ts_cap = 0;
    float *rho = nullptr;           // per listed event: frame-exit scale (see k_tile_fill)
    size_t rho_cap = 0;
    float2 *xyf = nullptr;          // per listed event: RN32 of the centred coordinates
    size_t xyf_cap = 0;
    int *order = nullptr;           // tiles with work, heaviest list first
    size_t order_cap = 0;
    int n_order = 0;
    unsigned int *ctr = nullptr;    // work-item counter
    size_t ctr_cap = 0;
    std::vector<int2> h_cnt;
};

FrontierTiles *tiles_new() { return new FrontierTiles(); }

void tiles_free(FrontierTiles *f)
{
    if (!f) return;
    for (void *p : {(void *)f->meta, (void *)f->rows, (void *)f->ang, (void *)f->start,
                    (void *)f->cnt, (void *)f->cursor, (void *)f->flag, (void *)f->xs,
                    (void *)f->ys, (void *)f->ts, (void *)f->rho, (void *)f->xyf, (void *)f->order,
                    (void *)f->ctr})
        if (p) cudaFree(p);
    delete f;
}

// Shared memory of the tile kernel for tiles of up to P pixels and max_rows rows.
struct TileQueue {
    SegDesc d[64];
    int ev[64];             // uncertain pairs: (listed event - start) << 5 | interval lane
    int off[65];
    unsigned char jj[64];   // interval lane of each queued segment
};
static size_t tile_smem_bytes(int P, int max_rows)
{
    const size_t words = (size_t)(P / 2) | 1;  // odd stride: lanes' images in distinct banks
    return 32 * words * 4 + (size_t)max_rows * sizeof(int4) + kTileWarps * sizeof(TileQueue);
}
static int tile_words(int P) { return (P / 2) | 1; }

// Build the disc + wedge partition of a W x H frame with tiles of <= P pixels.
static bool build_plan(FrontierTiles &f, int W, int H, int P)
{
    const long long M = (long long)W * H;
    const double cx = W / 2.0, cy = H / 2.0;
    std::vector<double> r(M), th(M);
    for (int iy = 0; iy < H; iy++)
        for (int ix = 0; ix < W; ix++) {
            const double qx = ix + 0.5 - cx, qy = iy + 0.5 - cy;
            r[(size_t)iy * W + ix] = std::hypot(qx, qy);
            th[(size_t)iy * W + ix] = std::atan2(qy, qx);
        }
    // disc: centres strictly inside R0, at most P of them
    std::vector<double> rs(r);
    double R0 = 0.0;
    if (M > P) {
        std::nth_element(rs.begin(), rs.begin() + P, rs.end());
        R0 = rs[P];
    } else {
        R0 = INFINITY;
    }
    std::vector<int> tile(M);
    std::vector<long long> rest;
    rest.reserve(M);
    double Rc = -1.0;
    for (long long p = 0; p < M; p++) {
        if (r[p] < R0) {
            tile[p] = 0;
            Rc = std::max(Rc, r[p]);
        } else {
            rest.push_back(p);
        }
    }
    std::sort(rest.begin(), rest.end(), [&](long long a, long long b) {
        if (th[a] != th[b]) return th[a] < th[b];
        if (r[a] != r[b]) return r[a] < r[b];
        return a < b;
    });
    const long long nr = (long long)rest.size();
    // at least 8 wedges: each spans < pi, so a row meets a wedge in one
    // interval, less the disc's chord: at most two runs of pixels
    const int S = nr ? (int)std::min<long long>(nr, std::max<long long>(8, (nr + P - 1) / P)) : 0;
    std::vector<double2> ang(S);
    double Rw = INFINITY;
    for (int k = 0; k < S; k++) {
        const long long a = k * nr / S, b = (k + 1) * nr / S;
        ang[k] = make_double2(th[rest[a]], th[rest[b - 1]]);
        for (long long i = a; i < b; i++) {
            tile[rest[i]] = 1 + k;
            Rw = std::min(Rw, r[rest[i]]);
        }
    }
    if (!S) Rw = 0.0;
    // per tile and row: one contiguous run of owned pixels
    const int T = 1 + S;
    std::vector<int> y0(T, INT32_MAX), y1(T, -1), npix(T, 0);
    for (int iy = 0; iy < H; iy++)
        for (int ix = 0; ix < W; ix++) {
            const int k = tile[(size_t)iy * W + ix];
            y0[k] = std::min(y0[k], iy);
            y1[k] = std::max(y1[k], iy);
            npix[k]++;
        }
    std::vector<int4> meta(T);
    std::vector<int4> rows;
    int max_rows = 0;
    for (int k = 0; k < T; k++) {
        if (npix[k] > P) return false;
        if (!npix[k]) {
            meta[k] = make_int4(0, 0, (int)rows.size(), 0);
            continue;
        }
        const int nrows = y1[k] - y0[k] + 1;
        meta[k] = make_int4(y0[k], nrows, (int)rows.size(), npix[k]);
        max_rows = std::max(max_rows, nrows);
        int base = 0;
        for (int iy = y0[k]; iy <= y1[k]; iy++) {
            int run[2][2] = {{1, 0}, {1, 0}};  // empty runs: x_lo = 1 > x_hi = 0
            int nrun = 0, ix = 0;
            while (ix < W) {
                if (tile[(size_t)iy * W + ix] != k) { ix++; continue; }
                const int xl = ix;
                while (ix < W && tile[(size_t)iy * W + ix] == k) ix++;
                if (nrun == 2) return false;  // three runs: this frame is not tiled
                run[nrun][0] = xl;
                run[nrun][1] = ix - 1;
                nrun++;
            }
            const int c0 = run[0][1] - run[0][0] + 1, c1 = run[1][1] - run[1][0] + 1;
            rows.push_back(make_int4((int)((unsigned)run[0][0] | ((unsigned)run[0][1] << 16)), base,
                                     (int)((unsigned)run[1][0] | ((unsigned)run[1][1] << 16)),
                                     base + c0));
            base += c0 + c1;
        }
    }
    f.W = W;
    f.H = H;
    f.P = P;
    f.S = S;
    f.Rc = Rc;
    f.Rw = Rw;
    f.max_rows = max_rows;
    f.h_meta = meta;
    if (ensure(f.meta, f.meta_cap, meta.size()) || ensure(f.rows, f.rows_cap, rows.size()) ||
        ensure(f.ang, f.ang_cap, ang.size()))
        return false;
    if (cudaMemcpy(f.meta, meta.data(), meta.size() * sizeof(int4), cudaMemcpyHostToDevice) ||
        cudaMemcpy(f.rows, rows.data(), rows.size() * sizeof(int4), cudaMemcpyHostToDevice) ||
        (S && cudaMemcpy(f.ang, ang.data(), ang.size() * sizeof(double2),
                         cudaMemcpyHostToDevice)))
        return false;
    return true;
}

// ---------------------------------------------------------------- binning
struct TileGeom {
    const double2 *ang;
    int S;
    double Rc, Rw;
};

__device__ __forceinline__ double circ_dist(double a, double b)
{
    const double d = fabs(a - b);
    return d > M_PI ? 2.0 * M_PI - d : d;
}

__device__ __forceinline__ double arc_dist(double th, double2 arc)
{
    if (th >= arc.x && th <= arc.y) return 0.0;
    return fmin(circ_dist(th, arc.x), circ_dist(th, arc.y));
}

// Calls f(tile, home) for every tile listing the event (xc, yc) = x - c;
// home is true for exactly the first.
template <class F>
__device__ __forceinline__ void for_each_tile(double xc, double yc, const TileGeom &g, F &&f)
{
    const double r = hypot(xc, yc);
    bool first = true;
    if (r <= g.Rc + kTileDelta + 1e-9) {
        f(0, true);
        first = false;
    }
    if (g.S == 0) return;
    const double th = atan2(yc, xc);
    const double phi = asin(fmin(1.0, kTileDelta / fmax(g.Rw, r - kTileDelta))) + 1e-9;
    int lo = 0, hi = g.S;  // first wedge starting after th
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (g.ang[mid].x <= th) lo = mid + 1;
        else hi = mid;
    }
    const int k0 = lo > 0 ? lo - 1 : g.S - 1;
    int visited = 0;
    for (int k = k0; visited < g.S; k = k > 0 ? k - 1 : g.S - 1) {
        if (arc_dist(th, g.ang[k]) > phi) break;
        f(1 + k, first);
        first = false;
        visited++;
    }
    for (int k = k0 + 1 < g.S ? k0 + 1 : 0; visited < g.S; k = k + 1 < g.S ? k + 1 : 0) {
        if (arc_dist(th, g.ang[k]) > phi) break;
        f(1 + k, first);
        first = false;
        visited++;
    }
}

__global__ void k_tile_count(const double *__restrict__ xc, const double *__restrict__ yc,
                             const double *__restrict__ t, long long n, TileGeom g, int T,
                             int2 *cnt, unsigned int *flag)
{
    extern __shared__ int hist[];  // [T][2]
    for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double x = xc[i], y = yc[i], tt = t[i];
        // the tiled path takes finite events within 1e5 px of the FOE (its
        // certified fp32 positions then stay below 1e11 px at any scale up to
        // 1e6, see tile_point); the rest of the windows take the global path
        if (!isfinite(tt) || !(fabs(x) <= 1e5) || !(fabs(y) <= 1e5)) {
            *flag = 1u;
            continue;
        }
        for_each_tile(x, y, g, [&](int k, bool home) { atomicAdd(hist + 2 * k + (home ? 0 : 1), 1); });
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * T; i += blockDim.x)
        if (hist[i]) atomicAdd((i & 1) ? &cnt[i >> 1].y : &cnt[i >> 1].x, hist[i]);
}

// cursor[2k] / [2k+1]: next home / foreign slot of tile k.  rho (rounded up
// to float) is the event's frame-exit scale: the ray from the FOE through the
// event leaves the closed frame at distance min(cx/|ux|, cy/|uy|) (unit
// direction u), so every point of it at scale s > rho = min(cx/|xc|, cy/|yc|)
// + 1.5/|x - c| lies more than 1.5 px beyond the frame.
__global__ void k_tile_fill(const double *__restrict__ xc, const double *__restrict__ yc,
                            const double *__restrict__ t, long long n, TileGeom g, double cx,
                            double cy, unsigned long long *cursor, double *xs, double *ys,
                            double *ts, float *rho, float2 *xyf)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double x = xc[i], y = yc[i], tt = t[i];
        const double r = hypot(x, y);
        const float q = r > 0.0 ? __double2float_ru(fmin(cx / fabs(x), cy / fabs(y)) + 1.5 / r)
                                : INFINITY;
        for_each_tile(x, y, g, [&](int k, bool home) {
            const unsigned long long p = atomicAdd(cursor + 2 * k + (home ? 0 : 1), 1ull);
            xs[p] = x;
            ys[p] = y;
            ts[p] = tt;
            rho[p] = q;
            xyf[p] = make_float2(__double2float_rn(x), __double2float_rn(y));
        });
    }
}

// ---------------------------------------------------------------- tile kernel
// Marks of one interval's image restricted to the tile: (x, y) -> local pixel
// through the tile's row table (two runs per row), u16 counters packed in
// pairs.  Shared-window addresses are 32-bit.
struct TileSink {
    unsigned img;    // shared address of this interval's image
    unsigned rows;   // shared address of the row table (int4 per row)
    int y0, nrows;
    __device__ __forceinline__ void operator()(long long, int x, int y) const
    {
        const int r = y - y0;
        if ((unsigned)r < (unsigned)nrows) {
            int e0, e1, e2, e3;
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3)
                         : "r"(rows + 16u * (unsigned)r));
            const int xl = e0 & 0xffff, xh = (int)((unsigned)e0 >> 16);
            const int xl2 = e2 & 0xffff, xh2 = (int)((unsigned)e2 >> 16);
            int l = -1;
            if (x >= xl && x <= xh) l = e1 + x - xl;
            else if (x >= xl2 && x <= xh2) l = e3 + x - xl2;
            EVD_CHECK(l < 2 * kTileMaxWords);
            if (l >= 0)
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(img + 4u * (unsigned)(l >> 1)),
                             "r"(1u << ((l & 1) << 4))
                             : "memory");
        }
    }
};

struct TileView {
    unsigned img;    // shared address of image 0; image j at img + 4 * j * words
    unsigned rows;
    int y0, nrows, words;
    __device__ __forceinline__ TileSink sink(int j) const
    {
        return TileSink{img + 4u * (unsigned)(j * words), rows, y0, nrows};
    }
};

// warp_drain_list for queued tile segments (slots [0, nq), nq < 64): rounds of
// 32 equal-length chunks, every lane marking into its segment's image.
__device__ __noinline__ void tile_drain(TileQueue &q, int nq, int W, int H, TileView v)
{
    const int lane = threadIdx.x & 31;
    const int c0 = lane < nq ? q.d[lane].chunks : 0;
    const int c1 = lane + 32 < nq ? q.d[lane + 32].chunks : 0;
    int i0 = c0, i1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v0 = __shfl_up_sync(0xffffffffu, i0, o);
        const int v1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= o) { i0 += v0; i1 += v1; }
    }
    const int t0 = __shfl_sync(0xffffffffu, i0, 31);
    i1 += t0;
    q.off[lane] = i0 - c0;
    q.off[lane + 32] = i1 - c1;
    const int total = __shfl_sync(0xffffffffu, i1, 31);
    if (lane == 0) q.off[64] = total;
    __syncwarp();
    int marks = 0;
    for (int base = 0; base < total; base += 32) {
        const int t = base + lane;
        bool active = false;
        int slot = 0;
        Cursor c;
        if (t < total) {
            int L = 0;
#pragma unroll
            for (int s = 32; s > 0; s >>= 1)
                if (L + s < 64 && q.off[L + s] <= t) L += s;
            slot = L;
            active = cursor_init(q.d[slot], t - q.off[L], c);
        }
        const SegDesc d = q.d[slot];
        TileSink sink = v.sink(q.jj[slot]);
        const bool live = active;
        if (active) active = cursor_head(d, c, W, H, sink, marks);
        while (__any_sync(0xffffffffu, active))
            if (active) active = cursor_step(d, c, W, H, sink, marks);
        if (live) cursor_tail(d, c, W, H, sink, marks);
    }
    __syncwarp();
}

// sure_segment_adj (evd_device.cuh) returning the certified cells as (x, y):
// (xa, ya) / (xb, yb), x = -1 for none.
__device__ __forceinline__ bool sure_cells(const Warped &a, const Warped &b, double ma, double mb,
                                           int W, int H, int &xa, int &ya, int &xb, int &yb,
                                           int &inside)
{
    const double sx = ma + mb + 1e-12 * (1.0 + fabs(a.x) + fabs(b.x));
    const double sy = ma + mb + 1e-12 * (1.0 + fabs(a.y) + fabs(b.y));
    xa = xb = -1;
    ya = yb = 0;
    if ((a.x < -sx && b.x < -sx) || (a.x > W + sx && b.x > W + sx) ||
        (a.y < -sy && b.y < -sy) || (a.y > H + sy && b.y > H + sy)) {
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
    if (ia) { xa = (int)fax; ya = (int)fay; }
    if (ib && (fax != fbx || fay != fby)) { xb = (int)fbx; yb = (int)fby; }
    return true;
}

struct TileArgs {
    const double *xs, *ys, *ts;  // listed events, tile-major
    const float *rho;            // their frame-exit scales
    const float2 *xyf;           // their centred coordinates rounded to float
    const long long *start;
    const int2 *cnt;             // (home, all)
    const int4 *meta;
    const int4 *rows;
    const int *order;
    int n_order, groups, K;
    const double *lo, *hi, *den_lo, *den_hi;
    double cx, cy;
    int W, H, words;
    float cxs, cys, Kxy, Wf, Hf;  // tile_point / tile_pair constants (kernel parameters:
                                  // read as constant-bank operands, no registers)
    unsigned int *ctr;
    unsigned long long *fi_out, *marks_s;
};

// One work item's state the out-of-line exact path needs.
struct TileItem {
    const double *xs, *ys, *ts;
    long long e0;
    int n_home;
    double lo, hi, dlo, dhi;   // this lane's interval
    double cx, cy;
    int W, H;
    TileView view;
};

// The exact path (reference arithmetic) for the last `take` uncertain pairs
// queued in q.ev: lanes take one pair each; fully_inside of home events into
// s_fi; multi-pixel segments queued and drained 32 at a time.  Returns the
// new queued-segment count.
__device__ __noinline__ int tile_exact(TileQueue &q, int nx, int take, int nq,
                                       const TileItem &it, unsigned long long *s_fi)
{
    const int lane = threadIdx.x & 31;
    const int code = lane < take ? q.ev[nx - take + lane] : -1;
    __syncwarp();
    const int j = code >= 0 ? (code & 31) : 0;
    const double lo_j = __shfl_sync(0xffffffffu, it.lo, j);
    const double hi_j = __shfl_sync(0xffffffffu, it.hi, j);
    const double dlo_j = __shfl_sync(0xffffffffu, it.dlo, j);
    const double dhi_j = __shfl_sync(0xffffffffu, it.dhi, j);
    TileSink sj = it.view.sink(j);
    SegDesc d;
    int c = 0, mk = 0;
    if (code >= 0) {
        const int el = code >> 5;
        const long long e = it.e0 + el;
        const double x = __ldg(it.xs + e), y = __ldg(it.ys + e), tt = __ldg(it.ts + e);
        const Warped wa = warp_event(x, y, tt, lo_j, dlo_j, it.cx, it.cy);
        const Warped wb = warp_event(x, y, tt, hi_j, dhi_j, it.cx, it.cy);
        if (el < it.n_home && fully_inside(wa.x, wa.y, wb.x, wb.y, it.W, it.H))
            atomicAdd(s_fi + j, 1ull);
        c = build_segment(wa.x, wa.y, wb.x, wb.y, it.W, it.H, 16, d, sj, mk);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, c > 0);
    if (c > 0) {
        const int slot = nq + __popc(bal & ((1u << lane) - 1u));
        EVD_CHECK(slot < 64);
        q.d[slot] = d;
        q.jj[slot] = (unsigned char)j;
    }
    nq += __popc(bal);
    if (nq >= 32) {
        __syncwarp();
        tile_drain(q, nq, it.W, it.H, it.view);
        nq = 0;
    }
    return nq;
}

// One endpoint warp of the filtered path: position, certification margin,
// certified cell (code) and the cell's local index in the tile (or -1).
// code = (fy + 2) << 16 | (fx + 2) when the exact position lies surely
// strictly inside cell (fx, fy) with -2 <= fx, fy <= 32000, else kFar.
constexpr unsigned kFar = 0xffffffffu;

// One endpoint of the filtered path in fp32.  The scale s = (1 + nu t) *
// RN(1 / den) is formed in binary64 (within 4.4e-16 |s| of the reference's
// RN((1 + nu t) / den): three roundings each), then the position in fp32,
// shifted by +8 px so every cell a certified point can touch has a positive
// index: X = RN32(RN32(xc) * RN32(s) + (cx + 8)), one FMA.  Against the
// reference's binary64 x' = RN(cx + RN(xc * s)):
//   |X - 8 - x'| <= |xc s| (2^-24 + 2^-24 + 2^-48 + 4.4e-16)   (RN32 of xc, s)
//                 + 2^-24 |X|                                  (the FMA)
//                 + 2^-53 (|xc s| + |x'|)                      (the reference)
//               <= 1.81e-7 |X| + 1.2e-7 (cx + 8) + 1e-12       (|xc s| <= |X| + cx + 8)
// so m = 1.9e-7 |X| + K, K = 1.25e-7 (c + 8) + 1e-9 (one fmaf; its own
// rounding is inside the 1.9 / 1.81 slack) bounds the error.  A coordinate is
// certified strictly inside its cell when 1 <= X <= 32000 and its fraction
// f = X - floor(X) (exact: Sterbenz) has f > m and f < 1 - 2m (RN32(1 - 2m)
// errs by <= 2^-25 < m since m >= 1.9e-7).
struct TilePoint {
    unsigned code;   // (iy + 8) << 16 | (ix + 8) of the certified cell, or kFar
    int l;           // its local pixel in the tile, or -1
    int out;         // certainly beyond the left / right / top / bottom edge (bits 0-3);
                     // bit 4: the certified cell is in the frame
};

// The hot path below is written branch-free (selects, non-short-circuit
// predicates, predicated shared REDs): the ALU pipe, not fp64, bounds the
// kernel (ncu), and every short-circuit branch costs a reconvergence pair.

// Local pixel of in-frame cell (x, y) in the tile, or -1 (not owned).  rows
// of an empty tile are never read (its items are never scheduled).
__device__ __forceinline__ int tile_local(const TileView &v, int x, int y, bool ok)
{
    const int r = y - v.y0;
    ok = ok & ((unsigned)r < (unsigned)v.nrows);
    const int rc = ok ? r : 0;
    int e0, e1, e2, e3;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3)
                 : "r"(v.rows + 16u * (unsigned)rc));
    const int xl = e0 & 0xffff, xh = (int)((unsigned)e0 >> 16);
    const int xl2 = e2 & 0xffff, xh2 = (int)((unsigned)e2 >> 16);
    const bool in1 = (x >= xl) & (x <= xh), in2 = (x >= xl2) & (x <= xh2);
    const int l = in1 ? e1 + x - xl : (in2 ? e3 + x - xl2 : -1);
    return ok ? l : -1;
}

// red.shared of pixel l's u16 counter when `on`
__device__ __forceinline__ void tile_mark(unsigned img, int l, bool on)
{
    EVD_CHECK(!on || (l >= 0 && l < 2 * kTileMaxWords));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                 "@p red.shared.add.u32 [%0], %1;\n\t}" ::"r"(img + 4u * (unsigned)(l >> 1)),
                 "r"(1u << ((l & 1) << 4)), "r"((unsigned)on)
                 : "memory");
}

__device__ __forceinline__ bool sure_frac(float X, float m)
{
    const float f = X - floorf(X);
    return (X >= 1.0f) & (X <= 32000.0f) & (f > m) & (f < 1.0f - 2.0f * m);
}

__device__ __forceinline__ TilePoint tile_point(float xf, float yf, double t, double nu,
                                                double rden, float cxs, float cys, float K,
                                                float Wf, float Hf, int W, int H,
                                                const TileView &v)
{
    TilePoint p;
    const float s = __double2float_rn(dmul(dadd(1.0, dmul(nu, t)), rden));
    const float X = fmaf(xf, s, cxs), Y = fmaf(yf, s, cys);
    const float mag = fmaxf(fabsf(X), fabsf(Y));
    const float m = fmaf(mag, 1.9e-7f, K);
    // Beyond an edge by the error bound plus 1e-3 px, which also covers the
    // reference's clip rounding, (|ax| + |bx|) 2^-50 < 1e-4 px while the
    // endpoints stay below 1e11 px (else no bit); the comparisons' own fp32
    // rounding near W + 8 is < 1.2e-4 px.
    const bool small = mag < 1e11f;
    p.out = (small & (X + m < 7.999f) ? 1 : 0) | (small & (X - m > Wf + 8.001f) ? 2 : 0) |
            (small & (Y + m < 7.999f) ? 4 : 0) | (small & (Y - m > Hf + 8.001f) ? 8 : 0);
    const bool sure = sure_frac(X, m) & sure_frac(Y, m);
    const int ix = sure ? (int)X : 0, iy = sure ? (int)Y : 0;  // shifted cell, >= 1
    p.code = sure ? (((unsigned)iy << 16) | (unsigned)ix) : kFar;
    const bool in = sure & (ix >= 8) & (ix < W + 8) & (iy >= 8) & (iy < H + 8);
    p.l = tile_local(v, ix - 8, iy - 8, in);
    p.out |= in ? 16 : 0;
    return p;
}

__device__ __forceinline__ bool code_in_frame(unsigned c, int W, int H)
{
    const int fx = (int)(c & 0xffffu) - 8, fy = (int)(c >> 16) - 8;
    return (fx >= 0) & (fx < W) & (fy >= 0) & (fy < H);
}

// Certified outcome of the segment a -> b (sure_segment_adj, evd_device.cuh,
// from the points' certified cells): false if uncertain; else (when `on`)
// marks the tile's pixels among the end cells and sets inside.  Off the
// frame: both endpoints beyond one edge (their `out` bits).
__device__ __forceinline__ bool tile_pair(const TilePoint &a, const TilePoint &b, int W, int H,
                                          unsigned img, bool on, int &inside)
{
    const bool off = (a.out & b.out & 15) != 0;
    // equal or edge-adjacent cells: codes differ by 0, +-1 or +-2^16 (both
    // halves of a certified code are in [1, 32000], so no borrow crosses)
    const unsigned u = a.code - b.code + 65536u;
    const bool adj = (u == 0u) | (u == 131072u) | (u - 65535u <= 2u);
    const bool cells = (a.code != kFar) & (b.code != kFar) & adj;
    const bool sure = off | cells;
    const bool mark = on & !off & cells;
    inside = (mark & ((a.out & b.out & 16) != 0)) ? 1 : 0;
    tile_mark(img, a.l, mark & (a.l >= 0));
    tile_mark(img, b.l, mark & (b.l >= 0) & (b.code != a.code));
    return sure;
}

// CONTIG: the intervals are contiguous (lo[k+1] == hi[k]); a group is 31
// intervals, lane j warps the event once at lo of its interval (lane 31 at hi
// of the last) and takes its segment's far end from lane j + 1.  Otherwise a
// group is 32 intervals and each lane warps the event at both ends.
template <bool CONTIG>
__global__ void __launch_bounds__(kTileThreads, 1) k_frontier_tiles(TileArgs a)
{
    constexpr int GS = CONTIG ? 31 : 32;
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned int *img = reinterpret_cast<unsigned int *>(smem);
    const int words = a.words;
    TileQueue *queues = reinterpret_cast<TileQueue *>(smem + 32 * (size_t)words * 4);
    int4 *rows = reinterpret_cast<int4 *>(queues + kTileWarps);
    __shared__ unsigned long long s_fi[32];
    __shared__ int s_item;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    TileQueue &wq = queues[warp];
    for (int i = threadIdx.x; i < 32 * words; i += blockDim.x) img[i] = 0u;
    const int W = a.W, H = a.H;
    const double cx = a.cx, cy = a.cy;
    const long long items = (long long)a.n_order * a.groups;
    const unsigned img_s = (unsigned)__cvta_generic_to_shared(img);
    const unsigned rows_s = (unsigned)__cvta_generic_to_shared(rows);
    for (;;) {
        if (threadIdx.x == 0) s_item = (int)atomicAdd(a.ctr, 1u);
        if (threadIdx.x < 32) s_fi[threadIdx.x] = 0ull;
        __syncthreads();
        const long long item = s_item;
        if (item >= items) break;
        const int tile = a.order[item / a.groups], g = (int)(item % a.groups);
        const int4 m = a.meta[tile];
        for (int i = threadIdx.x; i < m.y; i += blockDim.x) rows[i] = a.rows[m.z + i];
        __syncthreads();
        TileItem it;
        it.view = TileView{img_s, rows_s, m.x, m.y, words};
        it.xs = a.xs;
        it.ys = a.ys;
        it.ts = a.ts;
        it.e0 = a.start[tile];
        const int2 cn = a.cnt[tile];
        it.n_home = cn.x;
        it.cx = cx;
        it.cy = cy;
        it.W = W;
        it.H = H;
        // lane j evaluates interval g*GS + j
        const int k = g * GS + lane;
        const bool valid = lane < GS && k < a.K;
        const int kc = valid ? k : a.K - 1;
        it.lo = __ldg(a.lo + kc);
        it.hi = __ldg(a.hi + kc);
        it.dlo = __ldg(a.den_lo + kc);
        it.dhi = __ldg(a.den_hi + kc);
        // velocities this lane warps at: CONTIG: lo of its interval, or hi of
        // the interval before (the group's last point); else lo and hi
        double nu_a = it.lo, rden_a = ddiv(1.0, it.dlo);
        double nu_b = it.hi, rden_b = ddiv(1.0, it.dhi);
        bool has_pt = valid;
        if (CONTIG && !valid && k <= a.K && lane > 0) {
            // the point after the last valid interval (its hi)
            nu_a = __ldg(a.hi + k - 1);
            rden_a = ddiv(1.0, __ldg(a.den_hi + k - 1));
            has_pt = true;
        }
        // Whole-group rejection: the scale s(nu, t) = (1 + nu t) / (1 + nu tau)
        // decreases in nu (ds/dnu = (t - tau) / den^2 <= 0), so every endpoint
        // of the group's segments lies at scale >= s(hmax, t) along the
        // event's ray; beyond the frame-exit scale rho (+1.5 px) no sample of
        // any of them can touch an in-frame pixel (and none is fully inside).
        // Relative errors here are ~1e-15, the slack 1e-9; rounding in the
        // reference's clip is < 1e-3 px while |x'| < 1e12 (kappa).
        double hmax = has_pt ? (CONTIG ? nu_a : nu_b) : -INFINITY;
        double rhmax = CONTIG ? rden_a : rden_b;
        double smax = has_pt ? rden_a : 0.0;  // s(lo, 0) = 1 / den(lo): the largest scale
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double h2 = __shfl_xor_sync(0xffffffffu, hmax, o);
            const double r2 = __shfl_xor_sync(0xffffffffu, rhmax, o);
            if (h2 > hmax || (h2 == hmax && r2 > rhmax)) { hmax = h2; rhmax = r2; }
            smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
        }
        const double kappa = smax * (hypot(cx, cy) + 1.5) * 1e-12;
        const unsigned my_img = it.view.img + 4u * (unsigned)(lane * words);
        const float cxs = a.cxs, cys = a.cys, Kxy = a.Kxy, Wf = a.Wf, Hf = a.Hf;
        unsigned long long fi = 0;
        int nq = 0, nx = 0;  // queued segments / uncertain pairs (warp-uniform)
        // Events in chunks of 32: lane l loads event l of the chunk (coalesced),
        // tests the whole-group rejection for it, and the warp then walks only
        // the surviving events, broadcasting each from its lane.
        for (int c0 = warp * 32; c0 < cn.y; c0 += kTileWarps * 32) {
            const int el_l = c0 + lane;
            double tl = 0.0;
            float2 xyl = make_float2(0.0f, 0.0f);
            bool need = false;
            if (el_l < cn.y) {
                const long long e = it.e0 + el_l;
                tl = __ldg(a.ts + e);
                xyl = __ldg(a.xyf + e);
                const double rho = (double)__ldg(a.rho + e);
                const double smin = dmul(dadd(1.0, dmul(hmax, tl)), rhmax);
                need = !(smin > rho * (1.0 + 1e-9) && rho > kappa);
            }
            unsigned todo = __ballot_sync(0xffffffffu, need);
            while (todo) {
                const int i = __ffs(todo) - 1;
                todo &= todo - 1;
                const int el = c0 + i;
                const float x = __shfl_sync(0xffffffffu, xyl.x, i);
                const float y = __shfl_sync(0xffffffffu, xyl.y, i);
                const double tt = __shfl_sync(0xffffffffu, tl, i);
                TilePoint pa = tile_point(x, y, tt, nu_a, rden_a, cxs, cys, Kxy, Wf, Hf, W, H,
                                          it.view);
                TilePoint pb;
                if (CONTIG) {
                    pb.code = __shfl_down_sync(0xffffffffu, pa.code, 1);
                    pb.l = __shfl_down_sync(0xffffffffu, pa.l, 1);
                    pb.out = __shfl_down_sync(0xffffffffu, pa.out, 1);
                } else {
                    pb = tile_point(x, y, tt, nu_b, rden_b, cxs, cys, Kxy, Wf, Hf, W, H, it.view);
                }
                int ins;
                const bool sure = tile_pair(pa, pb, W, H, my_img, valid, ins);
                const bool unc = valid & !sure;
                fi += (el < cn.x) ? ins : 0;
                const unsigned bu = __ballot_sync(0xffffffffu, unc);
                if (unc) wq.ev[nx + __popc(bu & ((1u << lane) - 1u))] = (el << 5) | lane;
                nx += __popc(bu);
                if (nx >= 32) {
                    __syncwarp();
                    nq = tile_exact(wq, nx, 32, nq, it, s_fi);
                    nx -= 32;
                }
            }
        }
        while (nx > 0) {
            __syncwarp();
            const int take = nx < 32 ? nx : 32;
            nq = tile_exact(wq, nx, take, nq, it, s_fi);
            nx -= take;
        }
        if (nq > 0) {
            __syncwarp();
            tile_drain(wq, nq, W, H, it.view);
        }
        if (valid && fi) atomicAdd(s_fi + lane, fi);
        __syncthreads();
        // sum(H), sum(H^2) of each interval's tile image, leaving it zeroed
        const int nw = (m.w + 1) >> 1;
        for (int j = warp; j < GS; j += kTileWarps) {
            unsigned int *im = img + j * words;
            unsigned long long s1 = 0, s2 = 0;
            for (int w = lane; w < nw; w += 32) {
                const unsigned int v = im[w];
                if (v) {
                    const unsigned long long h0 = v & 0xffffu, h1 = v >> 16;
                    s1 += h0 + h1;
                    s2 += h0 * h0 + h1 * h1;
                    im[w] = 0u;
                }
            }
            s1 = warp_sum(s1);
            s2 = warp_sum(s2);
            const int kk = g * GS + j;
            if (lane == 0 && kk < a.K) {
                if (s1) {
                    atomicAdd(a.marks_s + 2 * kk, s1);
                    atomicAdd(a.marks_s + 2 * kk + 1, s2);
                }
                if (s_fi[j]) atomicAdd(a.fi_out + kk, s_fi[j]);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- host entry points
static int tile_capacity(int device, int max_rows_guess)
{
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const long long static_bytes = 32 * 8 + 16;  // s_fi, s_item
    const long long avail = optin - static_bytes - (long long)max_rows_guess * sizeof(int4) -
                            (long long)kTileWarps * sizeof(TileQueue);
    long long words = avail / (32 * 4);
    if (!(words & 1)) words--;
    const long long P = (words - 1) * 2;  // tile_words(P) = P/2 | 1 <= words
    return P > 64 ? (int)(P / 64 * 64) : 0;
}

cudaError_t tiles_bin(FrontierTiles *f, const double *xc, const double *yc, const double *t,
                      long long n, int W, int H, unsigned long long gen, bool *usable,
                      int *launches, cudaStream_t s)
{
    *usable = false;
    int dev = 0;
    cudaGetDevice(&dev);
    if (f->W != W || f->H != H) {
        f->plan_ok = false;
        f->gen = ~0ull;
        const int P = tile_capacity(dev, H);
        f->plan_ok = P > 0 && build_plan(*f, W, H, P);
        if (f->plan_ok) {
            f->W = W;
            f->H = H;
        } else {
            f->W = W;  // remember the failure for this frame
            f->H = H;
        }
    }
    if (!f->plan_ok) return cudaSuccess;
    if (f->gen == gen) {
        *usable = f->bin_ok;
        return cudaSuccess;
    }
    const int T = 1 + f->S;
    cudaError_t e;
    if ((e = ensure(f->cnt, f->cnt_cap, T)) || (e = ensure(f->start, f->start_cap, T)) ||
        (e = ensure(f->cursor, f->cursor_cap, 2 * (size_t)T)) ||
        (e = ensure(f->flag, f->flag_cap, 1)) || (e = ensure(f->order, f->order_cap, T)) ||
        (e = ensure(f->ctr, f->ctr_cap, 1)))
        return e;
    const TileGeom g{f->ang, f->S, f->Rc, f->Rw};
    cudaMemsetAsync(f->cnt, 0, T * sizeof(int2), s);
    cudaMemsetAsync(f->flag, 0, sizeof(unsigned int), s);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 4ll * sms));
    if (n > 0) {
        k_tile_count<<<blocks, 256, 2 * T * sizeof(int), s>>>(xc, yc, t, n, g, T, f->cnt, f->flag);
        (*launches)++;
    }
    f->h_cnt.resize(T);
    unsigned int flag = 0;
    if ((e = cudaMemcpyAsync(f->h_cnt.data(), f->cnt, T * sizeof(int2), cudaMemcpyDeviceToHost, s)) ||
        (e = cudaMemcpyAsync(&flag, f->flag, sizeof flag, cudaMemcpyDeviceToHost, s)) ||
        (e = cudaStreamSynchronize(s)))
        return e;
    f->gen = gen;
    f->bin_ok = false;
    if (flag) return cudaSuccess;  // non-finite events: global path
    std::vector<long long> start(T);
    std::vector<unsigned long long> cur(2 * (size_t)T);
    long long total = 0;
    std::vector<int> order;
    for (int k = 0; k < T; k++) {
        const int2 c = f->h_cnt[k];
        const long long all = (long long)c.x + c.y;
        if (all > kTileMaxEvents) return cudaSuccess;  // u16 counters could overflow
        f->h_cnt[k].y = (int)all;
        start[k] = total;
        cur[2 * k] = total;
        cur[2 * k + 1] = total + c.x;
        total += all;
        if (all > 0 && f->h_meta[k].w > 0) order.push_back(k);
    }
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return f->h_cnt[a].y > f->h_cnt[b].y; });
    if ((e = ensure(f->xs, f->xs_cap, total)) || (e = ensure(f->ys, f->ys_cap, total)) ||
        (e = ensure(f->ts, f->ts_cap, total)) || (e = ensure(f->rho, f->rho_cap, total)) ||
        (e = ensure(f->xyf, f->xyf_cap, total)))
        return e;
    if ((e = cudaMemcpyAsync(f->start, start.data(), T * sizeof(long long), cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(f->cnt, f->h_cnt.data(), T * sizeof(int2), cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(f->cursor, cur.data(), cur.size() * sizeof(unsigned long long),
                             cudaMemcpyHostToDevice, s)) ||
        (!order.empty() && (e = cudaMemcpyAsync(f->order, order.data(), order.size() * sizeof(int),
                                                cudaMemcpyHostToDevice, s))))
        return e;
    if (n > 0) {
        k_tile_fill<<<blocks, 256, 0, s>>>(xc, yc, t, n, g, W / 2.0, H / 2.0, f->cursor, f->xs,
                                           f->ys, f->ts, f->rho, f->xyf);
        (*launches)++;
    }
    if ((e = cudaStreamSynchronize(s))) return e;  // host vectors above are freed on return
    f->total = total;
    f->n_order = (int)order.size();
    f->bin_ok = true;
    *usable = true;
    return cudaGetLastError();
}

cudaError_t tiles_eval(FrontierTiles *f, const double *lo, const double *hi, const double *dlo,
                       const double *dhi, int K, bool contig, unsigned long long *fi_out,
                       unsigned long long *marks_s, int *launches, cudaStream_t s)
{
    if (f->n_order == 0 || K == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = tile_smem_bytes(f->P, f->max_rows);
    auto kern = contig ? k_frontier_tiles<true> : k_frontier_tiles<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e) return e;
    TileArgs a;
    a.xs = f->xs;
    a.ys = f->ys;
    a.ts = f->ts;
    a.rho = f->rho;
    a.xyf = f->xyf;
    a.start = f->start;
    a.cnt = f->cnt;
    a.meta = f->meta;
    a.rows = f->rows;
    a.order = f->order;
    a.n_order = f->n_order;
    a.groups = contig ? (K + 30) / 31 : (K + 31) / 32;
    a.K = K;
    a.lo = lo;
    a.hi = hi;
    a.den_lo = dlo;
    a.den_hi = dhi;
    a.cx = f->W / 2.0;
    a.cy = f->H / 2.0;
    a.W = f->W;
    a.H = f->H;
    a.cxs = (float)(a.cx + 8.0);  // exact: multiples of 1/2 below 2^23
    a.cys = (float)(a.cy + 8.0);
    a.Kxy = 1.25e-7f * std::max(a.cxs, a.cys) + 1e-9f;
    a.Wf = (float)f->W;
    a.Hf = (float)f->H;
    a.words = tile_words(f->P);
    a.ctr = f->ctr;
    a.fi_out = fi_out;
    a.marks_s = marks_s;
    if ((e = cudaMemsetAsync(f->ctr, 0, sizeof(unsigned int), s))) return e;
    const long long items = (long long)f->n_order * a.groups;
    const int grid = (int)std::min<long long>(sms, items);
    kern<<<grid, kTileThreads, smem, s>>>(a);
    (*launches)++;
    return cudaGetLastError();
}

void tiles_info(const FrontierTiles *f, long long *out)
{
    out[0] = f->plan_ok ? 1 + f->S : 0;
    out[1] = f->P;
    out[2] = f->bin_ok ? f->total : -1;
    out[3] = f->n_order;
}

}  // namespace evd

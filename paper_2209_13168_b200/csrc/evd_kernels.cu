// evd_kernels.cu -- sm_100a kernels of the BnB bound-evaluation hot path.
//
// Standalone kernels back the per-call entry points (accumulate_image,
// upper_bound_image, bound_terms, image_contrast, rasterize_segment,
// radial_warp); k_solve is the device-resident branch and bound
// (solver.py:79-123) that evaluates one node per grid-wide step.
#include <cfloat>
#include <cstdlib>
#include <atomic>
#include <climits>

#include "evd_device.cuh"
#include "evd_internal.h"

namespace evd {

// Compiled only into the diagnostic build (EVD_TRACE_BUILD, libevd_trace.so):
// the probes cost instruction-cache footprint in the per-node fixed phases.
#ifdef EVD_TRACE_BUILD
constexpr bool kTraceBuild = true;
#else
constexpr bool kTraceBuild = false;
#endif
constexpr int kThreads = 256;
#ifndef EVD_SOLVE_THREADS
#define EVD_SOLVE_THREADS 512
#define EVD_SOLVE_MINB 1
#endif
constexpr int kSolveThreads = EVD_SOLVE_THREADS;
#ifndef EVD_CHUNK
#define EVD_CHUNK 16
#endif
constexpr int kChunk = EVD_CHUNK;
// Chunk size of the 768-thread build (windows from 250 k events): 24 was best
// while every chunk paid a merge-path search (cfg 3 18.10 -> 17.96 ms vs 16);
// with continuing cursors (warp_drain) 16 is: cfg 3 15.79 -> 15.58 ms, cfg 5
// 125.4 -> 124.2 ms (12: 15.65 / 125.1, 8: 16.09 / 129.6, 32: 16.04 ms).  At
// 384 / 512 threads 16 stays (12: cfg 1 0.748 -> 0.755 ms, cfg 2 2.99 ->
// 2.98 ms).  Chunk size only moves the seams, never the marks.
#ifndef EVD_CHUNK_LARGE
#define EVD_CHUNK_LARGE 16
#endif
#ifndef EVD_DRAIN_CONT
#define EVD_DRAIN_CONT 1
#endif
#ifndef EVD_DRAIN_RELOAD
#define EVD_DRAIN_RELOAD 1
#endif
#ifndef EVD_DRAIN_CONT_MAXNT
#define EVD_DRAIN_CONT_MAXNT 1024
#endif
constexpr int chunk_for(int nt) { return nt >= 768 ? EVD_CHUNK_LARGE : kChunk; }
// warp_drain's continuing cursors (EVD_DRAIN_CONT; the segment re-read from
// shared memory each round, EVD_DRAIN_RELOAD): cfg 1 0.758 -> 0.748 ms, cfg 2
// 3.038 -> 2.985 ms, cfg 3 15.80 -> 15.77 ms, cfg 5 128.8 -> 125.6 ms; the
// cfg-2 root-width event pass 147 -> 128 us (tools/probe_events.py).  Kept
// per CTA size (EVD_DRAIN_CONT_MAXNT) for A/B.
template <int NT>
constexpr bool drain_cont() { return EVD_DRAIN_CONT && NT <= EVD_DRAIN_CONT_MAXNT; }
#ifndef EVD_PIX_CUT_THREADS
#define EVD_PIX_CUT_THREADS 128
#endif
// pixel phase: threads walking the point image's cut (the rest sum the
// segment images), by CTA size: 256 of 768 measured best for large windows
template <int NT>
constexpr int pix_cut_threads() { return NT >= 768 ? 2 * EVD_PIX_CUT_THREADS : EVD_PIX_CUT_THREADS; }
#ifndef EVD_BATCH_DIV
#define EVD_BATCH_DIV 1
#endif
#ifndef EVD_GUIDED_WIDTH
#define EVD_GUIDED_WIDTH (1.0 / 2)
#endif
constexpr double kGuidedWidth = EVD_GUIDED_WIDTH;  // nodes wider than this claim guided batches
constexpr double kFilterWidth = 1.0 / 64;  // node widths that try the filtered path

// SM count of the current device (contexts on several devices may share a
// process, one host thread each)
static int num_sms()
{
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

static int event_blocks(long long n)
{
    long long b = (n + kThreads - 1) / kThreads;
    const long long cap = (long long)num_sms() * 8;
    if (b > cap) b = cap;
    return b < 1 ? 1 : (int)b;
}

// Pixel increments are fire-and-forget L2 reductions.  The pointer reaches
// the sampler through shared memory (WarpQueue::img), where the compiler can
// no longer prove it global and emits a generic, value-returning ATOM; the
// explicit red.global keeps every mark a RED.
struct AtomicSink {
    unsigned int *img;
    __device__ __forceinline__ void operator()(long long p, int, int) const
    {
#ifdef EVD_NO_RED  // timing experiment only (profiles/no_red_ab_r02.txt): WRONG images
        if (p == -12345) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(img + p));
#else
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(img + p));
#endif
    }
};

// Per-warp queue of built segments: lane l owns slots 2l, 2l+1.
struct WarpQueue {
    long long ev[64];       // uncertain events awaiting the exact path
    SegDesc d[64];
    unsigned int *img[64];  // image each queued segment marks
    int off[65];  // exclusive prefix of chunk counts (per lane, or per slot for warp_drain_list)
    int na[32];   // chunks of the lane's first segment
};

// Build one segment and queue it in the lane's shared-memory slot for
// warp_drain (single-pixel and off-frame segments finish in build_segment).
// Returns the number of queued chunks.  Every multi-pixel segment is queued:
// a lane sampling its own short segment diverges from the others, and the
// extra sampler copy costs registers and I-cache (measured slower).
template <int C = kChunk>
__device__ __forceinline__ int segment_or_queue_inl(double ax, double ay, double bx, double by,
                                                    int W, int H, WarpQueue &q, int slot,
                                                    AtomicSink &sink, int &marks)
{
    SegDesc d;
    const int c = build_segment(ax, ay, bx, by, W, H, C, d, sink, marks);
    if (c == 0) return 0;
    EVD_CHECK(slot >= 0 && slot < 64);
    q.d[slot] = d;
    q.img[slot] = sink.img;
    return c;
}

// Out-of-line copy for the solve kernel, whose event loop calls it for both
// child segments: one copy keeps the hot loop inside the instruction cache.
// Plain-value interface (image pointer in, chunks | marks << 16 out): a
// reference to the caller's sink or mark counter would live in local memory.
template <int C = kChunk>
__device__ __noinline__ int segment_or_queue_ool(double ax, double ay, double bx, double by,
                                                 int W, int H, WarpQueue &q, int slot,
                                                 unsigned int *img)
{
    AtomicSink sink{img};
    int marks = 0;
    const int c = segment_or_queue_inl<C>(ax, ay, bx, by, W, H, q, slot, sink, marks);
    return c | (marks << 16);  // chunks <= (W + H + 4) / C < 2^16 (check_frame), marks <= 2
}
template <int C = kChunk>
__device__ __forceinline__ int segment_or_queue(double ax, double ay, double bx, double by, int W,
                                                int H, WarpQueue &q, int slot,
                                                const AtomicSink &sink, int &marks)
{
    const int r = segment_or_queue_ool<C>(ax, ay, bx, by, W, H, q, slot, sink.img);
    marks += r >> 16;
    return r & 0xffff;
}

// Sample every chunk the warp queued, in rounds of 32: all lanes position
// their cursors together, then step one item per iteration; chunks hold
// nearly equal item counts, so the lanes stay converged.
template <bool CONT = EVD_DRAIN_CONT>
__device__ __noinline__ int warp_drain(WarpQueue &q, int cA, int cB, int W, int H)
{
    const int lane = threadIdx.x & 31;
    int incl = cA + cB;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    q.off[lane + 1] = incl;
    if (lane == 0) q.off[0] = 0;
    q.na[lane] = cA;
    __syncwarp();
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int marks = 0;
    if (CONT) {
    // Lane l takes chunks l*R .. l*R + R-1, one per round: consecutive chunks
    // of a segment stay on one lane, whose cursor simply runs on (the state a
    // chunk's last step leaves is the state cursor_init would compute for the
    // next: same items, same lookahead, prev = the last midpoint's range), so
    // only a lane's first chunk of each segment pays the merge-path search.
    const int R = (total + 31) >> 5;
    int pslot = -1, pj = -1;
    Cursor c;
    SegDesc d;
    AtomicSink sink{nullptr};
    for (int r = 0; r < R; r++) {
        const int t = lane * R + r;
        bool active = false;
        if (t < total) {
            int L = 0;  // largest lane with off[L] <= t
#pragma unroll
            for (int s = 16; s > 0; s >>= 1)
                if (q.off[L + s] <= t) L += s;
            const int rr = t - q.off[L];
            const bool second = rr >= q.na[L];
            const int slot = 2 * L + (second ? 1 : 0), j = second ? rr - q.na[L] : rr;
            if (slot == pslot && j == pj + 1) {
#if EVD_DRAIN_RELOAD
                d = q.d[slot];  // not live across rounds
#endif
                const int N = d.X.n + d.Y.n + 2, m0 = j * d.csize;
                c.left = N - m0 < d.csize ? N - m0 : d.csize;
                c.fin = c.kind == 0 ? 1 : 0;  // the chunk holds only the trailing sample
                active = true;
            } else {
                d = q.d[slot];
                sink.img = q.img[slot];
                active = cursor_init(d, j, c);
            }
            pslot = slot;
            pj = j;
        }
        const bool live = active;
        if (active) active = cursor_head(d, c, W, H, sink, marks);
        while (__any_sync(0xffffffffu, active))
            if (active) active = cursor_step(d, c, W, H, sink, marks);
        if (live) cursor_tail(d, c, W, H, sink, marks);
    }
    } else {
    for (int base = 0; base < total; base += 32) {
        const int t = base + lane;
        bool active = false;
        int slot = 0;
        Cursor c;
        AtomicSink sink{nullptr};
        if (t < total) {
            int L = 0;  // largest lane with off[L] <= t
#pragma unroll
            for (int s = 16; s > 0; s >>= 1)
                if (q.off[L + s] <= t) L += s;
            const int r = t - q.off[L];
            const bool second = r >= q.na[L];
            slot = 2 * L + (second ? 1 : 0);
            sink.img = q.img[slot];
            active = cursor_init(q.d[slot], second ? r - q.na[L] : r, c);
        }
        const SegDesc d = q.d[slot];  // in registers for the walk
        const bool live = active;
        if (active) active = cursor_head(d, c, W, H, sink, marks);
        while (__any_sync(0xffffffffu, active))
            if (active) active = cursor_step(d, c, W, H, sink, marks);
        if (live) cursor_tail(d, c, W, H, sink, marks);
    }
    }
    __syncwarp();
    return marks;
}

// Sample the nq (< 64) segments pooled in slots [0, nq), in rounds of 32
// chunks.  Callers pool segments over several events and drain once 32 are
// waiting, so rounds run with full lanes.
__device__ __noinline__ int warp_drain_list(WarpQueue &q, int nq, int W, int H)
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
        AtomicSink sink{nullptr};
        if (t < total) {
            int L = 0;  // largest slot with off[L] <= t (empty slots share offsets)
#pragma unroll
            for (int s = 32; s > 0; s >>= 1)
                if (L + s < 64 && q.off[L + s] <= t) L += s;
            slot = L;
            sink.img = q.img[slot];
            active = cursor_init(q.d[slot], t - q.off[L], c);
        }
        const SegDesc d = q.d[slot];
        const bool live = active;
        if (active) active = cursor_head(d, c, W, H, sink, marks);
        while (__any_sync(0xffffffffu, active))
            if (active) active = cursor_step(d, c, W, H, sink, marks);
        if (live) cursor_tail(d, c, W, H, sink, marks);
    }
    __syncwarp();
    return marks;
}

// ---------------------------------------------------------------- elementwise
__global__ void k_center(const double *__restrict__ x, const double *__restrict__ y, long long n,
                         double cx, double cy, double *__restrict__ xc, double *__restrict__ yc)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        xc[i] = dsub(x[i], cx);  // the reference's (x - cx), geometry.py:87
        yc[i] = dsub(y[i], cy);
    }
}

__global__ void k_warp(const double *__restrict__ xc, const double *__restrict__ yc,
                       const double *__restrict__ t, long long n, double nu, double den,
                       double cx, double cy, double *__restrict__ xo, double *__restrict__ yo)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const Warped w = warp_event(xc[i], yc[i], t[i], nu, den, cx, cy);
        xo[i] = w.x;
        yo[i] = w.y;
    }
}

// warp_scale (geometry.py:70-75): s = (1 + nu*t) / denom
__global__ void k_scale(const double *__restrict__ t, long long n, double nu, double den,
                        double *__restrict__ s)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        s[i] = ddiv(dadd(1.0, dmul(nu, t[i])), den);
}

// accumulate_image (contrast.py:48-58): acc[0] += in-image events
__global__ void k_point_image(const double *__restrict__ xc, const double *__restrict__ yc,
                              const double *__restrict__ t, long long n, double nu, double den,
                              double cx, double cy, int W, int H, unsigned int *img,
                              unsigned long long *acc)
{
    unsigned long long v[1] = {0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const Warped w = warp_event(__ldg(xc + i), __ldg(yc + i), __ldg(t + i), nu, den, cx, cy);
        const long long p = floor_bin(w.x, w.y, W, H);
        if (p >= 0) {
            atomicAdd(img + p, 1u);
            v[0]++;
        }
    }
    block_add_u64<1>(v, acc);
}

// _bound_image_kernel (contrast.py:185-203) on warps at lo/hi, long segments
// spread over the warp: acc[0] += fully-inside segments, acc[1] += marks
__global__ void __launch_bounds__(kThreads) k_bound_image(
    const double *__restrict__ xc, const double *__restrict__ yc, const double *__restrict__ t,
    long long n, double lo, double den_lo, double hi, double den_hi, double cx, double cy, int W,
    int H, unsigned int *img, unsigned long long *acc)
{
    extern __shared__ __align__(16) unsigned char smem[];
    WarpQueue &wq = reinterpret_cast<WarpQueue *>(smem)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    unsigned long long v[2] = {0, 0};
    AtomicSink sink{img};
    const long long gsz = (long long)gridDim.x * blockDim.x;
    for (long long base = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); base < n;
         base += gsz) {
        const long long i = base + lane;
        int c = 0, marks = 0;
        if (i < n) {
            const double x = __ldg(xc + i), y = __ldg(yc + i), tt = __ldg(t + i);
            const Warped a = warp_event(x, y, tt, lo, den_lo, cx, cy);
            const Warped b = warp_event(x, y, tt, hi, den_hi, cx, cy);
            v[0] += fully_inside(a.x, a.y, b.x, b.y, W, H);
            c = segment_or_queue(a.x, a.y, b.x, b.y, W, H, wq, 2 * lane, sink, marks);
        }
        if (__any_sync(0xffffffffu, c != 0)) marks += warp_drain(wq, c, 0, W, H);
        v[1] += marks;
    }
    block_add_u64<2>(v, acc);
}

// ---------------------------------------------------------------- batched frontier
// bound_terms (contrast.py:241-251) for K intervals in one launch.  Lane j of
// a warp owns interval k0 + j of a group of 32 consecutive intervals and the
// warp walks events one at a time: every lane evaluates the same event (a
// broadcast load) at its own interval, so the 32 segments are neighbours along
// one trajectory and take the same branches.  An interval whose lower
// endpoint is its left neighbour's upper endpoint takes that warp by shuffle.
// Per-interval fully_inside / marks stay in registers; blocks are ordered
// group-major so a group's 32 images stay in L2 while it is in flight.
constexpr int kFrontGroup = 32;
#ifndef EVD_FRONT_BPG
#define EVD_FRONT_BPG 4  // event blocks per interval group, per SM
#endif

__global__ void __launch_bounds__(kThreads) k_frontier(
    const double *__restrict__ xc, const double *__restrict__ yc, const double *__restrict__ t,
    long long n, const double *__restrict__ lo, const double *__restrict__ hi,
    const double *__restrict__ den_lo, const double *__restrict__ den_hi, int K, double cx,
    double cy, int W, int H, unsigned int *images, long long M, int bpg,
    unsigned long long *fi_out)
{
    extern __shared__ __align__(16) unsigned char smem[];
    WarpQueue &wq = reinterpret_cast<WarpQueue *>(smem)[threadIdx.x >> 5];
    __shared__ unsigned long long s_fi[kFrontGroup];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int g = blockIdx.x / bpg, tb = blockIdx.x % bpg;
    const int k = g * kFrontGroup + lane;
    const bool valid = k < K;
    const int kc = valid ? k : K - 1;
    const double my_lo = __ldg(lo + kc), my_hi = __ldg(hi + kc);
    const double my_dlo = __ldg(den_lo + kc), my_dhi = __ldg(den_hi + kc);
    const double left_hi = __shfl_up_sync(0xffffffffu, my_hi, 1);
    const bool shared_lo = lane > 0 && my_lo == left_hi;
    unsigned int *img = images + (long long)kc * M;
    AtomicSink sink{img};
    if (threadIdx.x < kFrontGroup) s_fi[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long fi = 0;
    int nq = 0;  // segments pooled in wq (warp-uniform)
    const long long gw = (long long)tb * wpb + warp, nw = (long long)bpg * wpb;
    for (long long e = gw; e < n; e += nw) {
        const double x = __ldg(xc + e), y = __ldg(yc + e), tt = __ldg(t + e);
        const Warped b = warp_event(x, y, tt, my_hi, my_dhi, cx, cy);
        Warped a;
        a.x = __shfl_up_sync(0xffffffffu, b.x, 1);
        a.y = __shfl_up_sync(0xffffffffu, b.y, 1);
        if (!shared_lo) a = warp_event(x, y, tt, my_lo, my_dlo, cx, cy);
        // pool multi-pixel segments over events; drain 32+ at a time
        SegDesc d;
        int c = 0, m = 0;
        if (valid) {
            fi += fully_inside(a.x, a.y, b.x, b.y, W, H);
            c = build_segment(a.x, a.y, b.x, b.y, W, H, kChunk, d, sink, m);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, c > 0);
        if (c > 0) {
            const int slot = nq + __popc(bal & ((1u << lane) - 1u));
            EVD_CHECK(slot < 64);
            wq.d[slot] = d;
            wq.img[slot] = img;
        }
        nq += __popc(bal);
        if (nq >= 32) {
            __syncwarp();
            warp_drain_list(wq, nq, W, H);
            nq = 0;
        }
    }
    if (nq > 0) {
        __syncwarp();
        warp_drain_list(wq, nq, W, H);
    }
    if (valid && fi) atomicAdd(s_fi + lane, fi);
    __syncthreads();
    if (threadIdx.x < kFrontGroup && g * kFrontGroup + (int)threadIdx.x < K) {
        const int kk = g * kFrontGroup + threadIdx.x;
        if (s_fi[threadIdx.x]) atomicAdd(fi_out + kk, s_fi[threadIdx.x]);
    }
}

// k_frontier with a filtered first pass: each (event, interval) segment is
// warped with one multiplication by RN(1/den) and certified against a rounding
// margin (sure_segment: off-frame, or both endpoints surely in one pixel);
// the rest -- segments near pixel edges or crossing them -- are queued per
// warp as (event, interval) pairs and take the exact path 32 at a time with
// full lanes.  Same images and counts as k_frontier (every certified result
// is what the exact arithmetic gives).
__global__ void __launch_bounds__(kThreads) k_frontier_f(
    const double *__restrict__ xc, const double *__restrict__ yc, const double *__restrict__ t,
    long long n, const double *__restrict__ lo, const double *__restrict__ hi,
    const double *__restrict__ den_lo, const double *__restrict__ den_hi, int K, double cx,
    double cy, int W, int H, unsigned int *images, long long M, int bpg,
    unsigned long long *fi_out)
{
    extern __shared__ __align__(16) unsigned char smem[];
    WarpQueue &wq = reinterpret_cast<WarpQueue *>(smem)[threadIdx.x >> 5];
    __shared__ unsigned long long s_fi[kFrontGroup];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int g = blockIdx.x / bpg, tb = blockIdx.x % bpg;
    const int k = g * kFrontGroup + lane;
    const bool valid = k < K;
    const int kc = valid ? k : K - 1;
    const double my_lo = __ldg(lo + kc), my_hi = __ldg(hi + kc);
    const double my_dlo = __ldg(den_lo + kc), my_dhi = __ldg(den_hi + kc);
    const double my_rlo = ddiv(1.0, my_dlo), my_rhi = ddiv(1.0, my_dhi);
    const double left_hi = __shfl_up_sync(0xffffffffu, my_hi, 1);
    const bool shared_lo = lane > 0 && my_lo == left_hi;
    unsigned int *img = images + (long long)kc * M;
    AtomicSink sink{img};
    if (threadIdx.x < kFrontGroup) s_fi[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long fi = 0;
    int nq = 0;  // segments pooled in wq.d (warp-uniform)
    int nx = 0;  // uncertain (event, interval) pairs queued in wq.ev (warp-uniform)
    // the exact path for the last `take` queued pairs, with full lanes
    auto exact_batch = [&](int take) {
        const long long code = lane < take ? wq.ev[nx - take + lane] : -1;
        nx -= take;
        __syncwarp();
        const int j = code >= 0 ? (int)(code & 31) : 0;
        const double lo_j = __shfl_sync(0xffffffffu, my_lo, j);
        const double hi_j = __shfl_sync(0xffffffffu, my_hi, j);
        const double dlo_j = __shfl_sync(0xffffffffu, my_dlo, j);
        const double dhi_j = __shfl_sync(0xffffffffu, my_dhi, j);
        AtomicSink sj{images + (long long)(g * kFrontGroup + j) * M};
        SegDesc d;
        int c = 0, m = 0;
        if (code >= 0) {
            const long long e = code >> 5;
            const double x = __ldg(xc + e), y = __ldg(yc + e), tt = __ldg(t + e);
            const Warped a = warp_event(x, y, tt, lo_j, dlo_j, cx, cy);
            const Warped b = warp_event(x, y, tt, hi_j, dhi_j, cx, cy);
            const int ins = fully_inside(a.x, a.y, b.x, b.y, W, H);
            if (ins) atomicAdd(s_fi + j, (unsigned long long)ins);
            c = build_segment(a.x, a.y, b.x, b.y, W, H, kChunk, d, sj, m);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, c > 0);
        if (c > 0) {
            const int slot = nq + __popc(bal & ((1u << lane) - 1u));
            EVD_CHECK(slot < 64);
            wq.d[slot] = d;
            wq.img[slot] = sj.img;
        }
        nq += __popc(bal);
        if (nq >= 32) {
            __syncwarp();
            warp_drain_list(wq, nq, W, H);
            nq = 0;
        }
    };
    const long long gw = (long long)tb * wpb + warp, nw = (long long)bpg * wpb;
    for (long long e = gw; e < n; e += nw) {
        const double x = __ldg(xc + e), y = __ldg(yc + e), tt = __ldg(t + e);
        const Warped bq = warp_approx(x, y, tt, my_hi, my_rhi, cx, cy);
        const double mb = sure_margin(bq, cx, cy);
        Warped aq;
        aq.x = __shfl_up_sync(0xffffffffu, bq.x, 1);
        aq.y = __shfl_up_sync(0xffffffffu, bq.y, 1);
        double ma = __shfl_up_sync(0xffffffffu, mb, 1);
        if (!shared_lo) {
            aq = warp_approx(x, y, tt, my_lo, my_rlo, cx, cy);
            ma = sure_margin(aq, cx, cy);
        }
        bool unc = false;
        if (valid) {
            long long pix, pix2;
            int ins;
            if (sure_segment_adj(aq, bq, ma, mb, W, H, pix, pix2, ins)) {
                EVD_CHECK(pix < M && pix2 < M);
                if (pix >= 0) sink(pix, 0, 0);
                if (pix2 >= 0) sink(pix2, 0, 0);
                fi += ins;
            } else {
                unc = true;
            }
        }
        const unsigned bu = __ballot_sync(0xffffffffu, unc);
        if (unc) wq.ev[nx + __popc(bu & ((1u << lane) - 1u))] = e * 32 + lane;
        nx += __popc(bu);
        if (nx >= 32) {
            __syncwarp();
            exact_batch(32);
        }
    }
    while (nx > 0) {
        __syncwarp();
        exact_batch(nx < 32 ? nx : 32);
    }
    if (nq > 0) {
        __syncwarp();
        warp_drain_list(wq, nq, W, H);
    }
    if (valid && fi) atomicAdd(s_fi + lane, fi);
    __syncthreads();
    if (threadIdx.x < kFrontGroup && g * kFrontGroup + (int)threadIdx.x < K) {
        const int kk = g * kFrontGroup + threadIdx.x;
        if (s_fi[threadIdx.x]) atomicAdd(fi_out + kk, s_fi[threadIdx.x]);
    }
}

// marks = sum(H_bar) (upper_bound_image().in_image_events) and S_bar =
// sum(H_bar^2) per interval image (exact u64), leaving the images zeroed.
// marks_s points at [marks_k, s_bar_k] pairs.
__global__ void k_frontier_sums(unsigned int *images, long long M, int bpi,
                                unsigned long long *marks_s)
{
    const int k = blockIdx.x / bpi, part = blockIdx.x % bpi;
    unsigned int *img = images + (long long)k * M;
    unsigned long long v[2] = {0, 0};
    for (long long p = part * (long long)blockDim.x + threadIdx.x; p < M;
         p += (long long)bpi * blockDim.x) {
        const unsigned long long h = __ldcs(img + p);
        if (h) {
            v[0] += h;
            v[1] += h * h;
            img[p] = 0u;
        }
    }
    block_add_u64<2>(v, marks_s + 2 * k);
}

// acc[0] += sum(img), acc[1] += sum(img^2) -- exact integers (contrast.py:238,249)
__global__ void k_image_sums(const unsigned int *__restrict__ img, long long m,
                             unsigned long long *acc)
{
    unsigned long long v[2] = {0, 0};
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < m;
         p += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h = img[p];
        v[0] += h;
        v[1] += h * h;
    }
    block_add_u64<2>(v, acc);
}

// rasterize_segment (contrast.py:206-222) for k segments, one thread each
// (all chunks of size `chunk` in order): counts[j*M + p] is incremented once
// per mark, so a dedup failure would show as 2.
__global__ void k_raster_segments(const double *__restrict__ segs, int k, int W, int H,
                                  int chunk, unsigned int *counts)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    unsigned int *img = counts + (long long)j * W * H;
    auto sink = [img](long long p, int, int) { img[p] += 1u; };
    raster_segment(segs[4 * j], segs[4 * j + 1], segs[4 * j + 2], segs[4 * j + 3], W, H, chunk,
                   sink);
}

// ---------------------------------------------------------------- contrast tree
// Summands of image_contrast (contrast.py:64): (H_p - mu)**2 (numpy square).
struct SqU32 {
    typedef unsigned int raw;
    const unsigned int *img;
    double mu;
    __device__ __forceinline__ raw load(int i) const { return __ldcg(img + i); }
    __device__ __forceinline__ void clear(int) const {}
    __device__ __forceinline__ double term(raw h) const
    {
        const double d = dsub((double)h, mu);
        return dmul(d, d);
    }
};
struct SqU32Clear : SqU32 {  // and leave the pixel zeroed for the next BnB node
    __device__ __forceinline__ void clear(int i) const { const_cast<unsigned int *>(img)[i] = 0u; }
};
struct SqF64 {
    typedef double raw;
    const double *img;
    double mu;
    __device__ __forceinline__ raw load(int i) const { return __ldcg(img + i); }
    __device__ __forceinline__ void clear(int) const {}
    __device__ __forceinline__ double term(raw c) const
    {
        const double d = dsub(c, mu);
        return dmul(d, d);
    }
};

// Evaluate cut subtree c of the pairwise tree with threads [0, nt) of the
// block (a warp multiple) synchronised by `bar`; returns the subtree sum to
// every participating thread.
struct BlockBar {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct NamedBar {  // hardware barrier `id` over the first `nt` threads
    int id, nt;
    __device__ __forceinline__ void operator()() const
    {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory");
    }
};
__device__ __forceinline__ void bclock(const SolveArgs &a, long long it, int k);
template <class Q, class Bar = BlockBar>
__device__ double eval_cut(const TreeDev &T, int c, const Q &q, double *loc,
                           const SolveArgs &dbg_a, long long dbg_it, int nt = -1,
                           const Bar &bar = Bar{})
{
    if (kTraceBuild && dbg_a.btrace) bclock(dbg_a, dbg_it, 19);
    if (nt < 0) nt = blockDim.x;
    const int l0 = T.cut_leaf0[c], nl = T.cut_leaf0[c + 1] - l0;
    const int j = threadIdx.x & 7, ngroups = nt >> 3;
    if (kTraceBuild && dbg_a.btrace) {
        asm volatile("" ::"r"(nl));
        bclock(dbg_a, dbg_it, 16);
    }
    for (int i = threadIdx.x >> 3; i < nl; i += ngroups) {
        const int2 lf = T.leaves[l0 + i];
        if (dbg_a.btrace && i == 0) {
            asm volatile("" ::"r"(lf.x), "r"(lf.y));
            bclock(dbg_a, dbg_it, 17);
        }
        const double v = pairwise_leaf8(lf.x, lf.y, j, q);
        if (dbg_a.btrace && i == 0) {
            asm volatile("" ::"d"(v));
            bclock(dbg_a, dbg_it, 18);
        }
        if (j == 0) loc[i] = v;
    }
    if (kTraceBuild && dbg_a.btrace) bclock(dbg_a, dbg_it, 14);
    bar();
    if (kTraceBuild && dbg_a.btrace) bclock(dbg_a, dbg_it, 15);
    const int t0 = T.cut_trip0[c], ni = T.cut_trip0[c + 1] - t0;
    const int *lvl = T.cut_lvl + (long long)c * (kMaxLevels + 1);
    const int nlev = T.cut_nlev[c];
    if (ni <= nt) {
        // one internal node per thread, loaded once; its level is in .w
        const int4 tr = threadIdx.x < ni ? T.trip[t0 + threadIdx.x] : make_int4(0, 0, 0, -1);
        for (int h = 0; h < nlev; h++) {
            if (tr.w == h) loc[tr.x] = dadd(loc[tr.y], loc[tr.z]);
            bar();
        }
    } else {
        for (int h = 0; h < nlev; h++) {
            for (int k = lvl[h] + threadIdx.x; k < lvl[h + 1]; k += nt) {
                const int4 tr = T.trip[t0 + k];
                loc[tr.x] = dadd(loc[tr.y], loc[tr.z]);
            }
            bar();
        }
    }
    const double r = loc[ni > 0 ? nl + ni - 1 : 0];
    bar();
    return r;
}

// Combine the C cut sums through the top of the tree with one block.
__device__ double eval_top(const TreeDev &T, double *v)
{
    for (int i = threadIdx.x; i < T.C; i += blockDim.x) v[i] = __ldcg(T.cutval + i);
    __syncthreads();
    for (int h = 0; h < T.top_levels; h++) {
        for (int k = T.top_lvl[h] + threadIdx.x; k < T.top_lvl[h + 1]; k += blockDim.x) {
            const int4 tr = T.top[k];
            v[tr.x] = dadd(v[tr.y], v[tr.z]);
        }
        __syncthreads();
    }
    const double r = v[T.top_root];
    __syncthreads();
    return r;
}

__global__ void k_contrast_cuts_u32(const unsigned int *img, const unsigned long long *in_image,
                                    TreeDev T)
{
    __shared__ double loc[kCutSmem];
    const double mu = ddiv((double)*in_image, (double)T.M);  // EventImage.mean, contrast.py:35-36
    const double r = eval_cut(T, blockIdx.x, SqU32{img, mu}, loc, SolveArgs{}, 0);
    if (threadIdx.x == 0) T.cutval[blockIdx.x] = r;
}

// ---------------------------------------------------------------- batched points
// accumulate_image + image_contrast (contrast.py:48-64) at K velocities in one
// pass: lane j of a warp bins every event at velocity k0 + j (a broadcast load
// of the event), blocks ordered group-major like k_frontier.  The contrast of
// every image then follows from one cut-block per (image, cut) and one top
// block per image; the images are left zeroed.
__global__ void __launch_bounds__(kThreads) k_points_multi(
    const double *__restrict__ xc, const double *__restrict__ yc, const double *__restrict__ t,
    long long n, const double *__restrict__ nus, const double *__restrict__ dens, int K, double cx,
    double cy, int W, int H, unsigned int *images, long long M, int bpg,
    unsigned long long *in_out)
{
    __shared__ unsigned long long s_in[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int g = blockIdx.x / bpg, tb = blockIdx.x % bpg;
    const int k = g * 32 + lane;
    const bool valid = k < K;
    const int kc = valid ? k : K - 1;
    const double nu = __ldg(nus + kc), den = __ldg(dens + kc);
    unsigned int *img = images + (long long)kc * M;
    if (threadIdx.x < 32) s_in[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long inside = 0;
    const long long gw = (long long)tb * wpb + warp, nw = (long long)bpg * wpb;
    for (long long e = gw; e < n; e += nw) {
        const Warped w = warp_event(__ldg(xc + e), __ldg(yc + e), __ldg(t + e), nu, den, cx, cy);
        const long long p = floor_bin(w.x, w.y, W, H);
        if (valid && p >= 0) {
            atomicAdd(img + p, 1u);
            inside++;
        }
    }
    if (valid && inside) atomicAdd(s_in + lane, inside);
    __syncthreads();
    if (threadIdx.x < 32 && g * 32 + (int)threadIdx.x < K && s_in[threadIdx.x])
        atomicAdd(in_out + g * 32 + threadIdx.x, s_in[threadIdx.x]);
}

__global__ void k_contrast_cuts_multi(unsigned int *images, const unsigned long long *in_image,
                                      TreeDev T, double *cutvals)
{
    __shared__ double loc[kCutSmem];
    const int k = blockIdx.x / T.C, c = blockIdx.x % T.C;
    const double mu = ddiv((double)in_image[k], (double)T.M);
    const double r = eval_cut(T, c, SqU32Clear{{images + (long long)k * T.M, mu}}, loc,
                              SolveArgs{}, 0);
    if (threadIdx.x == 0) cutvals[(long long)k * T.C + c] = r;
}

__global__ void k_contrast_top_multi(TreeDev T, const double *cutvals, double *out)
{
    __shared__ double v[kCutSmem];
    const int k = blockIdx.x;
    for (int i = threadIdx.x; i < T.C; i += blockDim.x) v[i] = cutvals[(long long)k * T.C + i];
    __syncthreads();
    for (int h = 0; h < T.top_levels; h++) {
        for (int j = T.top_lvl[h] + threadIdx.x; j < T.top_lvl[h + 1]; j += blockDim.x) {
            const int4 tr = T.top[j];
            v[tr.x] = dadd(v[tr.y], v[tr.z]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = ddiv(dadd(0.0, v[T.top_root]), (double)T.M);
}

__global__ void k_contrast_cuts_f64(const double *img, double mu, TreeDev T)
{
    __shared__ double loc[kCutSmem];
    const double r = eval_cut(T, blockIdx.x, SqF64{img, mu}, loc, SolveArgs{}, 0);
    if (threadIdx.x == 0) T.cutval[blockIdx.x] = r;
}

// C = np.sum(q) / M, np.sum starting from 0.0 (contrast.py:64)
__global__ void k_contrast_top(TreeDev T, double *out)
{
    __shared__ double v[kCutSmem];
    const double s = eval_top(T, v);
    if (threadIdx.x == 0) *out = ddiv(dadd(0.0, s), (double)T.M);
}

// ---------------------------------------------------------------- BnB solve
// The solve is a replicated state machine: every block holds the same BnB
// control state (Replica, shared memory) and, after the grid barrier that
// completes a node's pixel reductions, every block computes the identical
// (deterministic) next step itself -- no serial leader, no release round.
// Global memory carries only what must be shared: images, per-node integer
// accumulators (double-buffered by parity), the cut sums of the contrast tree,
// and the frontier, whose writes block 0 commits one phase later (after the
// next barrier) so no block can still be reading the entries it replaces.

__device__ __forceinline__ long long globaltimer()
{
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Solve trace (globaltimer ns): trace[0] = kernel start, then kTraceSlots per
// node evaluation i (0 = root) at 1 + kTraceSlots*i + slot, see TraceSlot.
__device__ __forceinline__ void trace_point(const SolveArgs &a, long long it, int slot)
{
    if (!kTraceBuild) return;
    if (!a.trace || threadIdx.x != 0) return;
    if (slot < 0) a.trace[0] = globaltimer();
    else if (it < a.trace_iters) a.trace[1 + kTraceSlots * it + slot] = globaltimer();
}
__device__ __forceinline__ void trace_max(const SolveArgs &a, long long it, int slot)
{
    if (!kTraceBuild) return;
    if (!a.trace || threadIdx.x != 0 || it >= a.trace_iters) return;
    atomicMax(reinterpret_cast<unsigned long long *>(a.trace + 1 + kTraceSlots * it + slot),
              (unsigned long long)globaltimer());
}

__device__ __forceinline__ void btrace_point(const SolveArgs &a, long long it, int k)
{
    if (!kTraceBuild) return;
    if (!a.btrace || threadIdx.x != 0 || it >= kBTraceIters) return;
    a.btrace[(it * a.group_blocks + blockIdx.x) * kBTraceSlots + k] = globaltimer();
}
// sub-phase markers (SM cycles) in slots 4.. of the block trace
__device__ __forceinline__ void bclock(const SolveArgs &a, long long it, int k)
{
    if (!kTraceBuild) return;
    if (!a.btrace || threadIdx.x != 0 || it >= kBTraceIters) return;
    a.btrace[(it * a.group_blocks + blockIdx.x) * kBTraceSlots + k] = clock64();
}

// Barrier over a solver group of `blocks` CTAs on a monotone 64-bit arrival
// counter (no reset round trip): the n-th barrier completes when the counter
// reaches n * blocks.
__device__ __forceinline__ void grid_sync(unsigned long long *ctr, unsigned long long &target,
                                          int blocks)
{
    target += blocks;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// Overlapped upload: the group of window w waits (thread 0 of each CTA)
// until the copy stream has delivered the window's raw events, then gathers
// them into the solve layout with k_gather_windows' arithmetic (centred x, y;
// stream windows: t - start capped at tau, events.py:348; window lists: t as
// given, evd_set_events_list).  The raw stream is
// read through L2 (__ldcg: written by the copy engine during this kernel);
// the gathered region is read by the group only after the grid barrier that
// follows, and no other window shares its cache lines (padded offsets).
__device__ __noinline__ void gather_window(const SolveArgs &a, int w, long long off, long long n,
                                           int gb, int GB)
{
    const long long lo = a.s_lo[w];
    if (threadIdx.x == 0) {
        const unsigned long long need = (unsigned long long)(lo + n);
        const long long t0 = globaltimer();
        unsigned long long v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.ready) : "memory");
            if (v >= need) break;
            if (globaltimer() - t0 > kUploadTimeoutNs) {
                atomicExch(a.stall, 1u);
                break;
            }
            __nanosleep(500);
        }
    }
    __syncthreads();
    const double start = dmul((double)(a.k0 + w), a.tau);
    for (long long j = (long long)gb * blockDim.x + threadIdx.x; j < n;
         j += (long long)GB * blockDim.x) {
        const long long i = lo + j;
        a.gx[off + j] = dsub(__ldcg(a.sx + i), a.cx);
        a.gy[off + j] = dsub(__ldcg(a.sy + i), a.cy);
        const double tr = __ldcg(a.stt + i), d = dsub(tr, start);
        a.gt[off + j] = a.t_local ? tr : (d < a.tau ? d : a.tau);
    }
}

// One node's events on the exact path (k_solve's event phase; also timed
// alone by k_event_probe): every event, three warps (lo, centre, hi); point
// image at the centre, segment images of both children (root: of the root),
// segments sampled warp-cooperatively by warp_drain.  First round static, then
// warps take batches of 32 events from the node's work counter (acc[7]) so
// CTAs finish together.
struct EventJob {
    const double *xc, *yc, *tw;
    long long n;
    double lo, c, hi, den_lo, den_c, den_hi, cx, cy;
    int W, H;
    unsigned int *P, *A, *B;
    int mode;
    unsigned long long *acc;
    long long gsz;
    int gb;
    int guided;  // shrink claims as the counter runs out (wide nodes)
    // kModeRootCert: [0] += root_cells_lb, [1] += fully_inside of the root
    // segment (the root bound's certificate, k_solve_spec)
    unsigned long long *acc_root;
};

template <int C = kChunk, bool CONT = EVD_DRAIN_CONT>
__device__ __forceinline__ void event_pass_exact(const EventJob &j, WarpQueue &wq,
                                                 unsigned long long (&v)[4],
                                                 unsigned long long (&vex)[1])
{
    const int lane = threadIdx.x & 31, W = j.W, H = j.H;
    const double *xc = j.xc, *yc = j.yc, *tw = j.tw;
    const long long n = j.n, gsz = j.gsz;
    unsigned int *P = j.P;
    unsigned long long *acc = j.acc;
    AtomicSink sa{j.A}, sb{j.B};
    // One static batch of 32 events per warp, then batches from the node's
    // work counter.  Narrow nodes take batches of 32 (the pass is latency-
    // bound, a few batches per warp; claiming more at once was measured
    // slower, tools/probe_events.py).  Wide nodes, where one batch can hold
    // tens of microseconds of sampling, shrink their claims as the counter
    // runs out (guided self-scheduling, down to 4 events) so the warps finish
    // together; the sampler still spreads a small batch's chunks over all
    // 32 lanes.
    const long long warps = gsz >> 5;
    // batches of up to 32 events, fewer when the window cannot give every warp
    // one full batch: a small window is latency-bound, and more, shorter
    // batches keep all warps busy (cfg 1: 20k events on 2368 warps)
    unsigned long long rc0 = 0, rc1 = 0;  // kModeRootCert
    long long fb = n / (EVD_BATCH_DIV * warps);
    const int first = (int)(fb < 4 ? 4 : (fb > 32 ? 32 : fb));
    long long base = (j.gb * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5)) * first;
    int size = first;
    // (tried and measured slower, kept out: the next batch claimed and staged
    // into shared memory with cp.async while a batch is worked on, and the
    // first pass consuming batches as their upload chunks arrive -- DESIGN.md
    // §7, commits ce05e17 and 0d7c49a)
    while (base < n) {
        const long long i = base + lane;
        int cA = 0, cB = 0, dummy = 0;
        if (lane < size && i < n) {
            const double x = __ldg(xc + i), y = __ldg(yc + i), t = __ldg(tw + i);
            const Warped wl = warp_event(x, y, t, j.lo, j.den_lo, j.cx, j.cy);
            const Warped wc = warp_event(x, y, t, j.c, j.den_c, j.cx, j.cy);
            const Warped wh = warp_event(x, y, t, j.hi, j.den_hi, j.cx, j.cy);
            const long long p = floor_bin(wc.x, wc.y, W, H);
            if (p >= 0) {
                atomicAdd(P + p, 1u);
                v[0]++;
            }
            if (j.mode == kModeRoot) {
                v[1] += fully_inside(wl.x, wl.y, wh.x, wh.y, W, H);
                cA = segment_or_queue<C>(wl.x, wl.y, wh.x, wh.y, W, H, wq, 2 * lane, sa, dummy);
            } else {
                if (j.mode == kModeRootCert) {
                    rc0 += root_cells_lb(wl.x, wl.y, wh.x, wh.y, W, H);
                    rc1 += fully_inside(wl.x, wl.y, wh.x, wh.y, W, H);
                }
                v[1] += fully_inside(wl.x, wl.y, wc.x, wc.y, W, H);
                cA = segment_or_queue<C>(wl.x, wl.y, wc.x, wc.y, W, H, wq, 2 * lane, sa, dummy);
                v[2] += fully_inside(wc.x, wc.y, wh.x, wh.y, W, H);
                cB = segment_or_queue<C>(wc.x, wc.y, wh.x, wh.y, W, H, wq, 2 * lane + 1, sb, dummy);
            }
            vex[0]++;
        }
        if (__any_sync(0xffffffffu, (cA | cB) != 0)) dummy += warp_drain<CONT>(wq, cA, cB, W, H);
        v[3] += dummy;
        if (j.guided) {
            // claim size from the remaining events as last seen by this warp
            const long long rem = n - base;
            long long s = rem / (2 * warps);
            size = (int)(s < 4 ? 4 : (s > first ? first : s));
        }
        long long nb = 0;
        if (lane == 0) nb = warps * first + (long long)atomicAdd(acc + 7, (unsigned long long)size);
        base = __shfl_sync(0xffffffffu, nb, 0);
    }
    if (j.mode == kModeRootCert) {
        rc0 = warp_sum(rc0);
        rc1 = warp_sum(rc1);
        if (lane == 0) {
            if (rc0) atomicAdd(j.acc_root, rc0);
            if (rc1) atomicAdd(j.acc_root + 1, rc1);
        }
    }
}

// Diagnostics: the exact event pass of one child-node evaluation, timed alone
// (reps launches' worth in one kernel, each rep with its own work counter and
// scratch images; globaltimer span per rep in span[2*r], span[2*r+1]).
__global__ void __launch_bounds__(kSolveThreads, EVD_SOLVE_MINB)
    k_event_probe(EventJob j, int reps, unsigned long long *ctrs, unsigned long long *span,
                  unsigned int *scratch, long long M)
{
    extern __shared__ __align__(16) unsigned char smem[];
    WarpQueue &wq = reinterpret_cast<WarpQueue *>(smem)[threadIdx.x >> 5];
    for (int r = 0; r < reps; r++) {
        EventJob jr = j;
        jr.acc = ctrs + 8 * r;
        jr.gb = blockIdx.x;
        jr.P = scratch + (long long)(r % 2) * 3 * M;
        jr.A = jr.P + M;
        jr.B = jr.A + M;
        unsigned long long v[4] = {0, 0, 0, 0}, vex[1] = {0};
        __syncthreads();
        if (threadIdx.x == 0) atomicMin(span + 2 * r, (unsigned long long)globaltimer());
        event_pass_exact(jr, wq, v, vex);
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(span + 2 * r + 1, (unsigned long long)globaltimer());
        if (v[3] == 0xffffffffffffull) span[0] = 0;  // keep the counts live
    }
}

__device__ __forceinline__ bool better(double b1, long long c1, double b2, long long c2)
{
    // heapq order on (-c_bar, counter): larger bound first, FIFO among ties
    return b1 > b2 || (b1 == b2 && c1 < c2);
}

// 32-byte frontier entries moved as two 16-byte L2 (.cg) accesses
__device__ __forceinline__ void entry_store(FrontierEntry *dst, const FrontierEntry &e)
{
    const double2 *src = reinterpret_cast<const double2 *>(&e);
    __stcg(reinterpret_cast<double2 *>(dst), src[0]);
    __stcg(reinterpret_cast<double2 *>(dst) + 1, src[1]);
}
__device__ __forceinline__ FrontierEntry entry_load(const FrontierEntry *src)
{
    FrontierEntry e;
    double2 *d = reinterpret_cast<double2 *>(&e);
    d[0] = __ldcg(reinterpret_cast<const double2 *>(src));
    d[1] = __ldcg(reinterpret_cast<const double2 *>(src) + 1);
    return e;
}

// BnB control state, identical in every block.
struct Replica {
    double lo, hi, c, den_lo, den_c, den_hi;  // node under evaluation
    double r_lo, r_c, r_hi;                   // RN(1 / den) for the filtered path
    double mu;                                // point-image mean of the node (pixel phase)
    int mode, done, status, parity;
    double nu_hat, c_hat, bound_gap;
    long long iterations, bound_evals, point_evals, next_counter, fr_n, max_fr;
    unsigned long long marks;  // pixel increments of all images over the solve
    unsigned long long exact;  // events that took the exact (uncertain) path
    // this node's integer accumulators and pow(fi/M, 2) table values
    unsigned long long fiA, fiB, sA, sB;
    double p2A, p2B;
    // frontier writes of the last step, committed by block 0 after the next barrier
    int n_pending;
    long long pend_idx[3];
    FrontierEntry pend[3];
    // entries pushed by the current step (indices fr_n_before + k)
    int n_pushed;
    FrontierEntry pushed[2];
    double root_L;  // kModeRootCert: certified lower bound of the root's c_bar
};

constexpr int kFrView = 1024;  // frontier entries staged in shared memory per step

__device__ __forceinline__ void replica_push(const SolveArgs &a, Replica &R, long long n0,
                                             double bound, double lo, double hi)
{
    if (n0 + R.n_pushed >= a.fr_cap) {
        R.status = kStatusCapacity;
        R.done = 1;
        return;
    }
    const FrontierEntry e{bound, R.next_counter++, lo, hi};
    R.pushed[R.n_pushed] = e;
    R.pend_idx[R.n_pending] = n0 + R.n_pushed;
    R.pend[R.n_pending] = e;
    R.n_pending++;
    R.n_pushed++;
}

// One BnB step (solver.py:102-119 from the centre evaluation on): incumbent
// update with >=, both child bounds assembled as contrast.py:248-251, pruning
// with >=, the iteration cap, then the best-first pop and stop test of the
// next iteration.  Whole block; identical in every block.  Frontier entries
// [0, fr_n) are in `view` when fr_n <= kFrView (else read from global).
template <bool FILTER>
__device__ void bnb_step(const SolveArgs &a, Replica &R, double S, const FrontierEntry *view,
                         FrontierEntry *fr)
{
    const long long n0 = R.fr_n;
    const bool staged = n0 <= kFrView;
    if (threadIdx.x == 0) {
        const double M = (double)a.tree.M;
        const double C = ddiv(dadd(0.0, S), M);  // np.sum(...) / M
        R.n_pending = 0;
        R.n_pushed = 0;
        R.point_evals++;
        bool node = R.mode == kModeNode;
        if (R.mode == kModeRoot) {
            R.c_hat = C;
            R.nu_hat = R.c;
            const double cb = dsub(ddiv((double)R.sA, M), R.p2A);
            R.bound_evals++;
            replica_push(a, R, n0, cb, R.lo, R.hi);
        } else if (R.mode == kModeRootCert) {
            // solver.py:92-108 with the root bound certified (k_solve_spec's
            // kModeRootCert): the root is pushed and popped at once, then
            // evaluated as a node from this step's results
            R.c_hat = C;
            R.nu_hat = R.c;
            R.point_evals++;
            R.bound_evals++;
            R.next_counter++;
            if (n0 + 1 > R.max_fr) R.max_fr = n0 + 1;
            if (!(R.root_L - C > a.gamma + 1e-9 * fabs(C))) {
                R.status = kStatusRootCert;
                R.done = 1;
            } else {
                R.iterations++;
                node = true;
            }
        }
        if (node) {
            if (C >= R.c_hat) {  // solver.py:111
                R.nu_hat = R.c;
                R.c_hat = C;
            }
            const double cbA = dsub(ddiv((double)R.sA, M), R.p2A);
            const double cbB = dsub(ddiv((double)R.sB, M), R.p2B);
            R.bound_evals += 2;
            if (cbA >= R.c_hat) replica_push(a, R, n0, cbA, R.lo, R.c);
            if (cbB >= R.c_hat && !R.done) replica_push(a, R, n0, cbB, R.c, R.hi);
            if (R.iterations >= a.max_iter && !R.done) {
                R.status = kStatusIterLimit;
                R.done = 1;
            }
        }
    }
    __syncthreads();
    if (R.done) return;
    const long long n1 = n0 + R.n_pushed;
    if (n1 == 0) {  // queue exhausted: every interval pruned (solver.py:121-122)
        __syncthreads();
        if (threadIdx.x == 0) R.done = 1;
        __syncthreads();
        return;
    }
    auto entry = [&](long long i) -> FrontierEntry {
        if (i >= n0) return R.pushed[i - n0];
        return staged ? view[i] : entry_load(fr + i);
    };
    // best-first pop: argmax over the committed entries and this step's pushes
    // (by warp 0 alone for a frontier of up to 256 entries: no cross-warp pass)
    const bool small = n1 <= 256;
    if (small && threadIdx.x >= 32) {
        __syncthreads();
        __syncthreads();
        return;
    }
    __shared__ double r_b[32];
    __shared__ long long r_c[32], r_i[32];
    double bb = -DBL_MAX;
    long long bc = LLONG_MAX, bi = -1;
    const int stride = small ? 32 : (int)blockDim.x;
    for (long long i = threadIdx.x; i < n1; i += stride) {
        double b;
        long long c;
        if (i >= n0) { b = R.pushed[i - n0].bound; c = R.pushed[i - n0].counter; }
        else if (staged) { b = view[i].bound; c = view[i].counter; }
        else { b = __ldcg(&fr[i].bound); c = __ldcg(&fr[i].counter); }
        if (bi < 0 || better(b, c, bb, bc)) { bb = b; bc = c; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, bb, o);
        const long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || better(ob, oc, bb, bc))) { bb = ob; bc = oc; bi = oi; }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (!small && lane == 0) { r_b[wid] = bb; r_c[wid] = bc; r_i[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; !small && w < (int)(blockDim.x >> 5); w++)
            if (r_i[w] >= 0 && (bi < 0 || better(r_b[w], r_c[w], bb, bc))) {
                bb = r_b[w]; bc = r_c[w]; bi = r_i[w];
            }
        const FrontierEntry top = entry(bi);
        const long long last = n1 - 1;
        if (bi != last) {  // swap-remove: the last entry takes the popped slot
            R.pend_idx[R.n_pending] = bi;
            R.pend[R.n_pending] = entry(last);
            R.n_pending++;
        }
        R.fr_n = n1 - 1;
        if (n1 > R.max_fr) R.max_fr = n1;
        R.iterations++;
        const double gap = dsub(bb, R.c_hat);  // -(-c_bar) - c_hat
        if (gap <= a.gamma || dsub(top.hi, top.lo) < a.min_width) {
            R.bound_gap = (0.0 > gap) ? 0.0 : gap;  // Python max(gap, 0.0)
            R.done = 1;
        } else {
            const double c = dmul(0.5, dadd(top.lo, top.hi));  // VelocityInterval.center
            R.lo = top.lo;
            R.hi = top.hi;
            R.c = c;
            R.den_lo = dadd(1.0, dmul(top.lo, a.tau));
            R.den_c = dadd(1.0, dmul(c, a.tau));
            R.den_hi = dadd(1.0, dmul(top.hi, a.tau));
            if (FILTER) {  // the filtered path's approximate warps
                R.r_lo = ddiv(1.0, R.den_lo);
                R.r_c = ddiv(1.0, R.den_c);
                R.r_hi = ddiv(1.0, R.den_hi);
            }
            R.mode = kModeNode;
        }
    }
    __syncthreads();
}

// Per-block shared-memory copy of the reduction-tree metadata this block
// touches (its own cuts, and the top): after every barrier the L1 is
// invalidated, so tables left in global memory would cost a dependent L2
// round trip per tree level.
constexpr int kCacheCuts = 8, kCacheLeaves = 1024, kCacheTrips = 1024, kCacheTop = 1024;
struct TreeCache {
    int2 leaves[kCacheLeaves];
    int4 trip[kCacheTrips];
    int4 top[kCacheTop];
    int cut_leaf0[kCacheCuts + 1], cut_trip0[kCacheCuts + 1], cut_nlev[kCacheCuts];
    int cut_lvl[kCacheCuts * (kMaxLevels + 1)];
    int top_lvl[kMaxLevels + 1];
};

// Returns a TreeDev whose cut index q means global cut gb + q*GB
// (local = true), or the global tables when they do not fit (local = false).
__device__ TreeDev cache_tree(const TreeDev &g, TreeCache &tc, bool &local, int gb, int GB)
{
    __shared__ int s_ok, s_nq;
    if (threadIdx.x == 0) {
        int nq = g.C > gb ? (g.C - 1 - gb) / GB + 1 : 0;
        int ok = nq <= kCacheCuts && g.top_lvl[g.top_levels] <= kCacheTop &&
                 g.top_levels <= kMaxLevels;
        int nl = 0, nt = 0;
        for (int q = 0; ok && q < nq; q++) {
            const int c = gb + q * GB;
            tc.cut_leaf0[q] = nl;
            tc.cut_trip0[q] = nt;
            nl += g.cut_leaf0[c + 1] - g.cut_leaf0[c];
            nt += g.cut_trip0[c + 1] - g.cut_trip0[c];
            tc.cut_nlev[q] = g.cut_nlev[c];
        }
        ok = ok && nl <= kCacheLeaves && nt <= kCacheTrips;
        tc.cut_leaf0[nq] = nl;
        tc.cut_trip0[nq] = nt;
        s_ok = ok;
        s_nq = nq;
    }
    __syncthreads();
    local = s_ok != 0;
    if (!local) return g;  // does not fit: read the global tables
    const int nq = s_nq;
    for (int q = 0; q < nq; q++) {
        const int c = gb + q * GB;
        const int l0 = g.cut_leaf0[c], nl = g.cut_leaf0[c + 1] - l0;
        const int t0 = g.cut_trip0[c], nt = g.cut_trip0[c + 1] - t0;
        for (int i = threadIdx.x; i < nl; i += blockDim.x) tc.leaves[tc.cut_leaf0[q] + i] = g.leaves[l0 + i];
        for (int i = threadIdx.x; i < nt; i += blockDim.x) tc.trip[tc.cut_trip0[q] + i] = g.trip[t0 + i];
        for (int i = threadIdx.x; i <= kMaxLevels; i += blockDim.x)
            tc.cut_lvl[q * (kMaxLevels + 1) + i] = g.cut_lvl[(long long)c * (kMaxLevels + 1) + i];
    }
    const int ntop = g.top_lvl[g.top_levels];
    for (int i = threadIdx.x; i < ntop; i += blockDim.x) tc.top[i] = g.top[i];
    for (int i = threadIdx.x; i <= g.top_levels; i += blockDim.x) tc.top_lvl[i] = g.top_lvl[i];
    __syncthreads();
    TreeDev t = g;
    t.leaves = tc.leaves;
    t.cut_leaf0 = tc.cut_leaf0;
    t.cut_trip0 = tc.cut_trip0;
    t.cut_lvl = tc.cut_lvl;
    t.cut_nlev = tc.cut_nlev;
    t.trip = tc.trip;
    t.top = tc.top;
    t.top_lvl = tc.top_lvl;
    return t;
}

// Combine the C cut sums (already staged in v) through the top of the tree.
__device__ double top_combine(const TreeDev &T, double *v)
{
    const int levels = T.top_levels, ntop = T.top_lvl[levels];
    if (ntop <= (int)blockDim.x) {
        // one internal node per thread, loaded once; its level is in .w
        const int4 tr = threadIdx.x < ntop ? T.top[threadIdx.x] : make_int4(0, 0, 0, -1);
        for (int h = 0; h < levels; h++) {
            if (tr.w == h) v[tr.x] = dadd(v[tr.y], v[tr.z]);
            __syncthreads();
        }
    } else {
        for (int h = 0; h < levels; h++) {
            for (int k = T.top_lvl[h] + threadIdx.x; k < T.top_lvl[h + 1]; k += blockDim.x) {
                const int4 tr = T.top[k];
                v[tr.x] = dadd(v[tr.y], v[tr.z]);
            }
            __syncthreads();
        }
    }
    const double r = v[T.top_root];
    __syncthreads();
    return r;
}

constexpr size_t kQueueBytes = sizeof(WarpQueue) * (kSolveThreads / 32);
constexpr size_t kStepBytes = kCutSmem * sizeof(double) + kFrView * sizeof(FrontierEntry);
// dynamic shared memory of the solve kernels at NT threads per CTA: region A
// (warp queues | cut scratch + frontier view), then the cached cut plan
template <int NT>
struct SolveSmem {
    static constexpr size_t queue = sizeof(WarpQueue) * (NT / 32);
    static constexpr size_t region_a = queue > kStepBytes ? queue : kStepBytes;
};

// FEED: the windows arrive during the launch (SolveArgs' overlapped upload);
// a separate instantiation so the resident-window kernels keep their code
template <bool FILTER, int NT, bool FEED = false>
__global__ void __launch_bounds__(NT, 1) k_solve(SolveArgs a_param)
{
    constexpr size_t kRegionA = SolveSmem<NT>::region_a;
    constexpr int kPixCutThreads = pix_cut_threads<NT>();
    extern __shared__ __align__(16) unsigned char smem[];
#ifdef EVD_ARGS_SMEM
    __shared__ SolveArgs a_s;
    if (threadIdx.x == 0) a_s = a_param;
    __syncthreads();
    const SolveArgs &a = a_s;
#else
    const SolveArgs &a = a_param;
#endif
    // region A: warp queues (event phase) | cut scratch + frontier view (pixels, step)
    WarpQueue &wq = reinterpret_cast<WarpQueue *>(smem)[threadIdx.x >> 5];
    double *scratch = reinterpret_cast<double *>(smem);
    FrontierEntry *view = reinterpret_cast<FrontierEntry *>(smem + kCutSmem * sizeof(double));
    TreeCache &tc = *reinterpret_cast<TreeCache *>(smem + kRegionA);
    __shared__ Replica R;
    // this CTA's solver group: an independent solver over group_blocks CTAs
    const int GB = a.group_blocks;
    const int grp = blockIdx.x / GB, gb = blockIdx.x % GB;
    if (grp >= a.groups) return;
    const bool tracer = kTraceBuild && grp == 0 && a.trace != nullptr;
    unsigned long long *ctr = a.bar + 2 * grp;
    unsigned long long target = 0;
    SolveState *st = a.st + grp;
    FrontierEntry *fr = a.fr + (long long)grp * a.fr_cap;
    const long long M = a.tree.M;
    unsigned int *P = a.img + (long long)grp * 3 * M, *A = P + M, *B = A + M;
    const int lane = threadIdx.x & 31;
    const long long gtid = gb * (long long)blockDim.x + threadIdx.x;
    const long long gsz = (long long)GB * blockDim.x;
    const int W = a.W, H = a.H;
    bool local_cuts;
    TreeDev gtree = a.tree;
    gtree.cutval = a.tree.cutval + (long long)grp * a.tree.C;
    // the plan's pointers live in shared memory: kept in registers they are
    // spilled, and reloading them through L1 after an event phase cost
    // several L2 round trips per node (measured ~4k cycles)
    __shared__ TreeDev tree_s;
    {
        const TreeDev t = cache_tree(gtree, tc, local_cuts, gb, GB);
        if (threadIdx.x == 0) tree_s = t;
        __syncthreads();
    }
    const TreeDev &tree = tree_s;
    if (tracer && gb == 0) trace_point(a, 0, -1);

    for (int w = grp; w < a.n_windows; w += a.groups) {
        const long long off = a.offsets[w], n = FEED ? a.counts[w] : a.offsets[w + 1] - off;
        if (n == 0) {
            if (gb == 0 && threadIdx.x == 0) a.res[w].status = kStatusEmpty;
            continue;
        }
        if (FEED) gather_window(a, w, off, n, gb, GB);
        const double *xc = a.xc + off, *yc = a.yc + off, *tw = a.t + off;
        // fresh accumulators for the window: every CTA is past the previous
        // window's last step before block 0 clears them
        grid_sync(ctr, target, GB);
        if (gb == 0 && threadIdx.x == 0) {
            unsigned long long *z = &st->acc[0][0];
            for (int k = 0; k < 16; k++) __stcg(z + k, 0ull);
            __stcg(&st->sacc[0][1][0], 0ull);  // kModeRootCert sums
            __stcg(&st->sacc[0][1][1], 0ull);
        }
        grid_sync(ctr, target, GB);
        if (threadIdx.x == 0) {
            R.root_L = 0.0;
            R.lo = a.lo0;
            R.hi = a.hi0;
            R.c = a.c0;
            R.den_lo = a.den_lo0;
            R.den_c = a.den_c0;
            R.den_hi = a.den_hi0;
            R.r_lo = ddiv(1.0, R.den_lo);
            R.r_c = ddiv(1.0, R.den_c);
            R.r_hi = ddiv(1.0, R.den_hi);
            R.mode = a.root_cert ? kModeRootCert : kModeRoot;
            R.done = 0;
            R.status = kStatusOk;
            R.parity = 0;
            R.nu_hat = 0.0;
            R.c_hat = 0.0;
            R.bound_gap = 0.0;
            R.iterations = R.bound_evals = R.point_evals = R.next_counter = R.fr_n = R.max_fr = 0;
            R.marks = 0;
            R.exact = 0;
            R.n_pending = 0;
            R.n_pushed = 0;
        }
        __syncthreads();
        while (!R.done) {
            const int mode = R.mode, par = R.parity;
            const double lo = R.lo, hi = R.hi, c = R.c;
            const double den_lo = R.den_lo, den_c = R.den_c, den_hi = R.den_hi;
            const double r_lo = R.r_lo, r_c = R.r_c, r_hi = R.r_hi;
            const long long it = R.iterations;
            unsigned long long *acc = st->acc[par];
            const bool tr = tracer && w == 0;
            if (tr && gb == 0) trace_point(a, it, kTrB0Top);
            if (tr) btrace_point(a, it, 0);

            // event phase: every event, three warps (lo, centre, hi); point
            // image at the centre, segment images of both children (root: of
            // the root); short segments in the lane, long ones spread over the
            // warp.  First round static, then warps take batches of 32 events
            // from the node's work counter (acc[7]) so CTAs finish together.
            unsigned long long v[4] = {0, 0, 0, 0};  // in_image, fi A, fi B, marks
            unsigned long long vex[1] = {0};           // events on the exact path
            AtomicSink sa{A}, sb{B};
            // the filtered path pays off once segments are short; wide nodes
            // (and the FILTER=false kernel) go straight to the exact path --
            // both give the same images
            if (!FILTER || dsub(hi, lo) > kFilterWidth) {
                EventJob J{xc, yc, tw, n, lo, c, hi, den_lo, den_c, den_hi, a.cx, a.cy,
                           W, H, P, A, B, mode, acc, gsz, gb, dsub(hi, lo) > kGuidedWidth,
                           &st->sacc[0][1][0]};
                event_pass_exact<chunk_for(NT), drain_cont<NT>()>(J, wq, v, vex);
            } else {
                int nq = 0;  // uncertain events queued in wq.ev (warp-uniform)
                long long base = gb * (long long)blockDim.x + (threadIdx.x & ~31);
                while (true) {
                    const bool more = base < n;
                    int dummy = 0;
                    if (more) {
                        // filtered path: certify all three results from approximate
                        // warps; uncertain events are queued for the exact path
                        const long long i = base + lane;
                        bool exact = false;
                        if (i < n) {
                            const double x = __ldg(xc + i), y = __ldg(yc + i), t = __ldg(tw + i);
                            const Warped ql = warp_approx(x, y, t, lo, r_lo, a.cx, a.cy);
                            const Warped qc = warp_approx(x, y, t, c, r_c, a.cx, a.cy);
                            const Warped qh = warp_approx(x, y, t, hi, r_hi, a.cx, a.cy);
                            const double ml = sure_margin(ql, a.cx, a.cy);
                            const double mc = sure_margin(qc, a.cx, a.cy);
                            const double mh = sure_margin(qh, a.cx, a.cy);
                            long long pp, pa, pb = -1;
                            int ia, ib = 0;
                            const bool sure = sure_point(qc, mc, W, H, pp) &&
                                              (mode == kModeRoot
                                                   ? sure_segment(ql, qh, ml, mh, W, H, pa, ia)
                                                   : (sure_segment(ql, qc, ml, mc, W, H, pa, ia) &&
                                                      sure_segment(qc, qh, mc, mh, W, H, pb, ib)));
                            if (sure) {
                                if (pp >= 0) { atomicAdd(P + pp, 1u); v[0]++; }
                                if (pa >= 0) { atomicAdd(A + pa, 1u); dummy++; }
                                if (pb >= 0) { atomicAdd(B + pb, 1u); dummy++; }
                                v[1] += ia;
                                v[2] += ib;
                            } else {
                                exact = true;
                            }
                        }
                        const unsigned bal = __ballot_sync(0xffffffffu, exact);
                        if (exact) wq.ev[nq + __popc(bal & ((1u << lane) - 1u))] = i;
                        nq += __popc(bal);
                        __syncwarp();
                        long long nb = 0;
                        if (lane == 0) nb = gsz + (long long)atomicAdd(acc + 7, 32ull);
                        base = __shfl_sync(0xffffffffu, nb, 0);
                    }
                    if (nq >= 32 || (!more && nq > 0)) {
                        // exact path for 32 queued events at a time (full lanes)
                        const int take = nq < 32 ? nq : 32;
                        const long long i = lane < take ? wq.ev[nq - take + lane] : -1;
                        nq -= take;
                        __syncwarp();
                        int cA = 0, cB = 0;
                        if (i >= 0) {
                            vex[0]++;
                            const double x = __ldg(xc + i), y = __ldg(yc + i), t = __ldg(tw + i);
                            const Warped wl = warp_event(x, y, t, lo, den_lo, a.cx, a.cy);
                            const Warped wc = warp_event(x, y, t, c, den_c, a.cx, a.cy);
                            const Warped wh = warp_event(x, y, t, hi, den_hi, a.cx, a.cy);
                            const long long p = floor_bin(wc.x, wc.y, W, H);
                            if (p >= 0) {
                                atomicAdd(P + p, 1u);
                                v[0]++;
                            }
                            if (mode == kModeRoot) {
                                v[1] += fully_inside(wl.x, wl.y, wh.x, wh.y, W, H);
                                cA = segment_or_queue(wl.x, wl.y, wh.x, wh.y, W, H, wq, 2 * lane, sa,
                                                      dummy);
                            } else {
                                v[1] += fully_inside(wl.x, wl.y, wc.x, wc.y, W, H);
                                cA = segment_or_queue(wl.x, wl.y, wc.x, wc.y, W, H, wq, 2 * lane, sa,
                                                      dummy);
                                v[2] += fully_inside(wc.x, wc.y, wh.x, wh.y, W, H);
                                cB = segment_or_queue(wc.x, wc.y, wh.x, wh.y, W, H, wq, 2 * lane + 1,
                                                      sb, dummy);
                            }
                        }
                        if (__any_sync(0xffffffffu, (cA | cB) != 0))
                            dummy += warp_drain<drain_cont<NT>()>(wq, cA, cB, W, H);
                    }
                    v[3] += dummy;
                    if (!more && nq == 0) break;
                }
            }
            __syncthreads();
            if (tr && gb == 0) trace_point(a, it, kTrB0Events);
            if (tr) trace_max(a, it, kTrEventsMax);
            if (tr) btrace_point(a, it, 1);
            block_add_u64<4>(v, acc);
            block_add_u64<1>(vex, acc + 6);
            grid_sync(ctr, target, GB);
            if (tr) bclock(a, it, 4);
            if (tr && gb == 0) trace_point(a, it, kTrB0Pixels0);

            // pixel phase: contrast subtrees of the point image, exact sums of
            // squares of both segment images; every image is left zeroed
            // One thread per CTA reads the accumulators (all requests in flight
            // together) and broadcasts mu through shared memory: 512 threads
            // loading the same line after the barrier was measured ~4k cycles.
            if (threadIdx.x == 0) {
                const ulonglong2 a01 = __ldcg(reinterpret_cast<const ulonglong2 *>(acc));
                const unsigned long long a2 = __ldcg(acc + 2);
                if (gb == 0) {
                    for (int k = 0; k < R.n_pending; k++) entry_store(fr + R.pend_idx[k], R.pend[k]);
                    unsigned long long *nxt = st->acc[par ^ 1];
                    for (int k = 0; k < 8; k++) __stcg(nxt + k, 0ull);
                }
                R.fiA = a01.y;  // final after barrier 1; kept for the step
                R.fiB = a2;
                R.mu = ddiv((double)a01.x, (double)tree.M);
            }
            if (tr) bclock(a, it, 5);
            __syncthreads();
            const double mu = R.mu;
            if (tr) bclock(a, it, 13);
            // the point image's cut walk (first kPixCutThreads threads, named
            // barrier 1) runs beside the segment images' sums of squares (the
            // other warps, named barrier 2): independent latency chains
            if (threadIdx.x < kPixCutThreads) {
                for (int cut = gb, q = 0; cut < tree.C; cut += GB, q++) {
                    const double r = eval_cut(tree, local_cuts ? q : cut, SqU32Clear{{P, mu}}, scratch,
                                              a, tr ? it : kBTraceIters, kPixCutThreads,
                                              NamedBar{1, kPixCutThreads});
                    if (threadIdx.x == 0) __stcg(tree.cutval + cut, r);
                }
                if (threadIdx.x == 0) {  // pow(fi/M, 2) table values, needed by the step
                    R.p2A = __ldg(a.pow2 + R.fiA);
                    R.p2B = __ldg(a.pow2 + R.fiB);
                }
            } else {
                const int nt2 = blockDim.x - kPixCutThreads;
                const long long t2 = gb * (long long)nt2 + (threadIdx.x - kPixCutThreads);
                const long long s2 = (long long)GB * nt2;
                unsigned long long ws[2] = {0, 0};
                for (long long p = t2; p < tree.M; p += s2) {
                    const unsigned long long ha = __ldcg(A + p), hb = __ldcg(B + p);
                    if (ha) { ws[0] += ha * ha; A[p] = 0u; }
                    if (hb) { ws[1] += hb * hb; B[p] = 0u; }
                }
                __shared__ unsigned long long s_ws[32][2];
                const int wid = threadIdx.x >> 5;
                ws[0] = warp_sum(ws[0]);
                ws[1] = warp_sum(ws[1]);
                if (lane == 0) { s_ws[wid][0] = ws[0]; s_ws[wid][1] = ws[1]; }
                asm volatile("bar.sync 2, %0;" ::"r"(nt2) : "memory");
                if (threadIdx.x == kPixCutThreads) {
                    unsigned long long x0 = 0, x1 = 0;
                    for (int w2 = kPixCutThreads >> 5; w2 < (int)(blockDim.x >> 5); w2++) {
                        x0 += s_ws[w2][0];
                        x1 += s_ws[w2][1];
                    }
                    if (x0) atomicAdd(acc + 4, x0);
                    if (x1) atomicAdd(acc + 5, x1);
                }
            }
            if (tr) bclock(a, it, 6);
            if (tr) bclock(a, it, 7);
            if (tr) bclock(a, it, 8);
            if (tr && gb == 0) trace_point(a, it, kTrB0Pixels1);
            if (tr) trace_max(a, it, kTrPixelsMax);
            if (tr) btrace_point(a, it, 2);
            grid_sync(ctr, target, GB);
            if (tr) bclock(a, it, 9);
            if (tr && gb == 0) trace_point(a, it, kTrB0Step0);

            // step: every CTA stages the cut sums, this node's bound integers
            // and the frontier, finishes the contrast and takes the same step
            const long long n0 = R.fr_n;
            for (int i = threadIdx.x; i < tree.C; i += blockDim.x) scratch[i] = __ldcg(tree.cutval + i);
            if (n0 <= kFrView)
                for (long long i = threadIdx.x; i < n0; i += blockDim.x) view[i] = entry_load(fr + i);
            if (threadIdx.x == 0) {
                const ulonglong2 a23 = __ldcg(reinterpret_cast<const ulonglong2 *>(acc + 2));
                const ulonglong2 a45 = __ldcg(reinterpret_cast<const ulonglong2 *>(acc + 4));
                const ulonglong2 a67 = __ldcg(reinterpret_cast<const ulonglong2 *>(acc + 6));
                const unsigned long long in_image = __ldcg(acc);
                R.sA = a45.x;
                R.sB = a45.y;
                if (mode == kModeRootCert) {  // as k_solve_spec: S >= sum^2 / M
                    const double Md = (double)tree.M;
                    const double q = (double)__ldcg(&st->sacc[0][1][0]) / Md;
                    const double f = (double)__ldcg(&st->sacc[0][1][1]) / Md;
                    R.root_L = (q * q - f * f) * (1.0 - 1e-9);  // compared in bnb_step
                }
                R.marks += in_image + a23.y;
                R.exact += a67.x;
                if (tr && gb == 0 && it < a.trace_iters) {  // per-node work counters
                    a.trace[1 + kTraceSlots * it + kTrMarks] = (long long)a23.y;
                    a.trace[1 + kTraceSlots * it + kTrExact] = (long long)a67.x;
                }
            }
            __syncthreads();
            if (tr) bclock(a, it, 10);
            const double S = top_combine(tree, scratch);
            if (tr) bclock(a, it, 11);
            bnb_step<FILTER>(a, R, S, view, fr);
            if (tr) bclock(a, it, 12);
            if (threadIdx.x == 0) R.parity = par ^ 1;
            if (tr && gb == 0) trace_point(a, it, kTrB0Step1);
            if (tr) btrace_point(a, it, 3);
            __syncthreads();
        }
        if (gb == 0 && threadIdx.x == 0) {
            WindowResult &r = a.res[w];
            r.nu = R.nu_hat;
            r.contrast = R.c_hat;
            r.bound_gap = R.bound_gap;
            r.iterations = R.iterations;
            r.bound_evals = R.bound_evals;
            r.point_evals = R.point_evals;
            r.max_fr = R.max_fr;
            r.marks = R.marks;
            r.exact = R.exact;
            r.status = R.status;
            r.rounds = (int)R.point_evals;  // one node evaluation per round
        }
    }
}

// ---------------------------------------------------------------- speculative rounds
// k_solve_spec: the same best-first BnB, bit for bit, with up to kSpecK node
// evaluations per round.  Slot 0 is the node the reference pops next; slots
// 1.. are the best narrow frontier entries, evaluated speculatively (a node's
// results are a pure function of its interval).  The step then replays the
// reference's pops in order and consumes cached results until a pop finds
// none.  At cfg 1/2 a 4-slot round covers ~3.5 pops (the next pops are mostly
// the frontier's current best, rarely the newest children), so the per-round
// fixed costs (two grid barriers, the contrast reduction, the step) are paid
// ~3.5x less often.  The frontier is replicated in every CTA's shared memory.
constexpr int kSpecFr = 1024;     // frontier entries per CTA (shared memory)
constexpr int kSpecCache = 64;    // results of evaluated, not yet popped nodes
#ifndef EVD_SPEC_WIDTH
#define EVD_SPEC_WIDTH 1.0
#endif
constexpr double kSpecWidth = EVD_SPEC_WIDTH;  // only intervals this narrow are speculated

struct SpecSlot {
    double lo, hi, c, den_lo, den_c, den_hi;
    long long counter;
};
struct SpecRes {
    long long counter;
    double C, cbA, cbB;
};
struct SpecState {
    SpecSlot slot[kSpecK];
    int nslot, mode, done, status, parity;
    double nu_hat, c_hat, bound_gap;
    long long iterations, bound_evals, point_evals, next_counter, fr_n, max_fr;
    unsigned long long marks, exact;
    double mu[kSpecK];
    unsigned long long fiA[kSpecK], fiB[kSpecK];
    double pwA[kSpecK], pwB[kSpecK];  // mu_lower**2 of each child (the pow2 table)
    double S[kSpecK];
    SpecRes cache[kSpecCache];
    int ncache, cache_head;
    int cur;  // cache index of the node being processed (-1: slot results below)
    int rounds;
    int root_ok;  // kModeRootCert: the root bound is certified to exceed c_hat + gamma
    long long ev_next;  // evaluation-only launch: nodes handed to slots so far
};


// Frontier entries already chosen for a speculative slot carry this bit in
// their counter (set by the round's slot selection, masked wherever the
// counter is compared or copied), so the selection skips them in O(1)
// instead of searching the result cache per entry.
constexpr long long kSpecFlag = 1ll << 62;

// the result-cache index holding `counter`, or -1 (all 32 lanes of warp 0)
__device__ __forceinline__ int spec_find(const SpecState &Z, long long counter)
{
    const int lane = threadIdx.x & 31, nc = Z.ncache;
    int hit = -1;
    for (int k0 = 0; k0 < nc; k0 += 32) {
        const bool m = k0 + lane < nc && Z.cache[k0 + lane].counter == counter;
        const unsigned b = __ballot_sync(0xffffffffu, m);
        if (b) {
            hit = k0 + __ffs(b) - 1;
            break;
        }
    }
    return hit;
}

// warp-0 argmax over the shared frontier, skipping entries flagged by `skip`
template <class Skip>
__device__ __forceinline__ long long spec_argmax(const FrontierEntry *fr, long long n, Skip skip)
{
    double bb = -DBL_MAX;
    long long bc = LLONG_MAX, bi = -1;
    for (long long i = threadIdx.x & 31; i < n; i += 32) {
        const FrontierEntry &e = fr[i];
        if (skip(e)) continue;
        const long long ec = e.counter & ~kSpecFlag;
        if (bi < 0 || better(e.bound, ec, bb, bc)) { bb = e.bound; bc = ec; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, bb, o);
        const long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || better(ob, oc, bb, bc))) { bb = ob; bc = oc; bi = oi; }
    }
    return bi;
}

__device__ __forceinline__ void spec_set_slot(const SolveArgs &a, SpecSlot &s,
                                              const FrontierEntry &e)
{
    const double c = dmul(0.5, dadd(e.lo, e.hi));  // VelocityInterval.center
    s.lo = e.lo;
    s.hi = e.hi;
    s.c = c;
    s.den_lo = dadd(1.0, dmul(e.lo, a.tau));
    s.den_c = dadd(1.0, dmul(c, a.tau));
    s.den_hi = dadd(1.0, dmul(e.hi, a.tau));
    s.counter = e.counter & ~kSpecFlag;
}

// evaluation-only launch: the next round's slots from the node list
__device__ __forceinline__ void spec_eval_slots(const SolveArgs &a, SpecState &Z, int K)
{
    int ns = 0;
    while (ns < K && Z.ev_next < a.ev_n) {
        const long long i = Z.ev_next++;
        spec_set_slot(a, Z.slot[ns], FrontierEntry{0.0, i, a.ev_lo[i], a.ev_hi[i]});
        ns++;
    }
    Z.nslot = ns;
    Z.mode = kModeNode;
    if (ns == 0) Z.done = 1;
}

template <int NT, bool FEED = false>
__global__ void __launch_bounds__(NT, 1) k_solve_spec(SolveArgs a)
{
    constexpr size_t kRegionA = SolveSmem<NT>::region_a;
    constexpr int kPixCutThreads = pix_cut_threads<NT>();
    extern __shared__ __align__(16) unsigned char smem[];
    WarpQueue &wq = reinterpret_cast<WarpQueue *>(smem)[threadIdx.x >> 5];
    double *scratch = reinterpret_cast<double *>(smem);
    TreeCache &tc = *reinterpret_cast<TreeCache *>(smem + kRegionA);
    FrontierEntry *frs = reinterpret_cast<FrontierEntry *>(smem + kRegionA + sizeof(TreeCache));
    __shared__ SpecState Z;
    __shared__ unsigned long long s_acc[kSpecK][5];
    __shared__ int s_flag;
    const int GB = a.group_blocks;
    const int grp = blockIdx.x / GB, gb = blockIdx.x % GB;
    if (grp >= a.groups) return;
    unsigned long long *ctr = a.bar + 2 * grp;
    unsigned long long target = 0;
    SolveState *st = a.st + grp;
    const long long M = a.tree.M;
    const int K = a.spec_k;
    unsigned int *img0 = a.img + (long long)grp * 3 * kSpecK * M;  // slot s: P, A, B
    const int lane = threadIdx.x & 31;
    const long long gsz = (long long)GB * blockDim.x;
    const int W = a.W, H = a.H;
    bool local_cuts;
    TreeDev gtree = a.tree;
    gtree.cutval = a.tree.cutval + (long long)grp * kSpecK * a.tree.C;  // [slot][C]
    // this CTA walks cut (gb mod C) of slot (gb div C) whenever slots x cuts
    // fit the group (the plan aims at C <= GB / kSpecK): cache that cut
    __shared__ TreeDev tree_s;
    {
        const TreeDev t = cache_tree(gtree, tc, local_cuts, gb % gtree.C, GB);
        if (threadIdx.x == 0) tree_s = t;
        __syncthreads();
    }
    const TreeDev &tree = tree_s;
    const int C = tree.C;
    const int ntop = tree.top_lvl[tree.top_levels];

    for (int w = grp; w < a.n_windows; w += a.groups) {
        const long long off = a.offsets[w], n = FEED ? a.counts[w] : a.offsets[w + 1] - off;
        if (n == 0) {
            if (gb == 0 && threadIdx.x == 0) a.res[w].status = kStatusEmpty;
            continue;
        }
        if (FEED) gather_window(a, w, off, n, gb, GB);
        const double *xc = a.xc + off, *yc = a.yc + off, *tw = a.t + off;
        if (kTraceBuild && a.trace && grp == 0 && w == 0 && gb == 0) trace_point(a, 0, -1);
        grid_sync(ctr, target, GB);
        if (gb == 0 && threadIdx.x == 0) {
            unsigned long long *z = &st->sacc[0][0][0];
            for (int k = 0; k < 2 * kSpecK * 8; k++) __stcg(z + k, 0ull);
        }
        grid_sync(ctr, target, GB);
        if (threadIdx.x == 0) {
            Z.slot[0] = SpecSlot{a.lo0, a.hi0, a.c0, a.den_lo0, a.den_c0, a.den_hi0, -1};
            Z.nslot = 1;
            Z.mode = a.root_cert ? kModeRootCert : kModeRoot;
            Z.root_ok = 0;
            Z.done = 0;
            Z.ev_next = 0;
            if (a.ev_n > 0) spec_eval_slots(a, Z, K);
            Z.status = kStatusOk;
            Z.parity = 0;
            Z.nu_hat = Z.c_hat = Z.bound_gap = 0.0;
            Z.iterations = Z.bound_evals = Z.point_evals = Z.next_counter = Z.fr_n = Z.max_fr = 0;
            Z.marks = Z.exact = 0;
            Z.ncache = Z.cache_head = 0;
            Z.rounds = 0;
        }
        __syncthreads();
        while (!Z.done) {
            const int ns = Z.nslot, mode = Z.mode, par = Z.parity;
            unsigned long long (*sacc)[8] = st->sacc[par];
            // round timeline (trace build, window 0 of group 0): the same
            // slots as k_solve's per-node trace, one entry per round
            const long long it = Z.rounds;
            const bool tr = kTraceBuild && a.trace && grp == 0 && w == 0;
            if (tr && gb == 0) trace_point(a, it, kTrB0Top);
            if (threadIdx.x < kSpecK * 5) (&s_acc[0][0])[threadIdx.x] = 0;
            __syncthreads();
            // events: one pass per slot (each with its own work counter)
            for (int s = 0; s < ns; s++) {
                const SpecSlot sl = Z.slot[s];
                unsigned int *P = img0 + (long long)(3 * s) * M, *A = P + M, *B = A + M;
                unsigned long long v[4] = {0, 0, 0, 0}, vex[1] = {0};
                EventJob J{xc, yc, tw, n, sl.lo, sl.c, sl.hi, sl.den_lo, sl.den_c, sl.den_hi,
                           a.cx, a.cy, W, H, P, A, B, (s == 0 ? mode : kModeNode), sacc[s],
                           gsz, gb, dsub(sl.hi, sl.lo) > kGuidedWidth, sacc[1]};
                event_pass_exact<chunk_for(NT), drain_cont<NT>()>(J, wq, v, vex);
#pragma unroll
                for (int k = 0; k < 4; k++) v[k] = warp_sum(v[k]);
                vex[0] = warp_sum(vex[0]);
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        if (v[k]) atomicAdd(&s_acc[s][k], v[k]);
                    if (vex[0]) atomicAdd(&s_acc[s][4], vex[0]);
                }
            }
            __syncthreads();
            if (tr && gb == 0) trace_point(a, it, kTrB0Events);
            if (tr) trace_max(a, it, kTrEventsMax);
            if (threadIdx.x < ns * 5) {
                const int s = threadIdx.x / 5, k = threadIdx.x % 5;
                const unsigned long long x = s_acc[s][k];
                if (x) atomicAdd(&sacc[s][k == 4 ? 6 : k], x);
            }
            grid_sync(ctr, target, GB);
            if (tr && gb == 0) trace_point(a, it, kTrB0Pixels0);

            // pixels: per-slot accumulators, the point images' cut walks beside
            // the segment images' sums of squares
            // one thread per slot (the loads in parallel, not one after another)
            if (threadIdx.x < ns) {
                const int s = threadIdx.x;
                const ulonglong2 a01 = __ldcg(reinterpret_cast<const ulonglong2 *>(sacc[s]));
                const unsigned long long a2 = __ldcg(&sacc[s][2]);
                Z.mu[s] = ddiv((double)a01.x, (double)M);
                Z.fiA[s] = a01.y;
                Z.fiB[s] = a2;
                Z.pwA[s] = __ldg(a.pow2 + a01.y);  // prefetched for the step
                Z.pwB[s] = __ldg(a.pow2 + a2);
            }
            if (gb == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + kSpecK * 8)
                __stcg(&st->sacc[par ^ 1][0][0] + (threadIdx.x - 32), 0ull);
            __syncthreads();
            if (threadIdx.x < kPixCutThreads) {
                for (int p = gb; p < ns * C; p += GB) {
                    const int s = p / C, cut = p - s * C;
                    unsigned int *P = img0 + (long long)(3 * s) * M;
                    const bool mine = local_cuts && cut == gb % C;
                    const double r = eval_cut(mine ? tree : gtree, mine ? 0 : cut,
                                              SqU32Clear{{P, Z.mu[s]}}, scratch, a, kBTraceIters,
                                              kPixCutThreads, NamedBar{1, kPixCutThreads});
                    if (threadIdx.x == 0) __stcg(tree.cutval + (long long)s * C + cut, r);
                }
            } else {
                const int nt2 = blockDim.x - kPixCutThreads;
                const long long t2 = gb * (long long)nt2 + (threadIdx.x - kPixCutThreads);
                const long long s2 = (long long)GB * nt2;
                __shared__ unsigned long long s_ws[32][2 * kSpecK];
                const int wid = threadIdx.x >> 5;
                for (int s = 0; s < ns; s++) {
                    unsigned int *A = img0 + (long long)(3 * s + 1) * M, *B = A + M;
                    unsigned long long ws0 = 0, ws1 = 0;
                    for (long long p = t2; p < M; p += s2) {
                        const unsigned long long ha = __ldcg(A + p), hb = __ldcg(B + p);
                        if (ha) { ws0 += ha * ha; A[p] = 0u; }
                        if (hb) { ws1 += hb * hb; B[p] = 0u; }
                    }
                    ws0 = warp_sum(ws0);
                    ws1 = warp_sum(ws1);
                    if (lane == 0) { s_ws[wid][2 * s] = ws0; s_ws[wid][2 * s + 1] = ws1; }
                }
                asm volatile("bar.sync 2, %0;" ::"r"(nt2) : "memory");
                if (threadIdx.x < kPixCutThreads + 2 * ns) {
                    const int k = threadIdx.x - kPixCutThreads;
                    unsigned long long x = 0;
                    for (int w2 = kPixCutThreads >> 5; w2 < (int)(blockDim.x >> 5); w2++)
                        x += s_ws[w2][k];
                    if (x) atomicAdd(&sacc[k >> 1][4 + (k & 1)], x);
                }
            }
            if (tr) {
                __syncthreads();
                if (gb == 0) trace_point(a, it, kTrB0Pixels1);
                trace_max(a, it, kTrPixelsMax);
            }
            grid_sync(ctr, target, GB);
            if (tr && gb == 0) trace_point(a, it, kTrB0Step0);

            // step: finish every slot's contrast and bounds, then replay the
            // reference's pops while their results are known
            // each slot's child bounds and counts (one thread per slot, in the
            // CTA's last warp) while the other threads fetch the cut sums
            __shared__ double s_res[kSpecK][3];
            __shared__ unsigned long long s_cnt[kSpecK][2];
            const int sl0 = (int)blockDim.x - 32;
            if (threadIdx.x >= sl0 && threadIdx.x < sl0 + ns) {
                const int s = threadIdx.x - sl0;
                const double Md = (double)M;
                const ulonglong2 a45 = __ldcg(reinterpret_cast<const ulonglong2 *>(sacc[s] + 4));
                const ulonglong2 a23 = __ldcg(reinterpret_cast<const ulonglong2 *>(sacc[s] + 2));
                const unsigned long long a0 = __ldcg(sacc[s]), a6 = __ldcg(sacc[s] + 6);
                s_cnt[s][0] = a0 + a23.y;
                s_cnt[s][1] = a6;
                s_res[s][1] = dsub(ddiv((double)a45.x, Md), Z.pwA[s]);
                s_res[s][2] = dsub(ddiv((double)a45.y, Md), Z.pwB[s]);
            }
            if ((int)threadIdx.x < sl0)
                for (int i = threadIdx.x; i < ns * C; i += sl0)
                    scratch[(i / C) * (C + ntop) + (i % C)] = __ldcg(tree.cutval + i);
            __syncthreads();
            if (C > 1) {
                const int levels = tree.top_levels;
                const int4 tr = threadIdx.x < ns * ntop ? tree.top[threadIdx.x % ntop]
                                                        : make_int4(0, 0, 0, -1);
                double *vv = scratch + (threadIdx.x / (ntop > 0 ? ntop : 1)) * (C + ntop);
                if (ns * ntop <= (int)blockDim.x) {
                    for (int h = 0; h < levels; h++) {
                        if (tr.w == h) vv[tr.x] = dadd(vv[tr.y], vv[tr.z]);
                        __syncthreads();
                    }
                } else if (threadIdx.x == 0) {
                    Z.status = kStatusSpecOverflow;  // the host falls back to k_solve
                }
            }
            __syncthreads();
            // each slot's contrast, one thread per slot
            if (threadIdx.x < ns) {
                const int s = threadIdx.x;
                const double Sv = scratch[s * (C + ntop) + (C > 1 ? tree.top_root : 0)];
                s_res[s][0] = ddiv(dadd(0.0, Sv), (double)M);  // np.sum(...) / M
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                Z.rounds++;
                for (int s = 0; s < ns; s++) {
                    Z.marks += s_cnt[s][0];
#ifndef EVD_STEP_PROBE
                    if (tr && gb == 0 && it < a.trace_iters)  // round's marks, slots
                        a.trace[1 + kTraceSlots * it + kTrMarks] += (long long)s_cnt[s][0];
#endif
                    Z.exact += s_cnt[s][1];
                    const double Cs = s_res[s][0], cbA = s_res[s][1], cbB = s_res[s][2];
                    if (s == 0 && mode == kModeRoot) {
                        Z.S[0] = Cs;
                        Z.mu[0] = cbA;  // the root bound
                        continue;
                    }
                    if (s == 0 && mode == kModeRootCert) {
                        // solver.py:92-108 pushes the root with c_bar = S/M - mu_lower^2
                        // and pops it at once; only gap > gamma matters, and
                        // S >= (sum of root_cells_lb)^2 / M, mu_lower = fi / M
                        // (Cauchy-Schwarz over the M pixels), with a relative
                        // margin far above the reference's rounding of c_bar
                        const double Md = (double)M;
                        const double q = (double)__ldcg(&sacc[1][0]) / Md;
                        const double f = (double)__ldcg(&sacc[1][1]) / Md;
                        const double L = (q * q - f * f) * (1.0 - 1e-9);
                        Z.root_ok = (L - Cs > a.gamma + 1e-9 * fabs(Cs)) ? 1 : 0;
                    }
                    SpecRes &r = Z.cache[Z.cache_head];
                    r.counter = Z.slot[s].counter;
                    r.C = Cs;
                    r.cbA = cbA;
                    r.cbB = cbB;
                    if (s == 0) Z.cur = Z.cache_head;
                    Z.cache_head = (Z.cache_head + 1) % kSpecCache;
                    if (Z.ncache < kSpecCache) Z.ncache++;
                }
                if (Z.status == kStatusSpecOverflow) Z.done = 1;
                if (a.ev_n > 0) {  // evaluation only: results out, next slots in
                    if (gb == 0)
                        for (int s = 0; s < ns; s++) {
                            const long long i = Z.ev_next - ns + s;
                            a.ev_out[3 * i] = s_res[s][0];
                            a.ev_out[3 * i + 1] = s_res[s][1];
                            a.ev_out[3 * i + 2] = s_res[s][2];
                        }
                    Z.parity = par ^ 1;
                    spec_eval_slots(a, Z, K);
                }
            }
            __syncthreads();
#ifdef EVD_STEP_PROBE
            if (tr && gb == 0) trace_point(a, it, kTrMarks);
#endif
            if (threadIdx.x < 32 && !Z.done && a.ev_n == 0) {
                // warp 0: the pop loop.  The BnB state lives in registers,
                // identical in every lane (each lane computes the same values
                // from the same shared-memory reads); lane 0 writes the
                // frontier entries and, at the end, the state back to Z.
                SpecSlot node = Z.slot[0];
                bool root = mode == kModeRoot, rootc = mode == kModeRootCert;
                int stop = 0, next_uncached = 0;
                double c_hat = Z.c_hat, nu_hat = Z.nu_hat, bound_gap = Z.bound_gap;
                int fr_n = (int)Z.fr_n, cur = Z.cur, status = Z.status;
                long long next_counter = Z.next_counter, iterations = Z.iterations;
                long long point_evals = Z.point_evals, bound_evals = Z.bound_evals;
                long long max_fr = Z.max_fr;
                auto push = [&](double bound, double lo, double hi) {
                    if (fr_n >= kSpecFr || fr_n >= a.fr_cap) {
                        status = kStatusSpecOverflow;
                        stop = 1;
                    } else {
                        if (lane == 0) frs[fr_n] = FrontierEntry{bound, next_counter, lo, hi};
                        fr_n++;
                        next_counter++;
                    }
                };
                while (true) {
                    if (root) {  // solver.py:92-98
                        c_hat = Z.S[0];
                        nu_hat = node.c;
                        point_evals++;
                        bound_evals++;
                        push(Z.mu[0], node.lo, node.hi);
                    } else if (rootc) {
                        // solver.py:92-108 with the root bound certified: the
                        // root is pushed and popped (gap > gamma, width >=
                        // min_width, checked on the host), then evaluated from
                        // its cached result like any node
                        c_hat = Z.cache[cur].C;  // contrast_at(domain.center)
                        nu_hat = node.c;
                        point_evals++;
                        bound_evals++;
                        if (fr_n + 1 > max_fr) max_fr = fr_n + 1;
                        next_counter++;
                        if (!Z.root_ok) {
                            status = kStatusRootCert;
                            stop = 1;
                            break;
                        }
                        iterations++;
                        rootc = false;
                        continue;
                    } else {  // solver.py:109-119
                        const SpecRes &r = Z.cache[cur];
                        point_evals++;
                        if (r.C >= c_hat) {
                            nu_hat = node.c;
                            c_hat = r.C;
                        }
                        bound_evals += 2;
                        const double cbA = r.cbA, cbB = r.cbB;
                        if (cbA >= c_hat) push(cbA, node.lo, node.c);
                        if (!stop && cbB >= c_hat) push(cbB, node.c, node.hi);
                        if (!stop && iterations >= a.max_iter) {
                            status = kStatusIterLimit;
                            stop = 1;
                        }
                    }
                    if (fr_n > max_fr) max_fr = fr_n;
                    if (!stop && fr_n == 0) stop = 1;  // every interval pruned
                    if (stop) break;
                    __syncwarp();
                    const long long bi = spec_argmax(frs, fr_n, [](const FrontierEntry &) {
                        return false;
                    });
                    const FrontierEntry top = frs[bi];
                    const int hit = spec_find(Z, top.counter & ~kSpecFlag);
                    __syncwarp();
                    if (lane == 0) frs[bi] = frs[fr_n - 1];  // swap-remove
                    fr_n--;
                    iterations++;
                    const double gap = dsub(top.bound, c_hat);  // solver.py:105-108
                    if (gap <= a.gamma || dsub(top.hi, top.lo) < a.min_width) {
                        bound_gap = (0.0 > gap) ? 0.0 : gap;
                        stop = 1;
                        break;
                    }
                    spec_set_slot(a, node, top);
                    root = false;
                    __syncwarp();
                    if (hit >= 0) {
                        cur = hit;
                    } else {
                        next_uncached = 1;
                        break;
                    }
                }
#ifdef EVD_STEP_PROBE
                if (tr && gb == 0) trace_point(a, it, kTrExact);
#endif
                __syncwarp();
                int nslot = 1;
                if (!stop) {
                    // next round: the popped node, then the best narrow uncached
                    // entries of the frontier
                    for (int s = 1; s < K; s++) {
                        const long long bi = spec_argmax(frs, fr_n, [&](const FrontierEntry &e) {
                            if (dsub(e.hi, e.lo) > kSpecWidth) return true;
                            // never evaluated by the reference: popping it ends
                            // the search (solver.py:106-108; c_hat only grows)
                            if (dsub(e.bound, c_hat) <= a.gamma ||
                                dsub(e.hi, e.lo) < a.min_width)
                                return true;
                            // evaluated or scheduled already (its result is
                            // cached, or it is one of this round's slots)
                            return (e.counter & kSpecFlag) != 0;
                        });
                        if (bi < 0) break;
                        if (lane == 0) {
                            spec_set_slot(a, Z.slot[nslot], frs[bi]);
                            frs[bi].counter |= kSpecFlag;
                        }
                        nslot++;
                        __syncwarp();
                    }
                }
                if (lane == 0) {
                    Z.c_hat = c_hat;
                    Z.nu_hat = nu_hat;
                    Z.bound_gap = bound_gap;
                    Z.fr_n = fr_n;
                    Z.cur = cur;
                    Z.status = status;
                    Z.next_counter = next_counter;
                    Z.iterations = iterations;
                    Z.point_evals = point_evals;
                    Z.bound_evals = bound_evals;
                    Z.max_fr = max_fr;
                    if (stop) {
                        Z.done = 1;
                    } else {
                        Z.slot[0] = node;
                        Z.nslot = nslot;
                        Z.mode = kModeNode;
                        Z.parity = par ^ 1;
                    }
                }
            }
            __syncthreads();
            if (tr && gb == 0) {
                trace_point(a, it, kTrB0Step1);
#ifndef EVD_STEP_PROBE
                if (threadIdx.x == 0 && it < a.trace_iters)
                    a.trace[1 + kTraceSlots * it + kTrExact] = ns;  // slots this round
#endif
            }
        }
        // speculative slots' point images are summed (and cleared) every round;
        // segment images are cleared by the pixel phase: nothing is left dirty
        if (gb == 0 && threadIdx.x == 0) {
            WindowResult &r = a.res[w];
            r.nu = Z.nu_hat;
            r.contrast = Z.c_hat;
            r.bound_gap = Z.bound_gap;
            r.iterations = Z.iterations;
            r.bound_evals = Z.bound_evals;
            r.point_evals = Z.point_evals;
            r.max_fr = Z.max_fr;
            r.marks = Z.marks;
            r.exact = Z.exact;
            r.status = Z.status;
            r.rounds = Z.rounds;
        }
    }
}

// ---------------------------------------------------------------- launchers
constexpr size_t kBoundSmem = sizeof(WarpQueue) * (kThreads / 32);
template <int NT>
constexpr size_t solve_smem() { return SolveSmem<NT>::region_a + sizeof(TreeCache); }
template <int NT>
constexpr size_t spec_smem()
{
    return SolveSmem<NT>::region_a + sizeof(TreeCache) + kSpecFr * sizeof(FrontierEntry);
}

// Kernel attributes are per device: set them once for each device a context
// launches on (idempotent, so two threads racing on one device is harmless).
static std::atomic<unsigned long long> g_attrs{0};
static void set_attrs()
{
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (g_attrs.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(k_bound_image, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBoundSmem);
    cudaFuncSetAttribute(k_frontier, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBoundSmem);
    cudaFuncSetAttribute(k_frontier_f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBoundSmem);
    cudaFuncSetAttribute(k_solve<false, 384>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)solve_smem<384>());
    cudaFuncSetAttribute(k_solve<false, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)solve_smem<512>());
    cudaFuncSetAttribute(k_solve<false, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)solve_smem<768>());
    cudaFuncSetAttribute(k_solve<true, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)solve_smem<512>());
    cudaFuncSetAttribute(k_solve<false, 512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)solve_smem<512>());
    cudaFuncSetAttribute(k_solve_spec<512, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)spec_smem<512>());
    cudaFuncSetAttribute(k_event_probe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kQueueBytes);
    cudaFuncSetAttribute(k_solve_spec<384>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)spec_smem<384>());
    cudaFuncSetAttribute(k_solve_spec<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)spec_smem<512>());
    cudaFuncSetAttribute(k_solve_spec<768>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)spec_smem<768>());
    g_attrs.fetch_or(bit, std::memory_order_release);
}

void launch_center(const double *x, const double *y, long long n, double cx, double cy,
                   double *xc, double *yc, cudaStream_t s)
{
    k_center<<<event_blocks(n), kThreads, 0, s>>>(x, y, n, cx, cy, xc, yc);
}

void launch_warp(const double *xc, const double *yc, const double *t, long long n, double nu,
                 double den, double cx, double cy, double *xo, double *yo, cudaStream_t s)
{
    k_warp<<<event_blocks(n), kThreads, 0, s>>>(xc, yc, t, n, nu, den, cx, cy, xo, yo);
}

void launch_scale(const double *t, long long n, double nu, double den, double *s, cudaStream_t st)
{
    k_scale<<<event_blocks(n), kThreads, 0, st>>>(t, n, nu, den, s);
}

void launch_point_image(const double *xc, const double *yc, const double *t, long long n,
                        double nu, double den, double cx, double cy, int W, int H,
                        unsigned int *img, unsigned long long *acc, cudaStream_t s)
{
    k_point_image<<<event_blocks(n), kThreads, 0, s>>>(xc, yc, t, n, nu, den, cx, cy, W, H,
                                                       img, acc);
}

void launch_bound_image(const double *xc, const double *yc, const double *t, long long n,
                        double lo, double den_lo, double hi, double den_hi, double cx, double cy,
                        int W, int H, unsigned int *img, unsigned long long *acc,
                        cudaStream_t s)
{
    set_attrs();
    k_bound_image<<<event_blocks(n), kThreads, kBoundSmem, s>>>(xc, yc, t, n, lo, den_lo, hi,
                                                                den_hi, cx, cy, W, H, img, acc);
}

void launch_frontier(const double *xc, const double *yc, const double *t, long long n,
                     const double *lo, const double *hi, const double *den_lo,
                     const double *den_hi, int K, double cx, double cy, int W, int H,
                     unsigned int *images, long long M, unsigned long long *fi_out,
                     unsigned long long *marks_s, bool exact_only, cudaStream_t s)
{
    set_attrs();
    const int groups = (K + kFrontGroup - 1) / kFrontGroup;
    long long bpg = (n + kThreads - 1) / kThreads;
    if (bpg > (long long)num_sms() * EVD_FRONT_BPG) bpg = (long long)num_sms() * EVD_FRONT_BPG;
    if (bpg < 1) bpg = 1;
    if (exact_only)
        k_frontier<<<(unsigned)(groups * bpg), kThreads, kBoundSmem, s>>>(
            xc, yc, t, n, lo, hi, den_lo, den_hi, K, cx, cy, W, H, images, M, (int)bpg, fi_out);
    else
        k_frontier_f<<<(unsigned)(groups * bpg), kThreads, kBoundSmem, s>>>(
            xc, yc, t, n, lo, hi, den_lo, den_hi, K, cx, cy, W, H, images, M, (int)bpg, fi_out);
    long long bpi = (M + kThreads * 4 - 1) / (kThreads * 4);
    if (bpi < 1) bpi = 1;
    k_frontier_sums<<<(unsigned)(K * bpi), kThreads, 0, s>>>(images, M, (int)bpi, marks_s);
}

void launch_image_sums(const unsigned int *img, long long m, unsigned long long *acc,
                       cudaStream_t s)
{
    k_image_sums<<<event_blocks(m), kThreads, 0, s>>>(img, m, acc);
}

void launch_contrast_u32(const unsigned int *img, const unsigned long long *in_image,
                         const TreeDev &tree, double *out, cudaStream_t s)
{
    k_contrast_cuts_u32<<<tree.C, kThreads, 0, s>>>(img, in_image, tree);
    k_contrast_top<<<1, kThreads, 0, s>>>(tree, out);
}

void launch_points_multi(const double *xc, const double *yc, const double *t, long long n,
                         const double *nus, const double *dens, int K, double cx, double cy,
                         int W, int H, unsigned int *images, long long M,
                         unsigned long long *in_out, const TreeDev &tree, double *cutvals,
                         double *contrast, cudaStream_t s)
{
    const int groups = (K + 31) / 32;
    long long bpg = (n + kThreads - 1) / kThreads;
    if (bpg > (long long)num_sms() * EVD_FRONT_BPG) bpg = (long long)num_sms() * EVD_FRONT_BPG;
    if (bpg < 1) bpg = 1;
    k_points_multi<<<(unsigned)(groups * bpg), kThreads, 0, s>>>(xc, yc, t, n, nus, dens, K, cx,
                                                                 cy, W, H, images, M, (int)bpg,
                                                                 in_out);
    k_contrast_cuts_multi<<<(unsigned)((long long)K * tree.C), kThreads, 0, s>>>(images, in_out,
                                                                               tree, cutvals);
    k_contrast_top_multi<<<K, kThreads, 0, s>>>(tree, cutvals, contrast);
}

void launch_contrast_f64(const double *img, double mu, const TreeDev &tree, double *out,
                         cudaStream_t s)
{
    k_contrast_cuts_f64<<<tree.C, kThreads, 0, s>>>(img, mu, tree);
    k_contrast_top<<<1, kThreads, 0, s>>>(tree, out);
}

void launch_raster_segments(const double *segs, int k, int W, int H, int chunk,
                            unsigned int *counts, cudaStream_t s)
{
    k_raster_segments<<<(k + 127) / 128, 128, 0, s>>>(segs, k, W, H, chunk < 1 ? kChunk : chunk,
                                                      counts);
}

int solve_block_threads() { return kSolveThreads; }

int solve_grid_blocks(int device)
{
    set_attrs();
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve<true, 512>, 512,
                                                  solve_smem<512>());
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (per_sm < 1) per_sm = 1;
    return per_sm * sms;
}

// One CTA per SM at every block size (128 registers at 512 threads, 168 at
// 384, 85 at 768): fewer, fatter threads suit latency-bound small windows,
// more threads the sampler throughput of large ones (solve_threads_for).
cudaError_t launch_solve_spec(const SolveArgs &a, int blocks, int threads, cudaStream_t s)
{
    set_attrs();
    SolveArgs args = a;
    void *params[] = {&args};
    // the overlapped-upload variant (a.sx set) is built at 512 threads only
    if (a.sx || (threads != 384 && threads != 768)) threads = 512;
    const void *fn = a.sx           ? (const void *)k_solve_spec<512, true>
                   : threads == 384 ? (const void *)k_solve_spec<384>
                   : threads == 768 ? (const void *)k_solve_spec<768>
                                    : (const void *)k_solve_spec<512>;
    const size_t smem = threads == 384 ? spec_smem<384>()
                      : threads == 768 ? spec_smem<768>() : spec_smem<512>();
    return cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(threads), params, smem, s);
}

cudaError_t launch_solve(const SolveArgs &a, int blocks, int threads, cudaStream_t s)
{
    set_attrs();
    SolveArgs args = a;
    void *params[] = {&args};
    // the filtered path (opt-in) and the overlapped-upload variant (a.sx set)
    // are built at 512 threads only
    if (a.filter || a.sx || (threads != 384 && threads != 768)) threads = 512;
    const void *fn = a.sx             ? (const void *)k_solve<false, 512, true>
                   : a.filter         ? (const void *)k_solve<true, 512>
                   : threads == 384   ? (const void *)k_solve<false, 384>
                   : threads == 768   ? (const void *)k_solve<false, 768>
                                      : (const void *)k_solve<false, 512>;
    const size_t smem = threads == 384 ? solve_smem<384>()
                      : threads == 768 ? solve_smem<768>() : solve_smem<512>();
    return cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(threads), params, smem, s);
}

}  // namespace evd

namespace evd {
cudaError_t launch_event_probe(const double *xc, const double *yc, const double *t, long long n,
                               const double *nu3, const double *den3, double cx, double cy,
                               int W, int H, int blocks, int reps, unsigned long long *ctrs,
                               unsigned long long *span, unsigned int *scratch, cudaStream_t s)
{
    set_attrs();
    EventJob j{xc, yc, t, n, nu3[0], nu3[1], nu3[2], den3[0], den3[1], den3[2], cx, cy, W, H,
               nullptr, nullptr, nullptr, kModeNode, nullptr,
               (long long)blocks * kSolveThreads, 0, 1};
    k_event_probe<<<blocks, kSolveThreads, kQueueBytes, s>>>(j, reps, ctrs, span, scratch,
                                                             (long long)W * H);
    return cudaGetLastError();
}
}  // namespace evd

// ---------------------------------------------------------------- stream windowing
namespace evd {

// First index i in [0, n) with t[i] >= v (numpy searchsorted side="left").
__device__ __forceinline__ long long lower_bound_f64(const double *t, long long n, double v)
{
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (__ldg(t + mid) < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// batch_stream window bounds (events.py:341-347): window w is k = k0 + w,
// start = k * tau (Python int * float), events [searchsorted(start),
// searchsorted(start + tau)) of the time-sorted stream.
__global__ void k_window_bounds(const double *__restrict__ t, long long n, long long k0, int nw,
                                double tau, long long *__restrict__ lo, long long *__restrict__ hi)
{
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
        const double start = dmul((double)(k0 + w), tau);
        lo[w] = lower_bound_f64(t, n, start);
        hi[w] = lower_bound_f64(t, n, dadd(start, tau));
    }
}

// Concatenate the windows' events into the solve layout: centred x, y
// (geometry.py:87) and batch-local t = min(t - start, tau) (events.py:348).
__global__ void k_gather_windows(const double *__restrict__ x, const double *__restrict__ y,
                                 const double *__restrict__ t, const long long *__restrict__ lo,
                                 const long long *__restrict__ off, int nw, long long k0,
                                 double tau, double cx, double cy, double *__restrict__ xc,
                                 double *__restrict__ yc, double *__restrict__ tl)
{
    const long long total = off[nw];
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < total;
         j += (long long)gridDim.x * blockDim.x) {
        int a = 0, b = nw;  // largest w with off[w] <= j
        while (b - a > 1) {
            const int m = (a + b) >> 1;
            if (__ldg(off + m) <= j) a = m;
            else b = m;
        }
        const long long i = __ldg(lo + a) + (j - __ldg(off + a));
        const double start = dmul((double)(k0 + a), tau);
        xc[j] = dsub(__ldg(x + i), cx);
        yc[j] = dsub(__ldg(y + i), cy);
        const double d = dsub(__ldg(t + i), start);
        tl[j] = d < tau ? d : tau;
    }
}

void launch_window_bounds(const double *t, long long n, long long k0, int nw, double tau,
                          long long *lo, long long *hi, cudaStream_t s)
{
    const int blocks = std::max(1, std::min((nw + 255) / 256, num_sms() * 4));
    k_window_bounds<<<blocks, 256, 0, s>>>(t, n, k0, nw, tau, lo, hi);
}

void launch_gather_windows(const double *x, const double *y, const double *t,
                           const long long *lo, const long long *off, int nw, long long k0,
                           long long total, double tau, double cx, double cy, double *xc,
                           double *yc, double *tl, cudaStream_t s)
{
    k_gather_windows<<<event_blocks(total), kThreads, 0, s>>>(x, y, t, lo, off, nw, k0, tau, cx,
                                                               cy, xc, yc, tl);
}

}  // namespace evd

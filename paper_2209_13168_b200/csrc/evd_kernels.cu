// evd_kernels.cu -- sm_100a kernels of the BnB bound-evaluation hot path.
//
// Standalone kernels back the per-call entry points (accumulate_image,
// upper_bound_image, bound_terms, image_contrast, rasterize_segment,
// radial_warp); k_solve is the device-resident branch-and-bound
// (solver.py:79-123) that evaluates one node per grid-wide step.
#include <cfloat>
#include <climits>

#include "evd_device.cuh"
#include "evd_internal.h"

namespace evd {

constexpr int kThreads = 256;
constexpr int kSolveThreads = 512;

static int g_num_sms = 0;
static int num_sms()
{
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

static int event_blocks(long long n)
{
    long long b = (n + kThreads - 1) / kThreads;
    const long long cap = (long long)num_sms() * 8;
    if (b > cap) b = cap;
    return b < 1 ? 1 : (int)b;
}

struct AtomicSink {
    unsigned int *img;
    __device__ __forceinline__ void operator()(long long p) const { atomicAdd(img + p, 1u); }
};

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

// _bound_image_kernel (contrast.py:185-203) on warps at lo/hi:
// acc[0] += fully-inside segments, acc[1] += marks (= sum of the image)
__global__ void k_bound_image(const double *__restrict__ xc, const double *__restrict__ yc,
                              const double *__restrict__ t, long long n, double lo, double den_lo,
                              double hi, double den_hi, double cx, double cy, int W, int H,
                              unsigned int *img, unsigned long long *acc)
{
    unsigned long long v[2] = {0, 0};
    AtomicSink sink{img};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double x = __ldg(xc + i), y = __ldg(yc + i), tt = __ldg(t + i);
        const Warped a = warp_event(x, y, tt, lo, den_lo, cx, cy);
        const Warped b = warp_event(x, y, tt, hi, den_hi, cx, cy);
        v[0] += fully_inside(a.x, a.y, b.x, b.y, W, H);
        v[1] += raster_segment(a.x, a.y, b.x, b.y, W, H, sink);
    }
    block_add_u64<2>(v, acc);
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

// rasterize_segment (contrast.py:206-222) for k segments, one thread each:
// counts[j*M + p] is incremented once per mark (a dedup failure shows as 2).
__global__ void k_raster_segments(const double *__restrict__ segs, int k, int W, int H,
                                  unsigned int *counts)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    unsigned int *img = counts + (long long)j * W * H;
    auto sink = [img](long long p) { img[p] += 1u; };
    raster_segment(segs[4 * j], segs[4 * j + 1], segs[4 * j + 2], segs[4 * j + 3], W, H, sink);
}

// ---------------------------------------------------------------- contrast tree
// Summands of image_contrast (contrast.py:64): (H_p - mu)**2, numpy square.
struct SqU32 {
    const unsigned int *img;
    double mu;
    __device__ __forceinline__ double operator()(int i) const
    {
        const double d = dsub((double)__ldcg(img + i), mu);
        return dmul(d, d);
    }
};
struct SqU32Clear {  // same, and leaves the pixel zeroed for the next BnB node
    unsigned int *img;
    double mu;
    __device__ __forceinline__ double operator()(int i) const
    {
        const double d = dsub((double)__ldcg(img + i), mu);
        img[i] = 0u;
        return dmul(d, d);
    }
};
struct SqF64 {
    const double *img;
    double mu;
    __device__ __forceinline__ double operator()(int i) const
    {
        const double d = dsub(__ldcg(img + i), mu);
        return dmul(d, d);
    }
};

// Evaluate cut subtree c of the pairwise tree with the whole block; returns
// the subtree sum to every thread.
template <class Q>
__device__ double eval_cut(const TreeDev &T, int c, const Q &q, double *loc)
{
    const int l0 = T.cut_leaf0[c], nl = T.cut_leaf0[c + 1] - l0;
    const int j = threadIdx.x & 7, ngroups = blockDim.x >> 3;
    for (int i = threadIdx.x >> 3; i < nl; i += ngroups) {
        const int2 lf = T.leaves[l0 + i];
        const double v = pairwise_leaf8(lf.x, lf.y, j, q);
        if (j == 0) loc[i] = v;
    }
    __syncthreads();
    const int t0 = T.cut_trip0[c], ni = T.cut_trip0[c + 1] - t0;
    const int *lvl = T.cut_lvl + (long long)c * (kMaxLevels + 1);
    const int nlev = T.cut_nlev[c];
    for (int h = 0; h < nlev; h++) {
        for (int k = lvl[h] + threadIdx.x; k < lvl[h + 1]; k += blockDim.x) {
            const int4 tr = T.trip[t0 + k];
            loc[tr.x] = dadd(loc[tr.y], loc[tr.z]);
        }
        __syncthreads();
    }
    const double r = loc[ni > 0 ? nl + ni - 1 : 0];
    __syncthreads();
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
    const double r = eval_cut(T, blockIdx.x, SqU32{img, mu}, loc);
    if (threadIdx.x == 0) T.cutval[blockIdx.x] = r;
}

__global__ void k_contrast_cuts_f64(const double *img, double mu, TreeDev T)
{
    __shared__ double loc[kCutSmem];
    const double r = eval_cut(T, blockIdx.x, SqF64{img, mu}, loc);
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
__device__ __forceinline__ bool better(double b1, long long c1, double b2, long long c2)
{
    // heapq order on (-c_bar, counter): larger bound first, FIFO among ties
    return b1 > b2 || (b1 == b2 && c1 < c2);
}

__device__ void frontier_push(const SolveArgs &a, volatile SolveState *st, double bound,
                              double lo, double hi)
{
    const long long n = st->fr_n;
    if (n >= a.fr_cap) {
        st->status = kStatusCapacity;
        st->done = 1;
        return;
    }
    volatile FrontierEntry *e = a.fr + n;
    e->bound = bound;
    e->counter = st->next_counter;
    e->lo = lo;
    e->hi = hi;
    st->next_counter = st->next_counter + 1;
    st->fr_n = n + 1;
    if (n + 1 > st->max_fr) st->max_fr = n + 1;
}

// Pop the best frontier node and run the termination test (solver.py:102-108);
// otherwise make it the next node to evaluate.  Whole block.
__device__ void frontier_pop(const SolveArgs &a)
{
    volatile SolveState *st = a.st;
    __shared__ long long s_n;
    __shared__ double r_b[32];
    __shared__ long long r_c[32], r_i[32];
    if (threadIdx.x == 0) s_n = st->fr_n;
    __syncthreads();
    const long long n = s_n;
    if (n == 0) {  // queue exhausted: every interval pruned, gap closed (solver.py:121-122)
        if (threadIdx.x == 0) st->done = 1;
        return;
    }
    double bb = -DBL_MAX;
    long long bc = LLONG_MAX, bi = -1;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double b = __ldcg(&a.fr[i].bound);
        const long long c = __ldcg(&a.fr[i].counter);
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
    if (lane == 0) { r_b[wid] = bb; r_c[wid] = bc; r_i[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++)
            if (r_i[w] >= 0 && (bi < 0 || better(r_b[w], r_c[w], bb, bc))) {
                bb = r_b[w]; bc = r_c[w]; bi = r_i[w];
            }
        volatile FrontierEntry *e = a.fr + bi;
        const double lo = e->lo, hi = e->hi;
        volatile FrontierEntry *last = a.fr + (n - 1);
        e->bound = last->bound;
        e->counter = last->counter;
        e->lo = last->lo;
        e->hi = last->hi;
        st->fr_n = n - 1;
        st->iterations = st->iterations + 1;
        const double gap = dsub(bb, st->c_hat);  // -(-c_bar) - c_hat
        if (gap <= a.gamma || dsub(hi, lo) < a.min_width) {
            st->bound_gap = (0.0 > gap) ? 0.0 : gap;  // Python max(gap, 0.0)
            st->done = 1;
        } else {
            const double c = dmul(0.5, dadd(lo, hi));  // VelocityInterval.center
            st->lo = lo;
            st->hi = hi;
            st->c = c;
            st->den_lo = dadd(1.0, dmul(lo, a.tau));
            st->den_c = dadd(1.0, dmul(c, a.tau));
            st->den_hi = dadd(1.0, dmul(hi, a.tau));
            st->mode = kModeNode;
        }
    }
}

// Runs in the last block to arrive at the end of an iteration: finish the
// contrast of the centre, assemble the child bounds (contrast.py:248-251),
// incumbent update / pruning (solver.py:110-119), then pop the next node.
__device__ void leader_step(const SolveArgs &a, double *scratch)
{
    volatile SolveState *st = a.st;
    const double S = eval_top(a.tree, scratch);
    __shared__ int s_done;
    if (threadIdx.x == 0) {
        const double M = (double)a.tree.M;
        const double C = ddiv(dadd(0.0, S), M);
        const double lo = st->lo, hi = st->hi, c = st->c;
        const unsigned long long fiA = st->acc[1], fiB = st->acc[2];
        const unsigned long long sA = st->acc[3], sB = st->acc[4];
        st->point_evals = st->point_evals + 1;
        if (st->mode == kModeRoot) {
            st->c_hat = C;
            st->nu_hat = c;
            const double cb = dsub(ddiv((double)sA, M), a.pow2[fiA]);
            st->bound_evals = st->bound_evals + 1;
            frontier_push(a, st, cb, lo, hi);
        } else {
            if (C >= st->c_hat) {  // solver.py:111 uses >=
                st->nu_hat = c;
                st->c_hat = C;
            }
            const double cbA = dsub(ddiv((double)sA, M), a.pow2[fiA]);
            const double cbB = dsub(ddiv((double)sB, M), a.pow2[fiB]);
            st->bound_evals = st->bound_evals + 2;
            if (cbA >= st->c_hat) frontier_push(a, st, cbA, lo, c);
            if (cbB >= st->c_hat) frontier_push(a, st, cbB, c, hi);
            if (st->iterations >= a.max_iter && !st->done) {
                st->status = kStatusIterLimit;
                st->done = 1;
            }
        }
        for (int k = 0; k < 8; k++) st->acc[k] = 0ull;
        s_done = st->done;
    }
    __syncthreads();
    if (!s_done) frontier_pop(a);
}

__global__ void __launch_bounds__(kSolveThreads, 1) k_solve(SolveArgs a)
{
    __shared__ double scratch[kCutSmem];
    GridBar *bar = (GridBar *)a.bar;
    volatile SolveState *st = a.st;
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long gsz = (long long)gridDim.x * blockDim.x;
    const int W = a.W, H = a.H;
    while (true) {
        if (st->done) break;
        const int mode = st->mode;
        const double lo = st->lo, hi = st->hi, c = st->c;
        const double den_lo = st->den_lo, den_c = st->den_c, den_hi = st->den_hi;
        __syncthreads();

        // phase 1: every event, three warps (lo, centre, hi); point image at
        // the centre, segment images of both children (root: of the root)
        unsigned long long v[3] = {0, 0, 0};
        AtomicSink sa{a.A}, sb{a.B};
        for (long long i = gtid; i < a.n; i += gsz) {
            const double x = __ldg(a.xc + i), y = __ldg(a.yc + i), t = __ldg(a.t + i);
            const Warped wl = warp_event(x, y, t, lo, den_lo, a.cx, a.cy);
            const Warped wc = warp_event(x, y, t, c, den_c, a.cx, a.cy);
            const Warped wh = warp_event(x, y, t, hi, den_hi, a.cx, a.cy);
            const long long p = floor_bin(wc.x, wc.y, W, H);
            if (p >= 0) {
                atomicAdd(a.P + p, 1u);
                v[0]++;
            }
            if (mode == kModeRoot) {
                v[1] += fully_inside(wl.x, wl.y, wh.x, wh.y, W, H);
                raster_segment(wl.x, wl.y, wh.x, wh.y, W, H, sa);
            } else {
                v[1] += fully_inside(wl.x, wl.y, wc.x, wc.y, W, H);
                raster_segment(wl.x, wl.y, wc.x, wc.y, W, H, sa);
                v[2] += fully_inside(wc.x, wc.y, wh.x, wh.y, W, H);
                raster_segment(wc.x, wc.y, wh.x, wh.y, W, H, sb);
            }
        }
        block_add_u64<3>(v, (unsigned long long *)st->acc);
        grid_barrier(bar, [] {});

        // phase 2: contrast subtrees of the point image, exact sums of squares
        // of both segment images; every image is left zeroed
        const double mu = ddiv((double)st->acc[0], (double)a.tree.M);
        for (int cut = blockIdx.x; cut < a.tree.C; cut += gridDim.x) {
            const double r = eval_cut(a.tree, cut, SqU32Clear{a.P, mu}, scratch);
            if (threadIdx.x == 0) a.tree.cutval[cut] = r;
        }
        unsigned long long w[2] = {0, 0};
        for (long long p = gtid; p < a.tree.M; p += gsz) {
            const unsigned long long ha = __ldcg(a.A + p), hb = __ldcg(a.B + p);
            if (ha) { w[0] += ha * ha; a.A[p] = 0u; }
            if (hb) { w[1] += hb * hb; a.B[p] = 0u; }
        }
        block_add_u64<2>(w, (unsigned long long *)st->acc + 3);
        grid_barrier(bar, [&] { leader_step(a, scratch); });
    }
}

// ---------------------------------------------------------------- launchers
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
    k_bound_image<<<event_blocks(n), kThreads, 0, s>>>(xc, yc, t, n, lo, den_lo, hi, den_hi, cx,
                                                       cy, W, H, img, acc);
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

void launch_contrast_f64(const double *img, double mu, const TreeDev &tree, double *out,
                         cudaStream_t s)
{
    k_contrast_cuts_f64<<<tree.C, kThreads, 0, s>>>(img, mu, tree);
    k_contrast_top<<<1, kThreads, 0, s>>>(tree, out);
}

void launch_raster_segments(const double *segs, int k, int W, int H, unsigned int *counts,
                            cudaStream_t s)
{
    k_raster_segments<<<(k + 127) / 128, 128, 0, s>>>(segs, k, W, H, counts);
}

int solve_block_threads() { return kSolveThreads; }

int solve_grid_blocks(int device)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, kSolveThreads, 0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (per_sm < 1) per_sm = 1;
    return per_sm * sms;
}

cudaError_t launch_solve(const SolveArgs &a, int blocks, cudaStream_t s)
{
    SolveArgs args = a;
    void *params[] = {&args};
    return cudaLaunchCooperativeKernel((const void *)k_solve, dim3(blocks), dim3(kSolveThreads),
                                       params, 0, s);
}

}  // namespace evd

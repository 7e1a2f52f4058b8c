// evd_api.cu -- host side of the C ABI declared in include/evd.h.
//
// Owns device buffers per context, the fixed numpy pairwise-summation plan per
// image size, the libm pow table for the bound assembly, and the launch of the
// device-resident branch and bound.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/evd.h"
#include "evd_device.cuh"
#include "evd_internal.h"

using namespace evd;

namespace {

thread_local std::string g_thread_err;

template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t cap = 0;  // elements
    cudaError_t ensure(size_t n)
    {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(n, 1);
        cudaError_t e = cudaMalloc(&p, want * sizeof(T));
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Host plan of numpy's pairwise tree for M summands, uploaded as TreeDev.
struct TreePlan {
    long long M = -1;
    int cuts_target = -1;
    DevBuf<int2> leaves;
    DevBuf<int> cut_leaf0, cut_trip0, cut_lvl, cut_nlev, top_lvl;
    DevBuf<int4> trip, top;
    DevBuf<double> cutval;
    TreeDev dev{};
};

}  // namespace

struct evd_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    long long launches = 0;
    // resident window
    long long n = -1;
    int W = 0, H = 0;
    double tau = 0.0;
    DevBuf<double> xc, yc, t;
    // scratch
    DevBuf<unsigned int> img;          // 3 images (P, A, B) of the per-call entry points
    DevBuf<unsigned int> simg;         // solve images, per group (always left zeroed)
    DevBuf<unsigned long long> acc;    // 8 accumulators
    DevBuf<double> dscratch;           // misc device doubles
    DevBuf<double> evbuf;              // evd_eval_nodes: lo | hi | results
    DevBuf<double> wx, wy, wt, wxo, wyo;
    DevBuf<double> segs, fargs;
    DevBuf<unsigned int> fimg;          // batched-frontier images (kept zeroed)
    DevBuf<unsigned long long> facc;
    DevBuf<unsigned int> pimg;          // batched point images (kept zeroed)
    DevBuf<double> pargs;
    DevBuf<unsigned long long> pacc;
    DevBuf<unsigned int> seg_counts;
    TreePlan tree;
    // bound assembly table pow(f/M, 2)
    DevBuf<double> pow2;
    long long pow_m = -1, pow_n = -1;
    // solve
    DevBuf<SolveState> state;
    DevBuf<FrontierEntry> frontier;
    DevBuf<GridBar> bar;
    DevBuf<unsigned long long> bar2;   // per-group barrier counters
    DevBuf<long long> woff;            // window offsets
    DevBuf<WindowResult> wres;
    DevBuf<long long> trace, btrace;
    DevBuf<unsigned long long> probe_ctr, probe_span;  // evd_probe_events
    DevBuf<double> sx, sy, st;        // resident raw stream (evd_solve_stream, evd_load_bin)
    DevBuf<signed char> sp;           // its polarity (evd_load_bin)
    DevBuf<unsigned char> sbytes, sscratch;  // EVD1 body, decode scratch
    DevBuf<unsigned int> sflags;
    DevBuf<unsigned int> pcounts;        // evd_pixel_counts
    long long sn = -1;                // resident stream length (-1: none)
    int sW = 0, sH = 0;
    bool s_has_p = false;
    DevBuf<long long> wbounds;        // window lo, hi, offsets
    DevBuf<unsigned int> probe_img;
    long long trace_n = 0;
    bool trace_on = false;  // EVD_TRACE=1 at evd_create: record solve timelines
    int solve_blocks = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // resident-window generation (bumped whenever xc / yc / t change)
    unsigned long long gen = 0;
    // batched frontier (evd_eval_frontier)
    FrontierTiles *tiles = nullptr;
    int frontier_path = EVD_FRONTIER_AUTO;    // evd_set_option("frontier_path")
    long long frontier_budget = 8ll << 30;    // image bytes of the global-image paths
    int last_frontier_path = -1;
    // pinned staging for evd_set_events_list (two halves, double-buffered)
    unsigned char *stage = nullptr;
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    // evd_solve_stream from host arrays: the raw stream is uploaded on a copy
    // stream through a ring of pinned chunk slots while the solve runs
    bool stream_overlap = true;               // evd_set_option("stream_overlap")
    long long feed_chunk = 1ll << 16;         // events per chunk (option "stream_chunk")
    cudaStream_t copy = nullptr;
    cudaEvent_t feed_ev[8] = {};
    cudaEvent_t feed_start = nullptr;
    DevBuf<unsigned long long> feedw;         // [0] raw events delivered, [1] stall flag
    DevBuf<long long> feedb;                  // per window: raw lo, count, unpadded offsets
};

namespace {

int fail(evd_ctx *ctx, int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    g_thread_err = buf;
    return code;
}

#define CU(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(ctx, EVD_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),  \
                        __FILE__, __LINE__);                                                 \
    } while (0)

#define LAUNCHED(k)                                                                          \
    do {                                                                                     \
        ctx->launches += (k);                                                                \
        cudaError_t e_ = cudaGetLastError();                                                 \
        if (e_ != cudaSuccess)                                                               \
            return fail(ctx, EVD_ERR_CUDA, "kernel launch: %s (%s:%d)",                      \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                         \
    } while (0)

// ---- numpy pairwise tree plan (loops_utils.h.src pairwise_sum)
struct PNode {
    long long off, n;
    int l, r, h;
};

int pbuild(std::vector<PNode> &v, long long off, long long n)
{
    const int id = (int)v.size();
    v.push_back({off, n, -1, -1, 0});
    if (n > 128) {  // numpy: n2 = n / 2; n2 -= n2 % 8; pw(a, n2) + pw(a + n2, n - n2)
        long long n2 = n / 2;
        n2 -= n2 % 8;
        const int l = pbuild(v, off, n2);
        const int r = pbuild(v, off + n2, n - n2);
        v[id].l = l;
        v[id].r = r;
        v[id].h = 1 + std::max(v[l].h, v[r].h);
    }
    return id;
}

void pcuts(const std::vector<PNode> &v, int id, long long T, std::vector<int> &cuts)
{
    if (v[id].l < 0 || v[id].n <= T) {
        cuts.push_back(id);
        return;
    }
    pcuts(v, v[id].l, T, cuts);
    pcuts(v, v[id].r, T, cuts);
}

void pcollect(const std::vector<PNode> &v, int id, std::vector<int> &leaves,
              std::vector<int> &internals)
{
    if (v[id].l < 0) {
        leaves.push_back(id);
        return;
    }
    pcollect(v, v[id].l, leaves, internals);
    pcollect(v, v[id].r, leaves, internals);
    internals.push_back(id);
}

int ptop(const std::vector<PNode> &v, int id, const std::vector<int> &cut_index,
         std::vector<int> &top_nodes, std::vector<int> &top_h)
{
    // returns the height above the cut level; records top internals
    if (cut_index[id] >= 0) return 0;
    const int hl = ptop(v, v[id].l, cut_index, top_nodes, top_h);
    const int hr = ptop(v, v[id].r, cut_index, top_nodes, top_h);
    top_nodes.push_back(id);
    top_h.push_back(1 + std::max(hl, hr));
    return 1 + std::max(hl, hr);
}

int ensure_tree(evd_ctx *ctx, long long M, int cuts_target)
{
    TreePlan &tp = ctx->tree;
    if (tp.M == M && tp.cuts_target == cuts_target) return EVD_OK;
    if (M < 1 || M > (1ll << 30)) return fail(ctx, EVD_ERR_ARG, "image size %lld unsupported", M);
    std::vector<PNode> v;
    v.reserve((size_t)(2 * (M / 64 + 2)));
    pbuild(v, 0, M);
    long long T = std::max<long long>(128, (M + cuts_target - 1) / cuts_target);
    std::vector<int> cuts;
    std::vector<int> cut_index;
    // find a cut threshold whose subtrees and top fit the per-block scratch
    while (true) {
        cuts.clear();
        pcuts(v, 0, T, cuts);
        long long worst = 0;
        for (int c : cuts) worst = std::max<long long>(worst, 2 * (v[c].n / 64 + 1));
        // at most one cut per CTA: a CTA that owned two would evaluate them
        // back to back on every node's critical path (measured ~3 us/node)
        if (worst <= kCutSmem && 2 * (long long)cuts.size() <= kCutSmem &&
            (long long)cuts.size() <= std::max(cuts_target, 1))
            break;
        if (worst > kCutSmem) {
            if (2 * (long long)cuts.size() > kCutSmem)
                return fail(ctx, EVD_ERR_ARG, "image size %lld too large for the reduction plan", M);
            T = T * 3 / 4;  // never hit for practical sizes; keeps subtrees small
            if (T < 128) return fail(ctx, EVD_ERR_ARG, "reduction plan failed for M=%lld", M);
        } else {
            T *= 2;
        }
    }
    cut_index.assign(v.size(), -1);
    for (size_t c = 0; c < cuts.size(); c++) cut_index[cuts[c]] = (int)c;

    const int C = (int)cuts.size();
    std::vector<int2> leaves;
    std::vector<int> cut_leaf0{0}, cut_trip0{0}, cut_lvl((size_t)C * (kMaxLevels + 1), 0),
        cut_nlev(C, 0);
    std::vector<int4> trip;
    for (int c = 0; c < C; c++) {
        std::vector<int> lv, in;
        pcollect(v, cuts[c], lv, in);
        // local indices: leaves in order, internals sorted by height
        std::stable_sort(in.begin(), in.end(), [&](int a, int b) { return v[a].h < v[b].h; });
        auto find_local = [&](int node) -> int {
            for (size_t i = 0; i < lv.size(); i++)
                if (lv[i] == node) return (int)i;
            for (size_t i = 0; i < in.size(); i++)
                if (in[i] == node) return (int)(lv.size() + i);
            return -1;
        };
        for (int id : lv) leaves.push_back(make_int2((int)v[id].off, (int)v[id].n));
        int lvl = 0, level_h = 0;
        int *L = &cut_lvl[(size_t)c * (kMaxLevels + 1)];
        for (size_t i = 0; i < in.size(); i++) {
            const int id = in[i];
            const int rel = v[id].h;  // height above the leaves
            if (i == 0 || rel != level_h) {
                if (i > 0) lvl++;
                if (lvl >= kMaxLevels) return fail(ctx, EVD_ERR_ARG, "tree too deep");
                L[lvl] = (int)i;
                level_h = rel;
            }
            trip.push_back(make_int4((int)(lv.size() + i), find_local(v[id].l),
                                     find_local(v[id].r), lvl));  // .w: level
        }
        const int nlev = in.empty() ? 0 : lvl + 1;
        L[nlev] = (int)in.size();
        cut_nlev[c] = nlev;
        cut_leaf0.push_back((int)leaves.size());
        cut_trip0.push_back((int)trip.size());
    }
    // top of the tree above the cuts
    std::vector<int> top_nodes, top_h;
    std::vector<int4> top;
    std::vector<int> top_lvl;
    int top_root = 0, top_levels = 0;
    if (C > 1) {
        ptop(v, 0, cut_index, top_nodes, top_h);
        std::vector<int> order(top_nodes.size());
        for (size_t i = 0; i < order.size(); i++) order[i] = (int)i;
        std::stable_sort(order.begin(), order.end(),
                         [&](int a, int b) { return top_h[a] < top_h[b]; });
        std::vector<int> top_index(v.size(), -1);
        for (int c = 0; c < C; c++) top_index[cuts[c]] = c;
        for (size_t i = 0; i < order.size(); i++) top_index[top_nodes[order[i]]] = C + (int)i;
        int cur_h = -1;
        for (size_t i = 0; i < order.size(); i++) {
            const int id = top_nodes[order[i]];
            if (top_h[order[i]] != cur_h) {
                top_lvl.push_back((int)i);
                cur_h = top_h[order[i]];
            }
            top.push_back(make_int4(top_index[id], top_index[v[id].l], top_index[v[id].r],
                                    (int)top_lvl.size() - 1));  // .w: level
        }
        top_levels = (int)top_lvl.size();
        top_lvl.push_back((int)order.size());
        top_root = top_index[0];
        if (C + (long long)order.size() > kCutSmem) return fail(ctx, EVD_ERR_ARG, "top too large");
    } else {
        top_lvl.push_back(0);
    }
    CU(tp.leaves.ensure(leaves.size()));
    CU(tp.cut_leaf0.ensure(cut_leaf0.size()));
    CU(tp.cut_trip0.ensure(cut_trip0.size()));
    CU(tp.cut_lvl.ensure(cut_lvl.size()));
    CU(tp.cut_nlev.ensure(cut_nlev.size()));
    CU(tp.trip.ensure(std::max<size_t>(trip.size(), 1)));
    CU(tp.top.ensure(std::max<size_t>(top.size(), 1)));
    CU(tp.top_lvl.ensure(top_lvl.size()));
    CU(tp.cutval.ensure(C));
    auto up = [&](void *dst, const void *src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream)
                     : cudaSuccess;
    };
    CU(up(tp.leaves.p, leaves.data(), leaves.size() * sizeof(int2)));
    CU(up(tp.cut_leaf0.p, cut_leaf0.data(), cut_leaf0.size() * sizeof(int)));
    CU(up(tp.cut_trip0.p, cut_trip0.data(), cut_trip0.size() * sizeof(int)));
    CU(up(tp.cut_lvl.p, cut_lvl.data(), cut_lvl.size() * sizeof(int)));
    CU(up(tp.cut_nlev.p, cut_nlev.data(), cut_nlev.size() * sizeof(int)));
    CU(up(tp.trip.p, trip.data(), trip.size() * sizeof(int4)));
    CU(up(tp.top.p, top.data(), top.size() * sizeof(int4)));
    CU(up(tp.top_lvl.p, top_lvl.data(), top_lvl.size() * sizeof(int)));
    CU(cudaStreamSynchronize(ctx->stream));  // host vectors die at return
    TreeDev &d = tp.dev;
    d.M = (int)M;
    d.L = (int)leaves.size();
    d.C = C;
    d.leaves = tp.leaves.p;
    d.cut_leaf0 = tp.cut_leaf0.p;
    d.cut_trip0 = tp.cut_trip0.p;
    d.cut_lvl = tp.cut_lvl.p;
    d.cut_nlev = tp.cut_nlev.p;
    d.trip = tp.trip.p;
    d.top = tp.top.p;
    d.top_lvl = tp.top_lvl.p;
    d.top_levels = top_levels;
    d.top_root = top_root;
    d.cutval = tp.cutval.p;
    tp.M = M;
    tp.cuts_target = cuts_target;
    return EVD_OK;
}

// pow through a volatile pointer so the compiler cannot fold pow(x, 2.0) to x*x:
// CPython's float ** int calls libm pow(), which is not always x*x.
double (*volatile g_pow)(double, double) = pow;

void pow2_fill(long long m, long long n, double *out)
{
    const double dm = (double)m;
    for (long long f = 0; f <= n; f++) out[f] = g_pow((double)f / dm, 2.0);
}

int ensure_pow2(evd_ctx *ctx, long long m, long long n)
{
    if (ctx->pow_m == m && ctx->pow_n >= n) return EVD_OK;
    const long long want = std::max(n, 2 * std::max(ctx->pow_m == m ? ctx->pow_n : 0ll, 1024ll));
    std::vector<double> h((size_t)want + 1);
    pow2_fill(m, want, h.data());
    CU(ctx->pow2.ensure((size_t)want + 1));
    CU(cudaMemcpyAsync(ctx->pow2.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->pow_m = m;
    ctx->pow_n = want;
    return EVD_OK;
}

int need_events(evd_ctx *ctx)
{
    if (ctx->n < 0) return fail(ctx, EVD_ERR_STATE, "no events set (call evd_set_events first)");
    return EVD_OK;
}

int check_den(evd_ctx *ctx, double nu, double tau, double *den)
{
    *den = 1.0 + nu * tau;  // geometry.py:72
    if (!(*den > 0.0))
        return fail(ctx, EVD_ERR_CHEIRALITY, "1 + nu*tau = %.17g <= 0 (nu=%.17g, tau=%.17g)",
                    *den, nu, tau);
    return EVD_OK;
}

// Frame sizes the kernels support: pixel ids fit int (W*H < 2^31) and a
// segment's sample chunks fit the 16-bit field of segment_or_queue_ool's
// packed return (chunks <= (W + H + 4) / C with C >= 1).
int check_frame(evd_ctx *ctx, long long W, long long H)
{
    if (W + H + 4 >= 65536 || W * H >= (1ll << 31))
        return fail(ctx, EVD_ERR_ARG, "sensor %lldx%lld exceeds the supported frame (W+H < 65532, W*H < 2^31)",
                    W, H);
    return EVD_OK;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

int evd_create(int device, evd_ctx **out)
{
    evd_ctx *ctx = nullptr;
    if (!out) return fail(nullptr, EVD_ERR_ARG, "out is NULL");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(nullptr, EVD_ERR_CUDA, "no CUDA device: %s",
                    e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
    if (device < 0 || device >= count)
        return fail(nullptr, EVD_ERR_ARG, "device %d out of range (%d devices)", device, count);
    ctx = new evd_ctx();
    ctx->device = device;
    if (const char *t = getenv("EVD_TRACE")) ctx->trace_on = t[0] == '1';
    CU(cudaSetDevice(device));
    CU(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device));
    CU(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
    ctx->stream = ctx->own;
    CU(cudaEventCreate(&ctx->ev0));
    CU(cudaEventCreate(&ctx->ev1));
    CU(ctx->acc.ensure(8));
    CU(ctx->dscratch.ensure(64));
    *out = ctx;
    return EVD_OK;
}

void evd_destroy(evd_ctx *ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (DevBuf<double> *b : {&ctx->xc, &ctx->yc, &ctx->t, &ctx->dscratch, &ctx->evbuf, &ctx->wx, &ctx->wy,
                              &ctx->wt, &ctx->wxo, &ctx->wyo, &ctx->segs, &ctx->pow2})
        b->release();
    ctx->fargs.release();
    ctx->fimg.release();
    ctx->facc.release();
    ctx->pimg.release();
    ctx->pargs.release();
    ctx->pacc.release();
    ctx->img.release();
    ctx->simg.release();
    ctx->seg_counts.release();
    ctx->acc.release();
    ctx->state.release();
    ctx->frontier.release();
    ctx->bar.release();
    ctx->bar2.release();
    ctx->woff.release();
    ctx->wres.release();
    ctx->trace.release();
    ctx->btrace.release();
    ctx->probe_ctr.release();
    ctx->probe_span.release();
    ctx->probe_img.release();
    ctx->sx.release();
    ctx->sy.release();
    ctx->st.release();
    ctx->wbounds.release();
    ctx->sp.release();
    ctx->sbytes.release();
    ctx->sscratch.release();
    ctx->sflags.release();
    ctx->pcounts.release();
    TreePlan &tp = ctx->tree;
    tp.leaves.release();
    tp.cut_leaf0.release();
    tp.cut_trip0.release();
    tp.cut_lvl.release();
    tp.cut_nlev.release();
    tp.top_lvl.release();
    tp.trip.release();
    tp.top.release();
    tp.cutval.release();
    tiles_free(ctx->tiles);
    ctx->feedw.release();
    ctx->feedb.release();
    for (cudaEvent_t e : ctx->feed_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->feed_start) cudaEventDestroy(ctx->feed_start);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->stage) cudaFreeHost(ctx->stage);
    for (cudaEvent_t e : ctx->stage_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
}

const char *evd_last_error(const evd_ctx *ctx)
{
    return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

int evd_set_stream(evd_ctx *ctx, void *cuda_stream)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    ctx->stream = cuda_stream ? (cudaStream_t)cuda_stream : ctx->own;
    return EVD_OK;
}

int64_t evd_kernel_launches(const evd_ctx *ctx) { return ctx ? ctx->launches : -1; }

int64_t evd_window_generation(const evd_ctx *ctx) { return ctx ? (int64_t)ctx->gen : -1; }

int evd_device_sms(const evd_ctx *ctx) { return ctx ? ctx->sms : -1; }

int evd_set_events(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                   int32_t width, int32_t height, double tau)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (n < 0 || width < 1 || height < 1)
        return fail(ctx, EVD_ERR_ARG, "bad window: n=%lld %dx%d", (long long)n, width, height);
    if (int rc = check_frame(ctx, width, height)) return rc;
    if (!(tau > 0.0)) return fail(ctx, EVD_ERR_ARG, "batch duration tau must be positive");
    if (n > 0 && (!x || !y || !t)) return fail(ctx, EVD_ERR_ARG, "NULL event array");
    CU(cudaSetDevice(ctx->device));
    CU(ctx->xc.ensure(n));
    CU(ctx->yc.ensure(n));
    CU(ctx->t.ensure(n));
    if (n > 0) {
        // raw x, y land in the centred buffers and are centred in place
        CU(cudaMemcpyAsync(ctx->xc.p, x, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        CU(cudaMemcpyAsync(ctx->yc.p, y, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        CU(cudaMemcpyAsync(ctx->t.p, t, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        launch_center(ctx->xc.p, ctx->yc.p, n, width / 2.0, height / 2.0, ctx->xc.p, ctx->yc.p,
                      ctx->stream);
        LAUNCHED(1);
        // inputs are never retained (evd.h): the caller may reuse or free
        // x, y, t (pinned host or device memory) once this call returns
        CU(cudaStreamSynchronize(ctx->stream));
    }
    ctx->n = n;
    ctx->gen++;
    ctx->W = width;
    ctx->H = height;
    ctx->tau = tau;
    return EVD_OK;
}

int evd_set_events_list(evd_ctx *ctx, const double *const *x, const double *const *y,
                        const double *const *t, const int64_t *counts, int32_t k, int32_t width,
                        int32_t height, double tau)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (k < 0 || width < 1 || height < 1 || (k > 0 && (!x || !y || !t || !counts)))
        return fail(ctx, EVD_ERR_ARG, "bad evd_set_events_list arguments");
    if (int rc = check_frame(ctx, width, height)) return rc;
    if (!(tau > 0.0)) return fail(ctx, EVD_ERR_ARG, "batch duration tau must be positive");
    long long n = 0;
    for (int w = 0; w < k; w++) {
        if (counts[w] < 0 || (counts[w] > 0 && (!x[w] || !y[w] || !t[w])))
            return fail(ctx, EVD_ERR_ARG, "bad window %d", w);
        n += counts[w];
    }
    CU(cudaSetDevice(ctx->device));
    CU(ctx->xc.ensure(n));
    CU(ctx->yc.ensure(n));
    CU(ctx->t.ensure(n));
    // Host windows are gathered into two pinned halves while the other half's
    // copy runs: one host pass over the data, no host-side concatenation.
    const size_t half = 16u << 20;
    if (!ctx->stage) {
        CU(cudaHostAlloc(&ctx->stage, 2 * half, cudaHostAllocDefault));
        ctx->stage_bytes = 2 * half;
        CU(cudaEventCreateWithFlags(&ctx->stage_ev[0], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&ctx->stage_ev[1], cudaEventDisableTiming));
    }
    int cur = 0;
    size_t fill = 0;
    double *dst = nullptr;
    long long dpos = 0;  // element offset in dst of the half being filled
    auto flush = [&]() -> int {
        if (!fill) return EVD_OK;
        CU(cudaMemcpyAsync(dst + dpos, ctx->stage + cur * half, fill, cudaMemcpyHostToDevice,
                           ctx->stream));
        CU(cudaEventRecord(ctx->stage_ev[cur], ctx->stream));
        dpos += fill / sizeof(double);
        fill = 0;
        cur ^= 1;
        CU(cudaEventSynchronize(ctx->stage_ev[cur]));  // the next half is free again
        return EVD_OK;
    };
    for (int a = 0; a < 3 && n > 0; a++) {
        const double *const *src = a == 0 ? x : (a == 1 ? y : t);
        dst = a == 0 ? ctx->xc.p : (a == 1 ? ctx->yc.p : ctx->t.p);
        dpos = 0;
        for (int w = 0; w < k; w++) {
            size_t left = (size_t)counts[w] * sizeof(double);
            const unsigned char *p = reinterpret_cast<const unsigned char *>(src[w]);
            while (left) {
                const size_t take = std::min(left, half - fill);
                memcpy(ctx->stage + cur * half + fill, p, take);
                fill += take;
                p += take;
                left -= take;
                if (fill == half) {
                    if (int rc = flush()) return rc;
                }
            }
        }
        if (int rc = flush()) return rc;
    }
    if (n > 0) {
        launch_center(ctx->xc.p, ctx->yc.p, n, width / 2.0, height / 2.0, ctx->xc.p, ctx->yc.p,
                      ctx->stream);
        LAUNCHED(1);
        CU(cudaStreamSynchronize(ctx->stream));
    }
    ctx->n = n;
    ctx->gen++;
    ctx->W = width;
    ctx->H = height;
    ctx->tau = tau;
    return EVD_OK;
}

int evd_radial_warp(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                    double nu, double tau, int32_t width, int32_t height, double *x_out,
                    double *y_out)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    double den;
    int rc = check_den(ctx, nu, tau, &den);
    if (rc) return rc;
    if (n <= 0) return EVD_OK;
    CU(cudaSetDevice(ctx->device));
    CU(ctx->wx.ensure(n));
    CU(ctx->wy.ensure(n));
    CU(ctx->wt.ensure(n));
    CU(ctx->wxo.ensure(n));
    CU(ctx->wyo.ensure(n));
    CU(cudaMemcpyAsync(ctx->wx.p, x, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(ctx->wy.p, y, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(ctx->wt.p, t, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const double cx = width / 2.0, cy = height / 2.0;
    launch_center(ctx->wx.p, ctx->wy.p, n, cx, cy, ctx->wx.p, ctx->wy.p, ctx->stream);
    launch_warp(ctx->wx.p, ctx->wy.p, ctx->wt.p, n, nu, den, cx, cy, ctx->wxo.p, ctx->wyo.p,
                ctx->stream);
    LAUNCHED(2);
    CU(cudaMemcpyAsync(x_out, ctx->wxo.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(y_out, ctx->wyo.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return EVD_OK;
}

int evd_warp_scale(evd_ctx *ctx, const double *t, int64_t n, double nu, double tau,
                   double *s_out)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    double den;
    int rc = check_den(ctx, nu, tau, &den);
    if (rc) return rc;
    if (n <= 0) return EVD_OK;
    CU(cudaSetDevice(ctx->device));
    CU(ctx->wt.ensure(n));
    CU(ctx->wxo.ensure(n));
    CU(cudaMemcpyAsync(ctx->wt.p, t, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    launch_scale(ctx->wt.p, n, nu, den, ctx->wxo.p, ctx->stream);
    LAUNCHED(1);
    CU(cudaMemcpyAsync(s_out, ctx->wxo.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return EVD_OK;
}

}  // extern "C"

namespace {

static int point_images_batched(evd_ctx *ctx, const double *nu, int32_t k, int64_t *in_image,
                                double *contrast)
{
    int rc;
    const long long M = (long long)ctx->W * ctx->H;
    std::vector<double> host(2 * (size_t)k);
    for (int j = 0; j < k; j++) {
        host[j] = nu[j];
        if ((rc = check_den(ctx, nu[j], ctx->tau, &host[(size_t)k + j]))) return rc;
    }
    if ((rc = ensure_tree(ctx, M, ctx->sms))) return rc;
    // images of up to kb velocities at a time (the contrast pass leaves them zeroed)
    long long kb = std::max<long long>(32, (4ll << 30) / (M * 4)) / 32 * 32;
    kb = std::min<long long>(kb, (k + 31) / 32 * 32);
    if ((long long)ctx->pimg.cap < kb * M) {
        CU(ctx->pimg.ensure((size_t)(kb * M)));
        CU(cudaMemsetAsync(ctx->pimg.p, 0, ctx->pimg.cap * sizeof(unsigned int), ctx->stream));
    }
    CU(ctx->pargs.ensure(2 * (size_t)k + (size_t)kb * ctx->tree.dev.C + k));
    CU(ctx->pacc.ensure((size_t)k));
    CU(cudaMemcpyAsync(ctx->pargs.p, host.data(), host.size() * sizeof(double),
                       cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemsetAsync(ctx->pacc.p, 0, (size_t)k * sizeof(unsigned long long), ctx->stream));
    double *d_nu = ctx->pargs.p, *d_den = d_nu + k, *d_out = d_den + k, *d_cut = d_out + k;
    for (long long j0 = 0; j0 < k; j0 += kb) {
        const int kk = (int)std::min<long long>(kb, k - j0);
        launch_points_multi(ctx->xc.p, ctx->yc.p, ctx->t.p, ctx->n, d_nu + j0, d_den + j0, kk,
                            ctx->W / 2.0, ctx->H / 2.0, ctx->W, ctx->H, ctx->pimg.p, M,
                            ctx->pacc.p + j0, ctx->tree.dev, d_cut, d_out + j0, ctx->stream);
        LAUNCHED(3);
    }
    std::vector<unsigned long long> ins((size_t)k);
    CU(cudaMemcpyAsync(ins.data(), ctx->pacc.p, k * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, ctx->stream));
    if (contrast)
        CU(cudaMemcpyAsync(contrast, d_out, k * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (in_image)
        for (int j = 0; j < k; j++) in_image[j] = (int64_t)ins[j];
    return EVD_OK;
}

}  // namespace

extern "C" {

int evd_point_images(evd_ctx *ctx, const double *nu, int32_t k, int64_t *in_image,
                     double *contrast, uint32_t *counts)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    int rc = need_events(ctx);
    if (rc) return rc;
    if (k <= 0) return EVD_OK;
    CU(cudaSetDevice(ctx->device));
    if (!counts && k > 1) return point_images_batched(ctx, nu, k, in_image, contrast);
    const long long M = (long long)ctx->W * ctx->H;
    CU(cudaSetDevice(ctx->device));
    CU(ctx->img.ensure(3 * M));
    CU(ctx->acc.ensure(8));
    if (contrast && (rc = ensure_tree(ctx, M, ctx->sms))) return rc;
    const double cx = ctx->W / 2.0, cy = ctx->H / 2.0;
    for (int j = 0; j < k; j++) {
        double den;
        if ((rc = check_den(ctx, nu[j], ctx->tau, &den))) return rc;
        CU(cudaMemsetAsync(ctx->img.p, 0, M * sizeof(unsigned int), ctx->stream));
        CU(cudaMemsetAsync(ctx->acc.p, 0, 8 * sizeof(unsigned long long), ctx->stream));
        launch_point_image(ctx->xc.p, ctx->yc.p, ctx->t.p, ctx->n, nu[j], den, cx, cy, ctx->W,
                           ctx->H, ctx->img.p, ctx->acc.p, ctx->stream);
        LAUNCHED(1);
        if (contrast) {
            launch_contrast_u32(ctx->img.p, ctx->acc.p, ctx->tree.dev, ctx->dscratch.p,
                                ctx->stream);
            LAUNCHED(2);
            CU(cudaMemcpyAsync(contrast + j, ctx->dscratch.p, sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->stream));
        }
        unsigned long long hacc = 0;
        CU(cudaMemcpyAsync(&hacc, ctx->acc.p, sizeof hacc, cudaMemcpyDeviceToHost, ctx->stream));
        if (counts)
            CU(cudaMemcpyAsync(counts + (size_t)j * M, ctx->img.p, M * sizeof(unsigned int),
                               cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (in_image) in_image[j] = (int64_t)hacc;
    }
    return EVD_OK;
}

int evd_bound_images(evd_ctx *ctx, const double *lo, const double *hi, int32_t k,
                     uint64_t *s_bar, int64_t *fully_inside, uint64_t *marks, uint32_t *counts)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    int rc = need_events(ctx);
    if (rc) return rc;
    const long long M = (long long)ctx->W * ctx->H;
    CU(cudaSetDevice(ctx->device));
    CU(ctx->img.ensure(3 * M));
    CU(ctx->acc.ensure(8));
    const double cx = ctx->W / 2.0, cy = ctx->H / 2.0;
    for (int j = 0; j < k; j++) {
        if (lo[j] > hi[j]) return fail(ctx, EVD_ERR_ARG, "empty interval [%.17g, %.17g]", lo[j], hi[j]);
        double dl, dh;
        if ((rc = check_den(ctx, lo[j], ctx->tau, &dl))) return rc;
        if ((rc = check_den(ctx, hi[j], ctx->tau, &dh))) return rc;
        CU(cudaMemsetAsync(ctx->img.p, 0, M * sizeof(unsigned int), ctx->stream));
        CU(cudaMemsetAsync(ctx->acc.p, 0, 8 * sizeof(unsigned long long), ctx->stream));
        launch_bound_image(ctx->xc.p, ctx->yc.p, ctx->t.p, ctx->n, lo[j], dl, hi[j], dh, cx, cy,
                           ctx->W, ctx->H, ctx->img.p, ctx->acc.p, ctx->stream);
        launch_image_sums(ctx->img.p, M, ctx->acc.p + 2, ctx->stream);
        LAUNCHED(2);
        unsigned long long h[4];
        CU(cudaMemcpyAsync(h, ctx->acc.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        if (counts)
            CU(cudaMemcpyAsync(counts + (size_t)j * M, ctx->img.p, M * sizeof(unsigned int),
                               cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (h[1] != h[2])
            return fail(ctx, EVD_ERR_CUDA, "internal: marks %llu != image sum %llu", h[1], h[2]);
        if (fully_inside) fully_inside[j] = (int64_t)h[0];
        if (marks) marks[j] = h[2];
        if (s_bar) s_bar[j] = h[3];
    }
    return EVD_OK;
}

constexpr int kFrontierSmallK = 32;  // auto: per-interval passes up to this many intervals

int evd_eval_frontier(evd_ctx *ctx, const double *lo, const double *hi, int32_t k,
                      uint64_t *s_bar, int64_t *fully_inside, uint64_t *marks)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    int rc = need_events(ctx);
    if (rc) return rc;
    if (k < 0) return fail(ctx, EVD_ERR_ARG, "negative interval count");
    if (k == 0) return EVD_OK;
    const long long M = (long long)ctx->W * ctx->H;
    std::vector<double> host(4 * (size_t)k);
    bool nonpositive = true;  // every nu <= 0: the warp scale is >= 1 (tiled path)
    bool contig = true;       // lo[j+1] == hi[j]: adjacent intervals share an endpoint warp
    for (int j = 0; j < k; j++) {
        if (lo[j] > hi[j]) return fail(ctx, EVD_ERR_ARG, "empty interval [%.17g, %.17g]", lo[j], hi[j]);
        if ((rc = check_den(ctx, lo[j], ctx->tau, &host[2 * (size_t)k + j]))) return rc;
        if ((rc = check_den(ctx, hi[j], ctx->tau, &host[3 * (size_t)k + j]))) return rc;
        host[j] = lo[j];
        host[(size_t)k + j] = hi[j];
        nonpositive = nonpositive && hi[j] <= 0.0;
        if (j > 0 && lo[j] != hi[j - 1]) contig = false;
    }
    // A few intervals: one k_bound_image pass each (lane = event) beats the
    // frontier kernels (lane = interval, mostly idle lanes at small k): cfg 5
    // root 11.6 vs 21.5 ms, 32 intervals of width 1/16 30.7 vs 45.7 ms
    // (tools/probe_small_k.py)
    if (ctx->frontier_path == EVD_FRONTIER_PER_INTERVAL ||
        (ctx->frontier_path == EVD_FRONTIER_AUTO && k <= kFrontierSmallK)) {
        rc = evd_bound_images(ctx, lo, hi, k, s_bar, fully_inside, marks, nullptr);
        if (!rc) ctx->last_frontier_path = EVD_FRONTIER_PER_INTERVAL;
        return rc;
    }
    CU(cudaSetDevice(ctx->device));
    CU(ctx->fargs.ensure(4 * (size_t)k));
    CU(ctx->facc.ensure(3 * (size_t)k));
    CU(cudaMemcpyAsync(ctx->fargs.p, host.data(), host.size() * sizeof(double),
                       cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemsetAsync(ctx->facc.p, 0, 3 * (size_t)k * sizeof(unsigned long long), ctx->stream));
    const double *d_lo = ctx->fargs.p, *d_hi = d_lo + k, *d_dl = d_lo + 2 * k, *d_dh = d_lo + 3 * k;
    unsigned long long *f_fi = ctx->facc.p, *f_ms = f_fi + k;  // fi[k], then (marks, s_bar)[k]
    const int path = ctx->frontier_path;
    bool tiled = false;
    if ((path == EVD_FRONTIER_AUTO || path == EVD_FRONTIER_TILES) && nonpositive && ctx->n > 0) {
        if (!ctx->tiles) ctx->tiles = tiles_new();
        int nl = 0;
        CU(tiles_bin(ctx->tiles, ctx->xc.p, ctx->yc.p, ctx->t.p, ctx->n, ctx->W, ctx->H, ctx->gen,
                     &tiled, &nl, ctx->stream));
        LAUNCHED(nl);
    }
    if (path == EVD_FRONTIER_TILES && !tiled && ctx->n > 0)
        return fail(ctx, EVD_ERR_STATE, "tiled frontier does not apply to this window/intervals "
                                        "(frame not tileable, non-finite events, nu > 0 or a "
                                        "tile over 65535 events)");
    if (tiled) {
        int nl = 0;
        CU(tiles_eval(ctx->tiles, d_lo, d_hi, d_dl, d_dh, k, contig, f_fi, f_ms, &nl,
                      ctx->stream));
        LAUNCHED(nl);
        ctx->last_frontier_path = EVD_FRONTIER_TILES;
    } else if (ctx->n > 0) {
        // images of up to kb intervals at a time in HBM (kept zeroed between calls)
        const bool exact_only = path == EVD_FRONTIER_GLOBAL_EXACT;
        long long kb = std::max<long long>(1, ctx->frontier_budget / (M * 4));
        kb = std::min<long long>(kb, k);
        kb = (kb + kFrontGroupHost - 1) / kFrontGroupHost * kFrontGroupHost;
        if ((long long)ctx->fimg.cap < kb * M) {
            CU(ctx->fimg.ensure((size_t)(kb * M)));
            CU(cudaMemsetAsync(ctx->fimg.p, 0, ctx->fimg.cap * sizeof(unsigned int), ctx->stream));
        }
        for (long long j0 = 0; j0 < k; j0 += kb) {
            const int kk = (int)std::min<long long>(kb, k - j0);
            launch_frontier(ctx->xc.p, ctx->yc.p, ctx->t.p, ctx->n, d_lo + j0, d_hi + j0, d_dl + j0,
                            d_dh + j0, kk, ctx->W / 2.0, ctx->H / 2.0, ctx->W, ctx->H, ctx->fimg.p, M,
                            f_fi + j0, f_ms + 2 * j0, exact_only, ctx->stream);
            LAUNCHED(2);
        }
        ctx->last_frontier_path = exact_only ? EVD_FRONTIER_GLOBAL_EXACT : EVD_FRONTIER_GLOBAL;
    }
    std::vector<unsigned long long> out(3 * (size_t)k);
    CU(cudaMemcpyAsync(out.data(), ctx->facc.p, out.size() * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int j = 0; j < k; j++) {
        if (fully_inside) fully_inside[j] = (int64_t)out[j];
        if (marks) marks[j] = out[(size_t)k + 2 * j];
        if (s_bar) s_bar[j] = out[(size_t)k + 2 * j + 1];
    }
    return EVD_OK;
}

int evd_set_option(evd_ctx *ctx, const char *name, int64_t value)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!name) return fail(ctx, EVD_ERR_ARG, "option name is NULL");
    if (!strcmp(name, "frontier_path")) {
        if (value < EVD_FRONTIER_AUTO || value > EVD_FRONTIER_PER_INTERVAL)
            return fail(ctx, EVD_ERR_ARG, "frontier_path %lld out of range", (long long)value);
        ctx->frontier_path = (int)value;
        return EVD_OK;
    }
    if (!strcmp(name, "stream_overlap")) {
        if (value != 0 && value != 1) return fail(ctx, EVD_ERR_ARG, "stream_overlap must be 0 or 1");
        ctx->stream_overlap = value != 0;
        return EVD_OK;
    }
    if (!strcmp(name, "stream_chunk")) {
        if (value < 1024 || value > (1ll << 18))
            return fail(ctx, EVD_ERR_ARG, "stream_chunk must be in [1024, 262144] events");
        ctx->feed_chunk = value;
        return EVD_OK;
    }
    if (!strcmp(name, "frontier_image_budget")) {
        if (value < 1) return fail(ctx, EVD_ERR_ARG, "frontier_image_budget must be positive");
        ctx->frontier_budget = value;
        return EVD_OK;
    }
    return fail(ctx, EVD_ERR_ARG, "unknown option '%s'", name);
}

int evd_frontier_info(evd_ctx *ctx, int64_t *out)
{
    if (!ctx || !out) return fail(ctx, EVD_ERR_ARG, "NULL argument");
    long long v[4] = {0, 0, -1, 0};
    if (ctx->tiles) tiles_info(ctx->tiles, v);
    for (int i = 0; i < 4; i++) out[i] = v[i];
    out[4] = ctx->last_frontier_path;
    return EVD_OK;
}

int evd_image_contrast(evd_ctx *ctx, const double *counts, int64_t m, int64_t in_image,
                       double *contrast)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (m < 1) return fail(ctx, EVD_ERR_ARG, "image must have at least one pixel");
    CU(cudaSetDevice(ctx->device));
    int rc = ensure_tree(ctx, m, ctx->sms);
    if (rc) return rc;
    CU(ctx->wx.ensure(m));
    CU(cudaMemcpyAsync(ctx->wx.p, counts, m * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const double mu = (double)in_image / (double)m;  // EventImage.mean (contrast.py:35-36)
    launch_contrast_f64(ctx->wx.p, mu, ctx->tree.dev, ctx->dscratch.p, ctx->stream);
    LAUNCHED(2);
    CU(cudaMemcpyAsync(contrast, ctx->dscratch.p, sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return EVD_OK;
}

int evd_rasterize_segments(evd_ctx *ctx, const double *segs, int32_t k, int32_t width,
                           int32_t height, int32_t chunk, uint32_t *counts)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (width < 1 || height < 1 || k < 0) return fail(ctx, EVD_ERR_ARG, "bad raster request");
    if (int rc = check_frame(ctx, width, height)) return rc;
    if (k == 0) return EVD_OK;
    const size_t M = (size_t)width * height;
    CU(cudaSetDevice(ctx->device));
    CU(ctx->segs.ensure(4 * (size_t)k));
    CU(ctx->seg_counts.ensure(M * k));
    CU(cudaMemcpyAsync(ctx->segs.p, segs, 4 * k * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CU(cudaMemsetAsync(ctx->seg_counts.p, 0, M * k * sizeof(unsigned int), ctx->stream));
    launch_raster_segments(ctx->segs.p, k, width, height, chunk, ctx->seg_counts.p, ctx->stream);
    LAUNCHED(1);
    CU(cudaMemcpyAsync(counts, ctx->seg_counts.p, M * k * sizeof(unsigned int),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return EVD_OK;
}

}  // extern "C"

namespace {

// Run the device-resident BnB over n_windows windows of the resident events
// (window w = events [off[w], off[w+1])) with `groups` independent CTA groups.
// The filtered event path (approximate warps certified by error margins,
// exact fallback) was a win at ~1M events before the sampler's position-based
// chunks; it now measures 1-3% slower at every size (cfg 1, 2, 3, 5), so it is
// off unless EVD_SOLVE_FILTER=1 (kept: tested, and a base for other targets).
constexpr long long kFilterMinEvents = LLONG_MAX;
// 4 speculative slots below this, 2 above (cfg 5, 5.33 M events: 1 slot
// 138.1 ms, 2 slots 135.8, 3 137.4, 4 136.2 -- measured after the round-2
// step changes; before them 1 slot was best there)
constexpr long long kSpecMaxEvents = 2000000;
// CTA-size / slot-count policy for a whole-grid solve, from
// tools/threshold_sweep.py (subsampled cfg 2 / cfg 3 windows and cfg 1):
// 384 threads + 3 slots win at 20 k events, 512 + 4 slots at 50-150 k,
// 512 and 768 tie at 204 k, 768 + 4 slots wins from 400 k
constexpr long long kSmallWindow = 32768;     // 384-thread CTAs below this
constexpr long long kLargeWindow = 250000;    // 768-thread CTAs from this on

// Overlapped upload of a host stream into a running solve (evd_solve_stream):
// the device arrays k_solve / k_solve_spec gather from, and the host loop that
// feeds them (issued once, right after the first launch).
struct StreamFeed {
    const double *sx, *sy, *st;       // device: the raw events as they arrive
    const long long *s_lo, *counts;   // device, per window
    const long long *h_counts;        // host copy of counts
    long long k0;
    int t_local;                      // 1: t is window-local already (no shift)
    std::function<int()> upload;
};

// evd_eval_nodes: node intervals (device) and their results (device, 3 each)
struct EvalList {
    const double *lo, *hi;
    long long n;
    double *out;
};

// evd_solve_events: the window's upload, queued on the copy stream before
// the solve (run_windows calls it right before the launch)
struct Progressive {
    std::function<int()> upload;  // queues the window's copies on ctx->copy
};

static int run_windows(evd_ctx *ctx, const long long *off, int n_windows, int groups,
                       const evd_solve_params *params, std::vector<WindowResult> &out,
                       float *ms_out, StreamFeed *feed = nullptr, const EvalList *ev = nullptr,
                       Progressive *prog = nullptr)
{
    int rc;
    if (!(params->gamma > 0.0)) return fail(ctx, EVD_ERR_ARG, "gamma must be positive");
    const double tau = ctx->tau, eps = params->epsilon;
    if (!(eps >= 0.0 && eps < 1.0)) return fail(ctx, EVD_ERR_ARG, "epsilon must be in [0, 1)");
    // velocity_domain (geometry.py:61-67) and the first warps the reference makes
    const double lo0 = -(1.0 - eps) / tau, hi0 = 0.0, c0 = 0.5 * (lo0 + hi0);
    double den_c, den_lo, den_hi;
    if ((rc = check_den(ctx, c0, tau, &den_c))) return rc;    // contrast_at(center), solver.py:93
    if ((rc = check_den(ctx, lo0, tau, &den_lo))) return rc;  // bound_terms(domain), solver.py:97
    if ((rc = check_den(ctx, hi0, tau, &den_hi))) return rc;
    const long long M = (long long)ctx->W * ctx->H;
    CU(cudaSetDevice(ctx->device));
    if (!ctx->solve_blocks) ctx->solve_blocks = solve_grid_blocks(ctx->device);
    groups = std::max(1, std::min(groups, ctx->solve_blocks));
    const int GB = ctx->solve_blocks / groups;
    long long max_n = 0;
    for (int w = 0; w < n_windows; w++)
        max_n = std::max(max_n, feed ? feed->h_counts[w] : off[w + 1] - off[w]);
    // speculative rounds (k_solve_spec) unless EVD_SPEC_K=1 or the timeline
    // trace is on (k_solve has the probes)
    // (on the whole grid: 3 slots measured best with 384-thread CTAs, 4 above,
    // up to 2 M events -- cfg 3 20.07 -> 19.86 ms; 2 at cfg 5 (5.3 M), where
    // the wide nodes leave less fixed cost to save; small CTA groups have
    // little fixed cost to save)
    int spec_k = GB < 32 ? 1 : (max_n < kSmallWindow ? 3 : (max_n < kSpecMaxEvents ? 4 : 2));
    if (const char *e = getenv("EVD_SPEC_K")) spec_k = std::max(1, std::min(kSpecK, atoi(e)));
    if (ctx->trace_on && !getenv("EVD_TRACE_SPEC")) spec_k = 1;  // EVD_TRACE_SPEC=1: rounds
    // k_solve_spec certifies the root bound instead of rasterising it
    // (kModeRootCert) unless the root is narrower than min_interval_width
    // (then its exact bound is the result's bound_gap, solver.py:106-108)
    int root_cert = (hi0 - lo0 < params->min_interval_width || getenv("EVD_NO_ROOT_CERT")) ? 0 : 1;
    if (ev) root_cert = 0;
    // CTA size: small windows on the whole grid are latency-bound (384 fatter
    // threads), large ones sampler-throughput-bound (768); grouped solves and
    // the traced build stay at 512 (measured: cfg 1 1.10 -> 1.04 ms at 384,
    // cfg 3 21.5 -> 20.3 ms at 768, cfg 2 and cfg 4 best at 512)
    int threads = 512;
    if (GB >= 32 && !ctx->trace_on)
        threads = max_n < kSmallWindow ? 384 : (max_n >= kLargeWindow ? 768 : 512);
    if (const char *e = getenv("EVD_SOLVE_BLOCK")) threads = atoi(e);
    if ((rc = ensure_pow2(ctx, M, max_n))) return rc;
    if (ctx->simg.cap < (size_t)(3 * kSpecK * M * groups)) {  // the kernels leave them zeroed
        CU(ctx->simg.ensure((size_t)(3 * kSpecK * M * groups)));
        CU(cudaMemsetAsync(ctx->simg.p, 0, ctx->simg.cap * sizeof(unsigned int), ctx->stream));
    }
    CU(ctx->state.ensure(groups));
    CU(ctx->bar2.ensure(2 * (size_t)groups));
    if (ctx->trace_on) {
        CU(ctx->trace.ensure(1 + kTraceSlots * kTraceIters));
        CU(ctx->btrace.ensure((size_t)kBTraceIters * kBTraceMaxBlocks * kBTraceSlots));
        CU(cudaMemsetAsync(ctx->trace.p, 0, (1 + kTraceSlots * kTraceIters) * sizeof(long long),
                           ctx->stream));
    }
    CU(ctx->woff.ensure(n_windows + 1));
    CU(ctx->wres.ensure(n_windows));
    CU(cudaMemcpyAsync(ctx->woff.p, off, (n_windows + 1) * sizeof(long long),
                       cudaMemcpyHostToDevice, ctx->stream));
    long long cap = std::max<long long>(4096, (long long)(ctx->frontier.cap / groups));
    const long long need = params->max_iterations + 2;
    if (need > 0 && need < cap) cap = need;
    out.assign(n_windows, WindowResult{});
    std::vector<int> todo(n_windows);
    for (int w = 0; w < n_windows; w++) todo[w] = w;
    float total_ms = 0.f;
    while (true) {
        // cut plan: one cut per CTA, or per (slot, CTA) pair for speculative rounds
        if ((rc = ensure_tree(ctx, M, spec_k > 1 ? std::max(1, GB / spec_k) : GB))) return rc;
        CU(ctx->tree.cutval.ensure((size_t)ctx->tree.dev.C * kSpecK * groups));
        ctx->tree.dev.cutval = ctx->tree.cutval.p;
        CU(ctx->frontier.ensure((size_t)(cap * groups)));
        CU(cudaMemsetAsync(ctx->bar2.p, 0, 2 * groups * sizeof(unsigned long long), ctx->stream));
        CU(cudaMemsetAsync(ctx->wres.p, 0, n_windows * sizeof(WindowResult), ctx->stream));
        SolveArgs a{};
        a.xc = ctx->xc.p;
        a.yc = ctx->yc.p;
        a.t = ctx->t.p;
        a.offsets = ctx->woff.p;
        a.n_windows = n_windows;
        a.groups = groups;
        a.group_blocks = GB;
        a.W = ctx->W;
        a.H = ctx->H;
        a.cx = ctx->W / 2.0;
        a.cy = ctx->H / 2.0;
        a.tau = tau;
        a.lo0 = lo0;
        a.hi0 = hi0;
        a.c0 = c0;
        a.den_lo0 = den_lo;
        a.den_c0 = den_c;
        a.den_hi0 = den_hi;
        a.img = ctx->simg.p;
        a.tree = ctx->tree.dev;
        a.pow2 = ctx->pow2.p;
        a.gamma = params->gamma;
        a.min_width = params->min_interval_width;
        a.max_iter = params->max_iterations;
        a.st = ctx->state.p;
        a.fr = ctx->frontier.p;
        a.fr_cap = cap;
        a.bar = ctx->bar2.p;
        a.res = ctx->wres.p;
        a.trace = ctx->trace_on ? ctx->trace.p : nullptr;
        a.trace_iters = kTraceIters;
        a.btrace = ctx->trace_on ? ctx->btrace.p : nullptr;
        a.filter = (max_n >= kFilterMinEvents) ? 1 : 0;
        if (const char *f = getenv("EVD_SOLVE_FILTER")) a.filter = (f[0] == '1');  // tests / tuning
        a.spec_k = spec_k;
        a.root_cert = root_cert;
        if (ev) {
            a.ev_lo = ev->lo;
            a.ev_hi = ev->hi;
            a.ev_n = ev->n;
            a.ev_out = ev->out;
        }
        if (feed) {
            a.sx = feed->sx;
            a.sy = feed->sy;
            a.stt = feed->st;
            a.t_local = feed->t_local;
            a.s_lo = feed->s_lo;
            a.counts = feed->counts;
            a.ready = ctx->feedw.p;
            a.stall = reinterpret_cast<unsigned int *>(ctx->feedw.p + 1);
            a.gx = ctx->xc.p;
            a.gy = ctx->yc.p;
            a.gt = ctx->t.p;
            a.k0 = feed->k0;
        }
        const bool spec_launch = spec_k > 1 || ev || getenv("EVD_SPEC_FORCE");
        if (prog && prog->upload) {
            // the solve reads centred events from its first node on: upload,
            // then centre on the solve's stream
            const int urc = prog->upload();
            prog->upload = nullptr;
            if (urc) return urc;
            CU(cudaEventRecord(ctx->feed_start, ctx->copy));
            CU(cudaStreamWaitEvent(ctx->stream, ctx->feed_start, 0));
            launch_center(ctx->xc.p, ctx->yc.p, ctx->n, ctx->W / 2.0, ctx->H / 2.0, ctx->xc.p,
                          ctx->yc.p, ctx->stream);
            LAUNCHED(1);
        }
        CU(cudaEventRecord(ctx->ev0, ctx->stream));
        CU(spec_launch
               ? launch_solve_spec(a, groups * GB, threads, ctx->stream)
               : launch_solve(a, groups * GB, threads, ctx->stream));
        LAUNCHED(1);
        CU(cudaEventRecord(ctx->ev1, ctx->stream));
        if (feed && feed->upload) {
            // the solve waits on the chunks: feed them now (host copies into
            // pinned slots, device copies on ctx->copy)
            const int urc = feed->upload();
            feed->upload = nullptr;
            if (urc) {
                // release the waiting groups (their windows are garbage), then report
                cudaMemsetAsync(ctx->feedw.p, 0xff, sizeof(unsigned long long), ctx->copy);
                cudaStreamSynchronize(ctx->stream);
                return urc;
            }
        }
        std::vector<WindowResult> got(n_windows);
        CU(cudaMemcpyAsync(got.data(), ctx->wres.p, n_windows * sizeof(WindowResult),
                           cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        total_ms += ms;
        if (feed) {
            unsigned long long stall = 0;
            CU(cudaMemcpyAsync(&stall, ctx->feedw.p + 1, sizeof stall, cudaMemcpyDeviceToHost,
                               ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
            if (stall) return fail(ctx, EVD_ERR_CUDA, "stream upload did not arrive in time");
        }
        bool again = false, overflow = false, uncertified = false;
        for (int w : todo) {
            out[w] = got[w];
            if (got[w].status == kStatusCapacity) again = true;
            if (got[w].status == kStatusSpecOverflow) overflow = true;
            if (got[w].status == kStatusRootCert) uncertified = true;
        }
        if (uncertified) {  // a root bound near c_hat + gamma: rerun with it rasterised
            root_cert = 0;
            continue;
        }
        if (overflow) {  // the shared-memory frontier filled up: rerun without speculation
            spec_k = 1;
            continue;
        }
        if (!again) break;
        cap *= 8;  // frontier outgrew its buffer: rerun (the solve is deterministic)
    }
    ctx->trace_n = !ctx->trace_on ? 0 : 1 + kTraceSlots * std::min<long long>(out[0].iterations + 1, kTraceIters);
    if (ms_out) *ms_out = total_ms;
    return EVD_OK;
}

}  // namespace

extern "C" {

int evd_solve_events(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                     int32_t width, int32_t height, double tau, const evd_solve_params *params,
                     evd_solve_result *res)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!params || !res) return fail(ctx, EVD_ERR_ARG, "params/result is NULL");
    if (n < 0 || width < 1 || height < 1)
        return fail(ctx, EVD_ERR_ARG, "bad window: n=%lld %dx%d", (long long)n, width, height);
    if (int rc = check_frame(ctx, width, height)) return rc;
    if (!(tau > 0.0)) return fail(ctx, EVD_ERR_ARG, "batch duration tau must be positive");
    if (n > 0 && (!x || !y || !t)) return fail(ctx, EVD_ERR_ARG, "NULL event array");
    memset(res, 0, sizeof *res);
    if (n == 0) {
        ctx->n = 0;
        ctx->gen++;
        ctx->W = width;
        ctx->H = height;
        ctx->tau = tau;
        return fail(ctx, EVD_ERR_NO_EVENTS, "no events in batch");
    }
    CU(cudaSetDevice(ctx->device));
    CU(ctx->xc.ensure(n));
    CU(ctx->yc.ensure(n));
    CU(ctx->t.ensure(n));
    if (!ctx->copy) CU(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
    if (!ctx->feed_start) {
        CU(cudaEventCreateWithFlags(&ctx->feed_start, cudaEventDisableTiming));
        for (cudaEvent_t &e : ctx->feed_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ctx->n = n;
    ctx->gen++;
    ctx->W = width;
    ctx->H = height;
    ctx->tau = tau;
    // the copies start after everything queued so far (earlier readers of
    // the window buffers); run_windows queues them on the copy stream right
    // before the launch, the centring and the solve after them on ctx->stream
    CU(cudaEventRecord(ctx->feed_start, ctx->stream));
    CU(cudaStreamWaitEvent(ctx->copy, ctx->feed_start, 0));
    Progressive prog;
    prog.upload = [&]() -> int {
        CU(cudaMemcpyAsync(ctx->xc.p, x, n * sizeof(double), cudaMemcpyDefault, ctx->copy));
        CU(cudaMemcpyAsync(ctx->yc.p, y, n * sizeof(double), cudaMemcpyDefault, ctx->copy));
        CU(cudaMemcpyAsync(ctx->t.p, t, n * sizeof(double), cudaMemcpyDefault, ctx->copy));
        return EVD_OK;
    };
    const long long off[2] = {0, n};
    std::vector<WindowResult> out;
    float ms = 0.f;
    int rc = run_windows(ctx, off, 1, 1, params, out, &ms, nullptr, nullptr, &prog);
    // inputs are never retained: the copies are done before returning
    cudaError_t ce = cudaStreamSynchronize(ctx->copy);
    if (ce != cudaSuccess || (rc && rc != EVD_ERR_ITER_LIMIT)) {
        // a parameter error returns before the upload, a CUDA error may stop
        // it half-way: either way nothing is resident
        ctx->n = -1;
        ctx->gen++;
    }
    if (rc) return rc;
    if (ce != cudaSuccess) return fail(ctx, EVD_ERR_CUDA, "upload: %s", cudaGetErrorString(ce));
    const WindowResult &w = out[0];
    res->nu = w.nu;
    res->contrast = w.contrast;
    res->bound_gap = w.bound_gap;
    res->iterations = w.iterations;
    res->bound_evals = w.bound_evals;
    res->point_evals = w.point_evals;
    res->max_frontier = w.max_fr;
    res->marks = w.marks;
    res->exact_events = w.exact;
    res->rounds = w.rounds;
    res->device_ms = ms;
    if (w.status == kStatusIterLimit)
        return fail(ctx, EVD_ERR_ITER_LIMIT,
                    "iteration limit reached after %lld iterations (best nu=%.17g, contrast=%.17g)",
                    w.iterations, w.nu, w.contrast);
    return EVD_OK;
}

int evd_eval_nodes(evd_ctx *ctx, const double *lo, const double *hi, int64_t k,
                   double *contrast, double *cbar_lo, double *cbar_hi)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (k < 0 || (k > 0 && (!lo || !hi || !contrast || !cbar_lo || !cbar_hi)))
        return fail(ctx, EVD_ERR_ARG, "bad node list");
    int rc = need_events(ctx);
    if (rc) return rc;
    if (k == 0) return EVD_OK;
    if (ctx->n == 0) return fail(ctx, EVD_ERR_NO_EVENTS, "no events in batch");
    for (int64_t i = 0; i < k; i++) {
        if (!(lo[i] <= hi[i]))
            return fail(ctx, EVD_ERR_ARG, "empty interval [%.17g, %.17g]", lo[i], hi[i]);
        double d;
        if ((rc = check_den(ctx, lo[i], ctx->tau, &d))) return rc;
        if ((rc = check_den(ctx, hi[i], ctx->tau, &d))) return rc;
    }
    CU(cudaSetDevice(ctx->device));
    CU(ctx->evbuf.ensure((size_t)(5 * k)));
    std::vector<double> h(2 * k);
    std::copy(lo, lo + k, h.begin());
    std::copy(hi, hi + k, h.begin() + k);
    CU(cudaMemcpyAsync(ctx->evbuf.p, h.data(), 2 * k * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    const EvalList ev{ctx->evbuf.p, ctx->evbuf.p + k, k, ctx->evbuf.p + 2 * k};
    const evd_solve_params params{1.0, 1e-6, 0.0, 1};  // unused by an evaluation-only launch
    const long long off[2] = {0, ctx->n};
    std::vector<WindowResult> out;
    float ms = 0.f;
    if ((rc = run_windows(ctx, off, 1, 1, &params, out, &ms, nullptr, &ev))) return rc;
    std::vector<double> r(3 * k);
    CU(cudaMemcpyAsync(r.data(), ev.out, 3 * k * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < k; i++) {
        contrast[i] = r[3 * i];
        cbar_lo[i] = r[3 * i + 1];
        cbar_hi[i] = r[3 * i + 2];
    }
    return EVD_OK;
}

int evd_solve(evd_ctx *ctx, const evd_solve_params *params, evd_solve_result *res)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!params || !res) return fail(ctx, EVD_ERR_ARG, "params/result is NULL");
    int rc = need_events(ctx);
    if (rc) return rc;
    memset(res, 0, sizeof *res);
    if (ctx->n == 0) return fail(ctx, EVD_ERR_NO_EVENTS, "no events in batch");
    const long long off[2] = {0, ctx->n};
    std::vector<WindowResult> out;
    float ms = 0.f;
    if ((rc = run_windows(ctx, off, 1, 1, params, out, &ms))) return rc;
    const WindowResult &w = out[0];
    res->nu = w.nu;
    res->contrast = w.contrast;
    res->bound_gap = w.bound_gap;
    res->iterations = w.iterations;
    res->bound_evals = w.bound_evals;
    res->point_evals = w.point_evals;
    res->max_frontier = w.max_fr;
    res->marks = w.marks;
    res->exact_events = w.exact;
    res->rounds = w.rounds;
    res->device_ms = ms;
    if (w.status == kStatusIterLimit)
        return fail(ctx, EVD_ERR_ITER_LIMIT,
                    "iteration limit reached after %lld iterations (best nu=%.17g, contrast=%.17g)",
                    w.iterations, w.nu, w.contrast);
    return EVD_OK;
}

// Solve windows [offsets[w], offsets[w+1]) of the resident events (shared by
// evd_solve_windows and evd_solve_stream).
static int solve_offsets(evd_ctx *ctx, const long long *offsets, int n_windows, int groups,
                         const evd_solve_params *params, evd_window_result *results,
                         double *device_ms, StreamFeed *feed = nullptr)
{
    int rc;
    if (groups <= 0) {
        // auto: ~20 events per thread per group, at least one window per group
        // (cfg4, 2000 windows of ~20k events: 74 groups of 2 CTAs measured best;
        // smaller groups trade the grid barrier for per-thread event loops)
        long long tot = offsets[n_windows] - offsets[0];
        if (feed) {
            tot = 0;
            for (int w = 0; w < n_windows; w++) tot += feed->h_counts[w];
        }
        const double avg = (double)tot / n_windows;
        if (!ctx->solve_blocks) ctx->solve_blocks = solve_grid_blocks(ctx->device);
        const int per = std::max(1, (int)std::ceil(avg / (20.0 * solve_block_threads())));
        groups = std::max(1, std::min(n_windows, ctx->solve_blocks / per));
    }
    std::vector<WindowResult> out;
    float ms = 0.f;
    if ((rc = run_windows(ctx, offsets, n_windows, groups, params, out, &ms, feed))) return rc;
    for (int w = 0; w < n_windows; w++) {
        evd_window_result &r = results[w];
        r.nu = out[w].nu;
        r.contrast = out[w].contrast;
        r.bound_gap = out[w].bound_gap;
        r.iterations = out[w].iterations;
        r.bound_evals = out[w].bound_evals;
        r.point_evals = out[w].point_evals;
        r.max_frontier = out[w].max_fr;
        r.marks = out[w].marks;
        r.exact_events = out[w].exact;
        r.rounds = out[w].rounds;
        r.status = out[w].status == kStatusOk ? EVD_OK
                   : out[w].status == kStatusIterLimit ? EVD_ERR_ITER_LIMIT
                   : out[w].status == kStatusEmpty ? EVD_ERR_NO_EVENTS : EVD_ERR_CUDA;
        r.groups = groups;
    }
    if (device_ms) *device_ms = ms;
    return EVD_OK;
}

int evd_solve_windows(evd_ctx *ctx, const int64_t *offsets, int32_t n_windows, int32_t groups,
                      const evd_solve_params *params, evd_window_result *results,
                      double *device_ms)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!params || !results || !offsets || n_windows < 0)
        return fail(ctx, EVD_ERR_ARG, "bad evd_solve_windows arguments");
    int rc = need_events(ctx);
    if (rc) return rc;
    if (n_windows == 0) return EVD_OK;
    if (offsets[0] < 0 || offsets[n_windows] > ctx->n)
        return fail(ctx, EVD_ERR_ARG, "window offsets outside the resident events");
    for (int w = 0; w < n_windows; w++)
        if (offsets[w + 1] < offsets[w]) return fail(ctx, EVD_ERR_ARG, "offsets must be non-decreasing");
    return solve_offsets(ctx, (const long long *)offsets, n_windows, groups, params, results,
                         device_ms);
}

// Windows of the resident raw stream (sx, sy, st: time-sorted, sn events):
// bounds by device binary search, gather into the solve layout, one solve.
static int solve_resident_stream(evd_ctx *ctx, double tau, int groups,
                                 const evd_solve_params *params, evd_window_result *results,
                                 int capacity, int32_t *n_windows, int64_t *k0_out,
                                 double *device_ms)
{
    *n_windows = 0;
    *k0_out = 0;
    if (device_ms) *device_ms = 0.0;
    const long long n = ctx->sn;
    if (n == 0) return EVD_OK;  // batch_stream of an empty stream: no windows
    if (int rc = check_frame(ctx, ctx->sW, ctx->sH)) return rc;
    double tt[2];
    CU(cudaMemcpyAsync(tt, ctx->st.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(tt + 1, ctx->st.p + n - 1, sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    // events.py:341-342: k0 = int(floor(t[0] / tau)), k1 = int(floor(t[-1] / tau))
    const double f0 = std::floor(tt[0] / tau), f1 = std::floor(tt[1] / tau);
    if (!(f0 >= 0.0) || !(f1 >= f0) || f1 - f0 >= 2147483647.0)
        return fail(ctx, EVD_ERR_ARG, "timestamps must be sorted, non-negative and finite");
    const long long k0 = (long long)f0;
    const int nw = (int)((long long)f1 - k0 + 1);
    *n_windows = nw;
    *k0_out = k0;
    if (!results || capacity < nw)
        return fail(ctx, EVD_ERR_ARG, "stream spans %d windows, results hold %d", nw, capacity);
    CU(ctx->wbounds.ensure(3 * (size_t)nw + 1));
    long long *lo = ctx->wbounds.p, *hi = lo + nw, *off = hi + nw;
    launch_window_bounds(ctx->st.p, n, k0, nw, tau, lo, hi, ctx->stream);
    LAUNCHED(1);
    std::vector<long long> h(2 * (size_t)nw), o(nw + 1);
    CU(cudaMemcpyAsync(h.data(), lo, 2 * nw * sizeof(long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    o[0] = 0;
    for (int w = 0; w < nw; w++) o[w + 1] = o[w] + std::max(0LL, h[nw + w] - h[w]);
    const long long total = o[nw];
    // the windows' events, concatenated in the solve layout
    CU(ctx->xc.ensure(std::max(total, 1LL)));
    CU(ctx->yc.ensure(std::max(total, 1LL)));
    CU(ctx->t.ensure(std::max(total, 1LL)));
    CU(cudaMemcpyAsync(off, o.data(), (nw + 1) * sizeof(long long), cudaMemcpyHostToDevice,
                       ctx->stream));
    if (total > 0) {
        launch_gather_windows(ctx->sx.p, ctx->sy.p, ctx->st.p, lo, off, nw, k0, total, tau,
                              ctx->sW / 2.0, ctx->sH / 2.0, ctx->xc.p, ctx->yc.p, ctx->t.p,
                              ctx->stream);
        LAUNCHED(1);
    }
    ctx->n = total;
    ctx->gen++;
    ctx->W = ctx->sW;
    ctx->H = ctx->sH;
    ctx->tau = tau;
    if (total == 0) {  // every window empty
        for (int w = 0; w < nw; w++) {
            results[w] = evd_window_result{};
            results[w].status = EVD_ERR_NO_EVENTS;
        }
        return EVD_OK;
    }
    return solve_offsets(ctx, o.data(), nw, groups, params, results, device_ms);
}

// lower_bound of v in t[0, n) with k_window_bounds' loop (the same result on
// any input, sorted or not)
static long long host_lower_bound(const double *t, long long n, double v)
{
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (t[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Host event arrays in solve order: k pieces (one for a stream, one per window
// for a window list), concatenated they are the raw events the solve gathers.
struct HostPieces {
    const double *const *x, *const *y, *const *t;
    const long long *n;
    int k;
    bool pinned;  // one page-locked piece: DMA from it directly
};

// Solve windows whose raw events are still on the host, uploading them on
// ctx->copy while the solve runs: chunks of the concatenated pieces go
// through a ring of pinned slots (host memcpy, then H2D into dx / dy / dt),
// each followed by the count of raw events delivered; window w's group waits
// for its events (raw [lo[w], lo[w] + cnt[w])) and gathers them into the
// solve layout, which pads every window to 16 events.  On return (success or
// not) the copy stream is idle.
static int solve_fed(evd_ctx *ctx, const HostPieces &src, long long total_raw, double *dx,
                     double *dy, double *dt, const std::vector<long long> &lo,
                     const std::vector<long long> &cnt, long long k0, bool t_local, int groups,
                     const evd_solve_params *params, evd_window_result *results,
                     double *device_ms)
{
    const int nw = (int)cnt.size();
    std::vector<long long> pad(nw + 1);
    pad[0] = 0;
    for (int w = 0; w < nw; w++) pad[w + 1] = pad[w] + (cnt[w] + 15) / 16 * 16;
    CU(ctx->xc.ensure(std::max(pad[nw], 1LL)));
    CU(ctx->yc.ensure(std::max(pad[nw], 1LL)));
    CU(ctx->t.ensure(std::max(pad[nw], 1LL)));
    CU(ctx->feedw.ensure(2));
    CU(ctx->feedb.ensure(3 * (size_t)nw + 1));
    long long *d_lo = ctx->feedb.p, *d_cnt = d_lo + nw;
    if (!ctx->copy) CU(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
    if (!ctx->feed_start) {
        CU(cudaEventCreateWithFlags(&ctx->feed_start, cudaEventDisableTiming));
        for (cudaEvent_t &e : ctx->feed_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const size_t half = 16u << 20;
    if (!ctx->stage) {
        CU(cudaHostAlloc(&ctx->stage, 2 * half, cudaHostAllocDefault));
        ctx->stage_bytes = 2 * half;
        CU(cudaEventCreateWithFlags(&ctx->stage_ev[0], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&ctx->stage_ev[1], cudaEventDisableTiming));
    }
    CU(cudaMemsetAsync(ctx->feedw.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
    CU(cudaMemcpyAsync(d_lo, lo.data(), nw * sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(d_cnt, cnt.data(), nw * sizeof(long long), cudaMemcpyHostToDevice,
                       ctx->stream));
    // the copies start after everything queued so far (earlier readers of dx / dy / dt)
    CU(cudaEventRecord(ctx->feed_start, ctx->stream));
    CU(cudaStreamWaitEvent(ctx->copy, ctx->feed_start, 0));
    const int slots = 8;
    const long long S = std::min<long long>(ctx->feed_chunk, (long long)(2 * half / 8 / 32));
    const size_t slot_bytes = (size_t)S * 3 * sizeof(double) + 64;
    StreamFeed feed{dx, dy, dt, d_lo, d_cnt, cnt.data(), k0, t_local ? 1 : 0, nullptr};
    feed.upload = [&]() -> int {
        int p = 0;             // piece and position in it of the next raw event
        long long pp = 0;
        for (long long c0 = 0, c = 0; c0 < total_raw; c0 += S, c++) {
            const int sl = (int)(c % slots);
            if (c >= slots) CU(cudaEventSynchronize(ctx->feed_ev[sl]));  // slot free again
            const long long m = std::min(S, total_raw - c0);
            double *px = reinterpret_cast<double *>(ctx->stage + sl * slot_bytes);
            double *py = px + S, *pt = py + S;
            unsigned long long *val = reinterpret_cast<unsigned long long *>(pt + S);
            if (src.pinned) {
                px = const_cast<double *>(src.x[0] + c0);
                py = const_cast<double *>(src.y[0] + c0);
                pt = const_cast<double *>(src.t[0] + c0);
            } else {
                for (long long f = 0; f < m;) {
                    while (pp == src.n[p]) {
                        p++;
                        pp = 0;
                    }
                    const long long take = std::min(m - f, src.n[p] - pp);
                    memcpy(px + f, src.x[p] + pp, take * sizeof(double));
                    memcpy(py + f, src.y[p] + pp, take * sizeof(double));
                    memcpy(pt + f, src.t[p] + pp, take * sizeof(double));
                    f += take;
                    pp += take;
                }
            }
            *val = (unsigned long long)(c0 + m);
            CU(cudaMemcpyAsync(dx + c0, px, m * sizeof(double), cudaMemcpyHostToDevice, ctx->copy));
            CU(cudaMemcpyAsync(dy + c0, py, m * sizeof(double), cudaMemcpyHostToDevice, ctx->copy));
            CU(cudaMemcpyAsync(dt + c0, pt, m * sizeof(double), cudaMemcpyHostToDevice, ctx->copy));
            CU(cudaMemcpyAsync(ctx->feedw.p, val, sizeof *val, cudaMemcpyHostToDevice, ctx->copy));
            CU(cudaEventRecord(ctx->feed_ev[sl], ctx->copy));
        }
        return EVD_OK;
    };
    long long live = 0;
    for (int w = 0; w < nw; w++) live += cnt[w];
    int rc = EVD_OK;
    if (live == 0) {  // every window empty: nothing to solve, the events still go up
        rc = feed.upload();
        for (int w = 0; w < nw; w++) {
            results[w] = evd_window_result{};
            results[w].status = EVD_ERR_NO_EVENTS;
        }
        if (device_ms) *device_ms = 0.0;
    } else {
        rc = solve_offsets(ctx, pad.data(), nw, groups, params, results, device_ms, &feed);
    }
    CU(cudaStreamSynchronize(ctx->copy));
    return rc;
}

// evd_solve_stream from host arrays: the windows' bounds come from the host
// copy of t (k_window_bounds' search), the raw stream follows the launch
// (solve_fed), and the resident window set is re-gathered unpadded afterwards
// (the evd_set_events contract).
static int solve_stream_overlapped(evd_ctx *ctx, const double *x, const double *y,
                                   const double *t, long long n, bool pinned, double tau,
                                   int groups, const evd_solve_params *params,
                                   evd_window_result *results, int capacity, int32_t *n_windows,
                                   int64_t *k0_out, double *device_ms)
{
    // events.py:341-342 on the host copy of t
    const double f0 = std::floor(t[0] / tau), f1 = std::floor(t[n - 1] / tau);
    if (!(f0 >= 0.0) || !(f1 >= f0) || f1 - f0 >= 2147483647.0)
        return fail(ctx, EVD_ERR_ARG, "timestamps must be sorted, non-negative and finite");
    const long long k0 = (long long)f0;
    const int nw = (int)((long long)f1 - k0 + 1);
    *n_windows = nw;
    *k0_out = k0;
    if (!results || capacity < nw)
        return fail(ctx, EVD_ERR_ARG, "stream spans %d windows, results hold %d", nw, capacity);
    std::vector<long long> lo(nw), cnt(nw), o(nw + 1);
    o[0] = 0;
    for (int w = 0; w < nw; w++) {
        const double start = (double)(k0 + w) * tau;
        lo[w] = host_lower_bound(t, n, start);
        cnt[w] = std::max(0LL, host_lower_bound(t, n, start + tau) - lo[w]);
        o[w + 1] = o[w] + cnt[w];
    }
    ctx->W = ctx->sW;
    ctx->H = ctx->sH;
    ctx->tau = tau;
    ctx->gen++;
    ctx->n = 0;  // the resident window set is rebuilt below
    const HostPieces src{&x, &y, &t, &n, 1, pinned};
    int rc = solve_fed(ctx, src, n, ctx->sx.p, ctx->sy.p, ctx->st.p, lo, cnt, k0, false, groups,
                       params, results, device_ms);
    if (rc) return rc;
    const long long total = o[nw];
    if (total > 0) {
        long long *d_lo = ctx->feedb.p, *d_off = d_lo + 2 * nw;
        CU(cudaMemcpyAsync(d_off, o.data(), (nw + 1) * sizeof(long long), cudaMemcpyHostToDevice,
                           ctx->stream));
        launch_gather_windows(ctx->sx.p, ctx->sy.p, ctx->st.p, d_lo, d_off, nw, k0, total, tau,
                              ctx->sW / 2.0, ctx->sH / 2.0, ctx->xc.p, ctx->yc.p, ctx->t.p,
                              ctx->stream);
        LAUNCHED(1);
        CU(cudaStreamSynchronize(ctx->stream));
    }
    ctx->n = total;
    ctx->gen++;
    return EVD_OK;
}

int evd_solve_windows_list(evd_ctx *ctx, const double *const *x, const double *const *y,
                           const double *const *t, const int64_t *counts, int32_t k,
                           int32_t width, int32_t height, double tau, int32_t groups,
                           const evd_solve_params *params, evd_window_result *results,
                           double *device_ms)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (k < 0 || width < 1 || height < 1 || !params || (k > 0 && (!x || !y || !t || !counts || !results)))
        return fail(ctx, EVD_ERR_ARG, "bad evd_solve_windows_list arguments");
    if (int rc = check_frame(ctx, width, height)) return rc;
    if (!(tau > 0.0)) return fail(ctx, EVD_ERR_ARG, "batch duration tau must be positive");
    long long n = 0;
    std::vector<long long> lo(k), cnt(k);
    for (int w = 0; w < k; w++) {
        if (counts[w] < 0 || (counts[w] > 0 && (!x[w] || !y[w] || !t[w])))
            return fail(ctx, EVD_ERR_ARG, "bad window %d", w);
        lo[w] = n;
        cnt[w] = counts[w];
        n += counts[w];
    }
    if (device_ms) *device_ms = 0.0;
    CU(cudaSetDevice(ctx->device));
    if (!ctx->stream_overlap) {  // upload, then solve
        if (int rc = evd_set_events_list(ctx, x, y, t, counts, k, width, height, tau)) return rc;
        if (k == 0) return EVD_OK;
        std::vector<long long> o(k + 1);
        o[0] = 0;
        for (int w = 0; w < k; w++) o[w + 1] = o[w] + cnt[w];
        return solve_offsets(ctx, o.data(), k, groups, params, results, device_ms);
    }
    CU(ctx->wx.ensure(std::max(n, 1LL)));
    CU(ctx->wy.ensure(std::max(n, 1LL)));
    CU(ctx->wt.ensure(std::max(n, 1LL)));
    ctx->W = width;
    ctx->H = height;
    ctx->tau = tau;
    ctx->gen++;
    ctx->n = 0;  // the resident window set is rebuilt below
    if (k == 0) return EVD_OK;
    const HostPieces src{x, y, t, reinterpret_cast<const long long *>(counts), k, false};
    int rc = solve_fed(ctx, src, n, ctx->wx.p, ctx->wy.p, ctx->wt.p, lo, cnt, 0, true, groups,
                       params, results, device_ms);
    if (rc) return rc;
    // resident window set = the windows concatenated (as evd_set_events_list leaves it)
    if (n > 0) {
        launch_center(ctx->wx.p, ctx->wy.p, n, width / 2.0, height / 2.0, ctx->xc.p, ctx->yc.p,
                      ctx->stream);
        LAUNCHED(1);
        CU(cudaMemcpyAsync(ctx->t.p, ctx->wt.p, n * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    ctx->n = n;
    ctx->gen++;
    return EVD_OK;
}

int evd_solve_stream(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                     int32_t width, int32_t height, double tau, int32_t groups,
                     const evd_solve_params *params, evd_window_result *results,
                     int32_t capacity, int32_t *n_windows, int64_t *k0_out, double *device_ms)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!params || !n_windows || !k0_out || n < 0 || width < 1 || height < 1)
        return fail(ctx, EVD_ERR_ARG, "bad evd_solve_stream arguments");
    if (int rc = check_frame(ctx, width, height)) return rc;
    if (!(tau > 0.0)) return fail(ctx, EVD_ERR_ARG, "tau must be positive");
    if (n > 0 && (!x || !y || !t)) return fail(ctx, EVD_ERR_ARG, "NULL event array");
    CU(cudaSetDevice(ctx->device));
    CU(ctx->sx.ensure(std::max(n, (int64_t)1)));
    CU(ctx->sy.ensure(std::max(n, (int64_t)1)));
    CU(ctx->st.ensure(std::max(n, (int64_t)1)));
    // all three arrays in host memory: overlap their upload with the solve
    bool host = false, pinned = false;
    if (n > 0 && ctx->stream_overlap) {
        host = pinned = true;
        for (const double *q : {x, y, t}) {
            cudaPointerAttributes at{};
            CU(cudaPointerGetAttributes(&at, q));
            host = host && (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered);
            pinned = pinned && at.type == cudaMemoryTypeHost;
        }
    }
    if (host) {
        ctx->sn = n;
        ctx->sW = width;
        ctx->sH = height;
        ctx->s_has_p = false;
        return solve_stream_overlapped(ctx, x, y, t, n, pinned, tau, groups, params, results,
                                       capacity, n_windows, k0_out, device_ms);
    }
    if (n > 0) {
        CU(cudaMemcpyAsync(ctx->sx.p, x, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        CU(cudaMemcpyAsync(ctx->sy.p, y, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        CU(cudaMemcpyAsync(ctx->st.p, t, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
    }
    ctx->sn = n;
    ctx->sW = width;
    ctx->sH = height;
    ctx->s_has_p = false;
    return solve_resident_stream(ctx, tau, groups, params, results, capacity, n_windows, k0_out,
                                 device_ms);
}

int evd_solve_loaded_stream(evd_ctx *ctx, double tau, int32_t groups,
                            const evd_solve_params *params, evd_window_result *results,
                            int32_t capacity, int32_t *n_windows, int64_t *k0_out,
                            double *device_ms)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!params || !n_windows || !k0_out) return fail(ctx, EVD_ERR_ARG, "bad arguments");
    if (!(tau > 0.0)) return fail(ctx, EVD_ERR_ARG, "tau must be positive");
    if (ctx->sn < 0) return fail(ctx, EVD_ERR_STATE, "no stream loaded (evd_load_bin)");
    CU(cudaSetDevice(ctx->device));
    return solve_resident_stream(ctx, tau, groups, params, results, capacity, n_windows, k0_out,
                                 device_ms);
}

int evd_load_bin(evd_ctx *ctx, const uint8_t *data, int64_t size, int32_t *width,
                 int32_t *height, int64_t *n_out)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!width || !height || !n_out || (size > 0 && !data) || size < 0)
        return fail(ctx, EVD_ERR_ARG, "bad evd_load_bin arguments");
    // header <4sIIQ> (events.py:188-193)
    if (size < 20) return fail(ctx, EVD_ERR_FORMAT, "truncated BIN header");
    if (std::memcmp(data, "EVD1", 4) != 0) {
        char m[64];
        int k = 0;
        for (int i = 0; i < 4; i++) {
            const unsigned char c = data[i];
            if (c >= 32 && c < 127 && c != '\\' && c != '\'') m[k++] = (char)c;
            else k += std::snprintf(m + k, sizeof(m) - k, "\\x%02x", c);
        }
        m[k] = 0;
        return fail(ctx, EVD_ERR_FORMAT, "bad magic b'%s'", m);
    }
    uint32_t w, h;
    uint64_t count;
    std::memcpy(&w, data + 4, 4);
    std::memcpy(&h, data + 8, 4);
    std::memcpy(&count, data + 12, 8);
    if (count > (uint64_t)(size - 20) / 17)  // events.py:197-201
        return fail(ctx, EVD_ERR_FORMAT, "truncated BIN body: expected %llu records",
                    (unsigned long long)count);
    if (w < 1 || h < 1 || w > 2147483647u || h > 2147483647u)  // SensorGeometry (events.py:37-39)
        return fail(ctx, EVD_ERR_VALIDATION, "sensor dimensions must be positive, got %ux%u", w, h);
    const long long n = (long long)count;
    CU(cudaSetDevice(ctx->device));
    CU(ctx->sx.ensure(std::max(n, 1LL)));
    CU(ctx->sy.ensure(std::max(n, 1LL)));
    CU(ctx->st.ensure(std::max(n, 1LL)));
    CU(ctx->sp.ensure(std::max(n, 1LL)));
    ctx->sn = -1;
    if (n > 0) {
        CU(ctx->sbytes.ensure((size_t)n * 17));
        const size_t scratch = decode_scratch_bytes(n);
        CU(ctx->sscratch.ensure(scratch));
        CU(ctx->sflags.ensure(1));
        CU(cudaMemcpyAsync(ctx->sbytes.p, data + 20, (size_t)n * 17, cudaMemcpyHostToDevice,
                           ctx->stream));
        unsigned int flags = 0;
        int launches = 0;
        cudaError_t e = decode_bin(ctx->sbytes.p, n, (int)w, (int)h, ctx->sx.p, ctx->sy.p,
                                   ctx->st.p, ctx->sp.p, ctx->sscratch.p, ctx->sscratch.cap,
                                   ctx->sflags.p, &flags, &launches, ctx->stream);
        ctx->launches += launches;
        if (e != cudaSuccess) return fail(ctx, EVD_ERR_CUDA, "decode_bin: %s", cudaGetErrorString(e));
        // EventStream invariants, in the reference's order (events.py:67-81)
        if (flags & 2u) return fail(ctx, EVD_ERR_VALIDATION, "event coordinates must be finite");
        if (flags & 4u)
            return fail(ctx, EVD_ERR_VALIDATION, "event coordinates outside sensor geometry");
        if (flags & 8u) return fail(ctx, EVD_ERR_VALIDATION, "polarity must be +1 or -1");
    }
    ctx->sn = n;
    ctx->sW = (int)w;
    ctx->sH = (int)h;
    ctx->s_has_p = true;
    *width = (int32_t)w;
    *height = (int32_t)h;
    *n_out = n;
    return EVD_OK;
}

int evd_load_stream(evd_ctx *ctx, const double *x, const double *y, const double *t,
                    const int8_t *p, int64_t n, int32_t width, int32_t height)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (n < 0 || width < 1 || height < 1 || (n > 0 && (!x || !y || !t)))
        return fail(ctx, EVD_ERR_ARG, "bad evd_load_stream arguments");
    if (int rc = check_frame(ctx, width, height)) return rc;
    CU(cudaSetDevice(ctx->device));
    const long long m = std::max<long long>(n, 1);
    CU(ctx->sx.ensure(m));
    CU(ctx->sy.ensure(m));
    CU(ctx->st.ensure(m));
    CU(ctx->sp.ensure(m));
    if (n > 0) {
        CU(cudaMemcpyAsync(ctx->sx.p, x, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        CU(cudaMemcpyAsync(ctx->sy.p, y, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        CU(cudaMemcpyAsync(ctx->st.p, t, n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        if (p) CU(cudaMemcpyAsync(ctx->sp.p, p, n, cudaMemcpyDefault, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));  // inputs are never retained (evd.h)
    }
    ctx->sn = n;
    ctx->sW = width;
    ctx->sH = height;
    ctx->s_has_p = p != nullptr;
    return EVD_OK;
}

int evd_pixel_counts(evd_ctx *ctx, int64_t *counts)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (ctx->sn < 0) return fail(ctx, EVD_ERR_STATE, "no stream loaded");
    if (!counts) return fail(ctx, EVD_ERR_ARG, "counts is NULL");
    CU(cudaSetDevice(ctx->device));
    const long long M = (long long)ctx->sW * ctx->sH;
    CU(ctx->pcounts.ensure(M));
    int launches = 0;
    CU(pixel_counts_dev(ctx->sx.p, ctx->sy.p, ctx->sn, ctx->sW, ctx->sH, ctx->pcounts.p, &launches,
                        ctx->stream));
    ctx->launches += launches;
    std::vector<unsigned int> h(M);
    CU(cudaMemcpyAsync(h.data(), ctx->pcounts.p, M * sizeof(unsigned int), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (long long i = 0; i < M; i++) counts[i] = h[i];
    return EVD_OK;
}

int evd_stream_remove_hot_pixels(evd_ctx *ctx, double k, int64_t *n_out, double *threshold)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (!(k > 0.0)) return fail(ctx, EVD_ERR_ARG, "k must be positive");  // events.py:286-287
    if (ctx->sn < 0) return fail(ctx, EVD_ERR_STATE, "no stream loaded");
    if (!ctx->s_has_p) return fail(ctx, EVD_ERR_STATE, "the loaded stream has no polarity");
    if (n_out) *n_out = ctx->sn;
    if (threshold) *threshold = 0.0;
    if (ctx->sn == 0) return EVD_OK;  // events.py:288-289
    CU(cudaSetDevice(ctx->device));
    const long long n = ctx->sn, M = (long long)ctx->sW * ctx->sH;
    const size_t bytes = preprocess_scratch_bytes(n, M);
    CU(ctx->sscratch.ensure(bytes));
    long long kept = 0;
    double thr = 0.0;
    int launches = 0;
    cudaError_t e = remove_hot_pixels_dev(ctx->sx.p, ctx->sy.p, ctx->st.p, ctx->sp.p, n, ctx->sW,
                                          ctx->sH, k, ctx->sscratch.p, ctx->sscratch.cap, &kept,
                                          &thr, &launches, ctx->stream);
    ctx->launches += launches;
    if (e != cudaSuccess) return fail(ctx, EVD_ERR_CUDA, "remove_hot_pixels: %s", cudaGetErrorString(e));
    ctx->sn = kept;
    if (n_out) *n_out = kept;
    if (threshold) *threshold = thr;
    return EVD_OK;
}

int evd_stream_rescale(evd_ctx *ctx, int32_t width, int32_t height)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (width < 1 || height < 1)
        return fail(ctx, EVD_ERR_VALIDATION, "sensor dimensions must be positive, got %dx%d", width,
                    height);
    if (ctx->sn < 0) return fail(ctx, EVD_ERR_STATE, "no stream loaded");
    CU(cudaSetDevice(ctx->device));
    // events.py:305-312
    const double sx = (double)width / (double)ctx->sW, sy = (double)height / (double)ctx->sH;
    const double xmax = std::nextafter((double)width, 0.0), ymax = std::nextafter((double)height, 0.0);
    int launches = 0;
    CU(rescale_dev(ctx->sx.p, ctx->sy.p, ctx->sn, sx, sy, xmax, ymax, &launches, ctx->stream));
    ctx->launches += launches;
    ctx->sW = width;
    ctx->sH = height;
    return EVD_OK;
}

int evd_stream_copy(evd_ctx *ctx, double *x, double *y, double *t, int8_t *p)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (ctx->sn < 0) return fail(ctx, EVD_ERR_STATE, "no stream loaded");
    const long long n = ctx->sn;
    if (n == 0) return EVD_OK;
    CU(cudaSetDevice(ctx->device));
    if (x) CU(cudaMemcpyAsync(x, ctx->sx.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (y) CU(cudaMemcpyAsync(y, ctx->sy.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (t) CU(cudaMemcpyAsync(t, ctx->st.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (p) {
        if (!ctx->s_has_p) return fail(ctx, EVD_ERR_STATE, "the loaded stream has no polarity");
        CU(cudaMemcpyAsync(p, ctx->sp.p, n, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    return EVD_OK;
}

int evd_solve_trace(evd_ctx *ctx, int64_t *out, int64_t cap, int64_t *n)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    const long long k = std::min<long long>(cap, ctx->trace_n);
    if (n) *n = ctx->trace_n;
    if (k > 0 && ctx->trace.p) {
        CU(cudaMemcpy(out, ctx->trace.p, k * sizeof(long long), cudaMemcpyDeviceToHost));
    }
    return EVD_OK;
}

int evd_probe_events(evd_ctx *ctx, double lo, double hi, int32_t reps, double *span_ns)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (reps < 1 || reps > 1024 || !span_ns) return fail(ctx, EVD_ERR_ARG, "bad probe arguments");
    int rc = need_events(ctx);
    if (rc) return rc;
    const double nu3[3] = {lo, 0.5 * (lo + hi), hi};
    double den3[3];
    for (int k = 0; k < 3; k++)
        if ((rc = check_den(ctx, nu3[k], ctx->tau, den3 + k))) return rc;
    if (!ctx->solve_blocks) ctx->solve_blocks = solve_grid_blocks(ctx->device);
    const long long M = (long long)ctx->W * ctx->H;
    DevBuf<unsigned long long> &ctrs = ctx->probe_ctr, &span = ctx->probe_span;
    DevBuf<unsigned int> &scratch = ctx->probe_img;
    CU(ctrs.ensure(8 * (size_t)reps));
    CU(span.ensure(2 * (size_t)reps));
    CU(scratch.ensure(6 * (size_t)M));
    CU(cudaMemsetAsync(ctrs.p, 0, 8 * reps * sizeof(unsigned long long), ctx->stream));
    std::vector<unsigned long long> h(2 * (size_t)reps);
    for (int r = 0; r < reps; r++) { h[2 * r] = ~0ull; h[2 * r + 1] = 0; }
    CU(cudaMemcpyAsync(span.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemsetAsync(scratch.p, 0, 6 * M * sizeof(unsigned int), ctx->stream));
    const double cx = ctx->W / 2.0, cy = ctx->H / 2.0;
    CU(launch_event_probe(ctx->xc.p, ctx->yc.p, ctx->t.p, ctx->n, nu3, den3, cx, cy,
                          ctx->W, ctx->H, ctx->solve_blocks, reps, ctrs.p, span.p, scratch.p,
                          ctx->stream));
    LAUNCHED(1);
    CU(cudaMemcpyAsync(h.data(), span.p, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < reps; r++) span_ns[r] = (double)(h[2 * r + 1] - h[2 * r]);
    return EVD_OK;
}

int evd_solve_block_trace(evd_ctx *ctx, int64_t *out, int64_t cap, int32_t *blocks)
{
    if (!ctx) return fail(nullptr, EVD_ERR_ARG, "ctx is NULL");
    if (blocks) *blocks = ctx->solve_blocks;
    const long long k = std::min<long long>(cap, (long long)kBTraceIters * ctx->solve_blocks * kBTraceSlots);
    if (k > 0 && ctx->btrace.p)
        CU(cudaMemcpy(out, ctx->btrace.p, k * sizeof(long long), cudaMemcpyDeviceToHost));
    return EVD_OK;
}

int evd_pow2_table(int64_t m, int64_t n, double *out)
{
    if (m < 1 || n < 0 || !out) return fail(nullptr, EVD_ERR_ARG, "bad pow2 table request");
    pow2_fill(m, n, out);
    return EVD_OK;
}

}  // extern "C"

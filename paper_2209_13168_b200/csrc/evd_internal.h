// evd_internal.h -- structures shared by the host API (evd_api.cu) and the
// kernels (evd_kernels.cu).  Not part of the public C ABI (include/evd.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace evd {

constexpr int kMaxLevels = 32;    // heights of a numpy pairwise tree (log2(M/64)+1)
constexpr int kCutSmem = 4096;    // doubles of per-block scratch for a cut subtree / top

// Fixed numpy pairwise-summation tree over M pixels, split into C "cut"
// subtrees (evaluated one per block in parallel) and a top part (one block).
struct TreeDev {
    int M, L, C;
    const int2 *leaves;      // [L] (offset, n), left to right
    const int *cut_leaf0;    // [C+1] leaf range of each cut
    const int *cut_trip0;    // [C+1] triple range of each cut
    const int *cut_lvl;      // [C*(kMaxLevels+1)] per-cut level starts (relative)
    const int *cut_nlev;     // [C]
    const int4 *trip;        // (dst, l, r, -) local indices, sorted by height
    const int4 *top;         // (dst, l, r, -) in top index space (cuts 0..C-1, then internals)
    const int *top_lvl;      // [top_levels+1]
    int top_levels;
    int top_root;
    double *cutval;          // [C] scratch
};

struct alignas(32) FrontierEntry {
    double bound;
    long long counter;
    double lo, hi;
};

// kModeRootCert: the root round evaluates the root as a node (both children)
// and certifies its bound instead of rasterising it (k_solve_spec)
enum SolveMode : int { kModeRoot = 0, kModeNode = 1, kModeRootCert = 2 };
enum SolveStatus : int { kStatusOk = 0, kStatusIterLimit = 1, kStatusCapacity = 2 };

// Device-resident BnB state (one per context); host reads it back at the end.
#ifndef EVD_SPEC_KMAX
#define EVD_SPEC_KMAX 4
#endif
constexpr int kSpecK = EVD_SPEC_KMAX;  // node evaluations per speculative round (k_solve_spec)

struct SolveState {
    // node under evaluation
    double lo, hi, c, den_lo, den_c, den_hi;
    int mode, done;
    // per-node accumulators, double-buffered by node parity: 0 in_image,
    // 1 fully_inside A, 2 fully_inside B, 3 segment marks, 4 S_bar A, 5 S_bar B,
    // 6 exact-path events, 7 event work counter
    alignas(16) unsigned long long acc[2][8];  // 16-byte aligned: vector loads
    // incumbent and diagnostics
    double nu_hat, c_hat, bound_gap;
    long long iterations, bound_evals, point_evals, next_counter, fr_n, max_fr;
    int status, pad;
    unsigned long long marks;  // pixel increments of all images over the solve
    // speculative rounds (k_solve_spec): per-slot accumulators by round parity
    alignas(16) unsigned long long sacc[2][kSpecK][8];
};

// Result of one window of evd_solve_windows / evd_solve.
// kStatusRootCert: the root bound could not be certified (the host reruns
// with the root rasterised)
enum WindowStatus : int { kStatusEmpty = 3, kStatusSpecOverflow = 4, kStatusRootCert = 5 };
struct WindowResult {
    double nu, contrast, bound_gap;
    long long iterations, bound_evals, point_evals, max_fr;
    unsigned long long marks, exact;
    int status, rounds;  // rounds: grid-wide node-evaluation steps
};

struct SolveArgs {
    const double *xc, *yc, *t;   // centred events of all windows, concatenated
    const long long *offsets;     // [n_windows + 1] window w = [offsets[w], offsets[w+1])
    int n_windows;
    int groups, group_blocks;     // independent solver groups x CTAs per group
    int W, H;
    double cx, cy, tau;
    double lo0, hi0, c0, den_lo0, den_c0, den_hi0;  // root domain (host arithmetic)
    unsigned int *img;            // per group: P, A, B (u32, M each, zeroed)
    TreeDev tree;                 // cut plan for group_blocks CTAs; cutval: C per group
    const double *pow2;           // pow(fi / M, 2.0) via host libm, fi in [0, max n]
    double gamma, min_width;
    long long max_iter;
    SolveState *st;               // per group (accumulators)
    FrontierEntry *fr;            // per group, fr_cap entries each
    long long fr_cap;
    unsigned long long *bar;      // per group: barrier counter (stride 2)
    WindowResult *res;            // per window
    long long *trace;             // [1 + kTraceSlots*trace_iters] globaltimer ns (group 0, window 0)
    long long trace_iters;
    long long *btrace;            // [kBTraceIters][group_blocks][kBTraceSlots] (or null)
    int filter;                   // use the filtered (approximate-then-exact) event path
    int spec_k;                   // k_solve_spec: evaluations per round (1..kSpecK)
    int root_cert;                // k_solve_spec: certify the root bound (kModeRootCert)
    // evaluation-only launch (evd_eval_nodes; k_solve_spec, one window): the
    // nodes [ev_lo[i], ev_hi[i]] in rounds of spec_k slots, no BnB step;
    // ev_out[3 i .. 3 i + 2] = contrast at the centre, c_bar of both children
    const double *ev_lo, *ev_hi;
    long long ev_n;
    double *ev_out;
    // Overlapped stream upload (evd_solve_stream from host arrays; sx null:
    // the windows are already gathered).  The raw stream arrives in chunks on
    // a copy stream while the solve runs; *ready = raw events on the device.
    // Window w's group waits for ready >= s_lo[w] + counts[w], then gathers
    // the window into xc / yc / t at offsets[w] (offsets padded to 16 events:
    // no cache line holds two windows) before its first node.
    const double *sx, *sy, *stt;  // raw x, y, t
    const long long *s_lo, *counts;
    const unsigned long long *ready;
    double *gx, *gy, *gt;         // xc / yc / t, writable
    long long k0;
    int t_local;                  // t already window-local: gathered unchanged
    unsigned int *stall;          // set when an upload never arrived (the window is garbage)
};
constexpr long long kUploadTimeoutNs = 20000000000ll;  // 20 s

constexpr int kBTraceIters = 128;
constexpr int kBTraceSlots = 20;
constexpr int kBTraceMaxBlocks = 2048;

constexpr long long kTraceIters = 1 << 14;
constexpr int kTraceSlots = 10;
// per node evaluation: when ...
enum TraceSlot : int {
    kTrB0Top = 0,      // block 0 starts the node
    kTrB0Events = 1,   // block 0 finished its events
    kTrEventsMax = 2,  // the latest block finished its events (atomicMax)
    kTrB0Pixels0 = 3,  // block 0 left barrier 1
    kTrB0Pixels1 = 4,  // block 0 finished its pixels
    kTrPixelsMax = 5,  // the latest block finished its pixels (atomicMax)
    kTrB0Step0 = 6,    // block 0 left barrier 2
    kTrB0Step1 = 7,    // block 0 finished the BnB step
    kTrMarks = 8,      // segment-image marks of the node's children (a count, not a time)
    kTrExact = 9,      // events that took the exact path (a count)
};

// ---- kernel launchers (evd_kernels.cu); all asynchronous on `s` ----
void launch_center(const double *x, const double *y, long long n, double cx, double cy,
                   double *xc, double *yc, cudaStream_t s);
void launch_warp(const double *xc, const double *yc, const double *t, long long n, double nu,
                 double den, double cx, double cy, double *xo, double *yo, cudaStream_t s);
void launch_scale(const double *t, long long n, double nu, double den, double *s, cudaStream_t st);
void launch_point_image(const double *xc, const double *yc, const double *t, long long n,
                        double nu, double den, double cx, double cy, int W, int H,
                        unsigned int *img, unsigned long long *acc, cudaStream_t s);
void launch_bound_image(const double *xc, const double *yc, const double *t, long long n,
                        double lo, double den_lo, double hi, double den_hi, double cx, double cy,
                        int W, int H, unsigned int *img, unsigned long long *acc,
                        cudaStream_t s);
void launch_frontier(const double *xc, const double *yc, const double *t, long long n,
                     const double *lo, const double *hi, const double *den_lo,
                     const double *den_hi, int K, double cx, double cy, int W, int H,
                     unsigned int *images, long long M, unsigned long long *fi_out,
                     unsigned long long *marks_s, bool exact_only, cudaStream_t s);
constexpr int kFrontGroupHost = 32;
void launch_image_sums(const unsigned int *img, long long m, unsigned long long *acc,
                       cudaStream_t s);
void launch_contrast_u32(const unsigned int *img, const unsigned long long *in_image,
                         const TreeDev &tree, double *out, cudaStream_t s);
void launch_points_multi(const double *xc, const double *yc, const double *t, long long n,
                         const double *nus, const double *dens, int K, double cx, double cy,
                         int W, int H, unsigned int *images, long long M,
                         unsigned long long *in_out, const TreeDev &tree, double *cutvals,
                         double *contrast, cudaStream_t s);
void launch_contrast_f64(const double *img, double mu, const TreeDev &tree, double *out,
                         cudaStream_t s);
void launch_raster_segments(const double *segs, int k, int W, int H, int chunk, unsigned int *counts,
                            cudaStream_t s);
int solve_grid_blocks(int device);
int solve_block_threads();
// threads per CTA: 384, 512 or 768 (anything else runs at 512)
cudaError_t launch_solve(const SolveArgs &a, int blocks, int threads, cudaStream_t s);
cudaError_t launch_solve_spec(const SolveArgs &a, int blocks, int threads, cudaStream_t s);
cudaError_t decode_bin(const unsigned char *body_dev, long long n, int W, int H, double *x,
                       double *y, double *t, signed char *p, void *scratch, size_t scratch_bytes,
                       unsigned int *flags_dev, unsigned int *flags_host, int *launches,
                       cudaStream_t s);
size_t decode_scratch_bytes(long long n);
cudaError_t pixel_counts_dev(const double *x, const double *y, long long n, int W, int H,
                             unsigned int *counts, int *launches, cudaStream_t s);
cudaError_t remove_hot_pixels_dev(double *x, double *y, double *t, signed char *p, long long n,
                                  int W, int H, double k, void *scratch, size_t scratch_bytes,
                                  long long *n_out, double *threshold_out, int *launches,
                                  cudaStream_t s);
size_t preprocess_scratch_bytes(long long n, long long M);
cudaError_t rescale_dev(double *x, double *y, long long n, double sx, double sy, double xmax,
                        double ymax, int *launches, cudaStream_t s);
void launch_window_bounds(const double *t, long long n, long long k0, int nw, double tau,
                          long long *lo, long long *hi, cudaStream_t s);
void launch_gather_windows(const double *x, const double *y, const double *t,
                           const long long *lo, const long long *off, int nw, long long k0,
                           long long total, double tau, double cx, double cy, double *xc,
                           double *yc, double *tl, cudaStream_t s);
cudaError_t launch_event_probe(const double *xc, const double *yc, const double *t, long long n,
                               const double *nu3, const double *den3, double cx, double cy,
                               int W, int H, int blocks, int reps, unsigned long long *ctrs,
                               unsigned long long *span, unsigned int *scratch, cudaStream_t s);

// ---- tiled batched frontier (evd_frontier_tiles.cu) ----
struct FrontierTiles;
FrontierTiles *tiles_new();
void tiles_free(FrontierTiles *f);
// Bin the resident window (centred events) into the frame's angular tiles,
// once per window generation `gen`.  *usable = false when the tiled path does
// not apply to this window (frame not tileable, non-finite events, a tile
// listing more events than its u16 counters allow).
cudaError_t tiles_bin(FrontierTiles *f, const double *xc, const double *yc, const double *t,
                      long long n, int W, int H, unsigned long long gen, bool *usable,
                      int *launches, cudaStream_t s);
// bound_terms for K intervals (every hi <= 0) over the binned window
// (contig: lo[k+1] == hi[k] for every k, one warp per endpoint):
// fi_out[k] += fully_inside, marks_s[2k] += sum(H), marks_s[2k+1] += sum(H^2).
cudaError_t tiles_eval(FrontierTiles *f, const double *lo, const double *hi, const double *dlo,
                       const double *dhi, int K, bool contig, unsigned long long *fi_out,
                       unsigned long long *marks_s, int *launches, cudaStream_t s);
// out[0] tiles (0: frame not tiled), out[1] pixels per tile (max), out[2]
// listed events of the binned window (-1: not binned / not usable), out[3]
// tiles with work
void tiles_info(const FrontierTiles *f, long long *out);

}  // namespace evd

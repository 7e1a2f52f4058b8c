/*
 * evd.h -- C ABI of the B200 bound-evaluation library (libevd.so).
 *
 * Drop-in boundary for the hot path of the reference package `eventdiv`
 * (arXiv 2209.13168, /root/reference/pkg).  The reference exposes this path
 * only as Python functions; each entry point below names the reference
 * function it replaces (file:line under pkg/src/eventdiv/).  The Python mirror
 * of that interface is paper_2209_13168_b200/ (contrast.py, solver.py, ...),
 * bound through ctypes in paper_2209_13168_b200/_lib.py; INTEGRATION.md shows
 * how the reference package would bind the same symbols.
 *
 * Conventions
 *  - Plain pointers and sizes; host buffers are caller-owned and never retained.
 *  - Every call is synchronous w.r.t. its outputs (it returns after the
 *    results are in the caller's buffers) and runs on the context's stream.
 *  - Return value: EVD_OK or an EVD_ERR_* code; evd_last_error() has the text.
 *    No C++ exception crosses the ABI.
 *  - One context per (device, host thread).  Contexts are independent.
 *  - Arithmetic is IEEE binary64, round-to-nearest, no FMA contraction:
 *    integer images and bounds are bit-identical to the reference's.
 */
#ifndef EVD_H
#define EVD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct evd_ctx evd_ctx;

enum {
    EVD_OK = 0,
    EVD_ERR_CUDA = 1,         /* CUDA runtime failure (message has the CUDA error) */
    EVD_ERR_ARG = 2,          /* ValueError in the reference (bad tau/epsilon/sizes) */
    EVD_ERR_NO_EVENTS = 3,    /* NoEventsError, solver.py:32-33,88-89 */
    EVD_ERR_CHEIRALITY = 4,   /* CheiralityError, geometry.py:21-22,72-74 (1 + nu*tau <= 0) */
    EVD_ERR_ITER_LIMIT = 5,   /* IterationLimitError, solver.py:36-46,118-119; result holds the incumbent */
    EVD_ERR_STATE = 6,        /* call order (e.g. no events set) */
    EVD_ERR_FORMAT = 7,       /* malformed EVD1 file (EventFormatError, events.py:186-201) */
    EVD_ERR_VALIDATION = 8    /* stream invariant violated (EventValidationError, events.py:61-81) */
};

/* ---- context ----------------------------------------------------------- */
int evd_create(int device, evd_ctx **out);
void evd_destroy(evd_ctx *ctx);
/* Last error text for ctx (or for the calling thread when ctx is NULL). */
const char *evd_last_error(const evd_ctx *ctx);
/* Run subsequent work on a caller-owned cudaStream_t (NULL = the ctx's own stream). */
int evd_set_stream(evd_ctx *ctx, void *cuda_stream);
/* Number of kernels this context has launched so far. */
int64_t evd_kernel_launches(const evd_ctx *ctx);
/* Generation of the resident window: changes whenever a call replaces it
 * (evd_set_events, the stream solves).  A binding that keeps one window
 * resident across per-call entry points (bound_terms, contrast_at, ...)
 * re-uploads only when the generation or the caller's arrays changed. */
int64_t evd_window_generation(const evd_ctx *ctx);
/* SM count of the context's device. */
int evd_device_sms(const evd_ctx *ctx);

/* ---- event window (EventBatch, events.py:93-120) ---------------------- */
/* Copies one window's SoA events (x, y, t in [0, tau]) to device memory; they
 * stay resident for every following evaluation until the next call.  The
 * arrays may be host memory or device memory of the context's GPU (unified
 * addressing): a window broadcast to every rank's GPU (NCCL) is loaded without
 * a host round trip.  Likewise for evd_solve_stream / evd_load_stream. */
int evd_set_events(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                   int32_t width, int32_t height, double tau);

/* k windows given as separate host arrays, resident as one concatenation (window
 * w at offset counts[0] + ... + counts[w-1]) for evd_solve_windows: the arrays
 * are gathered through pinned staging while the previous chunk is copied, with
 * no host-side concatenation (estimate_stream_divergence, solver.py:139-162,
 * over a list of EventBatch). */
int evd_set_events_list(evd_ctx *ctx, const double *const *x, const double *const *y,
                        const double *const *t, const int64_t *counts, int32_t k, int32_t width,
                        int32_t height, double tau);

/* ---- motion model ------------------------------------------------------ */
/* radial_warp (geometry.py:78-87) of n arbitrary points. */
int evd_radial_warp(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                    double nu, double tau, int32_t width, int32_t height, double *x_out,
                    double *y_out);

/* warp_scale (geometry.py:70-75): s = (1 + nu*t) / (1 + nu*tau) for n times. */
int evd_warp_scale(evd_ctx *ctx, const double *t, int64_t n, double nu, double tau,
                   double *s_out);

/* ---- objective and bounds on the resident window ----------------------- */
/* accumulate_image (contrast.py:48-58) + image_contrast (contrast.py:61-64) /
 * contrast_at (solver.py:74-76) at k velocities.  counts (nullable) receives
 * k row-major (height, width) uint32 images. */
int evd_point_images(evd_ctx *ctx, const double *nu, int32_t k, int64_t *in_image,
                     double *contrast, uint32_t *counts);

/* upper_bound_image (contrast.py:231-238) / bound_terms (contrast.py:241-251)
 * for k intervals [lo_j, hi_j]: s_bar = sum(H_bar^2) (exact), fully_inside
 * (contrast.py:195-201), marks = sum(H_bar) (= upper_bound_image().in_image_events).
 * counts (nullable) receives k uint32 images.  c_bar is assembled by the
 * caller as s_bar/M - (fully_inside/M)**2 exactly as contrast.py:248-251. */
int evd_bound_images(evd_ctx *ctx, const double *lo, const double *hi, int32_t k,
                     uint64_t *s_bar, int64_t *fully_inside, uint64_t *marks,
                     uint32_t *counts);

/* Batched frontier: bound_terms (contrast.py:241-251) for k intervals in one
 * call over the resident window.  Same outputs as evd_bound_images without
 * images.  Paths (evd_set_option "frontier_path"):
 *  EVD_FRONTIER_TILES        the window is binned once into angular tiles
 *                            about the FOE (nu-invariant: the radial warp keeps
 *                            each event on its ray); each CTA evaluates a
 *                            (tile, 32 intervals) item with the 32 tile images
 *                            in shared memory and reduces them on chip -- no
 *                            image ever reaches HBM.  Needs every hi <= 0 and
 *                            finite events (the reference domain is [lo0, 0]);
 *  EVD_FRONTIER_GLOBAL       K x M u32 images in HBM (at most
 *                            "frontier_image_budget" bytes per launch, larger
 *                            k in chunks), filtered warp + exact fallback;
 *  EVD_FRONTIER_GLOBAL_EXACT the same with exact warps only;
 *  EVD_FRONTIER_PER_INTERVAL one evd_bound_images pass per interval (lane =
 *                            event: best for a few, wide intervals);
 *  EVD_FRONTIER_AUTO         per-interval up to 32 intervals, else tiles
 *                            when they apply, else global (default).
 * Every path returns identical integers. */
enum {
    EVD_FRONTIER_AUTO = 0,
    EVD_FRONTIER_TILES = 1,
    EVD_FRONTIER_GLOBAL = 2,
    EVD_FRONTIER_GLOBAL_EXACT = 3,
    EVD_FRONTIER_PER_INTERVAL = 4
};
int evd_eval_frontier(evd_ctx *ctx, const double *lo, const double *hi, int32_t k,
                      uint64_t *s_bar, int64_t *fully_inside, uint64_t *marks);

/* Per-context options: "frontier_path" (EVD_FRONTIER_*), "frontier_image_budget"
 * (bytes of HBM images per global-path launch, default 8 GiB), "stream_overlap"
 * (1, default: evd_solve_stream / evd_solve_windows_list upload host events
 * while the solve runs; 0: upload, then solve) and "stream_chunk" (events per
 * upload chunk, 1024..262144, default 65536). */
int evd_set_option(evd_ctx *ctx, const char *name, int64_t value);

/* Diagnostics of the tiled frontier: out[0] tiles of the frame (0: not
 * tiled), out[1] largest tile (pixels), out[2] events listed over all tiles
 * for the resident window (-1: not binned or not usable), out[3] tiles with
 * work, out[4] path of the last evd_eval_frontier call (EVD_FRONTIER_*). */
int evd_frontier_info(evd_ctx *ctx, int64_t *out);

/* image_contrast (contrast.py:61-64) of a caller image: np.sum((c - mean)**2)/M
 * with numpy's pairwise summation order; mean = in_image / m. */
int evd_image_contrast(evd_ctx *ctx, const double *counts, int64_t m, int64_t in_image,
                       double *contrast);

/* rasterize_segment (contrast.py:206-222) for k segments (ax, ay, bx, by);
 * counts receives k uint32 (height, width) mark images (each mark 0/1).
 * chunk: crossings per sampling chunk (0 = the kernels' default); any value
 * gives the same pixels -- exposed so tests can exercise chunk seams. */
int evd_rasterize_segments(evd_ctx *ctx, const double *segs, int32_t k, int32_t width,
                           int32_t height, int32_t chunk, uint32_t *counts);

/* ---- branch and bound (maximise_contrast_bnb, solver.py:79-123) -------- */
typedef struct {
    double gamma;               /* SolverParams.gamma (solver.py:51) */
    double epsilon;             /* SolverParams.epsilon */
    double min_interval_width;  /* SolverParams.min_interval_width */
    int64_t max_iterations;     /* SolverParams.max_iterations */
} evd_solve_params;

typedef struct {
    double nu;            /* BnbResult.nu */
    double contrast;      /* BnbResult.contrast */
    double bound_gap;     /* BnbResult.bound_gap */
    int64_t iterations;   /* BnbResult.iterations */
    int64_t bound_evals;  /* bound_terms evaluations (root + 2 per expanded node) */
    int64_t point_evals;  /* contrast_at evaluations */
    int64_t max_frontier; /* largest live queue */
    double device_ms;     /* device time of the solve (CUDA events on the ctx stream) */
    uint64_t marks;       /* pixel increments made in all images (atomic work) */
    uint64_t exact_events;/* event x node evaluations that needed the exact (division) path */
    int64_t rounds;       /* device rounds (grid-wide node-evaluation steps): < iterations
                             when speculative rounds evaluated several nodes at once */
} evd_solve_result;

/* The per-node work of maximise_contrast_bnb (solver.py:109-117) for k nodes
 * [lo[i], hi[i]] of the resident window: contrast_at(center) and
 * bound_terms(child).c_bar of both halves (VelocityInterval.split,
 * geometry.py:40-46), bit-identical to the reference's values; the nodes run
 * through the solve kernel's speculative rounds (several per event pass),
 * without a search.  Used by the host-driven exact BnB that splits a round's
 * nodes over GPUs (dist.solve_spec).  EVD_ERR_CHEIRALITY for an inadmissible
 * endpoint. */
int evd_eval_nodes(evd_ctx *ctx, const double *lo, const double *hi, int64_t k,
                   double *contrast, double *cbar_lo, double *cbar_hi);

/* Whole solve on the device for the resident window (one cooperative
 * persistent launch).  Returns EVD_ERR_ITER_LIMIT with the incumbent in *res
 * when max_iterations is reached. */
int evd_solve(evd_ctx *ctx, const evd_solve_params *params, evd_solve_result *res);

/* maximise_contrast_bnb (solver.py:79-123) for the window x, y, t (host,
 * pinned or device memory; evd_set_events' arguments) in one call: upload,
 * centring and solve are queued back to back with one host synchronisation.
 * Same results as evd_set_events + evd_solve; the window stays resident.  The
 * inputs are not retained. */
int evd_solve_events(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                     int32_t width, int32_t height, double tau, const evd_solve_params *params,
                     evd_solve_result *res);

/* Many windows in one launch (estimate_stream_divergence, solver.py:139-162):
 * window w is events [offsets[w], offsets[w+1]) of the resident event set
 * (evd_set_events with all windows concatenated; they share width, height,
 * tau).  The CTAs are split into `groups` independent solvers (0 = auto) that
 * take windows round-robin; each window is solved exactly as evd_solve.
 * results[w].status: EVD_OK, EVD_ERR_ITER_LIMIT (incumbent in the record),
 * or EVD_ERR_NO_EVENTS for an empty window. */
typedef struct {
    double nu, contrast, bound_gap;
    int64_t iterations, bound_evals, point_evals, max_frontier;
    uint64_t marks, exact_events;
    int32_t status;
    int32_t groups;   /* solver groups the launch used */
    int64_t rounds;   /* device rounds (see evd_solve_result) */
} evd_window_result;

int evd_solve_windows(evd_ctx *ctx, const int64_t *offsets, int32_t n_windows, int32_t groups,
                      const evd_solve_params *params, evd_window_result *results,
                      double *device_ms);

/* evd_set_events_list + evd_solve_windows in one call, the upload overlapped
 * with the solve: the solve is launched first, the host windows follow in
 * chunks on a copy stream, and each window's solver group starts once its
 * events have arrived (estimate_stream_divergence, solver.py:139-162, over a
 * list of EventBatch).  Results and the resident window set afterwards are
 * those of the two calls; device_ms includes the wait for the events. */
int evd_solve_windows_list(evd_ctx *ctx, const double *const *x, const double *const *y,
                           const double *const *t, const int64_t *counts, int32_t k,
                           int32_t width, int32_t height, double tau, int32_t groups,
                           const evd_solve_params *params, evd_window_result *results,
                           double *device_ms);

/* batch_stream + estimate_stream_divergence (events.py:330-359,
 * solver.py:139-162) for a whole time-sorted stream in one call: the raw
 * events go to the device once, the windows [k*tau, (k+1)*tau) are found by
 * binary search (on the host copy of t for host arrays, else on the device),
 * their events are gathered into the solve layout (centred x, y; batch-local
 * t = min(t - k*tau, tau)) and every window is solved in one evd_solve_windows
 * launch.  Host arrays are uploaded while the solve runs ("stream_overlap"):
 * each window's group gathers its events once they have arrived.  *n_windows = k1 - k0 + 1 (also
 * on EVD_ERR_ARG when `capacity` is too small), *k0 = floor(t[0] / tau);
 * results[w] describes window k0 + w (t_start = (k0 + w) * tau; status
 * EVD_ERR_NO_EVENTS for an empty window).  The stream becomes the context's
 * resident event set (as evd_set_events), windows concatenated. */
int evd_solve_stream(evd_ctx *ctx, const double *x, const double *y, const double *t, int64_t n,
                     int32_t width, int32_t height, double tau, int32_t groups,
                     const evd_solve_params *params, evd_window_result *results,
                     int32_t capacity, int32_t *n_windows, int64_t *k0, double *device_ms);

/* Same pipeline on the stream already resident in the context (the last
 * evd_solve_stream upload or evd_load_bin). */
int evd_solve_loaded_stream(evd_ctx *ctx, double tau, int32_t groups,
                            const evd_solve_params *params, evd_window_result *results,
                            int32_t capacity, int32_t *n_windows, int64_t *k0,
                            double *device_ms);

/* ---- EVD1 event files ------------------------------ */
/* parse_event_bin (events.py:186-206) + _from_columns (:128-134) on the
 * device: the 20-byte <4sIIQ> header is checked on the host, the packed
 * 17-byte records <u8 t_us, f4 x, f4 y, i1 p> are copied once and decoded on
 * the device (t = float64(t_us) * 1e-6, x, y widened exactly), stably sorted
 * by t when out of order, and checked against the EventStream invariants
 * (EVD_ERR_VALIDATION with the reference's message).  The stream stays
 * resident for evd_solve_loaded_stream / evd_stream_copy. */
int evd_load_bin(evd_ctx *ctx, const uint8_t *data, int64_t size, int32_t *width,
                 int32_t *height, int64_t *n);
/* Upload a host stream (time-sorted, validated as EventStream is) as the
 * resident stream; p (polarity) may be NULL. */
int evd_load_stream(evd_ctx *ctx, const double *x, const double *y, const double *t,
                    const int8_t *p, int64_t n, int32_t width, int32_t height);

/* ---- preprocessing of the resident stream ----------- */
/* pixel_counts (events.py:273-281): floor-binned per-pixel counts, H*W int64. */
int evd_pixel_counts(evd_ctx *ctx, int64_t *counts);
/* remove_hot_pixels (events.py:284-300): median and MAD of the nonzero counts
 * (device sorts; numpy's median of an even count = mean of the middle two),
 * threshold = med + k*mad, events on pixels above it dropped (stable).
 * *n = events kept; *threshold = the threshold (0 for an empty stream). */
int evd_stream_remove_hot_pixels(evd_ctx *ctx, double k, int64_t *n, double *threshold);
/* rescale_events (events.py:303-313): x * (W'/W), y * (H'/H), capped below W', H'. */
int evd_stream_rescale(evd_ctx *ctx, int32_t width, int32_t height);

/* Copy the resident stream to host arrays of n elements (any may be NULL). */
int evd_stream_copy(evd_ctx *ctx, double *x, double *y, double *t, int8_t *p);

/* Tracing is off unless the environment holds EVD_TRACE=1 when the context
 * is created (it costs a few percent).
 * Device timestamps (ns, %globaltimer) of the last solve (first window of
 * group 0): out[0] = start, then 10 slots per node evaluation (see
 * csrc/evd_internal.h TraceSlot: 8 timestamps, then the node's segment marks
 * and exact-path events).  *n receives the number of valid entries. */
int evd_solve_trace(evd_ctx *ctx, int64_t *out, int64_t cap, int64_t *n);

/* Per-block timestamps of the first 128 node evaluations of the last
 * evd_solve: out[(i*blocks + b)*4 + k], k = node start, events done, pixels
 * done, step done (diagnostics). */
int evd_solve_block_trace(evd_ctx *ctx, int64_t *out, int64_t cap, int32_t *blocks);

/* Diagnostics: the solve kernel's exact event pass for one child evaluation
 * of [lo, hi] (point image at the centre, both child segment images), run
 * `reps` times in one launch on the solve grid; span_ns[r] = device time of
 * rep r.  Results are discarded. */
int evd_probe_events(evd_ctx *ctx, double lo, double hi, int32_t reps, double *span_ns);

/* ---- helpers ----------------------------------------------------------- */
/* out[f] = pow(f / m, 2.0) through the process's libm pow(), f = 0..n: the
 * value CPython's `mu_lower**2` yields (contrast.py:250-251). */
int evd_pow2_table(int64_t m, int64_t n, double *out);

#ifdef __cplusplus
}
#endif

#endif /* EVD_H */

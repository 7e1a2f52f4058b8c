// evd_io.cu -- EVD1 binary event files decoded on the device (SURVEY §8(f)
// row 3): parse_event_bin (pkg/src/eventdiv/events.py:186-206) and
// _from_columns (:128-134) -- t = float64(t_us) * 1e-6, x, y widened from f32
// (exact), a stable sort by t, then the EventStream invariants (:61-81).
// The decoded stream stays resident for evd_solve_stream's windowing.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "evd_device.cuh"
#include "evd_internal.h"

namespace evd {

constexpr int kIoThreads = 256;

__device__ __forceinline__ unsigned long long load_u64_le(const unsigned char *p)
{
    unsigned long long v = 0;
#pragma unroll
    for (int k = 7; k >= 0; k--) v = (v << 8) | p[k];
    return v;
}
__device__ __forceinline__ float load_f32_le(const unsigned char *p)
{
    const unsigned int u = (unsigned int)p[0] | ((unsigned int)p[1] << 8) |
                           ((unsigned int)p[2] << 16) | ((unsigned int)p[3] << 24);
    return __uint_as_float(u);
}

// One 17-byte packed record <u8 t_us, f4 x, f4 y, i1 p> per thread; `unsorted`
// is set if some t[i] > t[i+1] (the sort is then needed).
__global__ void k_decode_bin(const unsigned char *__restrict__ body, long long n,
                             double *__restrict__ x, double *__restrict__ y,
                             double *__restrict__ t, signed char *__restrict__ p,
                             unsigned long long *__restrict__ key, unsigned int *flags)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned char *r = body + 17 * i;
        const double ti = dmul(__ull2double_rn(load_u64_le(r)), 1e-6);  // events.py:129
        x[i] = (double)load_f32_le(r + 8);
        y[i] = (double)load_f32_le(r + 12);
        t[i] = ti;
        p[i] = (signed char)r[16];
        key[i] = (unsigned long long)__double_as_longlong(ti);  // t >= 0: bit order = value order
        if (i + 1 < n) {
            const double tn = dmul(__ull2double_rn(load_u64_le(r + 17)), 1e-6);
            if (ti > tn) atomicOr(flags, 1u);
        }
    }
}

__global__ void k_iota(long long n, long long *__restrict__ v)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] = i;
}

// Apply the stable order: out[i] = in[perm[i]].
__global__ void k_permute(long long n, const long long *__restrict__ perm,
                          const double *__restrict__ xi, const double *__restrict__ yi,
                          const double *__restrict__ ti, const signed char *__restrict__ pi,
                          double *__restrict__ xo, double *__restrict__ yo, double *__restrict__ to,
                          signed char *__restrict__ po)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long s = perm[i];
        xo[i] = xi[s];
        yo[i] = yi[s];
        to[i] = ti[s];
        po[i] = pi[s];
    }
}

// EventStream invariants (events.py:61-81): bit 1 non-finite coordinate,
// bit 2 coordinate outside [0, W) x [0, H), bit 3 polarity not +-1.
__global__ void k_validate(long long n, const double *__restrict__ x, const double *__restrict__ y,
                           const signed char *__restrict__ p, int W, int H, unsigned int *flags)
{
    unsigned int f = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double xi = x[i], yi = y[i];
        if (!isfinite(xi) || !isfinite(yi)) f |= 2u;
        if (xi < 0.0 || xi >= (double)W || yi < 0.0 || yi >= (double)H) f |= 4u;
        if (p[i] != 1 && p[i] != -1) f |= 8u;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

static int io_blocks(long long n)
{
    long long b = (n + kIoThreads - 1) / kIoThreads;
    return (int)std::max(1LL, std::min(b, 148LL * 16));
}

cudaError_t decode_bin(const unsigned char *body_dev, long long n, int W, int H, double *x,
                       double *y, double *t, signed char *p, void *scratch, size_t scratch_bytes,
                       unsigned int *flags_dev, unsigned int *flags_host, int *launches,
                       cudaStream_t s)
{
    // scratch: key[n], key_alt[n], perm[n], perm_alt[n], x/y/t alt[3n], p alt[n], cub temp
    unsigned long long *key = (unsigned long long *)scratch, *key2 = key + n;
    long long *perm = (long long *)(key2 + n), *perm2 = perm + n;
    double *x2 = (double *)(perm2 + n), *y2 = x2 + n, *t2 = y2 + n;
    signed char *p2 = (signed char *)(t2 + n);
    unsigned char *tmp = (unsigned char *)p2 + ((n + 255) / 256) * 256;
    const size_t used = (size_t)(tmp - (unsigned char *)scratch);
    cudaError_t e;
    if ((e = cudaMemsetAsync(flags_dev, 0, sizeof(unsigned int), s))) return e;
    k_decode_bin<<<io_blocks(n), kIoThreads, 0, s>>>(body_dev, n, x, y, t, p, key, flags_dev);
    ++*launches;
    if ((e = cudaMemcpyAsync(flags_host, flags_dev, sizeof(unsigned int), cudaMemcpyDeviceToHost, s)))
        return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    if (*flags_host & 1u) {  // np.argsort(t, kind="stable") (events.py:133)
        k_iota<<<io_blocks(n), kIoThreads, 0, s>>>(n, perm);
        ++*launches;
        size_t need = 0;
        cub::DoubleBuffer<unsigned long long> kb(key, key2);
        cub::DoubleBuffer<long long> vb(perm, perm2);
        cub::DeviceRadixSort::SortPairs(nullptr, need, kb, vb, (int)n, 0, 64, s);
        if (used + need > scratch_bytes) return cudaErrorMemoryAllocation;
        if ((e = cub::DeviceRadixSort::SortPairs(tmp, need, kb, vb, (int)n, 0, 64, s))) return e;
        ++*launches;
        if ((e = cudaMemcpyAsync(x2, x, n * sizeof(double), cudaMemcpyDeviceToDevice, s))) return e;
        if ((e = cudaMemcpyAsync(y2, y, n * sizeof(double), cudaMemcpyDeviceToDevice, s))) return e;
        if ((e = cudaMemcpyAsync(t2, t, n * sizeof(double), cudaMemcpyDeviceToDevice, s))) return e;
        if ((e = cudaMemcpyAsync(p2, p, n, cudaMemcpyDeviceToDevice, s))) return e;
        k_permute<<<io_blocks(n), kIoThreads, 0, s>>>(n, vb.Current(), x2, y2, t2, p2, x, y, t, p);
        ++*launches;
    }
    if ((e = cudaMemsetAsync(flags_dev, 0, sizeof(unsigned int), s))) return e;
    k_validate<<<io_blocks(n), kIoThreads, 0, s>>>(n, x, y, p, W, H, flags_dev);
    ++*launches;
    if ((e = cudaMemcpyAsync(flags_host, flags_dev, sizeof(unsigned int), cudaMemcpyDeviceToHost, s)))
        return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    return cudaGetLastError();
}

size_t decode_scratch_bytes(long long n)
{
    size_t need = 0;
    cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
    cub::DoubleBuffer<long long> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, need, kb, vb, (int)std::max(n, 1LL), 0, 64);
    return (size_t)n * (8 * 4 + 24 + 1) + 256 + need + 1024;
}

// ---------------------------------------------------------------- preprocessing
struct NonZeroCount {
    __host__ __device__ bool operator()(unsigned int c) const { return c > 0; }
};

// pixel_counts (events.py:273-281): floor-binned per-pixel counts.
__global__ void k_pixel_counts(const double *__restrict__ x, const double *__restrict__ y,
                               long long n, int W, unsigned int *counts)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)floor(x[i]), iy = (int)floor(y[i]);  // in frame (validated)
        atomicAdd(counts + (long long)iy * W + ix, 1u);
    }
}

// |c - med| of the sorted nonzero counts, as doubles (exact: integers and
// half-integers), for the MAD.
__global__ void k_abs_dev(const unsigned int *__restrict__ v, long long n, double med,
                          double *__restrict__ d)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d[i] = fabs(dsub((double)v[i], med));
}

// keep[i] = the event's pixel is not hot (counts > threshold, events.py:294-298)
__global__ void k_keep_flags(const double *__restrict__ x, const double *__restrict__ y,
                             long long n, int W, const unsigned int *__restrict__ counts,
                             double threshold, unsigned char *__restrict__ keep)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)floor(x[i]), iy = (int)floor(y[i]);
        keep[i] = !((double)counts[(long long)iy * W + ix] > threshold);
    }
}

// rescale_events (events.py:303-313): x * (W'/W) capped at nextafter(W', 0).
__global__ void k_rescale(double *__restrict__ x, double *__restrict__ y, long long n,
                          double sx, double sy, double xmax, double ymax)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double a = dmul(x[i], sx), b = dmul(y[i], sy);
        x[i] = a < xmax ? a : xmax;  // np.minimum (no NaN: coordinates are finite)
        y[i] = b < ymax ? b : ymax;
    }
}

cudaError_t pixel_counts_dev(const double *x, const double *y, long long n, int W, int H,
                             unsigned int *counts, int *launches, cudaStream_t s)
{
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)W * H * sizeof(unsigned int), s);
    if (e) return e;
    if (n > 0) {
        k_pixel_counts<<<io_blocks(n), kIoThreads, 0, s>>>(x, y, n, W, counts);
        ++*launches;
    }
    return cudaGetLastError();
}

// Order statistic(s) numpy's median takes from a sorted array of n values.
template <class T>
static cudaError_t median_of_sorted(const T *sorted, long long n, double *out, cudaStream_t s)
{
    T a = 0, b = 0;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(&b, sorted + n / 2, sizeof(T), cudaMemcpyDeviceToHost, s))) return e;
    if (n % 2 == 0 &&
        (e = cudaMemcpyAsync(&a, sorted + n / 2 - 1, sizeof(T), cudaMemcpyDeviceToHost, s)))
        return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    // np.median: the middle value, or the mean of the two middle values
    *out = (n % 2) ? (double)b : ((double)a + (double)b) / 2.0;
    return cudaSuccess;
}

cudaError_t remove_hot_pixels_dev(double *x, double *y, double *t, signed char *p, long long n,
                                  int W, int H, double k, void *scratch, size_t scratch_bytes,
                                  long long *n_out, double *threshold_out, int *launches,
                                  cudaStream_t s)
{
    const long long M = (long long)W * H;
    // scratch: counts[M] u32, nz[M] u32, nz_sorted[M] u32, dev[M] f64, dev_sorted[M] f64,
    // keep[n] u8, x/y/t/p copies, counters, cub temp
    unsigned char *base = (unsigned char *)scratch;
    auto take = [&](size_t bytes) {
        unsigned char *r = base;
        base += (bytes + 255) / 256 * 256;
        return r;
    };
    unsigned int *counts = (unsigned int *)take(M * 4), *nz = (unsigned int *)take(M * 4);
    unsigned int *nzs = (unsigned int *)take(M * 4);
    double *dv = (double *)take(M * 8), *dvs = (double *)take(M * 8);
    unsigned char *keep = take(n);
    double *x2 = (double *)take(n * 8), *y2 = (double *)take(n * 8), *t2 = (double *)take(n * 8);
    signed char *p2 = (signed char *)take(n);
    long long *cnt = (long long *)take(64);
    unsigned char *tmp = base;
    const size_t avail = scratch_bytes - (size_t)(tmp - (unsigned char *)scratch);
    cudaError_t e;
    if ((e = pixel_counts_dev(x, y, n, W, H, counts, launches, s))) return e;
    // nonzero counts, sorted
    size_t need = 0;
    cub::DeviceSelect::If(nullptr, need, counts, nz, cnt, (int)M, NonZeroCount{}, s);
    if (need > avail) return cudaErrorMemoryAllocation;
    if ((e = cub::DeviceSelect::If(tmp, need, counts, nz, cnt, (int)M, NonZeroCount{}, s))) return e;
    ++*launches;
    long long nnz = 0;
    if ((e = cudaMemcpyAsync(&nnz, cnt, 8, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, nz, nzs, (int)nnz, 0, 32, s);
    if (need > avail) return cudaErrorMemoryAllocation;
    if ((e = cub::DeviceRadixSort::SortKeys(tmp, need, nz, nzs, (int)nnz, 0, 32, s))) return e;
    ++*launches;
    double med = 0.0, mad = 0.0;
    if ((e = median_of_sorted(nzs, nnz, &med, s))) return e;
    k_abs_dev<<<io_blocks(nnz), kIoThreads, 0, s>>>(nzs, nnz, med, dv);
    ++*launches;
    // non-negative doubles sort as their bit patterns
    need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, (unsigned long long *)dv,
                                   (unsigned long long *)dvs, (int)nnz, 0, 64, s);
    if (need > avail) return cudaErrorMemoryAllocation;
    if ((e = cub::DeviceRadixSort::SortKeys(tmp, need, (unsigned long long *)dv,
                                            (unsigned long long *)dvs, (int)nnz, 0, 64, s)))
        return e;
    ++*launches;
    if ((e = median_of_sorted(dvs, nnz, &mad, s))) return e;
    const double threshold = med + k * mad;  // events.py:292
    *threshold_out = threshold;
    k_keep_flags<<<io_blocks(n), kIoThreads, 0, s>>>(x, y, n, W, counts, threshold, keep);
    ++*launches;
    // stable compaction of the kept events
    if ((e = cudaMemcpyAsync(x2, x, n * 8, cudaMemcpyDeviceToDevice, s))) return e;
    if ((e = cudaMemcpyAsync(y2, y, n * 8, cudaMemcpyDeviceToDevice, s))) return e;
    if ((e = cudaMemcpyAsync(t2, t, n * 8, cudaMemcpyDeviceToDevice, s))) return e;
    if ((e = cudaMemcpyAsync(p2, p, n, cudaMemcpyDeviceToDevice, s))) return e;
    need = 0;
    cub::DeviceSelect::Flagged(nullptr, need, x2, keep, x, cnt, (int)n, s);
    if (need > avail) return cudaErrorMemoryAllocation;
    if ((e = cub::DeviceSelect::Flagged(tmp, need, x2, keep, x, cnt, (int)n, s))) return e;
    if ((e = cub::DeviceSelect::Flagged(tmp, need, y2, keep, y, cnt, (int)n, s))) return e;
    if ((e = cub::DeviceSelect::Flagged(tmp, need, t2, keep, t, cnt, (int)n, s))) return e;
    if ((e = cub::DeviceSelect::Flagged(tmp, need, p2, keep, p, cnt, (int)n, s))) return e;
    *launches += 4;
    if ((e = cudaMemcpyAsync(n_out, cnt, 8, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    return cudaGetLastError();
}

size_t preprocess_scratch_bytes(long long n, long long M)
{
    const int m = (int)std::max(M, 1LL), nn = (int)std::max(n, 1LL);
    size_t a = 0, b = 0, c = 0, d = 0;
    cub::DeviceSelect::If(nullptr, a, (unsigned int *)nullptr, (unsigned int *)nullptr,
                          (long long *)nullptr, m, NonZeroCount{});
    cub::DeviceRadixSort::SortKeys(nullptr, b, (unsigned int *)nullptr, (unsigned int *)nullptr, m,
                                   0, 32);
    cub::DeviceRadixSort::SortKeys(nullptr, c, (unsigned long long *)nullptr,
                                   (unsigned long long *)nullptr, m, 0, 64);
    cub::DeviceSelect::Flagged(nullptr, d, (double *)nullptr, (unsigned char *)nullptr,
                               (double *)nullptr, (long long *)nullptr, nn);
    const size_t tmp = std::max(std::max(a, b), std::max(c, d));
    const size_t fixed = (size_t)M * (4 + 4 + 4 + 8 + 8) + (size_t)n * (1 + 24 + 1) + 64 + 12 * 256;
    return fixed + tmp + 4096;
}

cudaError_t rescale_dev(double *x, double *y, long long n, double sx, double sy, double xmax,
                        double ymax, int *launches, cudaStream_t s)
{
    if (n > 0) {
        k_rescale<<<io_blocks(n), kIoThreads, 0, s>>>(x, y, n, sx, sy, xmax, ymax);
        ++*launches;
    }
    return cudaGetLastError();
}

}  // namespace evd

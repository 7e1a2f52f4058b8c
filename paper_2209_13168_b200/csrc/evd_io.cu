// evd_io.cu -- EVD1 binary event files decoded on the device (SURVEY §8(f)
// row 3): parse_event_bin (pkg/src/eventdiv/events.py:186-206) and
// _from_columns (:128-134) -- t = float64(t_us) * 1e-6, x, y widened from f32
// (exact), a stable sort by t, then the EventStream invariants (:61-81).
// The decoded stream stays resident for evd_solve_stream's windowing.
#include <cub/device/device_radix_sort.cuh>

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

}  // namespace evd

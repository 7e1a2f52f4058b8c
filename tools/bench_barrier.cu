// Microbenchmark of grid-barrier implementations for the persistent solve
// kernel (148 blocks x 512 threads, cooperative launch).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_barrier tools/bench_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

struct Bar {
    unsigned int count;
    unsigned int gen;
};

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_relaxed(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int atom_add_acqrel(unsigned int *p, unsigned int v)
{
    unsigned int old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(unsigned int *p, unsigned int v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// A: the solve kernel's first barrier (threadfence + nanosleep poll)
__device__ void bar_a(Bar *b)
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

// B: acq_rel atomic arrival, release store, acquire spin (no nanosleep)
template <bool SLEEP>
__device__ void bar_b(Bar *b)
{
    __shared__ unsigned int s_gen;
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int g = ld_relaxed(&b->gen);
        const unsigned int old = atom_add_acqrel(&b->count, 1u);
        s_gen = g;
        s_last = old == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __syncthreads();
        if (threadIdx.x == 0) {
            b->count = 0;
            st_release(&b->gen, s_gen + 1);
        }
    } else if (threadIdx.x == 0) {
        while (ld_acquire(&b->gen) == s_gen)
            if (SLEEP) __nanosleep(8);
    }
    __syncthreads();
}

// C: monotone counter, no reset: arrive with atom.add.release; target = round*G
__device__ void bar_c(unsigned int *ctr, unsigned int target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_acquire(ctr) < target) {
        }
    }
    __syncthreads();
}

__global__ void k_bar(int variant, int iters, Bar *b, unsigned int *ctr, long long *out)
{
    long long t0 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; i++) {
        if (variant == 0) bar_a(b);
        else if (variant == 1) bar_b<false>(b);
        else if (variant == 2) bar_b<true>(b);
        else if (variant == 3) bar_c(ctr, (unsigned)(i + 1) * gridDim.x);
        else cg::this_grid().sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[0] = t1 - t0;
    }
}

// L2 round-trip latency: one thread chasing dependent __ldcg loads
__global__ void k_chase(const unsigned int *p, int n, long long *out)
{
    long long t0, t1;
    unsigned int j = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; i++) j = __ldcg(p + j);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = t1 - t0;
    out[1] = j;
}

__global__ void k_fence(int n, long long *out, int kind)
{
    long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; i++) {
        if (kind == 0) __threadfence();
        else fence_acqrel();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main()
{
    Bar *b;
    unsigned int *ctr, *chain;
    long long *out;
    cudaMalloc(&b, sizeof(Bar));
    cudaMalloc(&ctr, 4);
    cudaMalloc(&out, 16);
    const int n = 1 << 22;
    cudaMalloc(&chain, n * 4);
    unsigned int *h = new unsigned int[n];
    for (int i = 0; i < n; i++) h[i] = (unsigned)((i + 1 + 7919 * 64) % n);
    cudaMemcpy(chain, h, n * 4, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char *names[] = {"A threadfence+nanosleep20", "B acq_rel spin", "B acq_rel nanosleep8",
                           "C monotone red.release", "cg grid.sync"};
    for (int threads : {512, 256}) {
        for (int v = 0; v < 5; v++) {
            for (int rep = 0; rep < 2; rep++) {
                cudaMemset(b, 0, sizeof(Bar));
                cudaMemset(ctr, 0, 4);
                int iters = 2000;
                void *args[] = {&v, &iters, &b, &ctr, &out};
                cudaError_t e = cudaLaunchCooperativeKernel((void *)k_bar, sms, threads, args);
                cudaDeviceSynchronize();
                long long ns = 0;
                cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
                if (rep) printf("%-28s blocks=%d threads=%d: %.3f us/barrier (%s)\n", names[v], sms,
                                threads, ns / 1e3 / iters, cudaGetErrorString(e));
            }
        }
    }
    k_chase<<<1, 1>>>(chain, 100000, out);
    cudaDeviceSynchronize();
    long long r[2];
    cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
    printf("L2 dependent-load latency: %.1f ns\n", r[0] / 100000.0);
    for (int kind = 0; kind < 2; kind++) {
        k_fence<<<1, 32>>>(10000, out, kind);
        cudaDeviceSynchronize();
        cudaMemcpy(r, out, 8, cudaMemcpyDeviceToHost);
        printf("%s: %.1f ns\n", kind ? "fence.acq_rel.gpu" : "__threadfence", r[0] / 10000.0);
    }
    return 0;
}

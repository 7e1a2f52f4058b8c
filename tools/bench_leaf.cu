// Microbenchmark: cost of one pairwise-sum leaf (8-lane group, <=128 u32
// pixels) as used by the solve's pixel phase.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_2209_13168_b200/csrc -o tools/bench_leaf tools/bench_leaf.cu
#include <cstdio>

#include "evd_device.cuh"

using namespace evd;

struct SqLoadOnly {
    typedef unsigned int raw;
    const unsigned int *img;
    double mu;
    __device__ raw load(int i) const { return __ldcg(img + i); }
    __device__ void clear(int) const {}
    __device__ double term(raw h) const { return (double)h; }
};
struct SqFull {
    typedef unsigned int raw;
    unsigned int *img;
    double mu;
    __device__ raw load(int i) const { return __ldcg(img + i); }
    __device__ void clear(int i) const { img[i] = 0u; }
    __device__ double term(raw h) const
    {
        const double d = evd::dsub((double)h, mu);
        return evd::dmul(d, d);
    }
};
struct SqPlain {
    typedef unsigned int raw;
    unsigned int *img;
    double mu;
    __device__ raw load(int i) const { return img[i]; }
    __device__ void clear(int i) const { img[i] = 0u; }
    __device__ double term(raw h) const
    {
        const double d = evd::dsub((double)h, mu);
        return evd::dmul(d, d);
    }
};

template <class Q>
__global__ void k_leaf(Q q, int leaf_n, long long *cyc, double *out)
{
    const int j = threadIdx.x & 7, g = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    __syncthreads();
    long long t0 = clock64();
    const double v = pairwise_leaf8(g * leaf_n, leaf_n, j, q);
    long long t1 = clock64();
    if (j == 0) out[g] = v;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main()
{
    const int M = 148 * 64 * 128;
    unsigned int *img;
    long long *cyc;
    double *out;
    cudaMalloc(&img, M * 4);
    cudaMalloc(&cyc, 8);
    cudaMalloc(&out, M);
    cudaMemset(img, 1, M * 4);
    for (int leaf : {64, 88, 128}) {
        for (int rep = 0; rep < 3; rep++) {
            long long c[3];
            k_leaf<<<148, 512>>>(SqLoadOnly{img, 0.5}, leaf, cyc, out);
            cudaMemcpy(&c[0], cyc, 8, cudaMemcpyDeviceToHost);
            k_leaf<<<148, 512>>>(SqFull{img, 0.5}, leaf, cyc, out);
            cudaMemcpy(&c[1], cyc, 8, cudaMemcpyDeviceToHost);
            k_leaf<<<148, 512>>>(SqPlain{img, 0.5}, leaf, cyc, out);
            cudaMemcpy(&c[2], cyc, 8, cudaMemcpyDeviceToHost);
            if (rep == 2)
                printf("leaf %3d: loads-only %lld cyc, ldcg+term+clear %lld, plain ld %lld\n", leaf,
                       c[0], c[1], c[2]);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

// Peak throughput of global u32 atomicAdd (RED, no return) into an image-sized
// buffer, the operation that builds every point / segment image.  Used as the
// atomic-roofline denominator (profiles/atomic_peak.json).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_atomics tools/bench_atomics.cu
#include <cstdio>

__global__ void k_red(unsigned int *img, unsigned int m, int per_thread, unsigned int seed)
{
    unsigned int x = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
#pragma unroll 8
    for (int i = 0; i < per_thread; i++) {
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        atomicAdd(img + (x % m), 1u);
    }
}

// neighbouring lanes hit neighbouring pixels (a segment walking the image)
__global__ void k_red_walk(unsigned int *img, unsigned int m, int per_thread, unsigned int seed)
{
    const unsigned int t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned int p = (t * 977u + seed) % m;
    for (int i = 0; i < per_thread; i++) {
        atomicAdd(img + p, 1u);
        p = (p + 1) % m;
    }
}

int main()
{
    unsigned int *img;
    cudaMalloc(&img, 64u << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, per = 256;
    const double total = (double)blocks * threads * per;
    printf("{");
    const char *sep = "";
    for (unsigned int m : {43200u, 89960u, 307200u, 921600u}) {
        cudaMemset(img, 0, m * 4);
        for (int kind = 0; kind < 2; kind++) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; rep++) {
                cudaEventRecord(a);
                if (kind == 0) k_red<<<blocks, threads>>>(img, m, per, 12345u + rep);
                else k_red_walk<<<blocks, threads>>>(img, m, per, 777u + rep);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("%s\"%s_m%u_gatomics_per_s\": %.2f", sep, kind ? "walk" : "random", m,
                   total / (best * 1e-3) / 1e9);
            sep = ", ";
        }
    }
    printf("}\n");
    return 0;
}

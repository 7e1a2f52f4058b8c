// Peak throughputs of the instruction classes that bound the hot path
// (profiles/fp64_peak.json): binary64 add / mul / fma (the warps, the
// certification margins), the IEEE division sequence __ddiv_rn (every exact
// warp, every Liang-Barsky quotient and grid crossing), floor (FRND.F64) and
// shared-memory u32 atomic adds with lanes in distinct banks (the tiled
// frontier's image marks), plus the u16-pair shared increment it uses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_fp64 tools/bench_fp64.cu
#include <cstdio>

constexpr int kChains = 8;  // independent dependency chains per thread

template <int OP>
__global__ void k_fp64(double *out, int iters, double a, double b)
{
    double v[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) v[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) {
            if (OP == 0) v[c] = __dadd_rn(v[c], a);
            if (OP == 1) v[c] = __dmul_rn(v[c], b);
            if (OP == 2) v[c] = __fma_rn(v[c], b, a);
            if (OP == 3) v[c] = __ddiv_rn(a, v[c] + 1.5);
            if (OP == 4) v[c] = floor(v[c] * b) + a;
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += v[c];
    if (s == 12345.678) out[0] = s;
}

// shared u32 atomics: lane l of warp w adds to word (l * 33 + i) % words
// (distinct banks), fire-and-forget like the tiled frontier's red.shared
__global__ void k_smem_red(unsigned *out, int iters, int words, int pair)
{
    extern __shared__ unsigned img[];
    for (int i = threadIdx.x; i < words; i += blockDim.x) img[i] = 0;
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(img);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned p = (unsigned)(lane * 33 + warp * 7) % words;
    for (int i = 0; i < iters; i++) {
        const unsigned inc = pair ? (1u << ((i & 1) << 4)) : 1u;
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base + 4u * p), "r"(inc) : "memory");
        p += 32 * 33;
        if (p >= (unsigned)words) p -= words;
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = img[0];
}

template <class F>
static float best_ms(F launch)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
    }
    return best;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *dout;
    unsigned *uout;
    cudaMalloc(&dout, 64);
    cudaMalloc(&uout, 1 << 20);
    const int blocks = sms * 4, threads = 512, iters = 4096;
    const double ops = (double)blocks * threads * iters * kChains;
    const char *names[] = {"dadd", "dmul", "dfma", "ddiv_rn", "floor_dmul_dadd"};
    printf("{\"sms\": %d, \"sm_clock_mhz_attr\": %d", sms, clk / 1000);
    float ms[5];
    ms[0] = best_ms([&] { k_fp64<0><<<blocks, threads>>>(dout, iters, 1e-9, 1.0000001); });
    ms[1] = best_ms([&] { k_fp64<1><<<blocks, threads>>>(dout, iters, 1e-9, 1.0000001); });
    ms[2] = best_ms([&] { k_fp64<2><<<blocks, threads>>>(dout, iters, 1e-9, 1.0000001); });
    ms[3] = best_ms([&] { k_fp64<3><<<blocks, threads>>>(dout, iters / 8, 1.25, 1.0); });
    ms[4] = best_ms([&] { k_fp64<4><<<blocks, threads>>>(dout, iters, 0.5, 1.0000001); });
    for (int k = 0; k < 5; k++) {
        const double n = k == 3 ? ops / 8 : ops;
        printf(", \"%s_g_per_s\": %.2f", names[k], n / (ms[k] * 1e-3) / 1e9);
    }
    // lanes per SM per clock at the attribute clock (a sanity scale, not a peak)
    printf(", \"dfma_lanes_per_sm_clk\": %.2f",
           ops / (ms[2] * 1e-3) / sms / (clk * 1e3));
    const int words = 40000, sm_threads = 512, sm_iters = 1 << 14;
    cudaFuncSetAttribute(k_smem_red, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4);
    const double reds = (double)sms * sm_threads * sm_iters;
    for (int pair = 0; pair < 2; pair++) {
        const float t = best_ms(
            [&] { k_smem_red<<<sms, sm_threads, words * 4>>>(uout, sm_iters, words, pair); });
        printf(", \"%s_g_per_s\": %.2f", pair ? "smem_red_u16pair" : "smem_red_u32",
               reds / (t * 1e-3) / 1e9);
    }
    printf(", \"how\": \"tools/bench_fp64.cu: %d CTAs x %d threads, %d independent chains per "
           "thread (fp64); %d CTAs x %d threads, one CTA per SM, lanes in distinct banks "
           "(shared RED); best of 4 after a warm-up, CUDA events\"}\n",
           blocks, threads, kChains, sms, sm_threads);
    return 0;
}

// Cost of the OU noise sample on B200: samples/s of the pieces of
// stream_xi (csrc/vxb_device.cuh) with one CTA of 1024 threads per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_2308_01241_b200/csrc -o mbnoise tools/microbench_noise.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "vxb_device.cuh"
using namespace vxb;

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint64_t root, uint32_t per_thread, float* out) {
    float acc = 0.0f;
    const uint64_t g0 = blockIdx.x * 1024ull + threadIdx.x;
    for (uint32_t t = 0; t < per_thread; ++t) {
        const uint64_t key = mix_key(root, g0);
        if (MODE == 0) acc += stream_xi(key, t);
        if (MODE == 1) acc += (float)stream_normal(key, t);
        if (MODE == 2) acc += (float)(stream_word(key, 2 * t) ^ stream_word(key, 2 * t + 1));
        if (MODE == 3) acc += (float)log(1.0 - stream_u01(key, 2 * t));
        if (MODE == 4) acc += (float)cos(6.283185307179586 * stream_u01(key, 2 * t + 1));
        if (MODE == 5) acc += (float)stream_u01(key, 2 * t) + (float)stream_u01(key, 2 * t + 1);
    }
    out[g0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sms * 1024 * sizeof(float));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint32_t pt = 256;
    const char* names[] = {"stream_xi (kernel's)", "stream_normal fast path", "2 splitmix words",
                           "words + log", "words + cos", "words -> 2 u01"};
    auto run = [&](auto kern, int m) {
        for (int w = 0; w < 2; ++w) {
            cudaEventRecord(a);
            kern<<<sms, 1024>>>(0x1234567ull, pt, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double n = (double)sms * 1024 * pt;
        printf("%-26s %.3g samples/s  %.2f ns per 6784-neuron tile-step per SM\n", names[m],
               n / (ms * 1e-3), ms * 1e6 / pt / 1024 * 6784 / 1000.0);
    };
    run(k<0>, 0); run(k<1>, 1); run(k<2>, 2); run(k<3>, 3); run(k<4>, 4); run(k<5>, 5);
    return 0;
}

// Large-sample noise parity check (test infrastructure, tests/test_noise_gpu.py):
// float xi = (float)stream_normal(mix_key(mix_key(seed, 1), gid), t) for
// gid in [0, G) and t in [t0, t0 + T), once with the device code the step
// kernel uses (paper_2308_01241_b200/csrc/vxb_device.cuh) and once on the
// host with glibc log/cos exactly as the reference evaluates it
// (rng.hpp:58-67, engine.cpp:551-553; compiled -ffp-contract=off).
// Prints one JSON line: samples, float mismatches and the first (gid, t) of
// them.  Argument 4 = 1 checks the fast path alone (no near-boundary
// correctly rounded recomputation).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false \
//        -Xcompiler -fopenmp,-ffp-contract=off -I paper_2308_01241_b200/csrc \
//        tests/native/noise_fliprate.cu -o noise_fliprate
//   ./noise_fliprate G T t0 [fast_only]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include <cuda_runtime.h>

#include "vxb_device.cuh"

using namespace vxb;

__global__ void xi_kernel(uint64_t root, uint64_t g0, uint32_t G, uint32_t T, uint64_t t0,
                          float* out, int fast_only) {
    const uint64_t n = (uint64_t)G * T;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t gid = g0 + i / T, t = t0 + i % T;
        out[i] = fast_only ? __double2float_rn(stream_normal(mix_key(root, gid), t))
                           : stream_xi(mix_key(root, gid), t);
    }
}

static double host_normal(uint64_t base, uint64_t k) {  // rng.hpp:63-67
    const double u1 = 1.0 - (double)(stream_word(base, 2 * k) >> 11) * 0x1.0p-53;
    const double u2 = (double)(stream_word(base, 2 * k + 1) >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

int main(int argc, char** argv) {
    const uint32_t G = argc > 1 ? (uint32_t)std::strtoul(argv[1], nullptr, 10) : 1000000;
    const uint32_t T = argc > 2 ? (uint32_t)std::strtoul(argv[2], nullptr, 10) : 1000;
    const uint64_t t0 = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 0;
    const uint64_t seed = 2;
    const uint64_t root = mix_key(seed, 1);  // rngstream::ou_noise
    const uint32_t gchunk = std::max<uint32_t>(1, (uint32_t)(200000000ull / T));
    const int fast_only = argc > 4 ? std::atoi(argv[4]) : 0;
    float* d = nullptr;
    if (cudaMalloc(&d, 4ull * gchunk * T) != cudaSuccess) return 2;
    std::vector<float> h((size_t)gchunk * T);
    unsigned long long fl = 0, total = 0;
    std::vector<std::pair<uint64_t, uint64_t>> bad;
    for (uint32_t g0 = 0; g0 < G; g0 += gchunk) {
        const uint32_t gn = std::min(gchunk, G - g0);
        xi_kernel<<<148 * 16, 256>>>(root, g0, gn, T, t0, d, fast_only);
        if (cudaDeviceSynchronize() != cudaSuccess) return 3;
        cudaMemcpy(h.data(), d, 4ull * gn * T, cudaMemcpyDeviceToHost);
#pragma omp parallel for reduction(+ : fl) schedule(static)
        for (long long i = 0; i < (long long)gn * T; ++i) {
            const uint64_t gid = g0 + (uint64_t)i / T, t = t0 + (uint64_t)i % T;
            const float x = (float)host_normal(mix_key(root, gid), t);
            if (x != h[i]) {
                ++fl;
#pragma omp critical
                if (bad.size() < 64) bad.emplace_back(gid, t);
            }
        }
        total += (unsigned long long)gn * T;
    }
    std::printf("{\"samples\": %llu, \"float_mismatch\": %llu, \"fast_only\": %d, \"mismatches\": [",
                total, fl, fast_only);
    for (size_t i = 0; i < bad.size(); ++i)
        std::printf("%s[%llu, %llu]", i ? ", " : "", (unsigned long long)bad[i].first,
                    (unsigned long long)bad[i].second);
    std::printf("]}\n");
    cudaFree(d);
    return 0;
}

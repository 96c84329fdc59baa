// Test infrastructure (tests/test_noise_gpu.py): the device double-double
// stream_normal_cr (correctly rounded log and cos, vxb_device.cuh) against
// glibc's stream_normal (rng.hpp:63-67) on the host, double for double, and
// the fast CUDA path beside it.  Prints one JSON line.
//   ./normal_cr_check N
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#include "vxb_device.cuh"

using namespace vxb;

__global__ void both_kernel(uint64_t root, uint64_t n, double* cr, double* fast) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = mix_key(root, i);
        cr[i] = stream_normal_cr(base, i * 7);
        fast[i] = stream_normal(base, i * 7);
    }
}

static double host_normal(uint64_t base, uint64_t k) {
    const double u1 = 1.0 - (double)(stream_word(base, 2 * k) >> 11) * 0x1.0p-53;
    const double u2 = (double)(stream_word(base, 2 * k + 1) >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
    const uint64_t root = mix_key(6, 3);
    double *dc = nullptr, *df = nullptr;
    if (cudaMalloc(&dc, 8 * n) != cudaSuccess || cudaMalloc(&df, 8 * n) != cudaSuccess) return 2;
    both_kernel<<<148 * 8, 256>>>(root, n, dc, df);
    if (cudaDeviceSynchronize() != cudaSuccess) return 3;
    std::vector<double> c(n), f(n);
    cudaMemcpy(c.data(), dc, 8 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(f.data(), df, 8 * n, cudaMemcpyDeviceToHost);
    unsigned long long mc = 0, mf = 0;
#pragma omp parallel for reduction(+ : mc, mf)
    for (long long i = 0; i < (long long)n; ++i) {
        const double h = host_normal(mix_key(root, (uint64_t)i), (uint64_t)i * 7);
        mc += c[i] != h;
        mf += f[i] != h;
    }
    std::printf("{\"samples\": %llu, \"cr_double_mismatch\": %llu, \"fast_double_mismatch\": %llu}\n",
                (unsigned long long)n, mc, mf);
    return 0;
}

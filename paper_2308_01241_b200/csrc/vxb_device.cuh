// vxb_device.cuh — device primitives of the simulation step.
//
// Counter-based noise (rng.hpp:32-67) and the exact-arithmetic helpers the
// fused neuron kernel uses so that every float/double operation rounds
// exactly like the reference build (-ffp-contract=off, CMakeLists.txt:11-14):
// every multiply and add below is an explicit round-to-nearest intrinsic, so
// no FMA contraction can happen regardless of nvcc flags.
#pragma once

#include <cstdint>

namespace vxb {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

// rng.hpp:32-37
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += kGolden;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// rng.hpp:40-42
__host__ __device__ __forceinline__ uint64_t mix_key(uint64_t a, uint64_t b) {
    return splitmix64(a ^ (b + kGolden + (a << 6) + (a >> 2)));
}

// rng.hpp:53-55
__host__ __device__ __forceinline__ uint64_t stream_word(uint64_t base, uint64_t k) {
    return splitmix64(base + k * kGolden);
}

#ifdef __CUDACC__

// rng.hpp:58-60: (word >> 11) * 2^-53, exact in double.
__device__ __forceinline__ double stream_u01(uint64_t base, uint64_t k) {
    return __dmul_rn(__ull2double_rn(stream_word(base, k) >> 11), 0x1.0p-53);
}

// rng.hpp:63-67: Box-Muller over words 2k, 2k+1.
//   u1 = 1 - u01(2k) (exact), u2 = u01(2k+1)
//   z  = sqrt(-2 log u1) * cos(2 pi u2)
// sqrt, the products and 1-u are IEEE round-to-nearest and therefore
// identical to the host; log and cos are the only non-IEEE operations
// ("noise parity").
__device__ __forceinline__ double stream_normal(uint64_t base, uint64_t k) {
    const double u1 = __dsub_rn(1.0, stream_u01(base, 2 * k));
    const double u2 = stream_u01(base, 2 * k + 1);
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    const double c = cos(__dmul_rn(6.283185307179586476925286766559, u2));
    return __dmul_rn(r, c);
}

// model.hpp:25-28: (float)((double)q * 2^-16) — one rounding to float.
__device__ __forceinline__ float dequantize(int64_t q) {
    return __double2float_rn(__dmul_rn(__ll2double_rn(q), 1.0 / 65536.0));
}

__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

#endif  // __CUDACC__

}  // namespace vxb

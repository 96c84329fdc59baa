// vxb_hemo.cuh — BOLD-proxy readout on the device.
//
// The assimilation caller turns every window's rate series into a BOLD
// sample per voxel (EnsembleMember::run_window -> window_bold,
// assim.cpp:51-71, 91-107): per step, the voxel's spike count (sum over its
// units, RateSeries::voxel_counts, stats.cpp:193-201) becomes a drive
// z = count / (voxel neurons * dt_s) / baseline_hz, and one forward-Euler step
// of the Balloon-Windkessel model (step_hemodynamics, hemo.cpp:19-41)
// advances the voxel's state; BOLD (bold_signal, hemo.cpp:43-47) is sampled
// every `sample_every` steps (bold_from_drive, hemo.cpp:49-62).  Here the
// per-unit counts never leave the device: after every chunk of the step
// kernel the voxel counts are summed from its rate rows and one thread per
// voxel runs the model over them, carrying the state between chunks and
// advance() calls.  On several GPUs each rank sums its own units, the ranks
// add their counts (one small all-gather per advance) and feed the totals
// back (vxb_hemo_feed_counts).
//
// The arithmetic is the reference's, operation for operation in IEEE double
// (no FMA contraction: the library is built with --fmad=false); pow() is
// CUDA's, within 1 ulp of glibc's, so states agree to ~1e-15 relative per
// step and BOLD to ~1e-12 over thousands of steps (tests/test_hemo_gpu.py).
#pragma once

#include <cstdint>

namespace vxb {

struct HemoParamsDev {  // HemoParams (hemo.hpp:10-23)
    double kappa, gamma, tau, alpha, e0, v0;
};
struct HemoStateDev {  // HemoState (hemo.hpp:25-30)
    double s, f, v, q;
};

// std::max(x, 1e-9) (NaN propagates as in the reference)
__device__ __forceinline__ double hemo_floor(double x) { return x < 1e-9 ? 1e-9 : x; }

// step_hemodynamics (hemo.cpp:19-41); false when the state is no longer finite
__device__ __forceinline__ bool hemo_step(HemoStateDev& h, double z, double dt_s,
                                          const HemoParamsDev& p) {
    const double f = hemo_floor(h.f);
    const double v = hemo_floor(h.v);
    const double extraction = 1.0 - pow(1.0 - p.e0, 1.0 / f);
    const double v_outflow = pow(v, 1.0 / p.alpha);
    const double ds = z - p.kappa * h.s - p.gamma * (f - 1.0);
    const double df = h.s;
    const double dv = (f - v_outflow) / p.tau;
    const double dq = (f * extraction / p.e0 - v_outflow * h.q / v) / p.tau;
    h.s += dt_s * ds;
    h.f += dt_s * df;
    h.v += dt_s * dv;
    h.q += dt_s * dq;
    return isfinite(h.s) && isfinite(h.f) && isfinite(h.v) && isfinite(h.q);
}

// bold_signal (hemo.cpp:43-47) with k1 = 7 E0, k2 = 2, k3 = 2 E0 - 0.2 (hemo.hpp:19-21)
__device__ __forceinline__ double hemo_bold(const HemoStateDev& h, const HemoParamsDev& p) {
    const double v = hemo_floor(h.v);
    return p.v0 * ((7.0 * p.e0) * (1.0 - h.q) + 2.0 * (1.0 - h.q / v) +
                   (2.0 * p.e0 - 0.2) * (1.0 - v));
}

// RateSeries::voxel_counts (stats.cpp:193-201) on the device for the rate
// rows of one chunk ([unit][steps]): counts[(t_base + t) * n_vox + v].  On
// several GPUs these are the rank's partial sums (its units only).
__global__ void voxel_counts_kernel(const uint32_t* __restrict__ rates, uint32_t steps,
                                    const uint32_t* __restrict__ vox_off,
                                    const uint32_t* __restrict__ vox_units, uint32_t n_vox,
                                    uint32_t t_base, uint32_t* __restrict__ counts) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < steps * n_vox;
         x += gridDim.x * blockDim.x) {
        const uint32_t t = x / n_vox, v = x - t * n_vox;
        uint32_t c = 0;
        for (uint32_t k = vox_off[v]; k < vox_off[v + 1]; ++k)
            c += rates[(size_t)vox_units[k] * steps + t];
        counts[(size_t)(t_base + t) * n_vox + v] = c;
    }
}

// window_bold's per-voxel loop (assim.cpp:58-66), one thread per voxel, over
// count rows [t_base, t_base + steps) of counts[step][voxel]: drive ->
// Euler step; BOLD at every (t + 1) % sample_every == 0 into
// out[sample][voxel].  A diverged voxel records the first failing
// (step << 32 | voxel) in *err and stops.
__global__ void hemo_counts_kernel(const uint32_t* __restrict__ counts, uint32_t t_base,
                                   uint32_t steps, const double* __restrict__ vox_n,
                                   uint32_t n_vox, HemoParamsDev p, double dt_s,
                                   double baseline_hz, uint32_t sample_every,
                                   HemoStateDev* __restrict__ state, double* __restrict__ out,
                                   unsigned long long* __restrict__ err) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_vox) return;
    HemoStateDev h = state[v];
    for (uint32_t t = t_base; t < t_base + steps; ++t) {
        const uint32_t c = counts[(size_t)t * n_vox + v];
        const double hz = vox_n[v] > 0 ? c / (vox_n[v] * dt_s) : 0.0;
        if (!hemo_step(h, hz / baseline_hz, dt_s, p)) {
            atomicMin(err, ((unsigned long long)t << 32) | v);
            break;
        }
        if ((t + 1) % sample_every == 0) out[(size_t)((t + 1) / sample_every - 1) * n_vox + v] = hemo_bold(h, p);
    }
    state[v] = h;
}

// bold_from_drive (hemo.cpp:49-62) over a given drive series, one thread
// per series (diagnostics: the reference's hemodynamics tests run on it).
__global__ void bold_drive_kernel(const double* __restrict__ z, uint32_t steps, uint32_t n_series,
                                  HemoParamsDev p, double dt_s, uint32_t sample_every,
                                  HemoStateDev* __restrict__ state, double* __restrict__ out,
                                  unsigned long long* __restrict__ err) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_series) return;
    HemoStateDev h = state[i];
    for (uint32_t t = 0; t < steps; ++t) {
        if (!hemo_step(h, z[(size_t)i * steps + t], dt_s, p)) {
            atomicMin(err, ((unsigned long long)t << 32) | i);
            break;
        }
        if ((t + 1) % sample_every == 0)
            out[(size_t)i * (steps / sample_every) + (t + 1) / sample_every - 1] = hemo_bold(h, p);
    }
    state[i] = h;
}

}  // namespace vxb

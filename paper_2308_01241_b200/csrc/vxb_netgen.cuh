// vxb_netgen.cuh — on-device synapse sampling (sample_synapses,
// netgen.cpp:51-192) writing straight into the delivery tables.
//
// Every draw is keyed by (seed, gid, slot) with the reference's stream tags
// (rng.hpp:17-28), so the sampled wiring does not depend on how targets are
// spread over warps, devices or passes: the count pass and the scatter pass
// re-draw identical sources.
#pragma once

#include <cstdint>

#include "vxb_device.cuh"

namespace vxb {

struct GenUnit {
    uint64_t gid_base;
    uint32_t neurons;
    uint32_t voxel;
    uint32_t worker;
    uint32_t local_base;     // on its worker (emit_tables, netgen.cpp:207-214)
    uint32_t exc;
    uint32_t dual;
    double split_ratio;
    double w_mean[4];
    double w_spread[4];
};

struct GenVoxel {
    uint32_t k_in;
    uint32_t m;              // inter picks ceil(rho K - 1e-9) (netgen.cpp:44-47)
    uint32_t unit_begin, unit_end;
    uint32_t e0, e1;         // in-edges [e0, e1)
    uint32_t pc_off;         // pop cdf rows: pc[pc_off + tp * pops + sp]
    uint32_t pt_off;         // pop cdf totals: pc[pt_off + tp]
    double in_total;
};

struct GenDev {
    uint64_t kv_root, kn_root, kp_root, kw_root;  // mix_key(seed, tag) for tags 3,4,5,6
    uint32_t n_units;
    const GenUnit* units;
    const GenVoxel* voxels;
    const double* e_cdf;
    const uint32_t* e_src;
    const uint64_t* e_nexc;
    const double* pc;
    const uint32_t* wbase;   // source index base per worker (global over all workers)
    const uint32_t* t_unit;  // target units of this shard, sorted by t_base
    const uint32_t* t_base;  // first target index of each target unit
    uint32_t n_t;
    unsigned int* err;       // 1 = self-redraw exhausted (netgen.cpp:151-154)
    unsigned int* wide;      // 1 = a row's Q16 sums need the int64 pending layout
};

// Categorical::pick (netgen.cpp:36-41): upper_bound over the cumulative weights.
__device__ __forceinline__ uint32_t cat_pick(const double* cdf, uint32_t n, double total,
                                             double u01) {
    const double x = __dmul_rn(u01, total);
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (x < cdf[mid])
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo < n ? lo : n - 1;
}

// NetworkLayout::unit_of_gid (layout.cpp:119-128)
__device__ __forceinline__ uint32_t gen_unit_of_gid(const GenDev& G, uint64_t gid) {
    uint32_t lo = 0, hi = G.n_units;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (gid < G.units[mid].gid_base)
            hi = mid;
        else
            lo = mid + 1;
    }
    uint32_t i = lo - 1;
    while (G.units[i].neurons == 0) --i;
    return i;
}

// quantize_weight (model.hpp:21-24)
__device__ __forceinline__ int32_t quantize(double w) {
    if (w < 0) w = 0;
    return (int32_t)llround(__dmul_rn(w, 65536.0));
}

// quantize(mean + spread * stream_normal(kw, idx)) (netgen.cpp:118-183): the
// fast normal unless w * 2^16 lies within 256 ulps of an llround half-way
// point, where CUDA's last-ulp log/cos could flip the integer; then the
// correctly rounded normal (vxb_device.cuh) decides, as glibc does.
__device__ __forceinline__ int32_t weight_q(double mean, double spread, uint64_t kw,
                                            uint64_t idx) {
    const double w = __dadd_rn(mean, __dmul_rn(spread, stream_normal(kw, idx)));
    const double x = __dmul_rn(w < 0 ? 0.0 : w, 65536.0);
    const double fr = __dsub_rn(x, floor(x));  // exact
    if (fabs(__dsub_rn(fr, 0.5)) > __dmul_rn(0x1p-44, x)) return (int32_t)llround(x);
    return quantize(__dadd_rn(mean, __dmul_rn(spread, stream_normal_cr(kw, idx))));
}

struct Drawn {
    uint32_t src_unit;
    uint64_t src_gid;
    uint32_t cls;
    int32_t wf, ws;
};

// One in-synapse slot k of target gid (netgen.cpp:126-183).
template <bool WEIGHTS>
__device__ __forceinline__ bool draw_synapse(const GenDev& G, const GenVoxel& V, uint32_t tgt_unit,
                                             uint64_t gid, uint64_t kv, uint64_t kn,
                                             uint64_t kp, uint64_t kw, uint32_t k, Drawn& d) {
    if (k < V.m) {
        const uint32_t pick = cat_pick(G.e_cdf + V.e0, V.e1 - V.e0, V.in_total, stream_u01(kv, k));
        const uint32_t sv = G.e_src[V.e0 + pick];
        const uint64_t n_exc = G.e_nexc[V.e0 + pick];
        uint64_t idx = stream_word(kn, (uint64_t)k * 64) % n_exc;
        // NetworkLayout::excitatory_gid (layout.cpp:137-144)
        const GenVoxel& S = G.voxels[sv];
        uint32_t u = S.unit_begin;
        for (; u < S.unit_end; ++u) {
            const GenUnit& U = G.units[u];
            if (!U.exc) continue;
            if (idx < U.neurons) break;
            idx -= U.neurons;
        }
        d.src_unit = u;
        d.src_gid = G.units[u].gid_base + idx;
    } else {
        const uint32_t pops = V.unit_end - V.unit_begin;
        const uint32_t tp = tgt_unit - V.unit_begin;
        const double* cdf = G.pc + V.pc_off + tp * pops;
        const double total = G.pc[V.pt_off + tp];
        uint32_t attempt = 0;
        for (;;) {
            const uint64_t word = (uint64_t)k * 64 + attempt;
            const uint32_t sp = cat_pick(cdf, pops, total, stream_u01(kp, word));
            const uint32_t su = V.unit_begin + sp;
            const uint64_t idx = stream_word(kn, word) % G.units[su].neurons;
            d.src_unit = su;
            d.src_gid = G.units[su].gid_base + idx;
            if (d.src_gid != gid) break;
            if (++attempt >= 63) {
                atomicExch(G.err, 1u);
                return false;
            }
        }
    }
    const GenUnit& SU = G.units[d.src_unit];
    d.cls = SU.exc ? 0u : 1u;
    d.wf = d.ws = 0;
    if (WEIGHTS) {
        const int rf = SU.exc ? 0 : 2, rs = SU.exc ? 1 : 3;
        bool want_fast = true, want_slow = true;
        if (!SU.dual) {
            want_fast = stream_u01(kw, (uint64_t)k * 6 + 4) < SU.split_ratio;
            want_slow = !want_fast;
        }
        if (want_fast)
            d.wf = weight_q(SU.w_mean[rf], SU.w_spread[rf], kw, (uint64_t)k * 3);
        if (want_slow)
            d.ws = weight_q(SU.w_mean[rs], SU.w_spread[rs], kw, (uint64_t)k * 3 + 1);
    }
    return true;
}

__device__ __forceinline__ uint32_t shard_index(const GenDev& G, uint32_t unit, uint64_t gid) {
    const GenUnit& U = G.units[unit];
    return G.wbase[U.worker] + U.local_base + (uint32_t)(gid - U.gid_base);
}

// mode 0: count per source; mode 1: scatter into the out-CSR; mode 2: write
// the in-rows of worker `only_worker` (SynEntry layout) for table export and
// the destination-worker masks of every source.
template <int MODE>
__global__ void gen_kernel(GenDev G, uint64_t gid_lo, uint64_t gid_hi,
                           unsigned long long* __restrict__ cnt,
                           uint32_t* __restrict__ tgt, uint64_t* __restrict__ w,
                           unsigned long long* __restrict__ have_mask,
                           uint32_t* __restrict__ inner, uint32_t only_worker,
                           const uint64_t* __restrict__ row_base, uint4* __restrict__ rows) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t it = gid_lo + warp; it < gid_hi; it += nwarps) {
        // modes 0/1 walk this shard's targets (index = shard-local target),
        // mode 2 walks every gid of the layout
        uint32_t u;
        uint64_t gid;
        uint32_t t_idx;
        if (MODE == 2) {
            gid = it;
            u = gen_unit_of_gid(G, gid);
            t_idx = 0;
        } else {
            uint32_t lo = 0, hi = G.n_t;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (G.t_base[mid] <= (uint32_t)it) lo = mid; else hi = mid;
            }
            u = G.t_unit[lo];
            gid = G.units[u].gid_base + (it - G.t_base[lo]);
            t_idx = (uint32_t)it;
        }
        const GenUnit& U = G.units[u];
        const GenVoxel V = G.voxels[U.voxel];
        const uint64_t kv = mix_key(G.kv_root, gid), kn = mix_key(G.kn_root, gid),
                       kp = mix_key(G.kp_root, gid), kw = mix_key(G.kw_root, gid);
        const bool mine = MODE == 2 && U.worker == only_worker;
        long long sf = 0, ss = 0;
        for (uint32_t k = lane; k < V.k_in; k += 32) {
            Drawn d;
            bool ok;
            if (MODE == 1 || mine)
                ok = draw_synapse<true>(G, V, u, gid, kv, kn, kp, kw, k, d);
            else
                ok = draw_synapse<false>(G, V, u, gid, kv, kn, kp, kw, k, d);
            if (!ok) continue;
            const uint32_t s_idx = shard_index(G, d.src_unit, d.src_gid);
            if (MODE == 0) {
                atomicAdd(cnt + s_idx, 1ull);
            } else if (MODE == 1) {
                const unsigned long long pos = atomicAdd(cnt + s_idx, 1ull);
                tgt[pos] = t_idx | (d.cls << 31);
                w[pos] = (uint64_t)(uint32_t)d.wf | ((uint64_t)(uint32_t)d.ws << 32);
                atomicOr(have_mask + s_idx, 1ull << U.worker);
                if (G.units[d.src_unit].worker == U.worker) atomicAdd(inner + s_idx, 1u);
                sf += d.wf;
                ss += d.ws;
            } else {
                atomicOr(have_mask + s_idx, 1ull << U.worker);
                if (mine) {
                    const GenUnit& S = G.units[d.src_unit];
                    const uint32_t local = U.local_base + (uint32_t)(gid - U.gid_base);
                    const uint64_t at = row_base[local] + k;
                    // SynEntry: src_local | src_worker,cls,pad | wq_fast | wq_slow
                    rows[at] = make_uint4(S.local_base + (uint32_t)(d.src_gid - S.gid_base),
                                          (uint32_t)S.worker | (d.cls << 16), (uint32_t)d.wf,
                                          (uint32_t)d.ws);
                }
            }
        }
        if (MODE == 1) {
            for (int o = 16; o; o >>= 1) {
                sf += __shfl_xor_sync(0xffffffffu, sf, o);
                ss += __shfl_xor_sync(0xffffffffu, ss, o);
            }
            if (lane == 0 && (sf >= (1ll << 32) || ss >= (1ll << 32))) atomicExch(G.wide, 1u);
        }
    }
}

}  // namespace vxb

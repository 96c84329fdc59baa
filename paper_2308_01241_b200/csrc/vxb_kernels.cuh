// vxb_kernels.cuh — sm_100a kernels of the voxel-network simulation step.
//
// One persistent cooperative kernel runs a whole chunk of steps.  Each grid
// phase ph does, for absolute steps tA = t0 + ph and tE = tA - 1:
//
//   F: for every neuron (static partition, thread-owned state)
//        E(tE)  gating with the pending buffer of S(tE-1), current, OU noise
//               (engine.cpp:539-559)
//        A(tA)  membrane / threshold / refractory / injection / forced spike
//               (engine.cpp:363-398), spiking neurons appended to the log
//   D: deliver S(tE) — the spikes A(tE) produced in the previous phase — into
//      the other pending buffer with integer atomics (engine.cpp:444-464)
//   grid barrier
//
// F and D of one phase touch disjoint pending buffers, so the delivery of a
// step overlaps the neuron update of the next: the one-step synaptic delay
// of the reference (test_engine.cpp:203-246) is the slack that makes the
// fusion legal.  Phase 0 of a chunk is A only, the last phase is E only, so
// the state between chunks (and between advance() calls) is exactly the
// reference's post-phase-E state.
#pragma once

#include <cstddef>
#include <cstdint>

#include "vxb_device.cuh"

namespace vxb {

// Per-segment parameters: a segment is a run of shard-local neurons with
// identical NeuronRecord parameters, unit, voxel, worker and consecutive gids.
// Reference populations give one segment per unit.
struct SegParams {
    int64_t gid_off;      // gid = local + gid_off
    uint32_t start;       // first shard-local index
    uint32_t unit;
    uint32_t voxel;
    uint32_t worker;
    uint32_t tref;        // refractory_steps
    float dt_over_c;      // dtf / C (engine.cpp:242)
    float g_leak, e_leak, v_th, v_reset;
    float decay[4];       // 1 - dtf / tau_u   (gating_kernel, model.hpp:69-71)
    float omega[4];
    float e_rev[4];
    float ou_mu;
    float ou_a;           // dtf / tau_ou
    float ou_b;           // sigma * sqrtf(2 dtf / tau_ou)  (ou_kernel, model.hpp:88-90)
    uint32_t sigma_pos;   // sigma > 0
    uint32_t pad[4];
};
static_assert(sizeof(SegParams) == 128, "SegParams layout");

// Device form of the segments: the float parameters are shared by every
// segment of a population (ParamSet, a handful per network) and a segment
// only keeps its unit, voxel, gid offset and parameter-set index (SegInfo),
// so networks with ~1000 units still keep the whole table in shared memory.
struct ParamSet {
    uint32_t tref;
    float dt_over_c, g_leak, e_leak, v_th, v_reset;
    float decay[4];
    float omega[4];
    float e_rev[4];
    float ou_mu, ou_a, ou_b;
    uint32_t sigma_pos;
    uint32_t pad[2];
};
static_assert(sizeof(ParamSet) == 96, "ParamSet layout");
struct SegInfo {
    int64_t gid_off;
    uint32_t unit, voxel, pset, pad;
};
static_assert(sizeof(SegInfo) == 24, "SegInfo layout");

// Refractory neurons hold V = V_reset (engine.cpp:364-367); the counter is
// kept in the V word as a negative NaN payload so the state is one word.
__host__ __device__ __forceinline__ bool is_refrac(uint32_t bits) {
    return (bits & 0xff800000u) == 0xff800000u && (bits & 0x007fffffu) != 0u;
}
__host__ __device__ __forceinline__ uint32_t refrac_bits(uint32_t r) { return 0xff800000u | r; }

struct Control {
    unsigned int bar_count;
    unsigned int bar_gen;
    unsigned int work;         // dynamic delivery work counter of the phase
    unsigned int spk_cursor;   // append cursor of the spike log
    unsigned long long err;    // min (step << 32 | local) of a divergence, ~0 = none
    unsigned long long flops_inner, flops_outer;
    unsigned int routed;       // CTAs that routed this phase's spikes (multi-GPU)
    // stop decision of the phase, taken once by the last CTA through the
    // barrier (hook) so every CTA leaves the loop at the same phase
    unsigned int stop;
    unsigned int rdone;        // tile_mp_kernel: CTAs done with the peers' batches (monotonic)
    unsigned int pad[3];
};

// Device-side state of the per-step spike-id exchange between ranks (one
// process per GPU).  Receive slots live in this rank's IPC-exported region,
// send slots are this rank's slots inside the peers' regions (NVLink P2P).
constexpr int kMaxShards = 64;  // dst masks are 64-bit (partition.hpp:35)
constexpr uint32_t kSlots = 4;  // exchange batches in flight per (sender, receiver)
struct Exchange {
    uint32_t rank, world;
    uint32_t cap_self;                    // ids per parity in my slots (= my neurons)
    uint32_t timeout;                     // peer + 1 whose batch never arrived, 0 = none
    uint32_t timeout_step;
    uint32_t peer_abort;                  // peer + 1 that aborted the run (engine.cpp:117-142)
    uint32_t pad0[2];
    unsigned long long timeout_ns;
    uint32_t src_base[kMaxShards + 1];    // global source index base per shard
    uint32_t cap[kMaxShards];             // neurons of shard h
    // Batches are buffered by step (slot = step % kSlots).  A batch is
    // published as soon as every CTA has routed its spikes (before the
    // phase's delivery ends), so a sender can be up to two phases ahead of
    // a receiver still reading the batch of step t - 1: four slots.
    uint32_t send_cnt[4][kMaxShards];     // ids queued per (slot, destination)
    uint32_t* rx_ids[kMaxShards];         // [kSlots * cap[h]] from source shard h
    uint32_t* rx_meta[kMaxShards];        // counts[kSlots], flag (= step + 1), abort word
    uint32_t* tx_ids[kMaxShards];         // my slot in peer d
    uint32_t* tx_meta[kMaxShards];
};

struct StepArgs {
    // sizes
    uint32_t n;             // shard neurons
    uint32_t nseg;
    uint32_t npset;
    uint32_t n_units;
    uint32_t steps;         // A steps in this chunk (phases = steps + 1)
    uint32_t t0;            // absolute step of the chunk's first A
    uint32_t rel0;          // index of t0 within the current advance()
    uint32_t adv_steps;     // steps of the whole advance() (trace stride)
    uint32_t spk_cap;       // spike log capacity
    uint32_t ring;          // spike log in ring mode (raster not recorded)
    uint32_t use_smem_seg;
    float dtf;
    uint64_t ou_root;       // mix_key(seed, rngstream::ou_noise)
    // parameters
    const ParamSet* pset;
    const SegInfo* sinfo;
    const uint32_t* seg_start;
    // state
    uint32_t* v;            // float bits or refractory code
    float4* j;
    float* i_ou;
    float* i_syn;
    const float4* g;
    void* pend0;            // pending buffers, parity of the step they hold
    void* pend1;
    // out-CSR
    const uint64_t* off;    // n + 1
    const uint32_t* inner;  // per source: entries whose target is on its worker
    const uint32_t* tgt;    // target | cls << 31
    const uint64_t* w;      // (u32)wq_fast | (u64)(u32)wq_slow << 32
    // spike log
    uint32_t* spk;
    uint32_t* seg_end;      // per phase: log end after that phase's A
    // readout
    uint32_t* rates;        // [unit][chunk step]
    uint32_t n_probes;
    const uint32_t* probe_local;  // sorted
    const uint32_t* probe_slot;
    float* probe_v;         // [slot][adv_steps]
    float* probe_i;
    const uint32_t* forced_off;   // [steps + 1]
    const uint32_t* forced_local; // sorted per step
    uint32_t has_forced;
    const uint32_t* inj_epoch;    // [steps], 0 = no injection active
    const float* inj_table;       // [(epoch-1) * n_voxels + voxel]
    uint32_t n_voxels;
    uint32_t has_inj;
    unsigned long long* phase_ns; // [steps + 2] globaltimer at phase ends
    Control* ctl;
    Exchange* ex;
    uint32_t world;
    unsigned long long* phase_wait;  // per phase: max over CTAs of the exchange wait (ns)
    unsigned long long* arrive;      // [phase][peer]: first globaltimer a CTA saw the peer's flag
    // L2-blocked delivery: targets split into n_blocks ranges delivered in
    // order; blk_off[s * (n_blocks + 1) + b] = row offset of block b
    uint32_t n_blocks;
    const uint32_t* blk_off;
    // dynamic delivery: per (phase parity, block, source list) chunk
    // counters; producers take chunks of spikes block-major so the grid
    // works on one L2 block at a time and balances itself (dyn != 0)
    uint32_t* work_ctr;
    uint32_t dyn;
    uint32_t stage_e;   // delivery ring: synapse entries per stage (SmemLayout)
    uint32_t ch_max;    // dynamic delivery of local spikes: most spikes per chunk (1 for
                        // long rows: the phase's last chunk ends sooner, config 2 79.4 ->
                        // 77.9 us/step); peers' batches (short rows here) take up to 32
    uint32_t f_policy;  // neuron-state stream in L2: 0 evict_normal, 1 evict_first, 2 evict_last
    // phase profile (VXB_PHASE_PROFILE): per (phase, CTA) globaltimer of the
    // end of this CTA's delivery and of its update, or null
    unsigned long long* prof;
    uint32_t early_publish;  // publish S(tA) once routed (else after the phase barrier)
    const unsigned long long* dst_mask;  // per local neuron: shards holding its targets
    // ---- SM-tile path (tile_kernel, vxb_tile.cuh) ----
    uint32_t tile_n;            // neurons per CTA tile (multiple of 32)
    uint32_t n_cons;            // consumer warps
    uint32_t n_noisew;          // tile_kernel: warps that start on the OU noise
    uint32_t q_total;           // queue items per parity
    const unsigned long long* tl_off;  // per global source: first tile segment (n_src + 1)
    const uint4* tl;            // tile segments {tile, first entry in row, length, 0}
    const uint32_t* q_base;     // per tile: first queue slot (tiles + 1)
    uint32_t* q_cnt;            // [sets][tiles] items queued per (step set, tile): 4 sets
                                // (tile_kernel, step & 3), 2 (tile_mp_kernel, parity)
    uint64_t* q;                // [sets][q_total] first entry | length << 40
    uint32_t src_self;          // global source index of shard-local neuron 0
    const uint64_t* tent;       // 8-byte tile entries (same indexing as tgt / w)
    float* i_ou_b;              // I_ou of odd steps (tile path; i_ou holds even steps)
    uint32_t n_tiles;           // tile_mp_kernel: tiles (T) and passes per CTA (P)
    uint32_t passes;
    uint32_t item_mode;         // 0: one queue item per warp, 1: one per lane
    // tile_kernel (no grid barrier): per phase, CTAs whose bucketing of that
    // phase's spikes is complete; the spike log is phase-strided (entries of
    // phase p at spk[p * n], per-phase counts in seg_end)
    uint32_t* bdone;
    // per CTA (128 B apart): the number of phases whose bucketing is complete,
    // written (red.max) by the CTA that completes a phase's count, polled by
    // one warp of each CTA — no hot line for 148 pollers
    uint32_t* bmail;
    uint32_t* routed;  // tile_kernel (MG): per phase, CTAs whose spikes are routed to the peers
};

__device__ __forceinline__ uint64_t ldg64(const uint64_t* p) {
    return (uint64_t)__ldg(reinterpret_cast<const unsigned long long*>(p));
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sense-counting grid barrier for a cooperative launch.  The last CTA to
// arrive runs `hook` (bookkeeping for the next phase) before releasing.
template <typename Hook, typename Post>
__device__ __forceinline__ void grid_barrier(Control* ctl, Hook hook, Post post) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = ld_acquire(&ctl->bar_gen);
        __threadfence();
        const unsigned int arrived = atomicAdd(&ctl->bar_count, 1u);
        if (arrived == gridDim.x - 1) {
            ctl->bar_count = 0;
            hook();
            __threadfence();
            st_release(&ctl->bar_gen, gen + 1);
            post();  // after the release: off the critical path of the grid
        } else {
            while (ld_acquire(&ctl->bar_gen) == gen) __nanosleep(40);
        }
    }
    __syncthreads();
}

// find_seg starting from a known segment lo (starts[lo] <= i): galloping
// search, O(log distance) — the update loop's neurons only move forward.
__device__ __forceinline__ uint32_t find_seg_from(const uint32_t* starts, uint32_t nseg,
                                                  uint32_t i, uint32_t lo) {
    uint32_t step = 1, hi = lo + 1;
    while (hi < nseg && starts[hi] <= i) {
        lo = hi;
        step <<= 1;
        hi = lo + step;
    }
    if (hi > nseg) hi = nseg;
    while (hi - lo > 1) {  // starts[lo] <= i < starts[hi] (hi == nseg: end)
        const uint32_t mid = (lo + hi) >> 1;
        if (starts[mid] <= i)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Index of the segment holding shard-local neuron i (largest start <= i).
__device__ __forceinline__ uint32_t find_seg(const uint32_t* starts, uint32_t nseg, uint32_t i) {
    uint32_t lo = 0, hi = nseg;  // invariant: starts[lo] <= i < starts[hi]
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (starts[mid] <= i)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// First index in sorted a[0..n) with a[k] >= x.
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

template <bool PACKED>
struct Pend;
template <>
struct Pend<true> {  // (AMPA|NMDA<<32, GABAA|GABAB<<32), carry-free by construction
    using T = ulonglong2;
};
template <>
struct Pend<false> {  // four signed int64 buckets, the reference's layout
    struct T {
        longlong2 lo, hi;
    };
};

constexpr int kMaxSmemSeg = 1024;   // segments kept in shared memory
constexpr int kMaxSmemPset = 32;    // parameter sets kept in shared memory
#ifndef VXB_THREADS
#define VXB_THREADS 256
#endif
#ifndef VXB_MINB
#define VXB_MINB 3
#endif
constexpr int kThreads = VXB_THREADS;
constexpr int kSpkStage = 1024;  // per-CTA spike staging before one log append
#ifndef VXB_DWARPS
#define VXB_DWARPS 3
#endif
static_assert(VXB_DWARPS >= 2, "delivery needs a producer warp and >= 1 consumer warp");
// L2 policies of the delivery: the synapse stream's bulk copies run with
// evict_normal (evict_first measured 2.8 % slower on config 2: 77.25 vs
// 75.1 us/step, equal on config 3); the pending buffers the atomics hit keep
// evict_last (evict_normal: config 2 110 us/step, config 3 3.5 vs 1.14 ms).
#ifndef VXB_POL_STREAM
#define VXB_POL_STREAM 1  // synapse stream: 0 evict_first, 1 evict_normal
#endif
#ifndef VXB_POL_KEEP
#define VXB_POL_KEEP 0    // pending buffers: 0 evict_last, 1 evict_normal
#endif
#ifndef VXB_PREFETCH
// L2 prefetch of the update state two chunks ahead: off since the state is
// kept evict_last (config 2 73.8 -> 71.6 us/step, silent 35.1 -> 31.9;
// config 3 1142 -> 1133 us/step)
#define VXB_PREFETCH 0
#endif
#ifndef VXB_DEPTH3
#define VXB_DEPTH3 0  // 1: update state loaded two chunks ahead (three register sets)
#endif
#ifndef VXB_STAGES
#define VXB_STAGES 4
#endif
#ifndef VXB_STAGE_E
#define VXB_STAGE_E 768
#endif
constexpr int kStages = VXB_STAGES;   // delivery pipeline depth (bulk copies in flight)
constexpr int kStageE = VXB_STAGE_E;  // synapse entries per stage (default; see SmemLayout)

// Stage metadata: the producer packs up to kSegPerStage row segments into
// one stage of the delivery ring.
constexpr int kSegPerStage = 16;
struct TStageMeta {
    uint32_t n;                       // entries in the stage
    uint32_t nseg;
    uint32_t end;                     // last stage of the phase
    uint32_t pad;
    uint32_t pre[kSegPerStage + 1];   // prefix of segment lengths
    uint32_t tb[kSegPerStage];        // first entry of segment i in the tgt buffer
    uint32_t wb[kSegPerStage];        // ... in the w buffer
};
constexpr uint32_t kMetaBytes = sizeof(TStageMeta);

// Dynamic shared memory carve-up of step_kernel.
// The stage size (entries) is chosen per launch: 1024 for L2-blocked
// networks (config 3: 1094 vs 1126 us/step), kStageE otherwise (config 2).
struct SmemLayout {
    uint32_t se, tb, wb;  // entries per stage, target / weight bytes per stage
    uint32_t tgt, w, bar, meta, pset, seg, start, spk, total;
    __host__ __device__ SmemLayout(uint32_t nseg_smem, uint32_t npset_smem,
                                   uint32_t stage_e = kStageE) {
        se = stage_e;
        tb = (se + 8) * 4;
        wb = (se + 4) * 8;
        tgt = 0;
        w = tgt + kStages * tb;
        bar = w + kStages * wb;
        meta = bar + 2 * kStages * 8;  // full barriers, then empty barriers
        pset = (meta + kStages * kMetaBytes + 127) & ~127u;
        seg = pset + npset_smem * (uint32_t)sizeof(ParamSet);
        start = seg + nseg_smem * (uint32_t)sizeof(SegInfo);
        spk = (start + (nseg_smem + 1) * 4 + 15) & ~15u;
        total = spk + kSpkStage * 4;
    }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "VXB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra VXB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity) : "memory");
}
// cp.async.bulk (TMA bulk copy) global -> shared, completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes),
        "r"(smem_u32(bar)), "l"(pol) : "memory");
}

// L2 eviction-priority policies (createpolicy): the synapse stream is read
// once per spike and must not evict the pending buffers the atomics hit.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void red_add(unsigned long long* p, uint64_t v, uint64_t pol) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;"
                 ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// Cache-hinted accesses of the neuron-update stream (policy chosen at run
// time: evict_first keeps the streamed state from displacing the pending
// buffers the delivery atomics hit; evict_normal otherwise).
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ldp(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ldp(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float4 ldp(const float4* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ ulonglong2 ldp_cg(const ulonglong2* p, uint64_t pol) {
    ulonglong2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void stp(uint32_t* p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stp(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stp(float4* p, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                 ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void stp_cg(ulonglong2* p, ulonglong2 v, uint64_t pol) {
    asm volatile("st.global.cg.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;"
                 ::"l"(p), "l"(v.x), "l"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}

// Delivery producer (lane 0 of the producer warp): packs row segments into
// the stage ring — long segments split, short ones packed up to
// kSegPerStage to a stage — so every bulk-copy round trip carries a full
// stage whatever the row lengths.  Copies are issued as segments are added
// (expect_tx per segment, one arrive at commit).
// Scratch of the warp-parallel stage packing (producer warp only).
constexpr int kMaxPieces = 2 * kSegPerStage;
struct BatchScratch {
    uint64_t sb0[32];                 // the warp's segments: first entry
    uint32_t slen[32];                //                      length
    uint64_t pb0[kMaxPieces];         // pieces laid out this round
    uint32_t ptake[kMaxPieces], pst[kMaxPieces], ptoff[kMaxPieces], pwoff[kMaxPieces];
    uint32_t np, ncom, more, com[2];
};

struct StageBuilder {
    uint32_t ctr;    // stages committed since launch (stage = ctr % kStages)
    uint32_t open;   // a stage is being filled
    uint32_t ns, toff, woff, total;

    __device__ __forceinline__ void begin(unsigned char* smem, const SmemLayout& L) {
        const uint32_t st = ctr % kStages;
        uint64_t* empty = reinterpret_cast<uint64_t*>(smem + L.bar) + kStages;
        mbar_wait(empty + st, ((ctr / kStages) & 1u) ^ 1u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        open = 1;
        ns = toff = woff = total = 0;
    }
    __device__ __forceinline__ void commit(unsigned char* smem, const SmemLayout& L, uint32_t end) {
        const uint32_t st = ctr % kStages;
        TStageMeta* m = reinterpret_cast<TStageMeta*>(smem + L.meta + st * kMetaBytes);
        m->pre[ns] = total;
        m->n = total;
        m->nseg = ns;
        m->end = end;
        mbar_arrive(reinterpret_cast<uint64_t*>(smem + L.bar) + st);
        ++ctr;
        open = 0;
    }
    __device__ __forceinline__ void add(const StepArgs& a, unsigned char* smem, const SmemLayout& L,
                                        uint64_t b0, uint64_t len, uint64_t pol) {
        while (len) {
            if (!open) begin(smem, L);
            const int room_t = (int)L.se - (int)toff, room_w = (int)L.se - 4 - (int)woff + 4;
            int room = room_t < room_w ? room_t : room_w;
            if (ns == (uint32_t)kSegPerStage || room <= 0) {
                commit(smem, L, 0);
                continue;
            }
            const uint32_t st = ctr % kStages;
            TStageMeta* m = reinterpret_cast<TStageMeta*>(smem + L.meta + st * kMetaBytes);
            const uint64_t take = min(len, (uint64_t)room);
            const uint64_t b1 = b0 + take;
            const uint64_t t0 = b0 & ~3ull, w0 = b0 & ~1ull;
            const uint32_t tn = (uint32_t)(((b1 + 3) & ~3ull) - t0);
            const uint32_t wn = (uint32_t)(((b1 + 1) & ~1ull) - w0);
            m->pre[ns] = total;
            m->tb[ns] = toff + (uint32_t)(b0 - t0);
            m->wb[ns] = woff + (uint32_t)(b0 - w0);
            uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar) + st;
            mbar_expect_tx_only(full, tn * 4 + wn * 8);
            bulk_g2s(smem + L.tgt + st * L.tb + toff * 4, a.tgt + t0, tn * 4, full, pol);
            bulk_g2s(smem + L.w + st * L.wb + woff * 8, a.w + w0, wn * 8, full, pol);
            total += (uint32_t)take;
            toff += tn;
            woff += wn;
            ++ns;
            b0 = b1;
            len -= take;
        }
    }
    // Warp-collective add of one segment per lane (len 0 = none).  Lane 0
    // lays the segments out over stages (metadata only, cheap scalar work),
    // all lanes then issue their pieces' bulk copies in parallel, and lane 0
    // commits the stages the round closed.  A round touches at most two
    // stages, so a deferred commit never holds a ring slot that this round
    // waits for (kStages >= 3).  StageBuilder state is meaningful in lane 0.
    __device__ __forceinline__ void add_batch(const StepArgs& a, unsigned char* smem,
                                              const SmemLayout& L, uint64_t my_b0,
                                              uint32_t my_len, uint64_t pol, BatchScratch& S,
                                              uint32_t lane) {
        if (!__any_sync(0xffffffffu, my_len != 0)) return;
        S.sb0[lane] = my_b0;
        S.slen[lane] = my_len;
        __syncwarp();
        uint32_t seg = 0, used = 0;  // lane 0's cursor over the warp's segments
        for (;;) {
            if (lane == 0) {
                uint32_t np = 0, ncom = 0, touched = open ? 1u : 0u;
                while (seg < 32) {
                    const uint32_t len = S.slen[seg] - used;
                    if (len == 0) {
                        ++seg;
                        used = 0;
                        continue;
                    }
                    if (!open) {
                        if (touched == 2) break;
                        begin(smem, L);
                        ++touched;
                    }
                    const int room_t = (int)L.se - (int)toff, room_w = (int)L.se - (int)woff;
                    const int room = room_t < room_w ? room_t : room_w;
                    const uint32_t st = ctr % kStages;
                    TStageMeta* m = reinterpret_cast<TStageMeta*>(smem + L.meta + st * kMetaBytes);
                    if (ns == (uint32_t)kSegPerStage || room <= 0) {  // close the stage
                        m->pre[ns] = total;
                        m->n = total;
                        m->nseg = ns;
                        m->end = 0;
                        S.com[ncom++] = st;
                        ++ctr;
                        open = 0;
                        continue;
                    }
                    const uint32_t take = min(len, (uint32_t)room);
                    const uint64_t b0 = S.sb0[seg] + used, b1 = b0 + take;
                    const uint64_t t0 = b0 & ~3ull, w0 = b0 & ~1ull;
                    m->pre[ns] = total;
                    m->tb[ns] = toff + (uint32_t)(b0 - t0);
                    m->wb[ns] = woff + (uint32_t)(b0 - w0);
                    S.pb0[np] = b0;
                    S.ptake[np] = take;
                    S.pst[np] = st;
                    S.ptoff[np] = toff;
                    S.pwoff[np] = woff;
                    ++np;
                    total += take;
                    toff += (uint32_t)(((b1 + 3) & ~3ull) - t0);
                    woff += (uint32_t)(((b1 + 1) & ~1ull) - w0);
                    ++ns;
                    used += take;
                }
                S.np = np;
                S.ncom = ncom;
                S.more = seg < 32;
            }
            __syncwarp();
            const uint32_t np = S.np;
            if (lane < np) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (uint32_t q = lane; q < np; q += 32) {
                const uint64_t b0 = S.pb0[q], b1 = b0 + S.ptake[q];
                const uint64_t t0 = b0 & ~3ull, w0 = b0 & ~1ull;
                const uint32_t tn = (uint32_t)(((b1 + 3) & ~3ull) - t0);
                const uint32_t wn = (uint32_t)(((b1 + 1) & ~1ull) - w0);
                const uint32_t st = S.pst[q];
                uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar) + st;
                mbar_expect_tx_only(full, tn * 4 + wn * 8);
                bulk_g2s(smem + L.tgt + st * L.tb + S.ptoff[q] * 4, a.tgt + t0, tn * 4,
                         full, pol);
                bulk_g2s(smem + L.w + st * L.wb + S.pwoff[q] * 8, a.w + w0, wn * 8, full,
                         pol);
            }
            __syncwarp();
            if (lane == 0)
                for (uint32_t k = 0; k < S.ncom; ++k)
                    mbar_arrive(reinterpret_cast<uint64_t*>(smem + L.bar) + S.com[k]);
            const uint32_t more = S.more;
            __syncwarp();
            if (!more) break;
        }
    }
};

// Routing of one warp's spikes to the peers (engine.cpp:416-437 + transport
// send): ids go straight into the peers' receive slots over NVLink P2P
// stores, positions reserved per destination with one atomic per warp and
// destination.  Called by the neuron-update warps when they flush their
// staged spikes; the counts and the step flag are published once per phase
// by exchange_publish.  Returns true if this thread stored anything remote.
__device__ __forceinline__ bool exchange_route(const StepArgs& a, uint32_t s, bool valid,
                                               uint32_t slot) {
    Exchange* ex = a.ex;
    const uint32_t lane = threadIdx.x & 31, world = ex->world, me = ex->rank;
    const unsigned long long m = valid ? (a.dst_mask[s] & ~(1ull << me)) : 0ull;
    bool sent = false;
    if (world <= 8) {  // one reservation round trip for all destinations
        unsigned ball[8];
#pragma unroll
        for (uint32_t d = 0; d < 8; ++d) ball[d] = d < world ? __ballot_sync(0xffffffffu, (m >> d) & 1ull) : 0u;
        unsigned mine = 0, cntl = 0;  // lane d < world: destination d's count
#pragma unroll
        for (uint32_t d = 0; d < 8; ++d)
            if (lane == d) cntl = __popc(ball[d]);
        if (lane < world && cntl) mine = atomicAdd(&ex->send_cnt[slot][lane], cntl);
#pragma unroll
        for (uint32_t d = 0; d < 8; ++d) {
            if (d >= world) break;
            const unsigned base = __shfl_sync(0xffffffffu, mine, d);
            if ((m >> d) & 1ull) {
                ex->tx_ids[d][slot * ex->cap_self + base + __popc(ball[d] & ((1u << lane) - 1u))] = s;
                sent = true;
            }
        }
        return sent;
    }
    for (uint32_t d = 0; d < world; ++d) {
        const bool want = (m >> d) & 1ull;
        const unsigned ball = __ballot_sync(0xffffffffu, want);
        if (!ball) continue;
        const int lead = __ffs(ball) - 1;
        unsigned base = 0;
        if ((int)lane == lead) base = atomicAdd(&ex->send_cnt[slot][d], (unsigned)__popc(ball));
        base = __shfl_sync(0xffffffffu, base, lead);
        if (want) {
            ex->tx_ids[d][slot * ex->cap_self + base + __popc(ball & ((1u << lane) - 1u))] = s;
            sent = true;
        }
    }
    return sent;
}

// Publish the batch of step t to every peer: counts, then the step flag
// with system-scope release.  An empty batch still publishes its flag: it is
// the reference's step barrier (engine.cpp:468-524).  Run by one thread after
// every CTA's routing is complete (the last CTA through the routing count).
__device__ __forceinline__ void exchange_publish(const StepArgs& a, uint32_t t) {
    Exchange* ex = a.ex;
    const uint32_t slot = t % kSlots, world = ex->world, me = ex->rank;
    __threadfence_system();
    for (uint32_t d = 0; d < world; ++d)
        if (d != me) ex->tx_meta[d][slot] = atomicExch(&ex->send_cnt[slot][d], 0u);
    __threadfence_system();
    for (uint32_t d = 0; d < world; ++d)
        if (d != me) st_release_sys(ex->tx_meta[d] + kSlots, t + 1);
}

// Wait for peer h's batch of step tE (receiver side of the step barrier);
// returns its id count.  recv_timeout_ms maps to a device-side timeout.
__device__ __forceinline__ uint32_t exchange_wait(const StepArgs& a, uint32_t h, uint32_t tE,
                                                 uint32_t slot, uint32_t ph) {
    Exchange* ex = a.ex;
    const uint32_t* meta = ex->rx_meta[h];
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(meta + kSlots) < tE + 1) {
        // a peer that failed never publishes again: its abort word ends the
        // wait at once (the reference's shared abort flag, engine.cpp:483-484)
        for (uint32_t q = 0; q < ex->world; ++q)
            if (q != ex->rank && ld_acquire_sys(ex->rx_meta[q] + kSlots + 1) != 0u) {
                atomicCAS(&ex->peer_abort, 0u, q + 1);
                return 0;
            }
        if (ex->timeout_ns && globaltimer() - t0 > ex->timeout_ns) {
            if (atomicCAS(&ex->timeout, 0u, h + 1) == 0u) ex->timeout_step = tE;
            return 0;
        }
        __nanosleep(64);
    }
    if (a.arrive) atomicMin(a.arrive + (size_t)ph * ex->world + h, (unsigned long long)globaltimer());
    return ld_acquire_sys(meta + slot);
}

// Tell every peer this rank stopped (divergence, timeout or a peer's abort):
// their waits for this rank's next batch end with the reference's "simulation
// aborted while waiting on the step barrier" instead of a 30 s timeout.
__device__ __forceinline__ void exchange_abort(const StepArgs& a) {
    Exchange* ex = a.ex;
    __threadfence_system();
    for (uint32_t d = 0; d < ex->world; ++d)
        if (d != ex->rank) st_release_sys(ex->tx_meta[d] + kSlots + 1, 1u);
}

// Per-neuron state the fused update reads (prefetched one neuron ahead).
template <bool PACKED>
struct NIn {
    uint32_t vb;
    float4 j;
    float iou;
    float4 g;
    ulonglong2 p0, p1;  // pending of S(tE-1); p1 only in the wide layout
    float isyn;
};

template <bool PACKED>
__device__ __forceinline__ void load_neuron(const StepArgs& a, uint32_t i, bool doE,
                                            const void* pend_rd, NIn<PACKED>& x, uint64_t pf,
                                            uint64_t pk) {
    x.vb = ldp(a.v + i, pf);
    x.iou = ldp(a.i_ou + i, pf);
    if (doE) {
        x.j = ldp(a.j + i, pf);
        x.g = ldp(a.g + i, pf);
        if constexpr (PACKED) {
            x.p0 = ldp_cg(reinterpret_cast<const ulonglong2*>(pend_rd) + i, pk);
        } else {
            x.p0 = ldp_cg(reinterpret_cast<const ulonglong2*>(pend_rd) + 2 * (size_t)i, pk);
            x.p1 = ldp_cg(reinterpret_cast<const ulonglong2*>(pend_rd) + 2 * (size_t)i + 1, pk);
        }
    } else {
        x.isyn = ldp(a.i_syn + i, pf);
    }
}

template <bool PACKED>
__global__ void __launch_bounds__(kThreads, VXB_MINB) step_kernel(StepArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemLayout L(a.use_smem_seg ? a.nseg : 0u, a.use_smem_seg ? a.npset : 0u, a.stage_e);
    ParamSet* s_pset = reinterpret_cast<ParamSet*>(smem + L.pset);
    SegInfo* s_seg = reinterpret_cast<SegInfo*>(smem + L.seg);
    uint32_t* s_start = reinterpret_cast<uint32_t*>(smem + L.start);
    uint32_t* s_spk = reinterpret_cast<uint32_t*>(smem + L.spk);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.bar);
    unsigned char* s_meta_base = smem + L.meta;
    __shared__ uint32_t s_nspk;
    __shared__ uint32_t s_fwork;  // next 32-neuron update chunk of the phase
    __shared__ uint32_t s_base;
    __shared__ int s_stop;
    __shared__ uint32_t s_hcnt[64];  // dynamic delivery: peer batch sizes of the phase
    __shared__ BatchScratch s_scr;   // producer warp: stage packing
    __shared__ unsigned long long s_tD, s_tF;  // phase profile

    const ParamSet* psp = a.pset;
    const SegInfo* segp = a.sinfo;
    const uint32_t* startp = a.seg_start;
    if (a.use_smem_seg) {
        for (uint32_t k = threadIdx.x; k < a.nseg; k += blockDim.x) {
            s_seg[k] = a.sinfo[k];
            s_start[k] = a.seg_start[k];
        }
        for (uint32_t k = threadIdx.x; k < a.npset; k += blockDim.x) s_pset[k] = a.pset[k];
        if (threadIdx.x == 0) s_start[a.nseg] = a.n;
        psp = s_pset;
        segp = s_seg;
        startp = s_start;
    }
    if (threadIdx.x == 0) {
        s_nspk = 0;
        s_fwork = 0;
        s_tD = s_tF = 0;
        for (int k = 0; k < kStages; ++k) {
            mbar_init(s_bar + k, 1);                          // full: producer + tx bytes
            mbar_init(s_bar + kStages + k, VXB_DWARPS > 1 ? VXB_DWARPS - 1 : 1);  // empty
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint32_t lane = threadIdx.x & 31;
    // Warp roles: the first VXB_DWARPS warps of every CTA run the delivery
    // pipeline (bulk copies + atomics, L2-atomic bound) and then join the
    // others on the neuron update, which every warp takes in 32-neuron
    // chunks of the CTA's contiguous neuron range.
    static_assert(VXB_DWARPS >= 2, "delivery needs a producer and a consumer warp");
    constexpr uint32_t kDT = VXB_DWARPS * 32;
    const bool roleD = threadIdx.x < kDT;
    const uint32_t d_cta = kDT;
    // this CTA's neurons: [c_lo, c_hi), multiples of 32 apart
    const uint32_t per = (((a.n + gridDim.x - 1) / gridDim.x) + 31u) & ~31u;
    const uint32_t c_lo = min(a.n, blockIdx.x * per), c_hi = min(a.n, c_lo + per);
    const uint32_t nch = (c_hi - c_lo + 31u) >> 5;
    Control* ctl = a.ctl;
    unsigned long long my_inner = 0, my_outer = 0;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_syn = VXB_POL_STREAM == 0 ? pol_stream : policy_evict_normal();
    const uint64_t pol_keep = VXB_POL_KEEP == 0 ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_f = a.f_policy == 1 ? pol_stream : a.f_policy == 2 ? pol_keep : policy_evict_normal();
    // the update's read + zeroing of the pending buffer: kept in L2 for the
    // next phase's atomics when the buffer fits; evict-first when it is
    // L2-blocked, or the zeroed lines would displace the live block
    const uint64_t pol_pz = a.n_blocks > 1 ? pol_stream : pol_keep;
    uint32_t g_item = 0;  // stages this CTA has consumed since launch (stage/parity)
    // warp-uniform cache of the parameter segment last looked up
    uint32_t seg_hint = 0, seg_lo = 1u, seg_nx = 0u;

    if (blockIdx.x == 0 && threadIdx.x == 0) a.phase_ns[0] = globaltimer();
    const uint32_t nph = a.steps + 1;
    for (uint32_t ph = 0; ph < nph; ++ph) {
        const bool doA = ph < a.steps;
        const bool doE = ph >= 1;
        const uint32_t tA = a.t0 + ph;
        const uint32_t tE = tA - 1;
        // pending buffer consumed by E(tE) holds S(tE-1): parity (tE-1)&1 == tA&1
        void* pend_rd = (tA & 1u) ? a.pend1 : a.pend0;
        // deliveries of S(tE) go to parity tE&1
        void* pend_wr = (tE & 1u) ? a.pend1 : a.pend0;
        const uint32_t inj_ep = (doA && a.has_inj) ? a.inj_epoch[ph] : 0u;
        uint32_t f_lo = 0, f_hi = 0;
        if (doA && a.has_forced) {
            f_lo = a.forced_off[ph];
            f_hi = a.forced_off[ph + 1];
        }
        const uint32_t log_base = a.ring ? (ph & 1u) * a.n : 0u;

        // D work of this phase: the rows of S(tE) (local spikes, then every
        // peer's batch)
        uint32_t d_lo = 0, d_cnt = 0, d_prev = 0;
        if (doE) {
            d_lo = (ph >= 2 && !a.ring) ? __ldcg(a.seg_end + ph - 2) : 0u;
            d_cnt = __ldcg(a.seg_end + ph - 1) - d_lo;
            d_prev = a.ring ? ((ph - 1) & 1u) * a.n : 0u;
        }

        // ------------------------------------------------------------ D
        unsigned long long wait_ns = 0;
        if (roleD && doE) {
            // Producer / consumer delivery pipeline: warp 0 lane 0 packs the
            // rows of this CTA's spikes (local list, then each peer's batch
            // once its step flag is set) into the stage ring with bulk copies;
            // the other delivery warps drain stages into the pending buffer
            // with red.add (L2 atomics).  full/empty mbarriers per stage.
            const uint32_t tslot = tE % kSlots;
            uint64_t* full = s_bar;
            uint64_t* empty = s_bar + kStages;
            if (threadIdx.x < 32) {
                // producer warp: 32 spikes' segment bounds per round trip,
                // lane 0 packs them; target blocks in order (L2 blocking)
                StageBuilder sbld{g_item, 0, 0, 0, 0, 0};
                const uint32_t B = a.n_blocks;
                if (a.dyn) {
                    // block-major dynamic chunks: every producer finishes
                    // its share of block b before block b + 1, so the
                    // grid's atomics stay inside one L2-resident block
                    const uint32_t W = a.world;
                    uint32_t* wc = a.work_ctr + (ph & 1u) * B * W;
                    if (blockIdx.x == 0)  // the other set serves phase ph + 1
                        for (uint32_t k = lane; k < B * W; k += 32)
                            a.work_ctr[((ph + 1) & 1u) * B * W + k] = 0u;
                    for (uint32_t blk = 0; blk < B; ++blk) {
                        for (uint32_t li = 0; li < W; ++li) {
                            const uint32_t h = (a.ex->rank + li) % W;
                            const uint32_t* ids = a.spk + d_prev + d_lo;
                            uint32_t cnt = d_cnt;
                            if (li) {
                                if (blk == 0 && lane == 0) {
                                    const unsigned long long w0 = globaltimer();
                                    s_hcnt[li] = exchange_wait(a, h, tE, tslot, ph);
                                    wait_ns += globaltimer() - w0;
                                }
                                __syncwarp();
                                cnt = s_hcnt[li];
                                ids = a.ex->rx_ids[h] + tslot * a.ex->cap[h];
                            }
                            const uint32_t sb = a.ex->src_base[h];
                            const uint32_t CH = max(1u, min(li ? 32u : a.ch_max, cnt / (8u * gridDim.x)));
                            uint32_t* ctr = wc + blk * W + li;
                            uint32_t nxt = 0;
                            if (lane == 0) nxt = atomicAdd(ctr, CH);
                            for (;;) {
                                const uint32_t c0 = __shfl_sync(0xffffffffu, nxt, 0);
                                if (c0 >= cnt) break;
                                if (lane == 0) nxt = atomicAdd(ctr, CH);  // in flight meanwhile
                                const uint32_t nl = min(CH, cnt - c0);
                                uint64_t sbeg = 0, slen = 0;
                                if (lane < nl) {
                                    const uint32_t s = sb + __ldcg(ids + c0 + lane);
                                    const uint64_t row = ldg64(a.off + s);
                                    if (B == 1) {
                                        sbeg = row;
                                        slen = ldg64(a.off + s + 1) - row;
                                    } else {
                                        const uint32_t* bo = a.blk_off + (size_t)s * (B + 1);
                                        const uint32_t lo = __ldg(bo + blk), hi = __ldg(bo + blk + 1);
                                        sbeg = row + lo;
                                        slen = hi - lo;
                                    }
                                    if (blk == 0) {
                                        const uint64_t len = ldg64(a.off + s + 1) - row;
                                        const uint32_t in = __ldg(a.inner + s);
                                        my_inner += 2ull * in;
                                        my_outer += 2ull * (len - in);
                                    }
                                }
                                if (B > 1) {  // short block segments: parallel issue
                                    sbld.add_batch(a, smem, L, sbeg, (uint32_t)slen, pol_syn, s_scr, lane);
                                } else {
                                    for (unsigned m = __ballot_sync(0xffffffffu, slen != 0); m; m &= m - 1) {
                                        const int l = __ffs(m) - 1;
                                        const uint64_t b0 = __shfl_sync(0xffffffffu, sbeg, l);
                                        const uint64_t ln = __shfl_sync(0xffffffffu, slen, l);
                                        if (lane == 0) sbld.add(a, smem, L, b0, ln, pol_syn);
                                    }
                                }
                            }
                        }
                    }
                } else {
                    for (uint32_t li = 0; li < a.world; ++li) {
                        const uint32_t h = (a.ex->rank + li) % a.world;
                        const uint32_t* ids = a.spk + d_prev + d_lo;
                        uint32_t cnt = d_cnt;
                        if (li) {
                            uint32_t c = 0;
                            if (lane == 0) {
                                const unsigned long long w0 = globaltimer();
                                c = exchange_wait(a, h, tE, tslot, ph);
                                wait_ns += globaltimer() - w0;
                            }
                            cnt = __shfl_sync(0xffffffffu, c, 0);
                            ids = a.ex->rx_ids[h] + tslot * a.ex->cap[h];
                        }
                        const uint32_t sb = a.ex->src_base[h];
                        const uint32_t mine = cnt > blockIdx.x ? (cnt - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
                        for (uint32_t blk = 0; blk < B; ++blk) {
                            for (uint32_t j0 = 0; j0 < mine; j0 += 32) {
                                const uint32_t j = j0 + lane;
                                uint64_t sbeg = 0, slen = 0;
                                if (j < mine) {
                                    const uint32_t s = sb + __ldcg(ids + blockIdx.x + j * gridDim.x);
                                    const uint64_t row = ldg64(a.off + s);
                                    if (B == 1) {
                                        sbeg = row;
                                        slen = ldg64(a.off + s + 1) - row;
                                    } else {
                                        const uint32_t* bo = a.blk_off + (size_t)s * (B + 1);
                                        const uint32_t lo = __ldg(bo + blk), hi = __ldg(bo + blk + 1);
                                        sbeg = row + lo;
                                        slen = hi - lo;
                                    }
                                    if (blk == 0) {
                                        const uint64_t len = ldg64(a.off + s + 1) - row;
                                        const uint32_t in = __ldg(a.inner + s);
                                        my_inner += 2ull * in;
                                        my_outer += 2ull * (len - in);
                                    }
                                }
                                if (B > 1) {  // short block segments: parallel issue
                                    sbld.add_batch(a, smem, L, sbeg, (uint32_t)slen, pol_syn, s_scr, lane);
                                } else {
                                    for (unsigned m = __ballot_sync(0xffffffffu, slen != 0); m; m &= m - 1) {
                                        const int l = __ffs(m) - 1;
                                        const uint64_t b0 = __shfl_sync(0xffffffffu, sbeg, l);
                                        const uint64_t ln = __shfl_sync(0xffffffffu, slen, l);
                                        if (lane == 0) sbld.add(a, smem, L, b0, ln, pol_syn);
                                    }
                                }
                            }
                        }
                    }
                }
                if (lane == 0) {
                    if (!sbld.open) sbld.begin(smem, L);
                    sbld.commit(smem, L, 1);  // end marker (possibly with data)
                }
                g_item = __shfl_sync(0xffffffffu, sbld.ctr, 0);
            } else if (threadIdx.x >= 32) {
                const uint32_t ct = threadIdx.x - 32, cn = d_cta - 32;
                for (;;) {
                    const uint32_t st = g_item % kStages;
                    mbar_wait(full + st, (g_item / kStages) & 1u);
                    ++g_item;
                    const TStageMeta* m = reinterpret_cast<const TStageMeta*>(s_meta_base + st * kMetaBytes);
                    const uint32_t n_e = m->n, last = m->end;
                    const uint32_t* tg = reinterpret_cast<const uint32_t*>(smem + L.tgt + st * L.tb);
                    const uint64_t* wv = reinterpret_cast<const uint64_t*>(smem + L.w + st * L.wb);
                    uint32_t sg = 0;
                    for (uint32_t e = ct; e < n_e; e += cn) {
                        while (e >= m->pre[sg + 1]) ++sg;
                        const uint32_t r = e - m->pre[sg];
                        const uint32_t t = tg[m->tb[sg] + r], tid = t & 0x7fffffffu, cls = t >> 31;
                        const uint64_t wq = wv[m->wb[sg] + r];
                        if constexpr (PACKED) {
                            red_add(reinterpret_cast<unsigned long long*>(pend_wr) + 2 * (size_t)tid + cls,
                                    wq, pol_keep);
                        } else {
                            unsigned long long* dst =
                                reinterpret_cast<unsigned long long*>(pend_wr) + 4 * (size_t)tid + 2 * cls;
                            red_add(dst, (uint64_t)(int64_t)(int32_t)(uint32_t)wq, pol_keep);
                            red_add(dst + 1, (uint64_t)(int64_t)(int32_t)(uint32_t)(wq >> 32), pol_keep);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + st);
                    if (last) break;
                }
            }
        }


        if (a.prof && roleD && lane == 0) atomicMax(&s_tD, (unsigned long long)globaltimer());

        // ------------------------------------------------------------ F
        // 32-neuron chunks from the CTA's counter; loads of the next chunk
        // are in flight while the current one is updated
        {
            NIn<PACKED> cur, nxt;
            // chunk pipeline: ch is being updated, chn's state is in flight
            // to registers, chn2's lines are being prefetched into L2
            auto grab = [&]() {
                uint32_t c = 0;
                if (lane == 0) c = atomicAdd(&s_fwork, 1u);
                return __shfl_sync(0xffffffffu, c, 0);
            };
            auto prefetch = [&](uint32_t c) {
                if (VXB_PREFETCH == 0 || c >= nch) return;
                const uint32_t b = c_lo + (c << 5);
                const char* q = nullptr;
                if (lane == 0) q = reinterpret_cast<const char*>(a.v + b);
                else if (lane == 1) q = reinterpret_cast<const char*>(a.i_ou + b);
                else if (lane < 6) q = reinterpret_cast<const char*>(a.j + b) + (lane - 2) * 128;
                else if (doE && lane < 10) q = reinterpret_cast<const char*>(a.g + b) + (lane - 6) * 128;
                else if (doE && lane < (PACKED ? 14u : 18u))
                    q = reinterpret_cast<const char*>(pend_rd) + (size_t)b * (PACKED ? 16 : 32) +
                        (lane - 10) * 128;
                else if (!doE && lane == 10) q = reinterpret_cast<const char*>(a.i_syn + b);
                if (q) asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
            };
            uint32_t ch = grab();
            uint32_t chn = grab();
            prefetch(chn);
            uint32_t i = c_lo + (ch << 5) + lane;
            // loads are unpredicated (a lane past the range re-reads a valid
            // neuron and ignores it): predicated asm loads made the compiler
            // spill the prefetched state around them
            const uint32_t i_safe = c_lo < a.n ? c_lo : 0u;
            if (nch) load_neuron<PACKED>(a, (ch < nch && i < c_hi) ? i : i_safe, doE, pend_rd, cur, pol_f, pol_pz);
#if VXB_DEPTH3
            NIn<PACKED> nx2;
            {
                const uint32_t i1 = c_lo + (chn << 5) + lane;
                if (chn < nch && i1 < c_hi)
                    load_neuron<PACKED>(a, i1, doE, pend_rd, nxt, pol_f, pol_pz);
            }
#endif
            while (ch < nch) {
                const uint32_t chn2 = grab();
                prefetch(chn2);
                const uint32_t inext = c_lo + (chn << 5) + lane;
#if VXB_DEPTH3
                {
                    const uint32_t i2 = c_lo + (chn2 << 5) + lane;
                    if (chn2 < nch && i2 < c_hi)
                        load_neuron<PACKED>(a, i2, doE, pend_rd, nx2, pol_f, pol_pz);
                }
#else
                load_neuron<PACKED>(a, (chn < nch && inext < c_hi) ? inext : i_safe, doE, pend_rd, nxt, pol_f,
                                    pol_pz);
#endif
                const bool live = i < c_hi;
                bool spiked = false;
                // parameter segment: warp-uniform cached range, a galloping
                // search when the chunk leaves it, a per-lane walk only for
                // lanes past a segment boundary
                uint32_t seg;
                {
                    const uint32_t w_lo = c_lo + (ch << 5);
                    const uint32_t w_last = min(w_lo + 31u, c_hi - 1u);
                    if (w_lo < seg_lo || w_last >= seg_nx) {
                        uint32_t s0 = 0;
                        if (lane == 0)
                            s0 = find_seg_from(startp, a.nseg, w_lo, w_lo >= seg_lo ? seg_hint : 0u);
                        seg_hint = __shfl_sync(0xffffffffu, s0, 0);
                        seg_lo = startp[seg_hint];
                        seg_nx = seg_hint + 1 < a.nseg ? startp[seg_hint + 1] : a.n;
                    }
                    seg = seg_hint;
                    const uint32_t il = live ? i : c_hi - 1u;
                    if (il >= seg_nx)
                        while (seg + 1 < a.nseg && startp[seg + 1] <= il) ++seg;
                }
                if (live) {
                    const SegInfo& S = segp[seg];
                    const ParamSet& P = psp[S.pset];
                    uint32_t vb = cur.vb;
                    const float v = is_refrac(vb) ? P.v_reset : __uint_as_float(vb);
                    float4 j = cur.j;
                    float iou = cur.iou;
                    float isyn;
                    if (doE) {
                        // gating_kernel (model.hpp:69-71) with deq(P_prev) (engine.cpp:543-546)
                        float p0, p1, p2, p3;
                        if constexpr (PACKED) {
                            p0 = dequantize_u32((uint32_t)(cur.p0.x & 0xffffffffull));
                            p1 = dequantize_u32((uint32_t)(cur.p0.x >> 32));
                            p2 = dequantize_u32((uint32_t)(cur.p0.y & 0xffffffffull));
                            p3 = dequantize_u32((uint32_t)(cur.p0.y >> 32));
                            stp_cg(reinterpret_cast<ulonglong2*>(pend_rd) + i, make_ulonglong2(0ull, 0ull), pol_pz);
                        } else {
                            p0 = dequantize((int64_t)cur.p0.x);
                            p1 = dequantize((int64_t)cur.p0.y);
                            p2 = dequantize((int64_t)cur.p1.x);
                            p3 = dequantize((int64_t)cur.p1.y);
                            ulonglong2* q = reinterpret_cast<ulonglong2*>(pend_rd) + 2 * (size_t)i;
                            stp_cg(q, make_ulonglong2(0ull, 0ull), pol_pz);
                            stp_cg(q + 1, make_ulonglong2(0ull, 0ull), pol_pz);
                        }
                        j.x = fadd(fmul(j.x, P.decay[0]), fmul(P.omega[0], p0));
                        j.y = fadd(fmul(j.y, P.decay[1]), fmul(P.omega[1], p1));
                        j.z = fadd(fmul(j.z, P.decay[2]), fmul(P.omega[2], p2));
                        j.w = fadd(fmul(j.w, P.decay[3]), fmul(P.omega[3], p3));
                        // current_kernel (model.hpp:73-81), u order, from 0.0f
                        const float4 g = cur.g;
                        float c = 0.0f;
                        c = fadd(c, fmul(fmul(g.x, j.x), fsub(P.e_rev[0], v)));
                        c = fadd(c, fmul(fmul(g.y, j.y), fsub(P.e_rev[1], v)));
                        c = fadd(c, fmul(fmul(g.z, j.z), fsub(P.e_rev[2], v)));
                        c = fadd(c, fmul(fmul(g.w, j.w), fsub(P.e_rev[3], v)));
                        isyn = c;
                        // ou_kernel (model.hpp:88-90) with xi = stream word tE (engine.cpp:551-558)
                        float xi = 0.0f;
                        if (P.sigma_pos) {
                            const uint64_t gid = (uint64_t)((int64_t)i + S.gid_off);
                            xi = stream_xi(mix_key(a.ou_root, gid), tE);
                        }
                        iou = fadd(fadd(iou, fmul(P.ou_a, fsub(P.ou_mu, iou))), fmul(P.ou_b, xi));
                        if (!doA) stp(a.i_syn + i, isyn, pol_f);
                        stp(a.j + i, j, pol_f);
                        stp(a.i_ou + i, iou, pol_f);
                    } else {
                        isyn = cur.isyn;
                    }
                    if (doA) {
                        // membrane_kernel + threshold (engine.cpp:363-385)
                        if (is_refrac(vb)) {
                            const uint32_t r = (vb & 0x007fffffu) - 1u;
                            vb = r ? refrac_bits(r) : __float_as_uint(P.v_reset);
                        } else {
                            float inoise = iou;
                            if (inj_ep) {
                                const float x =
                                    __ldg(a.inj_table + (size_t)(inj_ep - 1) * a.n_voxels + S.voxel);
                                if (x != 0.0f) inoise = fadd(iou, x);
                            }
                            const float nv = fadd(
                                v, fmul(P.dt_over_c,
                                        fadd(fadd(fmul(P.g_leak, fsub(P.e_leak, v)), isyn), inoise)));
                            if (!isfinite(nv)) {
                                atomicMin(&ctl->err, ((unsigned long long)tA << 32) | i);
                                vb = __float_as_uint(nv);
                            } else if (nv >= P.v_th) {
                                spiked = true;
                                vb = P.tref ? refrac_bits(P.tref) : __float_as_uint(P.v_reset);
                            } else {
                                vb = __float_as_uint(nv);
                            }
                        }
                        // forced spikes (engine.cpp:389-398): join unless already fired
                        if (f_hi > f_lo && !spiked) {
                            const uint32_t k =
                                f_lo + lower_bound_u32(a.forced_local + f_lo, f_hi - f_lo, i);
                            if (k < f_hi && __ldg(a.forced_local + k) == i) {
                                spiked = true;
                                vb = P.tref ? refrac_bits(P.tref) : __float_as_uint(P.v_reset);
                            }
                        }
                        stp(a.v + i, vb, pol_f);
                    }
                    // probes: V after A(tA), I_syn after E(tE) (engine.cpp:405-406, 564-565)
                    if (a.n_probes) {
                        uint32_t k = lower_bound_u32(a.probe_local, a.n_probes, i);
                        while (k < a.n_probes && __ldg(a.probe_local + k) == i) {
                            const size_t row = (size_t)__ldg(a.probe_slot + k) * a.adv_steps + a.rel0;
                            if (doE) a.probe_i[row + ph - 1] = isyn;
                            if (doA) a.probe_v[row + ph] = is_refrac(vb) ? P.v_reset : __uint_as_float(vb);
                            ++k;
                        }
                    }
                }
                // spike staging + rates (engine.cpp:400-404), warp aggregated
                bool overflow_route = false;
                const unsigned ball = __ballot_sync(0xffffffffu, spiked);
                if (ball) {
                    unsigned base = 0;
                    if (lane == 0) base = atomicAdd(&s_nspk, (unsigned)__popc(ball));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (spiked) {
                        const unsigned rank = __popc(ball & ((1u << lane) - 1u));
                        if (base + rank < kSpkStage)
                            s_spk[base + rank] = i;
                        else {  // staging full: straight to the log (and to the peers)
                            a.spk[log_base + atomicAdd(&ctl->spk_cursor, 1u)] = i;
                            if (a.world > 1) overflow_route = true;
                        }
                        const uint32_t unit = segp[seg].unit;
                        const unsigned peers = __match_any_sync(ball, unit);
                        if ((unsigned)__ffs(peers) - 1u == lane)
                            atomicAdd(&a.rates[(size_t)unit * a.steps + ph], (unsigned)__popc(peers));
                    }
                }
                if (a.world > 1 && __any_sync(0xffffffffu, overflow_route))
                    if (exchange_route(a, i, overflow_route, tA % kSlots)) __threadfence_system();
                cur = nxt;
#if VXB_DEPTH3
                nxt = nx2;
#endif
                ch = chn;
                chn = chn2;
                i = inext;
            }
        }
        if (a.prof && lane == 0) atomicMax(&s_tF, (unsigned long long)globaltimer());
        // flush the CTA's staged spikes with one log reservation
        __syncthreads();
        if (a.prof && threadIdx.x == 0) {
            a.prof[2 * ((size_t)ph * gridDim.x + blockIdx.x)] = s_tD;
            a.prof[2 * ((size_t)ph * gridDim.x + blockIdx.x) + 1] = s_tF;
        }
        const uint32_t nst = min(s_nspk, (uint32_t)kSpkStage);
        if (threadIdx.x == 0 && nst) s_base = atomicAdd(&ctl->spk_cursor, nst);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < nst; k += blockDim.x)
            a.spk[log_base + s_base + k] = s_spk[k];
        if (a.world > 1 && doA) {
            bool sent = false;
            const uint32_t nr = (nst + 31u) & ~31u;
            for (uint32_t k = threadIdx.x; k < nr; k += blockDim.x)
                sent |= exchange_route(a, k < nst ? s_spk[k] : 0u, k < nst, tA % kSlots);
            if (sent) __threadfence_system();
            // the batch S(tA) is complete once every CTA has routed: the last
            // CTA publishes it now, while the grid may still be delivering
            if (a.early_publish) {
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    if (atomicAdd(&ctl->routed, 1u) == gridDim.x - 1) {
                        ctl->routed = 0;
                        exchange_publish(a, tA);
                    }
                }
            }
        }

        if (threadIdx.x == 0 && wait_ns && a.phase_wait) atomicMax(a.phase_wait + ph, wait_ns);
        grid_barrier(
            ctl,
            [&] {
                if (doA) a.seg_end[ph] = ctl->spk_cursor;
                if (a.ring) ctl->spk_cursor = 0;  // next phase writes the other half
                a.phase_ns[ph + 1] = globaltimer();
                // one stop decision for the whole grid (L2-coherent reads of
                // the flags the phase may have raised)
                ctl->stop = (atomicAdd(&ctl->err, 0ull) != ~0ull ||
                             atomicAdd(&a.ex->timeout, 0u) != 0u ||
                             atomicAdd(&a.ex->peer_abort, 0u) != 0u) ? 1u : 0u;
            },
            [&] {
                if (a.world > 1) {
                    // a failed step publishes no batch (the reference's worker
                    // throws before phase B), so no peer can finish without it
                    if (ctl->stop)
                        exchange_abort(a);
                    else if (doA && !a.early_publish)
                        exchange_publish(a, tA);
                }
            });
        if (threadIdx.x == 0) {
            s_stop = (int)ld_acquire(&ctl->stop);
            s_nspk = 0;
            s_fwork = 0;
            s_tD = s_tF = 0;
        }
        __syncthreads();
        if (s_stop) break;
    }
    if (my_inner | my_outer) {
        atomicAdd(&ctl->flops_inner, my_inner);
        atomicAdd(&ctl->flops_outer, my_outer);
    }
}

// ------------------------------------------------------- out-CSR build
// Inverts the in-rows of the worker tables (engine.cpp:295-327) on the
// device: count per source, scan, scatter.

struct SynIn {  // == vxb_syn_entry
    uint32_t src_local;
    uint16_t src_worker;
    uint8_t cls;
    uint8_t pad;
    int32_t wq_fast;
    int32_t wq_slow;
};

__global__ void csr_count_kernel(const SynIn* __restrict__ e, uint64_t ne,
                                 const uint32_t* __restrict__ wbase,
                                 const uint32_t* __restrict__ wn, uint32_t nw,
                                 unsigned long long* __restrict__ cnt,
                                 unsigned int* __restrict__ bad) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < ne;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const SynIn x = e[k];
        if (x.src_worker >= nw || x.src_local >= wn[x.src_worker]) {
            atomicExch(bad, 1u);
            continue;
        }
        atomicAdd(cnt + wbase[x.src_worker] + x.src_local, 1ull);
    }
}

// One warp per target row.
__global__ void csr_scatter_kernel(const SynIn* __restrict__ e,
                                   const uint64_t* __restrict__ row_base, uint32_t rows,
                                   uint32_t dst_worker, uint32_t dst_base,
                                   const uint32_t* __restrict__ wbase,
                                   unsigned long long* __restrict__ cursor,
                                   uint32_t* __restrict__ tgt, uint64_t* __restrict__ w,
                                   unsigned long long* __restrict__ have_mask,
                                   uint32_t* __restrict__ inner,
                                   unsigned int* __restrict__ wide) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t base0 = row_base[0];
    for (uint64_t r = warp; r < rows; r += nwarps) {
        const uint64_t b = row_base[r] - base0, en = row_base[r + 1] - base0;
        long long sf = 0, ss = 0;
        bool neg = false;
        for (uint64_t k = b + lane; k < en; k += 32) {
            const SynIn x = e[k];
            const uint32_t src = wbase[x.src_worker] + x.src_local;
            const unsigned long long pos = atomicAdd(cursor + src, 1ull);
            tgt[pos] = (dst_base + (uint32_t)r) | (x.cls ? 0x80000000u : 0u);
            w[pos] = (uint64_t)(uint32_t)x.wq_fast | ((uint64_t)(uint32_t)x.wq_slow << 32);
            atomicOr(have_mask + src, 1ull << dst_worker);
            if (x.src_worker == dst_worker) atomicAdd(inner + src, 1u);
            sf += x.wq_fast;
            ss += x.wq_slow;
            neg |= (x.wq_fast < 0) || (x.wq_slow < 0);
        }
        for (int o = 16; o; o >>= 1) {
            sf += __shfl_xor_sync(0xffffffffu, sf, o);
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
        }
        neg = __any_sync(0xffffffffu, neg);
        if (lane == 0 && (neg || sf >= (1ll << 32) || ss >= (1ll << 32))) atomicExch(wide, 1u);
    }
}

// L2 blocking: per source, offsets (within its target-sorted row) of the
// first entry of every target block.
__global__ void block_offsets_kernel(const uint64_t* __restrict__ off,
                                     const uint32_t* __restrict__ tgt, uint32_t n_src,
                                     uint32_t n_blocks, uint32_t block_n,
                                     uint32_t* __restrict__ bo) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_src; s += gridDim.x * blockDim.x) {
        const uint64_t e0 = off[s], e1 = off[s + 1];
        uint32_t* o = bo + (size_t)s * (n_blocks + 1);
        o[0] = 0;
        uint64_t lo = e0;
        for (uint32_t b = 1; b < n_blocks; ++b) {
            const uint32_t bound = b * block_n;
            uint64_t hi = e1;  // first entry with target >= bound
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if ((tgt[mid] & 0x7fffffffu) < bound) lo = mid + 1; else hi = mid;
            }
            o[b] = (uint32_t)(lo - e0);
        }
        o[n_blocks] = (uint32_t)(e1 - e0);
    }
}

// crossing_matrix (netgen.cpp:331-355) from the out-CSR: synapses per
// (source worker, target worker).  Worker bases in shared memory, per-block
// counts in shared memory, flushed once per block.  One warp per row.
__global__ void crossing_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                                uint32_t n_src, const uint32_t* __restrict__ src_base,
                                const uint32_t* __restrict__ wbase, uint32_t W,
                                unsigned long long* __restrict__ out) {
    __shared__ uint32_t s_sb[65], s_wb[65];
    __shared__ unsigned int s_c[64 * 64];
    for (uint32_t k = threadIdx.x; k <= W; k += blockDim.x) {
        s_sb[k] = src_base[k];
        s_wb[k] = wbase[k];
    }
    for (uint32_t k = threadIdx.x; k < W * W; k += blockDim.x) s_c[k] = 0;
    __syncthreads();
    auto bin = [&](const uint32_t* b, uint32_t x) {  // last w with b[w] <= x
        uint32_t lo = 0, hi = W;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (b[mid] <= x) lo = mid; else hi = mid;
        }
        return lo;
    };
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t s = warp; s < n_src; s += nwarps) {
        const uint32_t sw = bin(s_sb, (uint32_t)s);
        for (uint64_t k = off[s] + lane; k < off[s + 1]; k += 32)
            atomicAdd(&s_c[sw * W + bin(s_wb, tgt[k] & 0x7fffffffu)], 1u);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < W * W; k += blockDim.x)
        if (s_c[k]) atomicAdd(out + k, (unsigned long long)s_c[k]);
}

__global__ void mask_check_kernel(const unsigned long long* __restrict__ have,
                                  const unsigned long long* __restrict__ mask, uint32_t n,
                                  unsigned long long* __restrict__ first_bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (have[i] != mask[i]) atomicMin(first_bad, (unsigned long long)i);
}

// Pack (step << 32 | local) keys of the spike log for the raster sort.
// Per-launch scratch clearing: up to kClearMax word arrays zeroed, and the
// control block reset (err = none) — one launch instead of a memset each.
constexpr int kClearMax = 12;
struct ClearList {
    uint32_t* p[kClearMax];
    uint64_t words[kClearMax];
    Control* ctl;
    int n;
};
__global__ void clear_kernel(ClearList cl) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (int k = 0; k < cl.n; ++k)
        for (uint64_t i = tid; i < cl.words[k]; i += nth) cl.p[k][i] = 0u;
    if (tid < sizeof(Control) / 4) {
        uint32_t* c = reinterpret_cast<uint32_t*>(cl.ctl);
        const uint32_t k = (uint32_t)tid;
        // err (~0 = none) sits at a fixed offset; everything else is zero
        const uint32_t e0 = (uint32_t)(offsetof(Control, err) / 4);
        c[k] = (k == e0 || k == e0 + 1) ? 0xffffffffu : 0u;
    }
}

// seg_end: cumulative log ends per step; stride != 0: the log is
// phase-strided (step s's entries at spk[s * stride], tile_kernel).
__global__ void raster_keys_kernel(const uint32_t* __restrict__ spk,
                                   const uint32_t* __restrict__ seg_end, uint32_t steps,
                                   uint64_t* __restrict__ keys, uint32_t stride) {
    for (uint32_t s = blockIdx.x; s < steps; s += gridDim.x) {
        const uint32_t lo = s ? seg_end[s - 1] : 0u, hi = seg_end[s];
        const uint32_t* src = stride ? spk + (size_t)s * stride - lo : spk;
        for (uint32_t k = lo + threadIdx.x; k < hi; k += blockDim.x)
            keys[k] = ((uint64_t)s << 32) | src[k];
    }
}

__global__ void debug_normal_kernel(const uint64_t* __restrict__ base,
                                    const uint64_t* __restrict__ k, uint64_t n,
                                    double* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = stream_normal(base[i], k[i]);
}

__global__ void debug_xi_kernel(const uint64_t* __restrict__ base,
                                const uint64_t* __restrict__ k, uint64_t n,
                                float* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = stream_xi(base[i], k[i]);
}

// Staged set_conductances (engine.cpp:829-844) applied in one launch before
// an advance: record r = {first staged value, destination float index
// (neuron * 4 + receptor), count}; records are sorted by their first value
// and never overlap, so every staged value has exactly one destination.
__global__ void cond_scatter_kernel(const float* __restrict__ vals,
                                    const uint4* __restrict__ rec, uint32_t n_rec,
                                    uint32_t total, float* __restrict__ g) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = n_rec;  // last record with rec.x <= i
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(&rec[mid].x) <= i) lo = mid;
            else hi = mid;
        }
        const uint4 r = rec[lo];
        g[(uint64_t)r.y + 4ull * (i - r.x)] = vals[i];
    }
}

}  // namespace vxb

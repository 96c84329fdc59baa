// vxb_tile.cuh — the SM-tile path of the simulation step, for shards whose
// pending sums fit in the GPU's shared memory (config 2: 1M neurons x 16 B
// = 16 MB over 148 SMs).
//
// One CTA per SM owns a contiguous tile of neurons: it updates them AND
// accumulates their pending synaptic input in shared memory, so delivery
// runs on the SMs' shared-memory atomics (two ATOMS.ADD.32 per event,
// measured 5.6e11 events/s chip-wide) instead of the L2 atomic units (the
// l2_atomic path's ceiling, ~1.9e11 red/s).  Rows are sorted by target and
// split at tile boundaries once at load: every (source, tile) segment is
// contiguous in the out-CSR.  When a neuron spikes (A(tA) of phase ph) the
// spiking lane appends one work item {first entry, length} per tile its row
// touches to that tile's queue; in phase ph + 1 each CTA streams exactly the
// segments of its own tile with TMA bulk copies and adds them into its
// shared-memory pending tile.  Every synapse entry is read once, by the CTA
// that owns its target; nothing is re-read or reduced twice.
//
// Phase ph of a chunk (tA = t0 + ph, tE = tA - 1), per CTA:
//   U  (all warps)    E(tE) + A(tA) of the tile's neurons: gating with the
//                     shared-memory pending P(S(tE-1)) (zeroed after the
//                     read), current, membrane; the OU current I_ou(tE) was
//                     already advanced in phase ph - 1 (see N).  Spikes of
//                     S(tA) are logged, counted and bucketed into the tile
//                     queues of parity tA.
//   then, concurrently:
//   C  (warps 0..C-1) consumers: take the segments queued for this tile in
//                     parity tE one per grab, stream their entries with
//                     plain loads (kTileUnroll in flight per lane; a TMA bulk
//                     copy per ~200-entry segment measured ~0.3 us of issue
//                     each, 9x slower) and add them into the pending tile
//                     with shared atomics — P(S(tE)), consumed by E(tA) in
//                     phase ph + 1.
//   N  (other warps)  advance I_ou to tA (fp64 Box-Muller noise, ou_kernel)
//                     for the tile, overlapping the delivery.
//   no grid barrier: a CTA goes on to phase ph + 1 as soon as its own C and N
//   are done (U(ph + 1) needs only its tile's pending sums and I_ou).  Only
//   the consumers of phase ph + 1 depend on the other CTAs — on their
//   bucketing of S(tA) — and wait for that phase's count (bdone[ph] == G).
//   Queues rotate over four step sets (tA & 3): a CTA can be bucketing
//   S(tA + 1) while a slower one still consumes S(tE); with four sets a
//   writer of set tA & 3 is provably behind every consumer of it.
// Moving the OU step one phase earlier is exact: I_ou(t) depends only on
// I_ou(t-1) and xi(gid, t) (ou_kernel, model.hpp:88-90; engine.cpp:551-558).
// Between chunks (and advance() calls) the state is the reference's
// post-phase-E state: the last phase does not advance I_ou, and the pending
// tile is written back to the global pending buffer of its parity.
#pragma once

#include "vxb_kernels.cuh"

namespace vxb {

#ifndef VXB_TILE_THREADS
// 32 warps at 64 registers: config 2 56.9 us/step vs 60.8 at 24 warps x 80
// registers (the update, noise and delivery are all latency-bound; more
// warps beat fewer spills), 67.9 at 20 x 96
#define VXB_TILE_THREADS 1024
#endif
constexpr int kTileThreads = VXB_TILE_THREADS;      // 24 warps: update, then consume / advance I_ou
#ifndef VXB_TILE_UNROLL
#define VXB_TILE_UNROLL 4
#endif
constexpr uint32_t kTileUnroll = VXB_TILE_UNROLL;  // synapse entries in flight per consumer lane
constexpr uint32_t kTileMaxGrid = 256;  // CTAs (tiles) the per-tile bucketing covers
#ifndef VXB_TILE_PREFETCH
#define VXB_TILE_PREFETCH 24
#endif
constexpr uint32_t kTilePrefetch = VXB_TILE_PREFETCH;  // queued segments prefetched ahead of the consumers
#ifndef VXB_TILE_BWARPS
// warps that route and bucket S(tA) after the update: 4 (config 2 at 2 / 4
// GPUs 3.82 -> 4.07e11 / 7.05 -> 7.51e11 events/s — the routing before the
// bucketing gets shorter; one GPU equal; 6 or 8 equal to 4)
#define VXB_TILE_BWARPS 4
#endif
constexpr uint32_t kTileBucketWarps = VXB_TILE_BWARPS;
constexpr uint32_t kTileProf = 8;       // phase-profile words per (phase, CTA)
#ifndef VXB_TILE_SCANW
#define VXB_TILE_SCANW 0  // consumer warps scanning the peers' batches (0 = all)
#endif
#ifndef VXB_TILE_SPIN0
#define VXB_TILE_SPIN0 64    // ns between mailbox polls (warp 0)
#endif
#ifndef VXB_TILE_SPIN1
#define VXB_TILE_SPIN1 128   // ns between polls of the posted phase (other warps)
#endif
#ifndef VXB_TILE_L1PF
#define VXB_TILE_L1PF 0                 // update: L1 prefetch of the chunk after next (no gain measured)
#endif
#ifndef VXB_TILE_FUSE_NOISE
// the OU step of I_ou(tA) inside the update loop instead of a separate pass
// (config 2: 55.5 vs 48.6 us/step — the update gets 14 us longer, the noise
// is better spread over the phase's idle warps)
#define VXB_TILE_FUSE_NOISE 0
#endif
constexpr uint32_t kTileQSets = 4;      // queue sets (step & 3), see the phase notes above
// queue item: first entry (bits 0-39) | segment length << 40
constexpr uint64_t kItemBeg = (1ull << 40) - 1;
constexpr uint32_t kTileMaxSeg = 64;    // a tile's parameter segments kept in shared memory
constexpr uint32_t kTileMaxPset = 32;

// Dynamic shared memory of tile_kernel.
struct TileLayout {
    uint32_t per;
    uint32_t pend, pset, seg, start, spk, total;
    __host__ __device__ explicit TileLayout(uint32_t per_) {
        per = per_;
        pend = 0;  // [parity][AMPA, NMDA, GABAA, GABAB][per] (u32)
        pset = (pend + 32 * per + 127) & ~127u;
        seg = pset + kTileMaxPset * (uint32_t)sizeof(ParamSet);
        start = seg + kTileMaxSeg * (uint32_t)sizeof(SegInfo);
        spk = (start + (kTileMaxSeg + 1) * 4 + 15) & ~15u;
        total = spk + kSpkStage * 4;
    }
};

// Streamed synapse entries: read once, not kept in L1, evict-first in L2.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p, uint64_t pol) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
                 : "=l"(v) : "l"(p), "l"(pol));
    return v;
}

// Warp-uniform parameter-segment lookup over the tile's segment table:
// starts[0..nseg) ascending, `end` = first neuron past the last segment.
// The cursor (last segment found and its range) lives in shared memory, one
// per warp: no registers stay live across the update loop for it (the
// kernel runs at 64 registers, and spills land in a 20 KB L1).
struct SegCursor {
    uint32_t hint, lo, nx, pad;
    __device__ __forceinline__ void reset() {
        hint = 0;
        lo = 1u;
        nx = 0u;
    }
    __device__ __forceinline__ uint32_t find(const uint32_t* starts, uint32_t nseg, uint32_t end,
                                             uint32_t w_lo, uint32_t w_last, uint32_t i_lane,
                                             uint32_t lane) {
        volatile SegCursor* c = this;
        uint32_t h = c->hint, l = c->lo, x = c->nx;
        if (w_lo < l || w_last >= x) {
            uint32_t s0 = 0;
            if (lane == 0) s0 = find_seg_from(starts, nseg, w_lo, w_lo >= l ? h : 0u);
            h = __shfl_sync(0xffffffffu, s0, 0);
            l = starts[h];
            x = h + 1 < nseg ? starts[h + 1] : end;
            __syncwarp();
            if (lane == 0) {
                c->hint = h;
                c->lo = l;
                c->nx = x;
            }
            __syncwarp();
        }
        uint32_t seg = h;
        if (i_lane >= x)
            while (seg + 1 < nseg && starts[seg + 1] <= i_lane) ++seg;
        return seg;
    }
};

// The same lookup with the cursor in registers (tile_mp_kernel).
struct SegCursorReg {
    uint32_t hint = 0, lo = 1u, nx = 0u;
    __device__ __forceinline__ uint32_t find(const uint32_t* starts, uint32_t nseg, uint32_t end,
                                             uint32_t w_lo, uint32_t w_last, uint32_t i_lane,
                                             uint32_t lane) {
        if (w_lo < lo || w_last >= nx) {
            uint32_t s0 = 0;
            if (lane == 0) s0 = find_seg_from(starts, nseg, w_lo, w_lo >= lo ? hint : 0u);
            hint = __shfl_sync(0xffffffffu, s0, 0);
            lo = starts[hint];
            nx = hint + 1 < nseg ? starts[hint + 1] : end;
        }
        uint32_t seg = hint;
        if (i_lane >= nx)
            while (seg + 1 < nseg && starts[seg + 1] <= i_lane) ++seg;
        return seg;
    }
};

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// 8-byte tile entry: bits 0-15 the word offset of its fast-receptor sum in
// the pending tile (AMPA: l, GABAA: 2 per + l for tile-local target l; the
// slow receptor's sum is `per` words further), bits 16-39 wq_slow, bits
// 40-63 wq_fast.  `bw` is the shared-memory address of the tile's parity
// buffer, per4 = 4 per: two shared reductions and four integer operations.
__device__ __forceinline__ void tile_add(uint32_t bw, uint32_t per4, uint64_t e) {
    const uint32_t q = bw + ((uint32_t)e & 0xffffu) * 4u;
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(q), "r"((uint32_t)(e >> 40)) : "memory");
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(q + per4),
                 "r"((uint32_t)(e >> 16) & 0xffffffu) : "memory");
}

// MG: one process per GPU (peers' batches, P2P routing); false: one GPU.
// EX: the advance has probes, forced spikes or injections; the variant
// without them keeps those paths (and their registers) out of the update.
template <bool MG, bool EX>
__global__ void __launch_bounds__(kTileThreads, 1) tile_kernel(StepArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const TileLayout L(a.tile_n);
    const uint32_t per = a.tile_n;
    uint32_t* s_pend = reinterpret_cast<uint32_t*>(smem + L.pend);  // [parity][receptor][per]
    uint32_t* s_spk = reinterpret_cast<uint32_t*>(smem + L.spk);
    __shared__ uint32_t s_nspk, s_fwork, s_nwork, s_iwork, s_base, s_nst;
    __shared__ uint32_t s_ravail, s_rdone;  // MG: peers' items reserved / scanning warps done
    __shared__ uint32_t s_ready;            // last phase whose queues this CTA knows final
    __shared__ int s_stop;
    __shared__ uint32_t s_seg_lo, s_nseg;
    __shared__ uint32_t s_hist[kTileMaxGrid], s_qb[kTileMaxGrid];  // per-tile bucketing
    // phase profile: update end, bucketing end, consumers end, noise end,
    // (start), bucketing pass 1 / reservations / pass 2 ends
    __shared__ unsigned long long s_t[kTileProf];

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t c_lo = min(a.n, blockIdx.x * per), c_hi = min(a.n, c_lo + per);
    const uint32_t nt = c_hi - c_lo;
    const uint32_t nch = (nt + 31u) >> 5;
    const uint32_t G = gridDim.x;
    Control* ctl = a.ctl;
    const uint32_t n_cons = a.n_cons;                       // warps that start on delivery
    const uint32_t n_nw = a.n_noisew;                       // warps that start on the noise
    // consumer warps that scan the peers' batches (MG)
    const uint32_t n_scan = VXB_TILE_SCANW ? min((uint32_t)VXB_TILE_SCANW, n_cons) : n_cons;
    const uint32_t n_upd = kTileThreads / 32 - n_cons - n_nw;  // warps that start on the update
    const bool upd_warp = warp >= n_cons + n_nw;
    const uint32_t ut = threadIdx.x - (n_cons + n_nw) * 32;    // index among update threads

    // parameter sets and the tile's segments in shared memory
    const ParamSet* psp = a.pset;
    const SegInfo* segp = a.sinfo;
    const uint32_t* startp = a.seg_start;
    uint32_t nseg = a.nseg, seg_end = a.n;
    if (threadIdx.x == 0) {
        uint32_t lo = 0, cnt = 0;
        if (nt) {
            lo = find_seg(a.seg_start, a.nseg, c_lo);
            const uint32_t hi = find_seg(a.seg_start, a.nseg, c_hi - 1);
            cnt = hi - lo + 1;
        }
        s_seg_lo = lo;
        s_nseg = cnt;
        s_nspk = s_fwork = s_nwork = s_iwork = 0;
        s_ravail = s_rdone = 0;
        s_ready = 0xffffffffu;
        for (uint32_t k = 0; k < kTileProf; ++k) s_t[k] = 0;
    }
    for (uint32_t k = threadIdx.x; k < kTileMaxGrid; k += blockDim.x) s_hist[k] = 0;
    __syncthreads();
    if (a.npset <= kTileMaxPset) {
        ParamSet* sp = reinterpret_cast<ParamSet*>(smem + L.pset);
        for (uint32_t k = threadIdx.x; k < a.npset; k += blockDim.x) sp[k] = a.pset[k];
        psp = sp;
    }
    if (s_nseg <= kTileMaxSeg) {
        SegInfo* ss = reinterpret_cast<SegInfo*>(smem + L.seg);
        uint32_t* st = reinterpret_cast<uint32_t*>(smem + L.start);
        for (uint32_t k = threadIdx.x; k < s_nseg; k += blockDim.x) {
            ss[k] = a.sinfo[s_seg_lo + k];
            st[k] = a.seg_start[s_seg_lo + k];
        }
        segp = ss;
        startp = st;
        nseg = s_nseg;
        seg_end = c_hi;
    }
    // pending tiles: parity (t0 - 1) holds P(S(t0 - 1)), delivered before this
    // chunk (moved out of the global buffer); parity t0 starts empty
    {
        const uint32_t pp = (a.t0 - 1u) & 1u;
        ulonglong2* gp = reinterpret_cast<ulonglong2*>(pp ? a.pend1 : a.pend0);
        uint32_t* B = s_pend + pp * 4 * per;
        uint32_t* Z = s_pend + (pp ^ 1u) * 4 * per;
        for (uint32_t l = threadIdx.x; l < per; l += blockDim.x) {
            ulonglong2 p = make_ulonglong2(0ull, 0ull);
            if (l < nt) {
                p = __ldcg(gp + c_lo + l);
                __stcg(gp + c_lo + l, make_ulonglong2(0ull, 0ull));
            }
            B[l] = (uint32_t)p.x;
            B[per + l] = (uint32_t)(p.x >> 32);
            B[2 * per + l] = (uint32_t)p.y;
            B[3 * per + l] = (uint32_t)(p.y >> 32);
            Z[l] = Z[per + l] = Z[2 * per + l] = Z[3 * per + l] = 0u;
        }
    }
    __syncthreads();

    const uint64_t pol_syn = policy_evict_first();  // synapse stream: read once
    const uint64_t pol_f = a.f_policy == 2 ? policy_evict_last() : policy_evict_normal();
    // FLOP tallies go straight to the control block (relaxed reductions, a
    // few per spike): no 64-bit accumulators held in every thread
    // (per-CTA 32-bit shared counters, flushed to the control block once per
    // phase: one global address hit per spike serialised in its L2 slice —
    // config 3 1.12 -> 1.53 ms/step; a CTA's tally of one phase is < 2^32,
    // the shard's synapses being < 2^40 over >= 148 CTAs)
    __shared__ uint32_t s_fl_in, s_fl_out;
    if (threadIdx.x == 0) s_fl_in = s_fl_out = 0u;
    auto add_flops = [&](uint64_t in, uint64_t out) {
        if (in) atomicAdd(&s_fl_in, (uint32_t)in);
        if (out) atomicAdd(&s_fl_out, (uint32_t)out);
    };
    auto flush_flops = [&]() {  // thread 0
        const uint32_t fi = *(volatile uint32_t*)&s_fl_in, fo = *(volatile uint32_t*)&s_fl_out;
        if (fi) atomicAdd(&ctl->flops_inner, (unsigned long long)fi);
        if (fo) atomicAdd(&ctl->flops_outer, (unsigned long long)fo);
        s_fl_in = s_fl_out = 0u;
    };
    __shared__ SegCursor s_cur[2][kTileThreads / 32];  // per warp: update, noise
    if (threadIdx.x < kTileThreads / 32) {
        s_cur[0][threadIdx.x].reset();
        s_cur[1][threadIdx.x].reset();
    }
    __syncthreads();
    SegCursor& cur_u = s_cur[0][warp];
    SegCursor& cur_n = s_cur[1][warp];

    // every CTA's bucketing of phase q is complete: tell each CTA's mailbox
    // (one fence, then relaxed reductions: a release per store would fence each)
    auto post_bucketed = [&](uint32_t q) {
        __threadfence();
        for (uint32_t c = 0; c < G; ++c)
            asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(a.bmail + 32 * c), "r"(q + 1) : "memory");
    };
    if (blockIdx.x == 0 && threadIdx.x == 0) a.phase_ns[0] = globaltimer();
    const uint32_t nph = a.steps + 1;
    for (uint32_t ph = 0; ph < nph; ++ph) {
        if (a.prof && threadIdx.x == 0) s_t[4] = globaltimer();
        const bool doA = ph < a.steps;
        const bool doE = ph >= 1;
        const uint32_t tA = a.t0 + ph;
        const uint32_t tE = tA - 1;
        const uint32_t inj_ep = (EX && doA && a.has_inj) ? a.inj_epoch[ph] : 0u;
        uint32_t f_lo = 0, f_hi = 0;
        if (doA && a.has_forced) {
            f_lo = a.forced_off[ph];
            f_hi = a.forced_off[ph + 1];
        }
        const size_t log_base = (size_t)ph * a.n;  // phase-strided log (not written in ring mode)
        // I_ou by parity of its step: U reads I_ou(tE), N writes I_ou(tA)
        const float* iou_rd = (tE & 1u) ? a.i_ou_b : a.i_ou;
        float* iou_wr = (tA & 1u) ? a.i_ou_b : a.i_ou;

        // N: advance I_ou to tA (ou_kernel, model.hpp:88-90, xi = stream word
        // tA, engine.cpp:551-558) for the tile: consumed by E(tA) in ph + 1
        // One 32-neuron chunk per call; false once the tile is done.
        auto noise_chunk = [&]() -> bool {
            if (!doA || VXB_TILE_FUSE_NOISE) return false;
            {
                uint32_t c = 0;
                if (lane == 0) c = atomicAdd(&s_nwork, 1u);
                c = __shfl_sync(0xffffffffu, c, 0);
                if (c >= nch) return false;
                const uint32_t w_lo = c_lo + (c << 5);
                const uint32_t i = w_lo + lane;
                const bool live = i < c_hi;
                const uint32_t seg = cur_n.find(startp, nseg, seg_end, w_lo, min(w_lo + 31u, c_hi - 1u),
                                                live ? i : c_hi - 1u, lane);
                if (live) {
                    const SegInfo& S = segp[seg];
                    const ParamSet& P = psp[S.pset];
                    float iou = ldp(iou_rd + i, pol_f);
                    float xi = 0.0f;
                    if (P.sigma_pos) {
                        const uint64_t gid = (uint64_t)((int64_t)i + S.gid_off);
                        xi = stream_xi(mix_key(a.ou_root, gid), tA);
                    }
                    iou = fadd(fadd(iou, fmul(P.ou_a, fsub(P.ou_mu, iou))), fmul(P.ou_b, xi));
                    stp(iou_wr + i, iou, pol_f);
                }
            }
            return true;
        };
        auto noise = [&]() {
            while (noise_chunk()) {
            }
        };
        // every CTA's bucketing of S(tE) (phase ph - 1) is complete: the
        // tile's queue of set tE & 3 is final.  A CTA that stops early
        // credits the phases it will not run, so this never waits on it.
        // One warp per CTA (warp 0, a consumer) polls the CTA's mailbox and
        // posts the phase in shared memory for the others.
        // Non-blocking form: true once the queues are final (warp 0 polls
        // the mailbox, the other warps read what it posted).
        auto bucketed = [&]() -> bool {
            uint32_t r = *reinterpret_cast<volatile uint32_t*>(&s_ready) == ph;
            if (!r && warp == 0) {
                if (lane == 0 && ld_acquire(a.bmail + 32 * blockIdx.x) >= ph) {
                    __threadfence_block();
                    *reinterpret_cast<volatile uint32_t*>(&s_ready) = ph;
                    r = 1;
                }
                r = __shfl_sync(0xffffffffu, r, 0);
            }
            if (r) __threadfence_block();
            return r != 0;
        };
        auto wait_bucketed = [&]() {
            // advance I_ou while the other CTAs finish their bucketing
            while (!bucketed())
                if (!noise_chunk()) break;
            if (*reinterpret_cast<volatile uint32_t*>(&s_ready) != ph) {
                if (lane == 0) {
                    if (warp == 0) {
                        while (ld_acquire(a.bmail + 32 * blockIdx.x) < ph) __nanosleep(VXB_TILE_SPIN0);
                        __threadfence_block();
                        *reinterpret_cast<volatile uint32_t*>(&s_ready) = ph;
                    } else {
                        while (*reinterpret_cast<volatile uint32_t*>(&s_ready) != ph) __nanosleep(VXB_TILE_SPIN1);
                        __threadfence_block();
                    }
                }
                __syncwarp();
            }
        };
        // C: deliver S(tE) into the pending tile of parity tE (one queued
        // segment per warp grab, kTileUnroll entries in flight per lane)
        // (MG: the peers' segments for this tile are appended after the
        // local items by the consumer warps, see R; a consumer that runs out
        // of local items takes them once every scanning warp is done)
        auto consume = [&]() {
            if (!doE) return;
            wait_bucketed();
            const uint32_t par = tE & 1u, set = tE & 3u;
            const uint32_t bw = smem_u32(s_pend + par * 4 * per), per4 = 4 * per;
            const uint32_t cnt0 = __ldcg(a.q_cnt + set * G + blockIdx.x);
            const uint64_t* items = a.q + (size_t)set * a.q_total + a.q_base[blockIdx.x];
            // queued items are final up to `cnt` (MG: plus the peers' items,
            // once every scanning warp is done)
            uint32_t cnt = cnt0;
            auto grab_item = [&]() {
                uint32_t it = 0;
                if (lane == 0) it = atomicAdd(&s_iwork, 1u);
                return __shfl_sync(0xffffffffu, it, 0);
            };
            // MG: wait until item `it` exists or the queue is complete
            auto resolve = [&](uint32_t it) -> bool {
                if (MG && it >= cnt)
                    for (;;) {
                        const bool done = *reinterpret_cast<volatile uint32_t*>(&s_rdone) == n_scan;
                        if (done) {
                            __threadfence_block();
                            cnt = cnt0 + *reinterpret_cast<volatile uint32_t*>(&s_ravail);
                        }
                        if (it < cnt || done) break;
                        __nanosleep(200);
                    }
                return it < cnt;
            };
            // the item descriptor and the one kTilePrefetch grabs ahead (its
            // segment is pulled into L2 when this one is processed)
            auto load_item = [&](uint32_t it, uint64_t& d, uint64_t& f) {
                d = __ldcg(reinterpret_cast<const unsigned long long*>(items + it));
                f = it + kTilePrefetch < cnt
                        ? __ldcg(reinterpret_cast<const unsigned long long*>(items + it + kTilePrefetch))
                        : 0ull;
            };
            uint32_t it = grab_item();
            uint64_t d = 0, f = 0;
            bool have = resolve(it);
            if (have) load_item(it, d, f);
            while (have) {
                // software pipeline: the next grab's descriptors are in
                // flight while this segment is delivered
                const uint32_t itn = grab_item();
                uint64_t dn = 0, fn = 0;
                const bool early = itn < cnt;
                if (early) load_item(itn, dn, fn);
                if (f) {  // no registers held: the entry loads below then wait on L2, not HBM
                    const uint64_t fb = f & kItemBeg;
                    const char* fp = reinterpret_cast<const char*>(a.tent + fb);
                    const char* fe = reinterpret_cast<const char*>(a.tent + fb + (f >> 40));
                    const char* ln = reinterpret_cast<const char*>(
                        reinterpret_cast<uintptr_t>(fp) & ~(uintptr_t)127) + 128 * lane;
                    if (ln < fe) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(ln));
                }
                const uint64_t* ev = a.tent + (d & kItemBeg) + lane;
                const uint32_t len = (uint32_t)(d >> 40);
                uint32_t k0 = 0;
                for (; k0 + 32 * kTileUnroll <= len; k0 += 32 * kTileUnroll) {  // full rounds
                    uint64_t e[kTileUnroll];
#pragma unroll
                    for (uint32_t u = 0; u < kTileUnroll; ++u) e[u] = ld_stream(ev + k0 + u * 32, pol_syn);
#pragma unroll
                    for (uint32_t u = 0; u < kTileUnroll; ++u) tile_add(bw, per4, e[u]);
                }
                if (k0 < len) {  // the tail: lanes past the end re-read the segment's first
                    // entry (unpredicated loads: a predicated asm load made the
                    // compiler spill the array around it) and add nothing
                    uint64_t e[kTileUnroll];
#pragma unroll
                    for (uint32_t u = 0; u < kTileUnroll; ++u)
                        e[u] = ld_stream(k0 + u * 32 + lane < len ? ev + k0 + u * 32 : ev - lane, pol_syn);
#pragma unroll
                    for (uint32_t u = 0; u < kTileUnroll; ++u)
                        if (k0 + u * 32 + lane < len) tile_add(bw, per4, e[u]);
                }
                if (early) {
                    have = true;
                } else {
                    have = resolve(itn);
                    if (have) load_item(itn, dn, fn);
                }
                d = dn;
                f = fn;
            }
        };
        // R (one process per GPU): the peers' batches of S(tE).  The consumer
        // warps of every CTA wait for each peer's flag (the reference's step
        // barrier, engine.cpp:468-524), scan a slice each of the batch for the
        // sources whose rows have a segment in the CTA's tile (the row's tile
        // list, ascending by tile) and append those segments to the tile's
        // queue after the local items (slots reserved in shared memory).
        auto scan_remote = [&]() {
            if (!MG || !doE) return;
            wait_bucketed();
            Exchange* ex = a.ex;
            const uint32_t set = tE & 3u, slot = tE % kSlots;
            const uint32_t cnt0 = __ldcg(a.q_cnt + set * G + blockIdx.x);
            uint64_t* items = a.q + (size_t)set * a.q_total + a.q_base[blockIdx.x] + cnt0;
            unsigned long long waited = 0;
            for (uint32_t li = 1; li < ex->world; ++li) {
                const uint32_t h = (ex->rank + li) % ex->world;
                uint32_t cnt = 0;
                if (lane == 0) {
                    const unsigned long long w0 = globaltimer();
                    cnt = exchange_wait(a, h, tE, slot, ph);
                    waited += globaltimer() - w0;
                }
                cnt = __shfl_sync(0xffffffffu, cnt, 0);
                const uint32_t* ids = ex->rx_ids[h] + (size_t)slot * ex->cap[h];
                const uint32_t sb = ex->src_base[h];
                // every scanning warp takes a slice of the batch
                for (uint32_t b0 = warp * 32; b0 < cnt; b0 += n_scan * 32) {
                    uint64_t item = 0;
                    if (b0 + lane < cnt) {
                        const uint32_t s = sb + __ldcg(ids + b0 + lane);
                        const uint64_t k1 = __ldg(a.tl_off + s + 1);
                        // the row's tile list is ascending: look at four
                        // segments per round trip
                        for (uint64_t kb = __ldg(a.tl_off + s); kb < k1; kb += 4) {
                            uint32_t tx[4];
#pragma unroll
                            for (uint32_t u = 0; u < 4; ++u) tx[u] = kb + u < k1 ? __ldg(&a.tl[kb + u].x) : 0xffffffffu;
                            uint32_t hit = 4;
#pragma unroll
                            for (uint32_t u = 0; u < 4; ++u)
                                if (hit == 4 && tx[u] == blockIdx.x) hit = u;
                            if (hit < 4) {
                                const uint4 sg = __ldg(a.tl + kb + hit);
                                item = (ldg64(a.off + s) + sg.y) | ((uint64_t)sg.z << 40);
                                add_flops(0, 2ull * sg.z);  // engine.cpp:459-463 (remote: outer)
                                break;
                            }
                            if (tx[3] != 0xffffffffu && tx[3] > blockIdx.x) break;
                        }
                    }
                    const unsigned ball = __ballot_sync(0xffffffffu, item != 0);
                    if (ball) {
                        uint32_t base = 0;
                        if (lane == 0) base = atomicAdd(&s_ravail, (uint32_t)__popc(ball));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (item) items[base + __popc(ball & ((1u << lane) - 1u))] = item;
                    }
                }
            }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) {
                atomicAdd(&s_rdone, 1u);  // the consumers take the peers' items once all warps are done
                if (waited && a.phase_wait) atomicMax(a.phase_wait + ph, waited);
            }
        };
        // deliveries of spike s of S(tA): the FLOP tally of its whole row
        // (engine.cpp:459-463) and, per tile its row touches, a queue item
        // {first entry, length} (one global reservation per (CTA, tile))
        auto tally = [&](uint32_t s) {
            const uint64_t row = ldg64(a.off + a.src_self + s);
            const uint64_t len = ldg64(a.off + a.src_self + s + 1) - row;
            const uint32_t in = __ldg(a.inner + a.src_self + s);
            add_flops(2ull * in, 2ull * (len - in));
            return row;
        };

        if (upd_warp) {
            // ------------------------------------------------ U (update)
            uint32_t* Br = s_pend + (tA & 1u) * 4 * per;  // P(S(tE - 1)), parity tA
            uint32_t vb_n = 0, iou_n = 0;
            float4 j_n, g_n;
            float isyn_n = 0.0f;
            auto grab = [&]() {
                uint32_t c = 0;
                if (lane == 0) c = atomicAdd(&s_fwork, 1u);
                return __shfl_sync(0xffffffffu, c, 0);
            };
            auto load = [&](uint32_t i) {
                vb_n = ldp(a.v + i, pol_f);
                iou_n = __float_as_uint(ldp(iou_rd + i, pol_f));
                if (doE) {
                    j_n = ldp(a.j + i, pol_f);
                    g_n = ldp(a.g + i, pol_f);
                } else {
                    isyn_n = ldp(a.i_syn + i, pol_f);
                }
            };
            // the chunk after next is grabbed early and its state pulled into
            // L1 (no registers held): the next chunk's register loads then
            // wait on L1, not on HBM/L2 — twice the update's bytes in flight
            auto prefetch = [&](uint32_t c) {
                if (!VXB_TILE_L1PF) return;
                const uint32_t k = c_lo + (c << 5) + lane;
                if (c < nch && k < c_hi) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.v + k));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(iou_rd + k));
                    if (doE) {
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.j + k));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.g + k));
                    }
                }
            };
            uint32_t ch = grab();
            uint32_t i = c_lo + (ch << 5) + lane;
            if (ch < nch && i < c_hi) load(i);
            uint32_t ch2 = VXB_TILE_L1PF ? grab() : 0u;
            prefetch(ch2);
            while (ch < nch) {
                const uint32_t vb0 = vb_n;
                const float iou = __uint_as_float(iou_n);
                float4 j = j_n;
                const float4 g = g_n;
                const float isyn_in = isyn_n;
                uint32_t chn;
                if (VXB_TILE_L1PF) {
                    chn = ch2;
                    ch2 = grab();
                    prefetch(ch2);
                } else {
                    chn = grab();
                }
                const uint32_t inext = c_lo + (chn << 5) + lane;
                if (chn < nch && inext < c_hi) load(inext);
                const bool live = i < c_hi;
                bool spiked = false;
                const uint32_t w_lo = c_lo + (ch << 5);
                const uint32_t seg = cur_u.find(startp, nseg, seg_end, w_lo, min(w_lo + 31u, c_hi - 1u),
                                                live ? i : c_hi - 1u, lane);
                uint32_t vb = vb0;
                if (live) {
                    const SegInfo& S = segp[seg];
                    const ParamSet& P = psp[S.pset];
                    const uint32_t l = i - c_lo;
                    const float v = is_refrac(vb) ? P.v_reset : __uint_as_float(vb);
                    float isyn;
                    if (doE) {
                        // gating_kernel (model.hpp:69-71) with deq(P_prev)
                        // (engine.cpp:543-546) from the shared pending tile
                        const float p0 = dequantize_u32(Br[l]);
                        const float p1 = dequantize_u32(Br[per + l]);
                        const float p2 = dequantize_u32(Br[2 * per + l]);
                        const float p3 = dequantize_u32(Br[3 * per + l]);
                        Br[l] = 0u;
                        Br[per + l] = 0u;
                        Br[2 * per + l] = 0u;
                        Br[3 * per + l] = 0u;
                        j.x = fadd(fmul(j.x, P.decay[0]), fmul(P.omega[0], p0));
                        j.y = fadd(fmul(j.y, P.decay[1]), fmul(P.omega[1], p1));
                        j.z = fadd(fmul(j.z, P.decay[2]), fmul(P.omega[2], p2));
                        j.w = fadd(fmul(j.w, P.decay[3]), fmul(P.omega[3], p3));
                        // current_kernel (model.hpp:73-81), u order, from 0.0f
                        float c = 0.0f;
                        c = fadd(c, fmul(fmul(g.x, j.x), fsub(P.e_rev[0], v)));
                        c = fadd(c, fmul(fmul(g.y, j.y), fsub(P.e_rev[1], v)));
                        c = fadd(c, fmul(fmul(g.z, j.z), fsub(P.e_rev[2], v)));
                        c = fadd(c, fmul(fmul(g.w, j.w), fsub(P.e_rev[3], v)));
                        isyn = c;
                        // I_ou(tE) was advanced by phase ph - 1 (N)
                        if (!doA) stp(a.i_syn + i, isyn, pol_f);
                        stp(a.j + i, j, pol_f);
                    } else {
                        isyn = isyn_in;
                    }
                    if (doA) {
                        // membrane_kernel + threshold (engine.cpp:363-385)
                        if (is_refrac(vb)) {
                            const uint32_t r = (vb & 0x007fffffu) - 1u;
                            vb = r ? refrac_bits(r) : __float_as_uint(P.v_reset);
                        } else {
                            float inoise = iou;
                            if (EX && inj_ep) {
                                const float x = __ldg(a.inj_table + (size_t)(inj_ep - 1) * a.n_voxels + S.voxel);
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
                        if (EX && f_hi > f_lo && !spiked) {
                            const uint32_t k = f_lo + lower_bound_u32(a.forced_local + f_lo, f_hi - f_lo, i);
                            if (k < f_hi && __ldg(a.forced_local + k) == i) {
                                spiked = true;
                                vb = P.tref ? refrac_bits(P.tref) : __float_as_uint(P.v_reset);
                            }
                        }
                        stp(a.v + i, vb, pol_f);
                        if (VXB_TILE_FUSE_NOISE) {  // N for this neuron (see the noise lambda)
                            float xi = 0.0f;
                            if (P.sigma_pos)
                                xi = stream_xi(mix_key(a.ou_root, (uint64_t)((int64_t)i + S.gid_off)), tA);
                            stp(iou_wr + i, fadd(fadd(iou, fmul(P.ou_a, fsub(P.ou_mu, iou))), fmul(P.ou_b, xi)),
                                pol_f);
                        }
                    }
                    // probes: V after A(tA), I_syn after E(tE) (engine.cpp:405-406, 564-565)
                    if (EX && a.n_probes) {
                        uint32_t k = lower_bound_u32(a.probe_local, a.n_probes, i);
                        while (k < a.n_probes && __ldg(a.probe_local + k) == i) {
                            const size_t row = (size_t)__ldg(a.probe_slot + k) * a.adv_steps + a.rel0;
                            if (doE) a.probe_i[row + ph - 1] = isyn;
                            if (doA) a.probe_v[row + ph] = is_refrac(vb) ? P.v_reset : __uint_as_float(vb);
                            ++k;
                        }
                    }
                }
                // spike log staging + rates (engine.cpp:400-404), warp aggregated
                bool ovf_route = false;
                const unsigned ball = __ballot_sync(0xffffffffu, spiked);
                if (ball) {
                    unsigned base = 0;
                    if (lane == 0) base = atomicAdd(&s_nspk, (unsigned)__popc(ball));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (spiked) {
                        const unsigned rank = __popc(ball & ((1u << lane) - 1u));
                        if (base + rank < kSpkStage) {
                            s_spk[base + rank] = i;  // bucketed after the update (B)
                        } else {  // staging full: log, route and bucket this spike directly
                            if (!a.ring) a.spk[log_base + atomicAdd(a.seg_end + ph, 1u)] = i;
                            ovf_route = MG;
                            const uint64_t row = tally(i);
                            const uint32_t set = tA & 3u;
                            const uint64_t k1 = __ldg(a.tl_off + a.src_self + i + 1);
                            for (uint64_t k = __ldg(a.tl_off + a.src_self + i); k < k1; ++k) {
                                const uint4 sg = __ldg(a.tl + k);
                                const uint32_t pos = atomicAdd(a.q_cnt + set * G + sg.x, 1u);
                                const uint64_t b = row + sg.y;
                                a.q[(size_t)set * a.q_total + __ldg(a.q_base + sg.x) + pos] =
                                    b | ((uint64_t)sg.z << 40);
                            }
                        }
                        const uint32_t unit = segp[seg].unit;
                        const unsigned peers = __match_any_sync(ball, unit);
                        if ((unsigned)__ffs(peers) - 1u == lane)
                            atomicAdd(&a.rates[(size_t)unit * a.steps + ph], (unsigned)__popc(peers));
                    }
                }
                if (MG && __any_sync(0xffffffffu, ovf_route))
                    if (exchange_route(a, i, ovf_route, tA % kSlots)) __threadfence_system();
                ch = chn;
                i = inext;
            }
            // the CTA's spikes of S(tA) are staged once every update warp is
            // here: the bucketing warps wait for that, the others go on
            const bool bucket_warp = warp >= kTileThreads / 32 - kTileBucketWarps;
            if (bucket_warp)
                named_sync(1, n_upd * 32);
            else
                asm volatile("bar.arrive 1, %0;" ::"r"(n_upd * 32) : "memory");
            if (a.prof && ut == 0) s_t[0] = globaltimer();

            // ------------------------------------------------ B (bucketing)
            // the staged spikes' tile segments: count per tile in shared
            // memory, one global reservation per (CTA, tile), then the items
            const uint32_t bt = threadIdx.x - (kTileThreads - 32 * kTileBucketWarps);
            const uint32_t nbt = 32 * kTileBucketWarps;
            const uint32_t nst = (doA && bucket_warp) ? min(s_nspk, (uint32_t)kSpkStage) : 0u;
            // MG first: the peers' ids of S(tA), P2P stores into their receive
            // slots (engine.cpp:416-437); the CTA that completes the phase's
            // routing count publishes the batch — before the bucketing, so
            // the peers can scan it ~10 us sooner
            if (MG && bucket_warp) {
                bool sent = false;
                const uint32_t nr = (nst + 31u) & ~31u;
                for (uint32_t k = bt; k < nr; k += nbt)
                    sent |= exchange_route(a, k < nst ? s_spk[k] : 0u, k < nst, tA % kSlots);
                (void)sent;
                // one system-scope fence for the CTA: it orders every bucket
                // thread's P2P stores (observed through the barrier) before
                // the routing count
                named_sync(2, nbt);
                if (bt == 0) {
                    __threadfence_system();
                    if (atomicAdd(a.routed + ph, 1u) == G - 1u && doA) {
                        __threadfence();
                        exchange_publish(a, tA);
                    }
                }
            }
            if (nst) {
                const uint32_t set = tA & 3u;
                for (uint32_t k = bt; k < nst; k += nbt) {
                    const uint32_t s = a.src_self + s_spk[k];
                    tally(s_spk[k]);
                    const uint64_t k1 = __ldg(a.tl_off + s + 1);
                    for (uint64_t q = __ldg(a.tl_off + s); q < k1; ++q) atomicAdd(&s_hist[__ldg(&a.tl[q].x)], 1u);
                }
                named_sync(2, nbt);
                if (a.prof && bt == 0) s_t[5] = globaltimer();
                {  // all of this thread's reservations in flight at once
                    constexpr uint32_t R = kTileMaxGrid / (32 * kTileBucketWarps);
                    uint32_t h[R], b[R];
#pragma unroll
                    for (uint32_t r = 0; r < R; ++r) h[r] = bt + r * nbt < G ? s_hist[bt + r * nbt] : 0u;
#pragma unroll
                    for (uint32_t r = 0; r < R; ++r)
                        if (h[r]) b[r] = atomicAdd(a.q_cnt + set * G + bt + r * nbt, h[r]);
#pragma unroll
                    for (uint32_t r = 0; r < R; ++r)
                        if (h[r]) {
                            s_qb[bt + r * nbt] = __ldg(a.q_base + bt + r * nbt) + b[r];
                            s_hist[bt + r * nbt] = 0u;
                        }
                }
                named_sync(2, nbt);
                if (a.prof && bt == 0) s_t[6] = globaltimer();
                uint64_t* qp = a.q + (size_t)set * a.q_total;
                for (uint32_t k = bt; k < nst; k += nbt) {
                    const uint32_t s = a.src_self + s_spk[k];
                    const uint64_t row = ldg64(a.off + s);
                    const uint64_t k1 = __ldg(a.tl_off + s + 1);
                    for (uint64_t q = __ldg(a.tl_off + s); q < k1; ++q) {
                        const uint4 sg = __ldg(a.tl + q);
                        const uint32_t pos = s_qb[sg.x] + atomicAdd(&s_hist[sg.x], 1u);
                        const uint64_t b = row + sg.y;
                        qp[pos] = b | ((uint64_t)sg.z << 40);
                    }
                }
                named_sync(2, nbt);
                if (a.prof && bt == 0) s_t[7] = globaltimer();
                for (uint32_t t = bt; t < G; t += nbt) s_hist[t] = 0u;
            }
            // this CTA's part of S(tA) is queued: count it; the CTA that
            // completes the count posts it to every CTA's mailbox
            if (bucket_warp) {
                named_sync(2, nbt);
                if (bt == 0) {
                    __threadfence();
                    if (MG) __threadfence_system();
                    const uint32_t old = atomicAdd(a.bdone + ph, 1u);
                    if (old == G - 1u) {
                        __threadfence();
                        post_bucketed(ph);
                    }
                }
            }
            if (a.prof && bt == 0) s_t[1] = globaltimer();
            noise();
            if (a.prof && lane == 0) atomicMax(&s_t[3], (unsigned long long)globaltimer());
            consume();
        } else if (warp < n_cons) {
            if (MG && warp < n_scan) scan_remote();
            consume();
            if (a.prof && lane == 0) atomicMax(&s_t[2], (unsigned long long)globaltimer());
            noise();
            if (a.prof && lane == 0) atomicMax(&s_t[3], (unsigned long long)globaltimer());
        } else {  // noise-first warps
            noise();
            if (a.prof && lane == 0) atomicMax(&s_t[3], (unsigned long long)globaltimer());
            consume();
            if (a.prof && lane == 0) atomicMax(&s_t[2], (unsigned long long)globaltimer());
        }

        // phase end (CTA-local): flush the staged spikes into the phase's log
        // segment, recycle the consumed queue set, take the stop decision
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t nst = min(s_nspk, (uint32_t)kSpkStage);
            s_nst = nst;
            s_nspk = 0;
            const unsigned long long now = globaltimer();
            if (a.prof) {
                for (uint32_t k = 0; k < kTileProf; ++k) {
                    a.prof[kTileProf * ((size_t)ph * G + blockIdx.x) + k] = s_t[k];
                    s_t[k] = 0;
                }
            }
            if (doE) a.q_cnt[(tE & 3u) * G + blockIdx.x] = 0u;  // serves S(tE + 4)
            flush_flops();
            if (nst && !a.ring) s_base = atomicAdd(a.seg_end + ph, nst);
            atomicMax(a.phase_ns + ph + 1, now);
            // divergence: every CTA runs through the phase of the earliest
            // diverging step (so the reported neuron is the smallest of that
            // step, as with a barrier), then stops; a peer's timeout or abort
            // stops at once.  A stopping CTA credits the bucketing counts of
            // the phases it skips, so no consumer waits on it.
            const unsigned long long e = atomicAdd(&ctl->err, 0ull);
            bool stop = e != ~0ull && (uint32_t)(e >> 32) <= tA;
            if (MG) stop = stop || atomicAdd(&a.ex->timeout, 0u) != 0u || atomicAdd(&a.ex->peer_abort, 0u) != 0u;
            if (stop) {
                for (uint32_t q = ph + 1; q < nph; ++q)
                    if (atomicAdd(a.bdone + q, 1u) == G - 1u) post_bucketed(q);
                if (MG) exchange_abort(a);
            }
            s_stop = stop ? 1 : 0;
            s_fwork = s_nwork = s_iwork = 0;
            s_ravail = s_rdone = 0;
        }
        __syncthreads();
        const uint32_t nst = s_nst;
        if (nst && !a.ring)
            for (uint32_t k = threadIdx.x; k < nst; k += blockDim.x) a.spk[log_base + s_base + k] = s_spk[k];
        if (s_stop) break;
        if (nst && !a.ring) __syncthreads();  // s_spk is restaged by the next phase
    }
    // the pending tile P(S(t_last)) back to the global buffer of its parity
    {
        const uint32_t tl = a.t0 + a.steps - 1u;
        ulonglong2* gp = reinterpret_cast<ulonglong2*>((tl & 1u) ? a.pend1 : a.pend0);
        const uint32_t* B = s_pend + (tl & 1u) * 4 * per;
        for (uint32_t l = threadIdx.x; l < nt; l += blockDim.x)
            __stcg(gp + c_lo + l,
                   make_ulonglong2((uint64_t)B[l] | ((uint64_t)B[per + l] << 32),
                                   (uint64_t)B[2 * per + l] | ((uint64_t)B[3 * per + l] << 32)));
    }
}

// 8-byte tile entries from the target-sorted out-CSR: the word offset of the
// fast receptor's sum in the pending tile (< 2^16) and both Q16 weights
// (< 2^24 each: checked, else the engine keeps the l2_atomic path).  flag[0]
// is set when an entry does not fit.
// tent == nullptr only checks; tent == w converts in place (each thread reads
// its entry before writing it).
__global__ void tile_entries_kernel(const uint32_t* __restrict__ tgt, const uint64_t* w,
                                    uint64_t n_syn, uint32_t per, uint64_t* tent,
                                    unsigned int* __restrict__ flag) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n_syn;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = tgt[k], tid = t & 0x7fffffffu;
        const uint64_t wq = w[k];
        const uint32_t wf = (uint32_t)wq, ws = (uint32_t)(wq >> 32);
        const uint32_t off = (t >> 31) * 2u * per + tid % per;  // fast receptor's word
        if (wf >= (1u << 24) || ws >= (1u << 24) || off + per >= (1u << 16)) atomicExch(flag, 1u);
        if (tent)
            tent[k] = ((uint64_t)(wf & 0xffffffu) << 40) | ((uint64_t)(ws & 0xffffffu) << 16) |
                      (off & 0xffffu);
    }
}

// ------------------------------------------------------- tile tables (load)
// Per source row (sorted by target): the runs of entries whose targets fall
// in one tile.  Pass 0 counts runs per source; pass 1 writes {tile, first
// entry (row-relative), length}.  One warp per source.
template <int PASS>
__global__ void tile_segments_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tgt,
                                     uint32_t n_src, uint32_t per,
                                     unsigned long long* __restrict__ cnt,   // PASS 0: [n_src]
                                     const unsigned long long* __restrict__ tl_off,  // PASS 1
                                     uint4* __restrict__ tl, uint32_t* __restrict__ tile_cap,
                                     unsigned int* __restrict__ too_long) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t s = warp; s < n_src; s += nwarps) {
        const uint64_t r0 = off[s], r1 = off[s + 1];
        uint32_t runs = 0;
        uint64_t out = PASS ? tl_off[s] : 0ull;
        uint32_t prev_tile = 0xffffffffu;
        for (uint64_t k0 = r0; k0 < r1; k0 += 32) {
            const uint64_t k = k0 + lane;
            const uint32_t t = k < r1 ? (tgt[k] & 0x7fffffffu) / per : 0xffffffffu;
            uint32_t up = __shfl_up_sync(0xffffffffu, t, 1);
            if (lane == 0) up = prev_tile;
            const bool start = k < r1 && t != up;
            const unsigned ball = __ballot_sync(0xffffffffu, start);
            if (PASS == 1 && start) {
                const uint64_t at = out + __popc(ball & ((1u << lane) - 1u));
                tl[at] = make_uint4(t, (uint32_t)(k - r0), 0u, 0u);
                atomicAdd(tile_cap + t, 1u);
            }
            out += __popc(ball);
            runs += __popc(ball);
            prev_tile = __shfl_sync(0xffffffffu, t, 31);
        }
        if (PASS == 0) {
            if (lane == 0) cnt[s] = runs;
        } else {
            __syncwarp();
            const uint64_t b = tl_off[s], e = tl_off[s + 1];
            for (uint64_t q = b + lane; q < e; q += 32) {
                const uint32_t beg = __ldcg(&tl[q].y);
                const uint32_t nxt = q + 1 < e ? __ldcg(&tl[q + 1].y) : (uint32_t)(r1 - r0);
                tl[q].z = nxt - beg;
                if (nxt - beg >= (1u << 24)) atomicExch(too_long, 1u);  // queue items hold 24 bits
            }
        }
    }
}

}  // namespace vxb

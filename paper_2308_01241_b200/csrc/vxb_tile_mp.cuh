// vxb_tile_mp.cuh — the SM-tile path for shards larger than one tile per SM
// (configs 3-5: 5-25M neurons on a GPU).
//
// The shard is cut into T tiles of `per` neurons; tile t belongs to CTA
// t % G (one CTA per SM) and is its pass t / G.  Delivery still runs on the
// SMs' shared-memory reductions, one tile at a time: per phase, for each of
// its passes a CTA adds the segments queued for that tile into its shared
// accumulator, then hands the tile's sums to the global pending buffer of
// parity tE (16 B per neuron, written once) and starts the next pass from
// zero.  The update reads P(S(tE-1)) from the global buffer of parity tA, so
// update and delivery of one phase touch disjoint buffers and run
// concurrently, as on the single-pass path (vxb_tile.cuh).
//
// Phase ph (tA = t0 + ph, tE = tA - 1), per CTA:
//   U  (update warps)    E(tE) + A(tA) over the CTA's neurons (all its tiles);
//                        S(tA) staged, logged, counted.
//   B  (2 update warps)  bucketing of the staged spikes into the destination
//                        tiles' queues of parity tA (one global reservation
//                        per (CTA, tile)); one process per GPU: the P2P routing
//                        of S(tA) to the peers and then R.
//   R  (MG)              the peers' batches of S(tE): CTA c takes ids c, c+G,
//                        ... of every batch and appends each row's tile
//                        segments to the destination tiles' queues (global
//                        atomics); every CTA then bumps ctl->rdone.
//   N  (update warps)    the OU step to tA (noise), by I_ou parity.
//   C  (consumer warps)  for each pass: the tile's items (local at once, the
//                        peers' once every CTA has bumped rdone), streamed into
//                        the shared accumulator; then the copy-out.
//   grid barrier.
// Items are consumed one per warp (long segments, config 2's shape) or one
// per lane (short segments: ~20 entries on the 200-voxel DTI-like networks),
// chosen at load from the mean segment length.
#pragma once

#include "vxb_tile.cuh"

namespace vxb {

constexpr int kMpThreads = 1024;
constexpr uint32_t kMpMaxTiles = 8192;
constexpr uint32_t kMpBucketWarps = 2;  // warps that bucket the peers' batches (R)

// Dynamic shared memory of tile_mp_kernel.
struct MpLayout {
    uint32_t per, tiles;
    uint32_t acc, hist, qb, pset, spk, total;
    __host__ __device__ MpLayout(uint32_t per_, uint32_t tiles_) {
        per = per_;
        tiles = tiles_;
        acc = 0;  // [AMPA, NMDA, GABAA, GABAB][per] (u32)
        hist = (acc + 16 * per + 127) & ~127u;
        qb = hist + 4 * tiles;
        pset = (qb + 4 * tiles + 127) & ~127u;
        spk = pset + kTileMaxPset * (uint32_t)sizeof(ParamSet);
        total = spk + kSpkStage * 4;
    }
};

template <bool MG>
__global__ void __launch_bounds__(kMpThreads, 1) tile_mp_kernel(StepArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t per = a.tile_n, T = a.n_tiles, P = a.passes;
    const MpLayout L(per, T);
    uint32_t* s_acc = reinterpret_cast<uint32_t*>(smem + L.acc);
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem + L.hist);
    uint32_t* s_qb = reinterpret_cast<uint32_t*>(smem + L.qb);
    uint32_t* s_spk = reinterpret_cast<uint32_t*>(smem + L.spk);
    __shared__ uint32_t s_nspk, s_fwork, s_nwork, s_iwork, s_base, s_pass_done;
    __shared__ int s_stop;
    __shared__ unsigned long long s_t[4];

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const uint32_t cpt = per >> 5;            // 32-neuron chunks per tile
    const uint32_t nch = P * cpt;             // chunks over the CTA's tiles
    Control* ctl = a.ctl;
    const uint32_t n_cons = a.n_cons;
    const uint32_t n_upd = kMpThreads / 32 - n_cons;
    const bool upd_warp = warp >= n_cons;
    const uint32_t ut = threadIdx.x - n_cons * 32;  // index among update threads
    const bool bucket_warp = warp >= kMpThreads / 32 - kMpBucketWarps;
    const uint32_t bt = threadIdx.x - (kMpThreads - 32 * kMpBucketWarps);
    const uint32_t nbt = 32 * kMpBucketWarps;

    const ParamSet* psp = a.pset;
    if (threadIdx.x == 0) {
        s_nspk = s_fwork = s_nwork = s_iwork = s_pass_done = 0;
        s_t[0] = s_t[1] = s_t[2] = s_t[3] = 0;
    }
    for (uint32_t k = threadIdx.x; k < T; k += blockDim.x) s_hist[k] = 0;
    for (uint32_t k = threadIdx.x; k < 4 * per; k += blockDim.x) s_acc[k] = 0;
    if (a.npset <= kTileMaxPset) {
        ParamSet* sp = reinterpret_cast<ParamSet*>(smem + L.pset);
        for (uint32_t k = threadIdx.x; k < a.npset; k += blockDim.x) sp[k] = a.pset[k];
        psp = sp;
    }
    __syncthreads();

    const uint64_t pol_syn = policy_evict_first();
    const uint64_t pol_f = a.f_policy == 2 ? policy_evict_last() : policy_evict_normal();
    unsigned long long my_inner = 0, my_outer = 0;
    SegCursorReg cur_u, cur_n;
    // neuron of chunk k of this CTA (tile k / cpt, pass-major)
    auto chunk_base = [&](uint32_t k) { return ((k / cpt) * G + c) * per + (k % cpt) * 32u; };

    if (blockIdx.x == 0 && threadIdx.x == 0) a.phase_ns[0] = globaltimer();
    const uint32_t nph = a.steps + 1;
    for (uint32_t ph = 0; ph < nph; ++ph) {
        const bool doA = ph < a.steps;
        const bool doE = ph >= 1;
        const uint32_t tA = a.t0 + ph;
        const uint32_t tE = tA - 1;
        const uint32_t inj_ep = (doA && a.has_inj) ? a.inj_epoch[ph] : 0u;
        uint32_t f_lo = 0, f_hi = 0;
        if (doA && a.has_forced) {
            f_lo = a.forced_off[ph];
            f_hi = a.forced_off[ph + 1];
        }
        const uint32_t log_base = a.ring ? (ph & 1u) * a.n : 0u;
        const float* iou_rd = (tE & 1u) ? a.i_ou_b : a.i_ou;
        float* iou_wr = (tA & 1u) ? a.i_ou_b : a.i_ou;

        // queue item of one tile segment of spike s (global source) -> tile queue
        auto enqueue = [&](uint32_t par, uint32_t tile, uint64_t item) {
            const uint32_t pos = atomicAdd(a.q_cnt + (size_t)par * T + tile, 1u);
            a.q[(size_t)par * a.q_total + __ldg(a.q_base + tile) + pos] = item;
        };

        if (upd_warp) {
            if (MG && bucket_warp) {
                // ------------------------------------------------ R (peers)
                if (MG && doE) {
                    Exchange* ex = a.ex;
                    const uint32_t par = tE & 1u, slot = tE % kSlots;
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
                        for (uint32_t k = c + (warp - (kMpThreads / 32 - kMpBucketWarps)) * G * 32 + lane * G;
                             k < cnt; k += G * nbt) {
                            const uint32_t s = sb + __ldcg(ids + k);
                            const uint64_t row = ldg64(a.off + s);
                            my_outer += 2ull * (ldg64(a.off + s + 1) - row);
                            const uint64_t k1 = __ldg(a.tl_off + s + 1);
                            for (uint64_t q = __ldg(a.tl_off + s); q < k1; ++q) {
                                const uint4 sg = __ldg(a.tl + q);
                                enqueue(par, sg.x, (row + sg.y) | ((uint64_t)sg.z << 40));
                            }
                        }
                    }
                    __threadfence();
                    named_sync(2, nbt);
                    if (bt == 0) {
                        atomicAdd(&ctl->rdone, 1u);
                        if (waited && a.phase_wait) atomicMax(a.phase_wait + ph, waited);
                    }
                }
            }
            // ------------------------------------------------ U (update)
            const ulonglong2* pr = reinterpret_cast<const ulonglong2*>((tA & 1u) ? a.pend1 : a.pend0);
            uint32_t vb_n = 0, iou_n = 0;
            float4 j_n, g_n;
            ulonglong2 p_n = make_ulonglong2(0ull, 0ull);
            float isyn_n = 0.0f;
            auto grab = [&]() {
                uint32_t x = 0;
                if (lane == 0) x = atomicAdd(&s_fwork, 1u);
                return __shfl_sync(0xffffffffu, x, 0);
            };
            auto load = [&](uint32_t i) {
                vb_n = ldp(a.v + i, pol_f);
                iou_n = __float_as_uint(ldp(iou_rd + i, pol_f));
                if (doE) {
                    j_n = ldp(a.j + i, pol_f);
                    g_n = ldp(a.g + i, pol_f);
                    p_n = ldp_cg(pr + i, pol_f);
                } else {
                    isyn_n = ldp(a.i_syn + i, pol_f);
                }
            };
            uint32_t ch = grab();
            uint32_t i = ch < nch ? chunk_base(ch) + lane : 0u;
            if (ch < nch && i < a.n) load(i);
            while (ch < nch) {
                const uint32_t vb0 = vb_n;
                const float iou = __uint_as_float(iou_n);
                float4 j = j_n;
                const float4 g = g_n;
                const ulonglong2 pq = p_n;
                const float isyn_in = isyn_n;
                const uint32_t chn = grab();
                const uint32_t inext = chn < nch ? chunk_base(chn) + lane : 0u;
                if (chn < nch && inext < a.n) load(inext);
                const uint32_t w_lo = chunk_base(ch);
                const bool live = i < a.n;
                bool spiked = false;
                uint32_t vb = vb0;
                if (w_lo < a.n) {
                    const uint32_t seg = cur_u.find(a.seg_start, a.nseg, a.n, w_lo,
                                                    min(w_lo + 31u, a.n - 1u), live ? i : a.n - 1u, lane);
                    if (live) {
                        const SegInfo S = a.sinfo[seg];
                        const ParamSet& Pp = psp[S.pset];
                        const float v = is_refrac(vb) ? Pp.v_reset : __uint_as_float(vb);
                        float isyn;
                        if (doE) {
                            const float p0 = dequantize((int64_t)(uint32_t)pq.x);
                            const float p1 = dequantize((int64_t)(uint32_t)(pq.x >> 32));
                            const float p2 = dequantize((int64_t)(uint32_t)pq.y);
                            const float p3 = dequantize((int64_t)(uint32_t)(pq.y >> 32));
                            j.x = fadd(fmul(j.x, Pp.decay[0]), fmul(Pp.omega[0], p0));
                            j.y = fadd(fmul(j.y, Pp.decay[1]), fmul(Pp.omega[1], p1));
                            j.z = fadd(fmul(j.z, Pp.decay[2]), fmul(Pp.omega[2], p2));
                            j.w = fadd(fmul(j.w, Pp.decay[3]), fmul(Pp.omega[3], p3));
                            float cc = 0.0f;
                            cc = fadd(cc, fmul(fmul(g.x, j.x), fsub(Pp.e_rev[0], v)));
                            cc = fadd(cc, fmul(fmul(g.y, j.y), fsub(Pp.e_rev[1], v)));
                            cc = fadd(cc, fmul(fmul(g.z, j.z), fsub(Pp.e_rev[2], v)));
                            cc = fadd(cc, fmul(fmul(g.w, j.w), fsub(Pp.e_rev[3], v)));
                            isyn = cc;
                            if (!doA) stp(a.i_syn + i, isyn, pol_f);
                            stp(a.j + i, j, pol_f);
                        } else {
                            isyn = isyn_in;
                        }
                        if (doA) {
                            if (is_refrac(vb)) {
                                const uint32_t r = (vb & 0x007fffffu) - 1u;
                                vb = r ? refrac_bits(r) : __float_as_uint(Pp.v_reset);
                            } else {
                                float inoise = iou;
                                if (inj_ep) {
                                    const float x = __ldg(a.inj_table + (size_t)(inj_ep - 1) * a.n_voxels + S.voxel);
                                    if (x != 0.0f) inoise = fadd(iou, x);
                                }
                                const float nv = fadd(
                                    v, fmul(Pp.dt_over_c,
                                            fadd(fadd(fmul(Pp.g_leak, fsub(Pp.e_leak, v)), isyn), inoise)));
                                if (!isfinite(nv)) {
                                    atomicMin(&ctl->err, ((unsigned long long)tA << 32) | i);
                                    vb = __float_as_uint(nv);
                                } else if (nv >= Pp.v_th) {
                                    spiked = true;
                                    vb = Pp.tref ? refrac_bits(Pp.tref) : __float_as_uint(Pp.v_reset);
                                } else {
                                    vb = __float_as_uint(nv);
                                }
                            }
                            if (f_hi > f_lo && !spiked) {
                                const uint32_t k = f_lo + lower_bound_u32(a.forced_local + f_lo, f_hi - f_lo, i);
                                if (k < f_hi && __ldg(a.forced_local + k) == i) {
                                    spiked = true;
                                    vb = Pp.tref ? refrac_bits(Pp.tref) : __float_as_uint(Pp.v_reset);
                                }
                            }
                            stp(a.v + i, vb, pol_f);
                        }
                        if (a.n_probes) {
                            uint32_t k = lower_bound_u32(a.probe_local, a.n_probes, i);
                            while (k < a.n_probes && __ldg(a.probe_local + k) == i) {
                                const size_t row = (size_t)__ldg(a.probe_slot + k) * a.adv_steps + a.rel0;
                                if (doE) a.probe_i[row + ph - 1] = isyn;
                                if (doA) a.probe_v[row + ph] = is_refrac(vb) ? Pp.v_reset : __uint_as_float(vb);
                                ++k;
                            }
                        }
                    }
                    bool ovf_route = false;
                    const unsigned ball = __ballot_sync(0xffffffffu, spiked);
                    if (ball) {
                        unsigned base = 0;
                        if (lane == 0) base = atomicAdd(&s_nspk, (unsigned)__popc(ball));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (spiked) {
                            const unsigned rank = __popc(ball & ((1u << lane) - 1u));
                            if (base + rank < kSpkStage) {
                                s_spk[base + rank] = i;
                            } else {  // staging full: log, route and bucket this spike directly
                                a.spk[log_base + atomicAdd(&ctl->spk_cursor, 1u)] = i;
                                ovf_route = MG;
                                const uint32_t s = a.src_self + i;
                                const uint64_t row = ldg64(a.off + s);
                                const uint64_t len = ldg64(a.off + s + 1) - row;
                                const uint32_t in = __ldg(a.inner + s);
                                my_inner += 2ull * in;
                                my_outer += 2ull * (len - in);
                                const uint64_t k1 = __ldg(a.tl_off + s + 1);
                                for (uint64_t k = __ldg(a.tl_off + s); k < k1; ++k) {
                                    const uint4 sg = __ldg(a.tl + k);
                                    enqueue(tA & 1u, sg.x, (row + sg.y) | ((uint64_t)sg.z << 40));
                                }
                            }
                            const uint32_t unit = a.sinfo[seg].unit;
                            const unsigned peers = __match_any_sync(ball, unit);
                            if ((unsigned)__ffs(peers) - 1u == lane)
                                atomicAdd(&a.rates[(size_t)unit * a.steps + ph], (unsigned)__popc(peers));
                        }
                    }
                    if (MG && __any_sync(0xffffffffu, ovf_route))
                        if (exchange_route(a, i, ovf_route, tA % kSlots)) __threadfence_system();
                }
                ch = chn;
                i = inext;
            }
            named_sync(1, n_upd * 32);  // the CTA's spikes of S(tA) are staged
            if (a.prof && ut == 0) s_t[0] = globaltimer();
            {
                // ------------------------------------------------ B (bucketing)
                // every update warp: a CTA holds ~1.4k spikes per step on
                // config 3 (45 on config 2)
                const uint32_t bt = ut, nbt = n_upd * 32;
                const uint32_t nst = doA ? min(s_nspk, (uint32_t)kSpkStage) : 0u;
                if (nst) {
                    const uint32_t par = tA & 1u;
                    for (uint32_t k = bt; k < nst; k += nbt) {
                        const uint32_t s = a.src_self + s_spk[k];
                        const uint64_t row = ldg64(a.off + s);
                        const uint64_t len = ldg64(a.off + s + 1) - row;
                        const uint32_t in = __ldg(a.inner + s);
                        my_inner += 2ull * in;
                        my_outer += 2ull * (len - in);
                        const uint64_t k1 = __ldg(a.tl_off + s + 1);
                        for (uint64_t q = __ldg(a.tl_off + s); q < k1; ++q) atomicAdd(&s_hist[__ldg(&a.tl[q].x)], 1u);
                    }
                    named_sync(4, nbt);
                    for (uint32_t t = bt; t < T; t += nbt) {
                        const uint32_t h = s_hist[t];
                        if (h) {
                            s_qb[t] = __ldg(a.q_base + t) + atomicAdd(a.q_cnt + (size_t)par * T + t, h);
                            s_hist[t] = 0u;
                        }
                    }
                    named_sync(4, nbt);
                    uint64_t* qp = a.q + (size_t)par * a.q_total;
                    for (uint32_t k = bt; k < nst; k += nbt) {
                        const uint32_t s = a.src_self + s_spk[k];
                        const uint64_t row = ldg64(a.off + s);
                        const uint64_t k1 = __ldg(a.tl_off + s + 1);
                        for (uint64_t q = __ldg(a.tl_off + s); q < k1; ++q) {
                            const uint4 sg = __ldg(a.tl + q);
                            const uint32_t pos = s_qb[sg.x] + atomicAdd(&s_hist[sg.x], 1u);
                            qp[pos] = (row + sg.y) | ((uint64_t)sg.z << 40);
                        }
                    }
                    named_sync(4, nbt);
                    for (uint32_t t = bt; t < T; t += nbt) s_hist[t] = 0u;
                    if (MG) {
                        bool sent = false;
                        const uint32_t nr = (nst + 31u) & ~31u;
                        for (uint32_t k = bt; k < nr; k += nbt)
                            sent |= exchange_route(a, k < nst ? s_spk[k] : 0u, k < nst, tA % kSlots);
                        if (sent) __threadfence_system();
                    }
                }
            }
            if (a.prof && ut == 0) s_t[1] = globaltimer();
            // ------------------------------------------------ N (OU step)
            if (doA) {
                for (;;) {
                    uint32_t k = 0;
                    if (lane == 0) k = atomicAdd(&s_nwork, 1u);
                    k = __shfl_sync(0xffffffffu, k, 0);
                    if (k >= nch) break;
                    const uint32_t w_lo = chunk_base(k);
                    if (w_lo >= a.n) continue;
                    const uint32_t ii = w_lo + lane;
                    const bool live = ii < a.n;
                    const uint32_t seg = cur_n.find(a.seg_start, a.nseg, a.n, w_lo, min(w_lo + 31u, a.n - 1u),
                                                    live ? ii : a.n - 1u, lane);
                    if (live) {
                        const SegInfo S = a.sinfo[seg];
                        const ParamSet& Pp = psp[S.pset];
                        float iou = ldp(iou_rd + ii, pol_f);
                        float xi = 0.0f;
                        if (Pp.sigma_pos) xi = stream_xi(mix_key(a.ou_root, (uint64_t)((int64_t)ii + S.gid_off)), tA);
                        iou = fadd(fadd(iou, fmul(Pp.ou_a, fsub(Pp.ou_mu, iou))), fmul(Pp.ou_b, xi));
                        stp(iou_wr + ii, iou, pol_f);
                    }
                }
            }
            if (a.prof && lane == 0) atomicMax(&s_t[3], (unsigned long long)globaltimer());
        } else if (doE) {
            // ------------------------------------------------ C (consumers)
            const uint32_t par = tE & 1u;
            const uint32_t bw = smem_u32(s_acc), per4 = 4 * per;
            const uint32_t ct = threadIdx.x, cn = n_cons * 32;
            ulonglong2* gout = reinterpret_cast<ulonglong2*>(par ? a.pend1 : a.pend0);
            for (uint32_t p = 0; p < P; ++p) {
                const uint32_t t = p * G + c;
                if (t >= T) break;
                const uint64_t* items = a.q + (size_t)par * a.q_total + __ldg(a.q_base + t);
                const uint32_t* cntp = a.q_cnt + (size_t)par * T + t;
                // local items are complete (queued before the phase barrier);
                // the peers' are complete once every CTA bumped rdone
                bool final_cnt = !MG;
                uint32_t cnt = __ldcg(cntp);
                for (;;) {
                    uint32_t it = 0;
                    if (lane == 0) it = atomicAdd(&s_iwork, a.item_mode ? 32u : 1u);
                    it = __shfl_sync(0xffffffffu, it, 0);
                    // (MG) a grab that reaches past the items known so far
                    // waits for the peers' items (or for the count to be final)
                    const uint32_t span = a.item_mode ? 32u : 1u;
                    while (it + span > cnt && !final_cnt) {
                        if (ld_acquire(&ctl->rdone) >= G * ph) {
                            final_cnt = true;
                        } else {
                            __nanosleep(200);
                        }
                        cnt = ld_acquire(cntp);
                    }
                    if (it >= cnt) break;
                    if (a.item_mode) {  // one item per lane (short segments)
                        uint64_t d = 0;
                        if (it + lane < cnt) d = __ldcg(reinterpret_cast<const unsigned long long*>(items + it + lane));
                        const uint64_t* ev = a.tent + (d & kItemBeg);
                        const uint32_t len = (uint32_t)(d >> 40);
                        for (uint32_t k = 0; __any_sync(0xffffffffu, k < len); ++k)
                            if (k < len) tile_add(bw, per4, __ldg(reinterpret_cast<const unsigned long long*>(ev + k)));
                    } else {  // one item per warp
                        const uint64_t d = __ldcg(reinterpret_cast<const unsigned long long*>(items + it));
                        const uint64_t* ev = a.tent + (d & kItemBeg) + lane;
                        const uint32_t len = (uint32_t)(d >> 40);
                        uint32_t k0 = 0;
                        for (; k0 + 32 * kTileUnroll <= len; k0 += 32 * kTileUnroll) {
                            uint64_t e[kTileUnroll];
#pragma unroll
                            for (uint32_t u = 0; u < kTileUnroll; ++u) e[u] = ld_stream(ev + k0 + u * 32, pol_syn);
#pragma unroll
                            for (uint32_t u = 0; u < kTileUnroll; ++u) tile_add(bw, per4, e[u]);
                        }
                        for (; k0 < len; k0 += 32)
                            if (k0 + lane < len) tile_add(bw, per4, ld_stream(ev + k0, pol_syn));
                    }
                }
                // every consumer warp is past this pass's items: hand the tile over
                named_sync(3, cn);
                const uint32_t lo = t * per, nt = min(per, a.n - lo);
                for (uint32_t l = ct; l < nt; l += cn) {
                    __stcg(gout + lo + l,
                           make_ulonglong2((uint64_t)s_acc[l] | ((uint64_t)s_acc[per + l] << 32),
                                           (uint64_t)s_acc[2 * per + l] | ((uint64_t)s_acc[3 * per + l] << 32)));
                    s_acc[l] = s_acc[per + l] = s_acc[2 * per + l] = s_acc[3 * per + l] = 0u;
                }
                if (ct == 0) {
                    s_iwork = 0;
                    *const_cast<uint32_t*>(cntp) = 0u;  // serves S(tE + 2)
                }
                named_sync(3, cn);
            }
            if (a.prof && lane == 0) atomicMax(&s_t[2], (unsigned long long)globaltimer());
        }

        // flush the CTA's staged spikes with one log reservation
        __syncthreads();
        if (a.prof && threadIdx.x == 0)
            for (int k = 0; k < 4; ++k) {
                a.prof[4 * ((size_t)ph * G + blockIdx.x) + k] = s_t[k];
                s_t[k] = 0;
            }
        const uint32_t nst = min(s_nspk, (uint32_t)kSpkStage);
        if (threadIdx.x == 0 && nst) s_base = atomicAdd(&ctl->spk_cursor, nst);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < nst; k += blockDim.x) a.spk[log_base + s_base + k] = s_spk[k];

        grid_barrier(
            ctl,
            [&] {
                if (doA) a.seg_end[ph] = ctl->spk_cursor;
                if (a.ring) ctl->spk_cursor = 0;
                a.phase_ns[ph + 1] = globaltimer();
                ctl->stop = (atomicAdd(&ctl->err, 0ull) != ~0ull ||
                             (MG && (atomicAdd(&a.ex->timeout, 0u) != 0u ||
                                     atomicAdd(&a.ex->peer_abort, 0u) != 0u))) ? 1u : 0u;
            },
            [&] {
                if (MG) {
                    if (ctl->stop)
                        exchange_abort(a);
                    else if (doA)
                        exchange_publish(a, tA);
                }
            });
        if (threadIdx.x == 0) {
            s_stop = (int)ld_acquire(&ctl->stop);
            s_nspk = s_fwork = s_nwork = s_iwork = 0;
        }
        __syncthreads();
        if (s_stop) break;
    }
    if (my_inner | my_outer) {
        atomicAdd(&ctl->flops_inner, my_inner);
        atomicAdd(&ctl->flops_outer, my_outer);
    }
}

}  // namespace vxb

// vxb_engine.cu — host side of the B200 simulation step and the C ABI of
// include/vxb.h.
//
// The engine mirrors voxsim::SimInstance (engine.hpp:68-89, engine.cpp):
//   load      (engine.cpp:175-293)  -> Engine::load: validation with the same
//             error kinds/messages, per-segment parameter tables, SoA state
//             upload, out-CSR built on the device (engine.cpp:295-344)
//   advance   (engine.cpp:763-827)  -> Engine::advance: one cooperative
//             persistent kernel per chunk of steps (vxb_kernels.cuh), results
//             read back into RunResult-shaped buffers
//   set_conductances / membrane_snapshot (engine.cpp:829-849)
// All workers of the tables are concatenated on one device ("shard"): worker
// w occupies shard-local indices [wbase[w], wbase[w] + n_w), so the raster's
// (step, worker, local) order is the shard-local order.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include "vxb.h"
#include "vxb_hemo.cuh"
#include "vxb_kernels.cuh"
#include "vxb_netgen.cuh"
#include "vxb_tile.cuh"
#include "vxb_tile_mp.cuh"

namespace {

using namespace vxb;

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SimError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// hemo.cpp:37-40: raised by the BOLD readout; the simulation itself stays usable
struct HemoError : SimError {
    using SimError::SimError;
};

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            throw SimError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" + \
                           #x + ")");                                                  \
    } while (0)

thread_local std::string g_create_error;

// Tuning / diagnostic knobs.  They change the schedule (never the results),
// so they are read only when VXB_TUNING=1 is set, and every knob applied is
// recorded in the engine's schedule report (vxb_schedule_info) — a stray
// value in the environment cannot change a run silently.
const char* knob(const char* name, std::string* log) {
    const char* on = std::getenv("VXB_TUNING");
    if (!on || std::atoi(on) == 0) return nullptr;
    const char* v = std::getenv(name);
    if (v && log) *log += std::string(*log->c_str() ? "," : "") + "\"" + name + "\":\"" + v + "\"";
    return v;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    // Reference-counted allocation: ensemble members view the donor's
    // read-only tables (share), and the memory is freed only when the last
    // engine holding it is destroyed, whatever the destruction order.
    std::shared_ptr<void> mem;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void release() {
        mem.reset();
        p = nullptr;
        n = 0;
    }
    void share(const DevBuf& o) {
        mem = o.mem;
        p = o.p;
        n = o.n;
    }
    void alloc(size_t count) {
        release();
        if (!count) return;
        T* q = nullptr;
        CK(cudaMalloc(&q, count * sizeof(T)));
        mem = std::shared_ptr<void>(q, [](void* x) { cudaFree(x); });
        p = q;
        n = count;
    }
    void reserve(size_t count) {  // grow-only: no free/sync when it already fits
        if (count > n) alloc(count);
    }
    void zero(cudaStream_t s) {
        if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

// Page-locked host staging buffer (grow-only).
template <typename T>
struct HostBuf {
    T* p = nullptr;
    size_t n = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    void reserve(size_t count) {
        if (count <= n) return;
        count = std::max(count, 2 * n);  // geometric growth
        T* q = nullptr;
        CK(cudaMallocHost(&q, count * sizeof(T)));
        if (p) {
            std::memcpy(q, p, n * sizeof(T));
            cudaFreeHost(p);
        }
        p = q;
        n = count;
    }
};

// Copies the prefix of finite, non-negative values of v into dst and
// returns its length (NaN fails both compares; -0.0 passes, as in the
// reference).  Block-wise: each 1024-value block is checked branch-free and
// then copied while it is still in cache, so the caller's buffer is read
// from memory once.  dst == nullptr only validates.
uint32_t copy_valid_prefix(float* dst, const float* v, uint32_t n) {
    for (uint32_t b = 0; b < n; b += 1024) {
        const uint32_t e = std::min(n, b + 1024);
        int bad = 0;
        for (uint32_t i = b; i < e; ++i) {
            const float x = v[i];
            bad |= !((x >= 0.0f) & (x <= 3.402823466e38f));
        }
        uint32_t end = e;
        if (bad)
            for (end = b; end < e; ++end)
                if (!(v[end] >= 0.0f && v[end] <= 3.402823466e38f)) break;
        if (dst) std::memcpy(dst + b, v + b, 4ull * (end - b));
        if (end < e) return end;
    }
    return n;
}

struct Probe {
    uint64_t gid;
    uint32_t local;  // shard-local
};

struct Engine {
    // ---------------------------------------------------------- static
    uint16_t workers = 1;
    uint32_t n_units = 0, n_voxels = 0;
    uint64_t seed = 0;
    double dt_ms = 1.0;
    float dtf = 1.0f;
    bool record_raster = true, record_timings = true;
    uint16_t workers_per_node = 4;
    int device = 0;
    std::vector<vxb_unit> units;
    std::vector<uint16_t> unit_worker;
    std::vector<uint32_t> unit_local_base;
    std::vector<uint32_t> wbase;  // per worker, shard-local base (size workers+1)
    uint32_t n = 0;
    std::vector<SegParams> segs;
    std::vector<uint32_t> seg_start;
    std::vector<Probe> probes;
    uint32_t n_probe_dev = 0;  // probes on this device
    std::vector<std::pair<uint32_t, uint32_t>> forced;  // (abs step, shard-local)
    std::vector<vxb_injection> injections;
    bool packed = true;
    uint64_t n_syn = 0;
    // sharding (one process per GPU): this engine holds worker `rank` of
    // `world`; world == 1 holds every worker of the tables on one device
    uint32_t rank = 0, world = 1;
    uint16_t local_lo = 0, local_hi = 0;  // local worker range
    std::vector<uint32_t> src_base;       // global source index base per worker
    uint32_t n_src = 0;
    int recv_timeout_ms = 30000;
    DevBuf<Exchange> d_ex;
    Exchange h_ex{};
    DevBuf<unsigned char> d_rx;           // receive region (IPC-exported)
    std::vector<size_t> rx_slot_off;      // my region: byte offset of the slot of shard h
    std::vector<void*> peer_base;         // IPC-mapped peer regions
    DevBuf<unsigned long long> d_mask;    // per local neuron: shards with targets
    std::vector<unsigned long long> h_mask;
    std::vector<unsigned long long> have_src;  // per global source: workers holding targets here
    bool use_smem_seg = true;
    uint32_t smem_bytes = 0;
    std::string knobs;  // tuning knobs applied (VXB_TUNING=1), JSON members
    uint32_t ch_max = 1;
    bool early_publish = false;
    // SM-tile path (vxb_tile.cuh): pending sums in shared memory, one CTA per
    // SM; chosen when the shard fits on chip (tile_path), else l2_atomic
    bool tile_path = false;
    uint32_t tile_per = 0, tile_cons = 12, tile_smem = 0, tile_grid = 0;
    uint32_t tile_noisew = 0;  // tile_kernel: warps that start on the OU noise
    bool tile_mp = false;                  // several tiles per SM (tile_mp_kernel)
    // queue sets: tile_kernel rotates four (no grid barrier), tile_mp_kernel two
    uint32_t q_sets() const { return tile_mp ? 2u : kTileQSets; }
    uint32_t tile_T = 0, tile_passes = 1, tile_items = 0;
    uint64_t q_total = 0;
    DevBuf<unsigned long long> d_tl_off;
    DevBuf<uint4> d_tl;
    DevBuf<uint32_t> d_qbase, d_qcnt;
    DevBuf<uint64_t> d_q;
    DevBuf<uint64_t> d_tent;   // 8-byte tile entries (replace tgt / w on this path)
    DevBuf<float> d_iou_b;     // I_ou of odd steps (i_ou holds even steps)
    void setup_tiles();
    void init_tile_state();
    std::string schedule_info() const;

    // ---------------------------------------------------------- device
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int grid = 0;
    DevBuf<ParamSet> d_pset;
    DevBuf<SegInfo> d_sinfo;
    uint32_t npset = 0;
    DevBuf<uint32_t> d_seg_start;
    DevBuf<uint32_t> d_v;
    DevBuf<float4> d_j;
    DevBuf<float> d_iou, d_isyn;
    DevBuf<float4> d_g;
    DevBuf<unsigned char> d_pend0, d_pend1;
    DevBuf<uint64_t> d_off;
    DevBuf<uint32_t> d_inner;
    DevBuf<uint32_t> d_tgt;
    DevBuf<uint64_t> d_w;
    DevBuf<uint32_t> d_spk;
    DevBuf<uint32_t> d_seg_end;
    DevBuf<uint32_t> d_bdone;  // tile_kernel: per phase, CTAs done bucketing
    DevBuf<uint32_t> d_routed;  // tile_kernel (MG): per phase, CTAs done routing
    DevBuf<uint32_t> d_bmail;  // tile_kernel: per CTA (32 words apart), phases bucketed
    DevBuf<uint32_t> d_rates;
    DevBuf<uint32_t> d_probe_local, d_probe_slot;
    DevBuf<float> d_probe_v, d_probe_i;
    DevBuf<uint32_t> d_forced_off, d_forced_local;
    DevBuf<uint32_t> d_inj_epoch;
    DevBuf<float> d_inj_table;
    bool has_forced = false, has_inj = false;  // tables of the current advance
    DevBuf<unsigned long long> d_phase_ns;
    DevBuf<unsigned long long> d_phase_wait;
    DevBuf<unsigned long long> d_arrive;    // [phase][peer] first flag observation (globaltimer)
    double exchange_arrival_ms = 0;         // last advance: sum over phases of the last
                                            // peer's arrival after the phase start
    double exchange_wait_ms = 0;  // last advance: sum over phases of the max CTA wait
    DevBuf<Control> d_ctl;
    DevBuf<uint64_t> d_keys, d_keys_sorted;
    DevBuf<unsigned char> d_cub_tmp;

    // ---------------------------------------------------------- run state
    uint32_t step_done = 0;
    bool failed = false;
    std::string err;

    // last advance
    uint32_t res_steps = 0;
    uint32_t res_start = 0;
    std::vector<uint64_t> raster_keys;  // (rel step << 32 | shard-local), sorted
    // spikes are logged per step (linear log, sorted keys) when the raster or
    // the timing rows' wire-byte counters need them
    bool log_spikes() const { return record_raster || record_timings; }
    std::vector<unsigned long long> dst_full;  // world == 1: full dst mask per shard-local neuron
    std::vector<uint64_t> wire_sent;           // world > 1: [step][dst worker] bytes sent
    std::vector<uint64_t> phase_wait_all;      // per phase of the last advance: max CTA wait (ns)
    std::vector<uint64_t> crossing;            // [src worker][dst worker] synapses held here
    void compute_crossing();
    void account_wire_bytes(uint32_t steps);
    std::vector<uint32_t> rates;        // [unit][steps]
    std::vector<float> probe_v, probe_i;
    vxb_flops flops{};
    uint64_t total_spikes = 0;
    std::vector<vxb_step_timings> timings;
    double device_ms = 0;
    uint64_t h2d = 0, d2h = 0, launches = 0;

    // set_conductances staging (flushed by the next advance): one record per
    // (unit, receptor) = {first staged value, dst float index, count, key}
    HostBuf<float> h_cstage;
    std::vector<uint4> cond_rec;
    std::vector<int32_t> cond_slot;  // [unit * 4 + receptor] -> record, -1 if none
    size_t cond_total = 0;
    DevBuf<float> d_cstage;
    DevBuf<uint4> d_crec;
    uint32_t stage_conductances(uint32_t unit, int receptor, const float* values, uint32_t n);
    int32_t& slot_of(uint32_t unit, int receptor);
    void stage_batch(uint32_t count, const uint32_t* units_, const int32_t* receptors,
                     const float* const* values, const uint32_t* ns, uint32_t* failed);
    void flush_conductances(bool sync);

    // BOLD-proxy readout on the device (vxb_hemo.cuh), enabled by
    // vxb_set_hemodynamics: per-voxel Balloon-Windkessel state carried across
    // advances, BOLD samples of the last advance [sample][voxel]
    bool hemo_on = false;
    HemoParamsDev hemo_p{};
    double hemo_baseline = 1.0;
    uint32_t hemo_every = 1;
    DevBuf<HemoStateDev> d_hemo;
    DevBuf<uint32_t> d_vox_off, d_vox_units;
    DevBuf<double> d_vox_n, d_bold;
    DevBuf<uint32_t> d_vcounts;            // [steps][voxels] of the last advance
    DevBuf<unsigned long long> d_hemo_err;
    std::vector<double> bold;
    std::vector<uint32_t> vcounts;         // voxel counts of the last advance (this rank's units)
    void run_hemo(uint32_t t_base, uint32_t steps);
    bool fetch_bold();                     // false: a voxel's state diverged
    void set_hemodynamics(const vxb_hemo_params& p, double baseline_hz, uint32_t sample_every,
                          const vxb_hemo_state* init);

    ~Engine() {
        for (void* p : peer_base)
            if (p) cudaIpcCloseMemHandle(p);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (stream) cudaStreamDestroy(stream);
    }

    void load(const vxb_network* net, const vxb_options* opt, const vxb_netspec* gen = nullptr,
              uint32_t rank_ = 0, uint32_t world_ = 1);
    void setup_exchange();
    void sort_rows();
    void build_blocks();
    bool rows_sorted = false;
    uint32_t n_blocks = 1, block_n = 0;
    DevBuf<uint32_t> d_blk;
    DevBuf<uint32_t> d_work;  // dynamic delivery chunk counters [2][blocks][world]
    bool dyn = false;
    uint32_t stage_e = 0;     // delivery ring entries per stage
    bool big_pend = false;    // pending buffer of 384 MB+ (few, large L2 blocks)
    uint32_t f_policy = 0;    // neuron-state stream: 0 evict_normal, 1 evict_first, 2 evict_last
    bool local(uint32_t w) const { return w >= local_lo && w < local_hi; }
    void build_csr(const vxb_network* net);
    void generate_csr(const vxb_netspec& spec);
    // ensemble members (assim.cpp's EnsembleMember on one device): the
    // synapse tables are read-only during a run, so members view the donor's
    // out-CSR instead of building their own (12 GB for config 2)
    const Engine* donor = nullptr;
    void share_tables(const Engine& d);
    std::vector<unsigned long long> gen_have_mask;  // dst masks of generated tables
    void advance(uint32_t steps);
    uint32_t advance_begin(uint32_t steps);
    void launch_chunk(uint32_t t0, uint32_t rel0, uint32_t steps, uint32_t adv_steps, int grid_ctas);
    void finish_chunk(uint32_t rel0, uint32_t steps, uint32_t adv_steps);
    void chunk_post(uint32_t rel0, uint32_t cs, std::vector<unsigned long long>& phase_ns_all);
    void advance_end(uint32_t steps, const std::vector<unsigned long long>& phase_ns_all);
    bool prof = false;
    DevBuf<unsigned long long> d_prof;
    uint32_t seg_of(uint32_t local) const {
        return (uint32_t)(std::upper_bound(seg_start.begin(), seg_start.end(), local) -
                          seg_start.begin()) -
               1;
    }
    // layout.cpp:119-128
    const vxb_unit& unit_of_gid(uint64_t gid, uint32_t* uid) const {
        uint64_t total = 0;
        for (const auto& u : units) total = std::max<uint64_t>(total, u.gid_base + u.neurons);
        if (gid >= total || units.empty()) throw SimError("gid out of range");
        size_t lo = 0, hi = units.size();
        while (lo < hi) {
            size_t mid = (lo + hi) / 2;
            if (gid < units[mid].gid_base)
                hi = mid;
            else
                lo = mid + 1;
        }
        size_t i = lo - 1;
        while (units[i].neurons == 0) --i;
        *uid = (uint32_t)i;
        return units[i];
    }
};

std::string fmt(const char* f, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, f);
    vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

// NeuronParams::validate (model.cpp:7-26)
void validate_params(const vxb_neuron& r, float dtf) {
    if (!(r.capacitance > 0)) throw ConfigError("neuron params: capacitance must be > 0");
    if (r.g_leak < 0) throw ConfigError("neuron params: leak conductance must be >= 0");
    if (!(r.v_reset < r.v_threshold))
        throw ConfigError("neuron params: V_reset must be below V_th");
    for (int u = 0; u < 4; ++u) {
        if (!(r.tau[u] > 0)) throw ConfigError("neuron params: receptor tau must be > 0");
        if (!(dtf < r.tau[u]))
            throw ConfigError(
                "neuron params: dt must be below every receptor tau (explicit Euler)");
        if (r.g[u] < 0 || r.omega[u] < 0)
            throw ConfigError(
                "neuron params: receptor conductance and jump weights must be >= 0");
    }
    if (r.e_rev[0] <= r.v_threshold || r.e_rev[1] <= r.v_threshold)
        throw ConfigError("neuron params: excitatory reversals must lie above V_th");
    if (r.e_rev[2] >= r.e_leak || r.e_rev[3] >= r.e_leak)
        throw ConfigError("neuron params: inhibitory reversals must lie below E_L");
}

SegParams make_seg(const vxb_neuron& r, uint32_t start, uint32_t worker, float dtf) {
    SegParams s;
    std::memset(&s, 0, sizeof s);
    s.gid_off = (int64_t)r.gid - (int64_t)start;
    s.start = start;
    s.unit = r.unit;
    s.voxel = r.voxel;
    s.worker = worker;
    s.tref = r.refractory_steps;
    // Host float arithmetic, one rounding per operation, as at the
    // reference's load / kernel sites.
    volatile float c = r.capacitance;
    s.dt_over_c = dtf / c;  // engine.cpp:242
    s.g_leak = r.g_leak;
    s.e_leak = r.e_leak;
    s.v_th = r.v_threshold;
    s.v_reset = r.v_reset;
    for (int u = 0; u < 4; ++u) {
        volatile float q = dtf / r.tau[u];
        s.decay[u] = 1.0f - q;  // gating_kernel: j * (1 - dt / tau)
        s.omega[u] = r.omega[u];
        s.e_rev[u] = r.e_rev[u];
    }
    s.ou_mu = r.ou_mean;
    s.ou_a = dtf / r.ou_tau;  // ou_kernel: (dt / tau)
    volatile float two_dt = 2.0f * dtf;
    volatile float ratio = two_dt / r.ou_tau;
    volatile float sq = std::sqrt((float)ratio);
    s.ou_b = r.ou_sigma * sq;  // sigma * sqrt(2 dt / tau)
    s.sigma_pos = r.ou_sigma > 0 ? 1u : 0u;
    return s;
}

bool same_params(const SegParams& s, const vxb_neuron& r, uint32_t local, uint32_t worker,
                 float dtf) {
    SegParams t = make_seg(r, local, worker, dtf);
    t.start = s.start;
    t.gid_off = (int64_t)r.gid - (int64_t)local;
    return std::memcmp(&s, &t, sizeof s) == 0;
}

void Engine::load(const vxb_network* net, const vxb_options* opt, const vxb_netspec* gen,
                  uint32_t rank_, uint32_t world_) {
    if (!net || !opt) throw ConfigError("null network or options");
    if (net->n_workers == 0) throw ConfigError("no worker tables");
    if (net->n_workers > 64) throw ConfigError("worker counts above 64 are unsupported");
    workers = (uint16_t)net->n_workers;
    rank = rank_;
    world = world_;
    if (world > 1 && world != workers)
        throw ConfigError("distributed engines need one worker per rank");
    if (rank >= world) throw ConfigError("rank out of range");
    local_lo = world > 1 ? (uint16_t)rank : 0;
    local_hi = world > 1 ? (uint16_t)(rank + 1) : workers;
    recv_timeout_ms = opt->recv_timeout_ms;
    n_units = net->n_units;
    n_voxels = net->n_voxels;
    seed = net->workers[0].seed;
    units.assign(net->units, net->units + n_units);
    unit_worker.assign(net->unit_worker, net->unit_worker + n_units);
    unit_local_base.assign(net->unit_local_base, net->unit_local_base + n_units);

    dt_ms = opt->dt_ms;
    if (!(opt->dt_ms > 0.0)) throw ConfigError("dt must be positive");
    if (opt->workers_per_node == 0) throw ConfigError("workers_per_node must be >= 1");
    workers_per_node = opt->workers_per_node;
    const std::string sched = opt->scheduler ? opt->scheduler : "cuda";
    if (sched != "cuda" && sched != "threads" && sched != "loopback")
        throw ConfigError("unknown scheduler: " + sched);
    dtf = (float)opt->dt_ms;
    for (uint32_t k = 0; k < opt->n_injections; ++k) {
        const vxb_injection& inj = opt->injections[k];
        if (inj.voxel >= n_voxels) throw ConfigError("injection voxel out of range");
        if (inj.to_step < inj.from_step) throw ConfigError("injection interval is reversed");
        injections.push_back(inj);
    }
    record_raster = opt->record_raster != 0;
    record_timings = opt->record_timings != 0;

    // shard-local layout and parameter segments
    wbase.assign(workers + 1, 0);
    src_base.assign(workers + 1, 0);
    uint64_t wsum = 0, ssum = 0;  // 64-bit sums, checked before narrowing
    for (uint16_t wi = 0; wi < workers; ++wi) {
        const vxb_worker_table& t = net->workers[wi];
        if (t.worker != wi || t.worker_count != workers)
            throw ConfigError("worker table ids are inconsistent");
        wsum += local(wi) ? t.n_neurons : 0u;
        ssum += t.n_neurons;
        if (ssum >= (1ull << 32))
            throw ConfigError("global neuron ids exceed 32-bit source addressing");
        if (wsum >= (1ull << 31)) throw ConfigError("more than 2^31 neurons on one device");
        wbase[wi + 1] = (uint32_t)wsum;
        src_base[wi + 1] = (uint32_t)ssum;
    }
    n_src = src_base[workers];
    n = wbase[workers];
    std::vector<uint32_t> h_v(n);
    std::vector<float4> h_g(n);
    std::vector<float> h_iou(n);
    std::vector<unsigned long long> h_mask(n);
    for (uint16_t wi = local_lo; wi < local_hi; ++wi) {
        const vxb_worker_table& t = net->workers[wi];
        for (uint32_t i = 0; i < t.n_neurons; ++i) {
            const vxb_neuron& r = t.neurons[i];
            validate_params(r, dtf);
            if (r.unit >= n_units || r.voxel >= n_voxels)
                throw ConfigError("neuron record references unknown unit/voxel");
            if (r.refractory_steps >= (1u << 23))
                throw ConfigError("refractory_steps above 2^23 are unsupported");
            const uint32_t loc = wbase[wi] + i;
            bool extend = !segs.empty() && segs.back().worker == wi &&
                          (int64_t)r.gid - (int64_t)loc == segs.back().gid_off &&
                          same_params(segs.back(), r, loc, wi, dtf);
            if (!extend) {
                segs.push_back(make_seg(r, loc, wi, dtf));
                seg_start.push_back(loc);
            }
            // Non-finite v_init: keep it non-finite but outside the
            // refractory code space, so step 0 diverges like the reference.
            float vi = r.v_init;
            uint32_t bits;
            std::memcpy(&bits, &vi, 4);
            if (!std::isfinite(vi)) bits = 0x7f800000u;
            h_v[loc] = bits;
            h_g[loc] = make_float4(r.g[0], r.g[1], r.g[2], r.g[3]);
            h_iou[loc] = r.ou_mean;  // stationary start (engine.cpp:265)
            h_mask[loc] = r.dst_mask;
        }
    }

    // device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw SimError("no CUDA device available (the cuda scheduler has no CPU fallback)");
    device = opt->device >= 0 ? opt->device : 0;
    if (opt->device < 0) CK(cudaGetDevice(&device));
    if (device >= ndev) throw ConfigError("CUDA device out of range");
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));

    {  // device segment tables: shared parameter sets + per-segment info
        std::vector<ParamSet> ps;
        std::vector<SegInfo> si(segs.size());
        for (size_t k = 0; k < segs.size(); ++k) {
            const SegParams& g = segs[k];
            ParamSet p;
            std::memset(&p, 0, sizeof p);
            p.tref = g.tref;
            p.dt_over_c = g.dt_over_c;
            p.g_leak = g.g_leak;
            p.e_leak = g.e_leak;
            p.v_th = g.v_th;
            p.v_reset = g.v_reset;
            for (int r = 0; r < 4; ++r) {
                p.decay[r] = g.decay[r];
                p.omega[r] = g.omega[r];
                p.e_rev[r] = g.e_rev[r];
            }
            p.ou_mu = g.ou_mu;
            p.ou_a = g.ou_a;
            p.ou_b = g.ou_b;
            p.sigma_pos = g.sigma_pos;
            size_t idx = 0;
            while (idx < ps.size() && std::memcmp(&ps[idx], &p, sizeof p) != 0) ++idx;
            if (idx == ps.size()) ps.push_back(p);
            si[k] = SegInfo{g.gid_off, g.unit, g.voxel, (uint32_t)idx, 0u};
        }
        npset = (uint32_t)ps.size();
        d_pset.alloc(std::max<size_t>(1, ps.size()));
        d_sinfo.alloc(std::max<size_t>(1, si.size()));
        if (!ps.empty())
            CK(cudaMemcpyAsync(d_pset.p, ps.data(), ps.size() * sizeof(ParamSet),
                               cudaMemcpyHostToDevice, stream));
        if (!si.empty())
            CK(cudaMemcpyAsync(d_sinfo.p, si.data(), si.size() * sizeof(SegInfo),
                               cudaMemcpyHostToDevice, stream));
    }
    d_seg_start.alloc(seg_start.size());
    CK(cudaMemcpyAsync(d_seg_start.p, seg_start.data(), seg_start.size() * 4,
                       cudaMemcpyHostToDevice, stream));
    d_v.alloc(n);
    d_j.alloc(n);
    d_iou.alloc(n);
    d_isyn.alloc(n);
    d_g.alloc(n);
    CK(cudaMemcpyAsync(d_v.p, h_v.data(), 4ull * n, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_g.p, h_g.data(), 16ull * n, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_iou.p, h_iou.data(), 4ull * n, cudaMemcpyHostToDevice, stream));
    d_j.zero(stream);
    d_isyn.zero(stream);

    // out-CSR + mask consistency
    if (donor) {
        share_tables(*donor);
    } else if (gen) {
        generate_csr(*gen);  // consistent by construction
    } else {
        build_csr(net);
        if (world == 1) dst_full = h_mask;
        DevBuf<unsigned long long> d_mask, d_bad;
        d_mask.alloc(n);
        d_bad.alloc(1);
        CK(cudaMemcpyAsync(d_mask.p, h_mask.data(), 8ull * n, cudaMemcpyHostToDevice, stream));
        const unsigned long long init = ~0ull;
        CK(cudaMemcpyAsync(d_bad.p, &init, 8, cudaMemcpyHostToDevice, stream));
        // have_mask was left in d_keys by build_csr
        if (n)
            mask_check_kernel<<<1184, 256, 0, stream>>>(
                reinterpret_cast<unsigned long long*>(d_keys.p), d_mask.p, n, d_bad.p);
        CK(cudaGetLastError());
        unsigned long long bad = 0;
        CK(cudaMemcpyAsync(&bad, d_bad.p, 8, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (bad != ~0ull) {
            unsigned long long have = 0;
            CK(cudaMemcpy(&have, reinterpret_cast<unsigned long long*>(d_keys.p) + bad, 8,
                          cudaMemcpyDeviceToHost));
            const uint32_t s = (uint32_t)(std::upper_bound(wbase.begin(), wbase.end(),
                                                           (uint32_t)bad) - wbase.begin()) - 1;
            const uint64_t diff = have ^ h_mask[bad];
            int d = 0;
            while (!((diff >> d) & 1ull)) ++d;
            throw SimError(fmt("destination mask inconsistent with tables (worker %u neuron %u "
                               "-> worker %d)",
                               s, (unsigned)(bad - wbase[s]), d));
        }
    }
    d_keys.release();
    if (donor)
        crossing = donor->crossing;
    else
        compute_crossing();
    if (world == 1 && dst_full.empty() && !have_src.empty())  // generated tables
        dst_full.assign(have_src.begin(), have_src.begin() + n);

    const size_t pend_bytes = (packed ? 16ull : 32ull) * n;
    d_pend0.alloc(pend_bytes);
    d_pend1.alloc(pend_bytes);
    d_pend0.zero(stream);
    d_pend1.zero(stream);
    d_ctl.alloc(1);

    // probes and forced spikes (engine.cpp:276-290)
    for (uint32_t s = 0; s < opt->n_probes; ++s) {
        uint32_t uid;
        const vxb_unit& u = unit_of_gid(opt->probe_gids[s], &uid);
        const uint32_t loc = local(unit_worker[uid])
                                 ? wbase[unit_worker[uid]] + unit_local_base[uid] +
                                       (uint32_t)(opt->probe_gids[s] - u.gid_base)
                                 : UINT32_MAX;  // recorded by the rank that owns it
        probes.push_back({opt->probe_gids[s], loc});
    }
    for (uint32_t f = 0; f < opt->n_forced; ++f) {
        uint32_t uid;
        const vxb_unit& u = unit_of_gid(opt->forced_spikes[f].gid, &uid);
        if (!local(unit_worker[uid])) continue;
        const uint32_t loc = wbase[unit_worker[uid]] + unit_local_base[uid] +
                             (uint32_t)(opt->forced_spikes[f].gid - u.gid_base);
        forced.push_back({opt->forced_spikes[f].step, loc});
    }
    std::sort(forced.begin(), forced.end());
    forced.erase(std::unique(forced.begin(), forced.end()), forced.end());
    n_probe_dev = 0;
    if (!probes.empty()) {
        std::vector<std::pair<uint32_t, uint32_t>> ps;
        for (uint32_t s = 0; s < probes.size(); ++s)
            if (probes[s].local != UINT32_MAX) ps.push_back({probes[s].local, s});
        std::sort(ps.begin(), ps.end());
        std::vector<uint32_t> pl, pslot;
        for (auto& x : ps) {
            pl.push_back(x.first);
            pslot.push_back(x.second);
        }
        n_probe_dev = (uint32_t)pl.size();
        d_probe_local.alloc(std::max<size_t>(1, pl.size()));
        d_probe_slot.alloc(std::max<size_t>(1, pslot.size()));
        CK(cudaMemcpyAsync(d_probe_local.p, pl.data(), 4 * pl.size(), cudaMemcpyHostToDevice,
                           stream));
        CK(cudaMemcpyAsync(d_probe_slot.p, pslot.data(), 4 * pslot.size(),
                           cudaMemcpyHostToDevice, stream));
    }

    // transport (engine.cpp:292, transport.cpp:124-128)
    const std::string tr = opt->transport ? opt->transport : "queue";
    if (tr != "queue" && tr != "nvlink") throw ConfigError("unknown transport: " + tr);

    setup_exchange();
    if (!donor) {
        setup_tiles();
        if (!tile_path) build_blocks();
    }
    if (tile_path) init_tile_state();
    // dynamic chunks win on one device (+8% config 2, config 3 2.0 -> 1.5 s
    // per bio-s), with peers when there is one block (config 2 at 4 GPUs
    // +4%) and with peers over three or more blocks (config 5 at 4 GPUs
    // 3.98 -> 3.71 ms/step, config 3 at 2 GPUs 634 -> 609 us/step); with
    // peers and two blocks of a mid-size shard the static deal is far better
    // (config 3 at 4 GPUs, 80 MB of pending sums: 333 vs 579 us/step), of a
    // big one the dynamic (config 5 at 4 GPUs: 3.50 vs 4.99 ms/step)
    dyn = world == 1 || n_blocks == 1 || n_blocks >= 3 || big_pend;
    if (const char* env = knob("VXB_DYN", &knobs)) dyn = std::atoi(env) != 0;
    // chunks of one local spike on one GPU when a row segment averages >= 512
    // entries (in-degree per L2 block; config 2: 1000), else up to 32
    // (config 3's short L2-block segments: 1.14 ms per step at 32, 1.31 ms at
    // 13, 6.2 at 1; config 2 on 2 GPUs: 2.44e11 events/s at 32, 2.37e11 at 1)
    ch_max = (world == 1 && n && (double)n_syn / n / n_blocks >= 512.0) ? 1u : 32u;
    if (const char* env = knob("VXB_CHMAX", &knobs))  // a chunk is one warp's lanes: <= 32
        ch_max = (uint32_t)std::min(32, std::max(1, std::atoi(env)));
    // publishing S(t) as soon as every CTA has routed it (before the phase's
    // own delivery ends) measured slower: config 2 at 4 GPUs 4.23e11 vs
    // 4.72e11 events/s
    if (const char* ep = knob("VXB_EARLY_PUBLISH", &knobs)) early_publish = std::atoi(ep) != 0;

    // cooperative grid
    use_smem_seg = segs.size() <= (size_t)kMaxSmemSeg && npset <= (uint32_t)kMaxSmemPset;
    // bigger stages for L2-blocked delivery (short block segments per row)
    stage_e = n_blocks > 1 ? 1024u : (uint32_t)kStageE;
    if (const char* env = knob("VXB_STAGE_ENTRIES", &knobs))
        stage_e = (uint32_t)std::max(64, std::atoi(env));
    smem_bytes = SmemLayout(use_smem_seg ? (uint32_t)segs.size() : 0u,
                            use_smem_seg ? npset : 0u, stage_e).total;
    int sms = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const void* kfn = packed ? (const void*)step_kernel<true> : (const void*)step_kernel<false>;
    CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
    if (packed)
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<true>, kThreads,
                                                         smem_bytes));
    else
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<false>, kThreads,
                                                         smem_bytes));
    if (per_sm < 1) throw SimError("step kernel cannot be resident on this device");
    grid = sms * per_sm;
    if (knob("VXB_VERBOSE", nullptr))
        std::fprintf(stderr,
                     "vxb: n=%u n_src=%u syn=%llu segs=%zu psets=%u smem_seg=%d smem=%u B "
                     "grid=%d (%d/SM) blocks=%u packed=%d dyn=%d\n",
                     n, n_src, (unsigned long long)n_syn, segs.size(), npset, (int)use_smem_seg,
                     smem_bytes, grid, per_sm, n_blocks, (int)packed, (int)dyn);
    // L2 residency of the pending buffers: evict_last lines are retained
    // within the persisting carve-out, so size it to the device maximum
    // (VXB_PERSIST=0 leaves the driver default)
    {
        const char* env = knob("VXB_PERSIST", &knobs);
        if (!env || std::atoi(env) != 0) {
            int mx = 0;
            CK(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, device));
            if (mx > 0) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mx));
        }
        // the update's state (v, j, i_ou, g: 40 B/neuron) is kept evict_last
        // too when it fits in L2 beside both pending buffers (config 2: 72 MB,
        // 75.3 -> 74.0 us/step; config 3's 1.4 GB would only thrash: 1.14 ->
        // 1.20 ms); VXB_FPOL = 0/1/2 forces evict_normal / first / last
        int l2 = 0;
        CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
        const uint64_t keep = (uint64_t)n * (40 + 2 * (packed ? 16 : 32));
        f_policy = keep <= (uint64_t)l2 * 3 / 4 ? 2u : 0u;
        if (const char* fp = knob("VXB_FPOL", &knobs)) f_policy = (uint32_t)std::atoi(fp);
    }
    CK(cudaStreamSynchronize(stream));
}

void Engine::build_csr(const vxb_network* net) {
    DevBuf<unsigned long long> cnt;  // counts, then cursors
    cnt.alloc((size_t)n + 1);
    cnt.zero(stream);
    DevBuf<uint32_t> d_wbase, d_wn;
    d_wbase.alloc(workers);
    d_wn.alloc(workers);
    std::vector<uint32_t> wn(workers);
    for (uint16_t w = 0; w < workers; ++w) wn[w] = net->workers[w].n_neurons;
    CK(cudaMemcpyAsync(d_wbase.p, src_base.data(), 4ull * workers, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_wn.p, wn.data(), 4ull * workers, cudaMemcpyHostToDevice, stream));
    DevBuf<unsigned int> flags;  // [0] bad source, [1] needs wide accumulators
    flags.alloc(2);
    flags.zero(stream);

    n_syn = 0;
    for (uint16_t w = 0; w < workers; ++w) n_syn += net->workers[w].n_synapses;
    // stage all in-rows once (16 B / synapse), then count and scatter
    std::vector<std::unique_ptr<DevBuf<SynIn>>> stage(workers);
    std::vector<std::unique_ptr<DevBuf<uint64_t>>> rb(workers);
    for (uint16_t w = 0; w < workers; ++w) {
        const vxb_worker_table& t = net->workers[w];
        stage[w] = std::make_unique<DevBuf<SynIn>>();
        rb[w] = std::make_unique<DevBuf<uint64_t>>();
        stage[w]->alloc(t.n_synapses);
        rb[w]->alloc((size_t)t.n_neurons + 1);
        if (t.n_synapses)
            CK(cudaMemcpyAsync(stage[w]->p, t.synapses, 16ull * t.n_synapses,
                               cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(rb[w]->p, t.row_base, 8ull * (t.n_neurons + 1),
                           cudaMemcpyHostToDevice, stream));
        if (t.n_synapses)
            csr_count_kernel<<<2368, 256, 0, stream>>>(stage[w]->p, t.n_synapses, d_wbase.p,
                                                       d_wn.p, workers, cnt.p + 1, flags.p);
        CK(cudaGetLastError());
    }
    unsigned int bad = 0;
    CK(cudaMemcpyAsync(&bad, flags.p, 4, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (bad) throw SimError("synapse entry references a nonexistent source");

    // exclusive offsets: off[0] = 0, off[i+1] = sum(cnt[0..i])
    d_off.alloc((size_t)n + 1);
    {
        size_t tmp = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt.p + 1,
                                         reinterpret_cast<unsigned long long*>(d_off.p) + 1, n,
                                         stream));
        DevBuf<unsigned char> t;
        t.alloc(tmp ? tmp : 1);
        CK(cub::DeviceScan::InclusiveSum(t.p, tmp, cnt.p + 1,
                                         reinterpret_cast<unsigned long long*>(d_off.p) + 1, n,
                                         stream));
        CK(cudaMemsetAsync(d_off.p, 0, 8, stream));
    }
    CK(cudaMemcpyAsync(cnt.p, d_off.p, 8ull * n, cudaMemcpyDeviceToDevice, stream));
    d_tgt.alloc(n_syn + 4);  // +pad: bulk copies read 16-byte aligned supersets
    d_w.alloc(n_syn + 2);
    d_inner.alloc(n);
    d_inner.zero(stream);
    d_keys.alloc(n);  // reused as have_mask for the consistency check
    d_keys.zero(stream);
    for (uint16_t w = 0; w < workers; ++w) {
        const vxb_worker_table& t = net->workers[w];
        if (t.n_neurons)
            csr_scatter_kernel<<<2368, 256, 0, stream>>>(
                stage[w]->p, rb[w]->p, t.n_neurons, w, wbase[w], d_wbase.p, cnt.p, d_tgt.p,
                d_w.p, reinterpret_cast<unsigned long long*>(d_keys.p), d_inner.p, flags.p + 1);
        CK(cudaGetLastError());
    }
    unsigned int wide = 0;
    CK(cudaMemcpyAsync(&wide, flags.p + 1, 4, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    packed = wide == 0;
}

// ------------------------------------------------------------ generation
// Host half of on-device generation: the per-neuron records of emit_tables
// (netgen.cpp:242-298) with the reference's own libm calls, and the sampling
// tables the device draws from (netgen.cpp:60-100).

double h_stream_u01(uint64_t base, uint64_t k) {
    return (double)(stream_word(base, k) >> 11) * 0x1.0p-53;
}
double h_stream_normal(uint64_t base, uint64_t k) {  // rng.hpp:63-67, glibc
    const double u1 = 1.0 - h_stream_u01(base, 2 * k);
    const double u2 = h_stream_u01(base, 2 * k + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

struct GenHost {
    std::vector<uint32_t> unit_local_base;
    std::vector<std::vector<vxb_neuron>> recs;  // per worker
    std::vector<uint64_t> nsyn;                 // per worker
    std::vector<vxb_worker_table> tables;
    std::vector<GenUnit> gunits;
    std::vector<GenVoxel> gvox;
    std::vector<double> e_cdf, pc;
    std::vector<uint32_t> e_src;
    std::vector<uint64_t> e_nexc;
    vxb_network net{};
    uint64_t total_neurons = 0;
};

// local_worker >= 0: draw the neuron records of that worker only (one
// process per GPU); the other workers contribute their sizes.
void build_gen_host(const vxb_netspec& s, GenHost& h, int local_worker = -1) {
    if (s.n_workers == 0) throw ConfigError("partition with zero workers");
    if (s.n_workers > 64)
        throw ConfigError("worker count exceeds the routing mask limit of 64");
    if (s.n_voxels == 0) throw ConfigError("layout with zero voxels");
    const uint32_t U = s.n_units;
    std::vector<uint32_t> fill(s.n_workers, 0), nunits(s.n_workers, 0);
    h.unit_local_base.assign(U, 0);
    for (uint32_t u = 0; u < U; ++u) {
        const uint16_t w = s.unit_worker[u];
        if (w >= s.n_workers) throw ConfigError("partition worker id out of range");
        h.unit_local_base[u] = fill[w];
        fill[w] += s.units[u].neurons;
        nunits[w] += 1;
    }
    for (uint32_t w = 0; w < s.n_workers; ++w)
        if (nunits[w] == 0)
            throw ConfigError("worker " + std::to_string(w) + " has no units assigned");
    for (uint32_t u = 0; u < U; ++u) h.total_neurons += s.units[u].neurons;
    if (h.total_neurons > 0xffffffffull)
        throw ConfigError("global neuron ids exceed 32-bit source addressing");
    for (uint32_t e = 0; e < s.n_edges; ++e) {
        const vxb_gen_edge& x = s.edges[e];
        if (x.src >= s.n_voxels || x.dst >= s.n_voxels)
            throw ConfigError("edge endpoint out of range");
        if (e && (x.dst < s.edges[e - 1].dst ||
                  (x.dst == s.edges[e - 1].dst && x.src <= s.edges[e - 1].src)))
            throw ConfigError("edges must be sorted by (dst, src), unique");
    }

    // sampling tables
    std::vector<uint64_t> exc_count(s.n_voxels, 0);  // layout.cpp:130-135
    for (uint32_t v = 0; v < s.n_voxels; ++v)
        for (uint32_t u = s.voxels[v].unit_begin; u < s.voxels[v].unit_end; ++u)
            if (s.units[u].excitatory) exc_count[v] += s.units[u].neurons;
    h.gunits.resize(U);
    for (uint32_t u = 0; u < U; ++u) {
        const vxb_unit& x = s.units[u];
        const vxb_gen_population& p = s.unit_pops[u];
        GenUnit& g = h.gunits[u];
        std::memset(&g, 0, sizeof g);
        g.gid_base = x.gid_base;
        g.neurons = x.neurons;
        g.voxel = x.voxel;
        g.worker = s.unit_worker[u];
        g.local_base = h.unit_local_base[u];
        g.exc = x.excitatory ? 1u : 0u;
        g.dual = p.dual_receptor ? 1u : 0u;
        g.split_ratio = p.split_ratio;
        for (int r = 0; r < 4; ++r) {
            g.w_mean[r] = p.weight_mean[r];
            g.w_spread[r] = p.weight_spread[r];
        }
    }
    h.gvox.resize(s.n_voxels);
    uint32_t e = 0;
    for (uint32_t v = 0; v < s.n_voxels; ++v) {
        const vxb_gen_voxel& x = s.voxels[v];
        GenVoxel& g = h.gvox[v];
        std::memset(&g, 0, sizeof g);
        g.k_in = x.k_in;
        g.m = (uint32_t)std::ceil(x.rho * x.k_in - 1e-9);
        g.unit_begin = x.unit_begin;
        g.unit_end = x.unit_end;
        g.e0 = (uint32_t)h.e_cdf.size();
        double acc = 0.0;
        for (; e < s.n_edges && s.edges[e].dst == v; ++e) {
            const double wgt = s.edges[e].weight;
            if (!(wgt >= 0.0)) throw ConfigError("negative categorical weight");
            acc += wgt;
            h.e_cdf.push_back(acc);
            h.e_src.push_back(s.edges[e].src);
            h.e_nexc.push_back(exc_count[s.edges[e].src]);
            if (g.m > 0 && wgt > 0 && exc_count[s.edges[e].src] == 0)
                throw ConfigError("voxel " + std::to_string(s.edges[e].src) +
                                  " has no excitatory neurons but is an in-edge source");
        }
        g.e1 = (uint32_t)h.e_cdf.size();
        g.in_total = acc;
        if (g.m > 0 && !(acc > 0.0))
            throw ConfigError("voxel " + std::to_string(v) +
                              ": rho > 0 but no weighted inter-voxel in-edges");
        const uint32_t pops = x.unit_end - x.unit_begin;
        const uint32_t reg = x.region;
        if (reg >= 4 || s.intra_pops[reg] != pops)
            throw ConfigError("population matrix size does not match region layout");
        g.pc_off = (uint32_t)h.pc.size();
        std::vector<double> totals(pops);
        for (uint32_t tp = 0; tp < pops; ++tp) {
            double a = 0.0;
            for (uint32_t sp = 0; sp < pops; ++sp) {
                const double wgt = s.intra[reg][tp * pops + sp] *
                                   (double)s.units[x.unit_begin + sp].neurons;
                if (!(wgt >= 0.0)) throw ConfigError("negative categorical weight");
                a += wgt;
                h.pc.push_back(a);
            }
            totals[tp] = a;
            if (g.m < g.k_in && !(a > 0.0))
                throw ConfigError("voxel " + std::to_string(v) + " population " +
                                  std::to_string(tp) +
                                  ": intra picks required but matrix row is empty");
        }
        g.pt_off = (uint32_t)h.pc.size();
        h.pc.insert(h.pc.end(), totals.begin(), totals.end());
    }

    // per-neuron records (emit_tables, netgen.cpp:251-298)
    h.recs.assign(s.n_workers, {});
    h.nsyn.assign(s.n_workers, 0);
    for (uint32_t w = 0; w < s.n_workers; ++w) h.recs[w].reserve(fill[w]);
    const uint64_t init_key = mix_key(mix_key(s.seed, 2), 0);  // rngstream::init_state
    for (uint32_t u = 0; u < U; ++u) {
        const vxb_unit& x = s.units[u];
        const vxb_gen_population& p = s.unit_pops[u];
        const uint16_t w = s.unit_worker[u];
        const uint32_t k_in = s.voxels[x.voxel].k_in;
        h.nsyn[w] += (uint64_t)x.neurons * k_in;
        if (local_worker >= 0 && w != (uint32_t)local_worker) continue;
        std::array<uint64_t, 4> gbase;
        for (int r = 0; r < 4; ++r)  // sample_conductances (netgen.cpp:318-329), salt 0
            gbase[r] = mix_key(mix_key(mix_key(mix_key(s.seed, 7), 0), u), (uint64_t)r);
        for (uint32_t j = 0; j < x.neurons; ++j) {
            vxb_neuron r;
            std::memset(&r, 0, sizeof r);
            r.gid = x.gid_base + j;
            r.voxel = x.voxel;
            r.unit = u;
            r.pop = x.pop;
            r.excitatory = x.excitatory;
            r.row_len = k_in;
            r.capacitance = p.capacitance;
            r.g_leak = p.g_leak;
            r.e_leak = p.e_leak;
            r.v_threshold = p.v_threshold;
            r.v_reset = p.v_reset;
            r.refractory_steps = p.refractory_steps;
            for (int q = 0; q < 4; ++q) {
                r.e_rev[q] = p.e_rev[q];
                r.tau[q] = p.tau[q];
                r.omega[q] = p.omega[q];
                r.g[q] = (float)std::exp(p.g_location[q] +
                                         p.g_scale[q] * h_stream_normal(gbase[q], j));
            }
            r.ou_mean = p.ou_mean;
            r.ou_sigma = p.ou_sigma;
            r.ou_tau = p.ou_tau;
            const double u01 = h_stream_u01(init_key, r.gid);
            const float span = p.v_threshold - p.v_reset;  // float subtraction, as the reference
            r.v_init = (float)((double)p.v_reset + u01 * (double)span);
            h.recs[w].push_back(r);
        }
    }
    h.tables.resize(s.n_workers);
    for (uint32_t w = 0; w < s.n_workers; ++w) {
        vxb_worker_table& t = h.tables[w];
        std::memset(&t, 0, sizeof t);
        t.worker = (uint16_t)w;
        t.worker_count = (uint16_t)s.n_workers;
        t.n_neurons = fill[w];
        t.seed = s.seed;
        t.n_synapses = h.nsyn[w];
        t.neurons = h.recs[w].empty() ? nullptr : h.recs[w].data();
    }
    h.net.n_workers = s.n_workers;
    h.net.n_units = U;
    h.net.n_voxels = s.n_voxels;
    h.net.workers = h.tables.data();
    h.net.unit_worker = s.unit_worker;
    h.net.unit_local_base = h.unit_local_base.data();
    h.net.units = s.units;
}

struct GenDevTables {
    DevBuf<GenUnit> units;
    DevBuf<GenVoxel> vox;
    DevBuf<double> e_cdf, pc;
    DevBuf<uint32_t> e_src, wbase;
    DevBuf<uint64_t> e_nexc;
    DevBuf<unsigned int> flags;  // [0] err, [1] wide
    GenDev G{};

    void upload(const GenHost& h, const vxb_netspec& s, const std::vector<uint32_t>& wb,
                cudaStream_t st) {
        auto up = [&](auto& buf, const auto& vec) {
            buf.alloc(std::max<size_t>(1, vec.size()));
            if (!vec.empty())
                CK(cudaMemcpyAsync(buf.p, vec.data(), vec.size() * sizeof(vec[0]),
                                   cudaMemcpyHostToDevice, st));
        };
        up(units, h.gunits);
        up(vox, h.gvox);
        up(e_cdf, h.e_cdf);
        up(pc, h.pc);
        up(e_src, h.e_src);
        up(e_nexc, h.e_nexc);
        up(wbase, wb);
        flags.alloc(2);
        flags.zero(st);
        G.kv_root = mix_key(s.seed, 3);  // rngstream::pick_voxel
        G.kn_root = mix_key(s.seed, 4);  // rngstream::pick_neuron
        G.kp_root = mix_key(s.seed, 5);  // rngstream::pick_pop
        G.kw_root = mix_key(s.seed, 6);  // rngstream::weight
        G.n_units = s.n_units;
        G.units = units.p;
        G.voxels = vox.p;
        G.e_cdf = e_cdf.p;
        G.e_src = e_src.p;
        G.e_nexc = e_nexc.p;
        G.pc = pc.p;
        G.wbase = wbase.p;
        G.err = flags.p;
        G.wide = flags.p + 1;
    }
    void check(cudaStream_t st, unsigned int* wide_out) {
        unsigned int f[2] = {0, 0};
        CK(cudaMemcpyAsync(f, flags.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (f[0])
            throw ConfigError("cannot draw a non-self intra-voxel source (population too small)");
        if (wide_out) *wide_out = f[1];
    }
};

thread_local GenHost* g_gen_host = nullptr;

void Engine::generate_csr(const vxb_netspec& spec) {
    GenHost& h = *g_gen_host;
    GenDevTables T;
    // target units of this device, in shard-local order
    std::vector<std::pair<uint32_t, uint32_t>> tu;  // (shard base, unit)
    for (uint32_t u = 0; u < spec.n_units; ++u)
        if (local(spec.unit_worker[u]) && spec.units[u].neurons)
            tu.push_back({wbase[spec.unit_worker[u]] + h.unit_local_base[u], u});
    std::sort(tu.begin(), tu.end());
    std::vector<uint32_t> t_base, t_unit;
    for (auto& x : tu) {
        t_base.push_back(x.first);
        t_unit.push_back(x.second);
    }
    std::vector<uint32_t> sb(src_base.begin(), src_base.end() - 1);
    T.upload(h, spec, sb, stream);
    DevBuf<uint32_t> d_tb, d_tu;
    d_tb.alloc(std::max<size_t>(1, t_base.size()));
    d_tu.alloc(std::max<size_t>(1, t_unit.size()));
    if (!t_base.empty()) {
        CK(cudaMemcpyAsync(d_tb.p, t_base.data(), 4 * t_base.size(), cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_tu.p, t_unit.data(), 4 * t_unit.size(), cudaMemcpyHostToDevice, stream));
    }
    T.G.t_base = d_tb.p;
    T.G.t_unit = d_tu.p;
    T.G.n_t = (uint32_t)t_base.size();
    n_syn = 0;
    for (uint32_t w = local_lo; w < local_hi; ++w) n_syn += h.nsyn[w];
    DevBuf<unsigned long long> cnt;
    cnt.alloc((size_t)n_src + 1);
    cnt.zero(stream);
    const int blocks = 148 * 8, threads = 256;
    if (n)
        gen_kernel<0><<<blocks, threads, 0, stream>>>(T.G, 0, n, cnt.p + 1, nullptr, nullptr,
                                                      nullptr, nullptr, 0, nullptr, nullptr);
    CK(cudaGetLastError());
    T.check(stream, nullptr);
    d_off.alloc((size_t)n_src + 1);
    {
        size_t tmp = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt.p + 1,
                                         reinterpret_cast<unsigned long long*>(d_off.p) + 1, n_src,
                                         stream));
        DevBuf<unsigned char> t;
        t.alloc(tmp ? tmp : 1);
        CK(cub::DeviceScan::InclusiveSum(t.p, tmp, cnt.p + 1,
                                         reinterpret_cast<unsigned long long*>(d_off.p) + 1, n_src,
                                         stream));
        CK(cudaMemsetAsync(d_off.p, 0, 8, stream));
    }
    CK(cudaMemcpyAsync(cnt.p, d_off.p, 8ull * n_src, cudaMemcpyDeviceToDevice, stream));
    d_tgt.alloc(n_syn + 4);
    d_w.alloc(n_syn + 2);
    d_inner.alloc(std::max<uint32_t>(1, n_src));
    d_inner.zero(stream);
    d_keys.alloc(std::max<uint32_t>(1, n_src));  // have_mask per global source
    d_keys.zero(stream);
    if (n)
        gen_kernel<1><<<blocks, threads, 0, stream>>>(
            T.G, 0, n, cnt.p, d_tgt.p, d_w.p, reinterpret_cast<unsigned long long*>(d_keys.p),
            d_inner.p, 0, nullptr, nullptr);
    CK(cudaGetLastError());
    unsigned int wide = 0;
    T.check(stream, &wide);
    packed = wide == 0;
    have_src.assign(n_src, 0);
    if (n_src)
        CK(cudaMemcpyAsync(have_src.data(), d_keys.p, 8ull * n_src, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
}

// A member engine views the donor's out-CSR, L2-block offsets and tallies;
// its own load() built the neuron state from the same network, so only the
// table sizes need to agree.
void Engine::share_tables(const Engine& d) {
    if (d.world != 1 || world != 1) throw ConfigError("ensemble members need a one-GPU donor");
    if (d.device != device) throw ConfigError("ensemble members must run on the donor's device");
    if (d.n != n || d.n_src != n_src || d.workers != workers || d.n_units != n_units)
        throw ConfigError("ensemble member network does not match the donor's");
    n_syn = d.n_syn;
    packed = d.packed;
    have_src = d.have_src;
    d_off.share(d.d_off);
    d_inner.share(d.d_inner);
    d_tgt.share(d.d_tgt);
    d_w.share(d.d_w);
    d_blk.share(d.d_blk);
    rows_sorted = d.rows_sorted;
    n_blocks = d.n_blocks;
    block_n = d.block_n;
    tile_path = d.tile_path;
    tile_per = d.tile_per;
    tile_cons = d.tile_cons;
    tile_noisew = d.tile_noisew;
    tile_mp = d.tile_mp;
    tile_T = d.tile_T;
    tile_passes = d.tile_passes;
    tile_items = d.tile_items;
    tile_smem = d.tile_smem;
    tile_grid = d.tile_grid;
    q_total = d.q_total;
    d_tl_off.share(d.d_tl_off);
    d_tl.share(d.d_tl);
    d_qbase.share(d.d_qbase);
    d_tent.share(d.d_tent);
}

// Exchange state: receive region (one slot per peer: ids[kSlots][n_h],
// counts[kSlots], flag), per-neuron destination masks, device control block.
void Engine::setup_exchange() {
    std::memset(&h_ex, 0, sizeof h_ex);
    h_ex.rank = rank;
    h_ex.world = world;
    h_ex.cap_self = world > 1 ? src_base[rank + 1] - src_base[rank] : 0;
    h_ex.timeout_ns = recv_timeout_ms > 0 ? (unsigned long long)recv_timeout_ms * 1000000ull : 0;
    for (uint32_t w = 0; w <= workers && w <= (uint32_t)kMaxShards; ++w)
        h_ex.src_base[w] = world > 1 ? src_base[w] : 0u;
    if (world > 1) {
        rx_slot_off.assign(world, 0);
        size_t off = 0;
        for (uint32_t hh = 0; hh < world; ++hh) {
            h_ex.cap[hh] = src_base[hh + 1] - src_base[hh];
            rx_slot_off[hh] = off;
            if (hh != rank) off += ((4ull * kSlots * h_ex.cap[hh] + 15) & ~15ull) + 32;
        }
        d_rx.alloc(std::max<size_t>(16, off));
        d_rx.zero(stream);
        for (uint32_t hh = 0; hh < world; ++hh) {
            if (hh == rank) continue;
            unsigned char* b = d_rx.p + rx_slot_off[hh];
            h_ex.rx_ids[hh] = reinterpret_cast<uint32_t*>(b);
            h_ex.rx_meta[hh] = reinterpret_cast<uint32_t*>(b + ((4ull * kSlots * h_ex.cap[hh] + 15) & ~15ull));
        }
        peer_base.assign(world, nullptr);
    }
    // own bit: local neurons with targets on this rank
    h_mask.assign(n, 0);
    if (!have_src.empty())
        for (uint32_t i = 0; i < n; ++i)
            h_mask[i] = have_src[src_base[local_lo] + i] ? (1ull << rank) : 0ull;
    d_mask.alloc(std::max<uint32_t>(1, n));
    d_mask.zero(stream);
    if (n) CK(cudaMemcpyAsync(d_mask.p, h_mask.data(), 8ull * n, cudaMemcpyHostToDevice, stream));
    d_ex.alloc(1);
    CK(cudaMemcpyAsync(d_ex.p, &h_ex, sizeof h_ex, cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));
}

// Sort every out-row by target (low bits only: the class bit rides along).
// Rows are sorted in slices of <= 2^28 entries through slice-sized scratch
// buffers, so the sort needs ~3 GB extra HBM whatever the table size.
void Engine::sort_rows() {
    if (rows_sorted || n_syn == 0) return;
    int end_bit = 1;
    while ((1ull << end_bit) < n) ++end_bit;
    std::vector<uint64_t> hoff((size_t)n_src + 1);
    CK(cudaMemcpyAsync(hoff.data(), d_off.p, 8ull * (n_src + 1), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    const uint64_t kSlice = 1ull << 28;
    uint64_t biggest = 0;
    for (uint32_t s0 = 0; s0 < n_src;) {  // slice bounds
        uint32_t s1 = s0;
        while (s1 < n_src && hoff[s1 + 1] - hoff[s0] <= kSlice) ++s1;
        if (s1 == s0) s1 = s0 + 1;
        biggest = std::max(biggest, hoff[s1] - hoff[s0]);
        s0 = s1;
    }
    DevBuf<uint32_t> t2;
    DevBuf<uint64_t> w2;
    DevBuf<unsigned long long> rel;
    DevBuf<unsigned char> tmpbuf;
    t2.alloc(std::max<uint64_t>(1, biggest));
    w2.alloc(std::max<uint64_t>(1, biggest));
    for (uint32_t s0 = 0; s0 < n_src;) {
        uint32_t s1 = s0;
        while (s1 < n_src && hoff[s1 + 1] - hoff[s0] <= kSlice) ++s1;
        if (s1 == s0) s1 = s0 + 1;
        const uint64_t base = hoff[s0];
        const uint64_t items = hoff[s1] - base;
        if (items > 1) {
            if (items >= (1ull << 31)) throw SimError("a single out-row exceeds 2^31 entries");
            std::vector<unsigned long long> hr(s1 - s0 + 1);
            for (uint32_t i = s0; i <= s1; ++i) hr[i - s0] = hoff[i] - base;
            if (rel.n < hr.size()) rel.alloc(hr.size());
            CK(cudaMemcpyAsync(rel.p, hr.data(), 8 * hr.size(), cudaMemcpyHostToDevice, stream));
            size_t tmp = 0;
            CK(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp, d_tgt.p + base, t2.p,
                                                        d_w.p + base, w2.p, (int)items,
                                                        (int)(s1 - s0), rel.p, rel.p + 1, 0,
                                                        end_bit, stream));
            if (tmpbuf.n < tmp) tmpbuf.alloc(tmp);
            CK(cub::DeviceSegmentedRadixSort::SortPairs(tmpbuf.p, tmp, d_tgt.p + base, t2.p,
                                                        d_w.p + base, w2.p, (int)items,
                                                        (int)(s1 - s0), rel.p, rel.p + 1, 0,
                                                        end_bit, stream));
            CK(cudaMemcpyAsync(d_tgt.p + base, t2.p, 4 * items, cudaMemcpyDeviceToDevice, stream));
            CK(cudaMemcpyAsync(d_w.p + base, w2.p, 8 * items, cudaMemcpyDeviceToDevice, stream));
            CK(cudaStreamSynchronize(stream));  // rel / scratch reused by the next slice
        }
        s0 = s1;
    }
    rows_sorted = true;
}

constexpr uint32_t kTileMinNeurons = 400000;

// SM-tile path: every CTA (one per SM) owns a contiguous tile of neurons and
// keeps their pending sums in shared memory (vxb_tile.cuh).  Eligible when
// both parities of the pending tile fit in a CTA's shared memory (shards up
// to ~1M neurons on 148 SMs) with carry-free packed sums; with one process
// per GPU the peers' spikes are delivered by every CTA from the received
// batches.  Rows are sorted by target and cut into per-tile segments here,
// once.
void Engine::setup_tiles() {
    tile_path = false;
    const char* force = knob("VXB_PATH", &knobs);
    if (force && std::string(force) == "l2") return;
    if (!packed || n == 0) return;
    // small shards stay on the l2_atomic path: the tile kernel's per-phase
    // fixed costs (bucketing round trips, per-tile queues) dominate there
    // (config-2 shape, 100k neurons: l2 17 vs tile 24 us/step; 1M neurons:
    // tile 53.5 vs l2 72)
    const bool force_tile = force && (std::string(force) == "tile" || std::string(force) == "mp");
    if (!force_tile && n < kTileMinNeurons) return;
    int sms = 0, optin = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    // consumer warps at the start of a phase: 12 on one GPU (8 / 10: 44.0 /
    // 43.4 vs 42.9 us/step); 6 with peers, where the consumers also scan the
    // peers' batches and more update and bucketing throughput pays (config 2
    // at 4 GPUs: 6 / 8 / 12 / 16 -> 7.92 / 7.80 / 7.44 / 7.02e11 events/s)
    tile_cons = world > 1 ? 6u : 12u;
    if (const char* c = knob("VXB_TILE_CONS", &knobs))
        tile_cons = (uint32_t)std::min(20, std::max(1, std::atoi(c)));
    if (const char* c = knob("VXB_TILE_NOISEW", &knobs))
        tile_noisew = (uint32_t)std::min(8, std::max(0, std::atoi(c)));
    cudaFuncAttributes fa1, fa2;
    CK(cudaFuncGetAttributes(&fa1, (const void*)tile_kernel<true, true>));
    CK(cudaFuncGetAttributes(&fa2, (const void*)tile_mp_kernel<true>));
    // one tile per SM (both pending parities in shared memory) when it fits,
    // else several tiles per SM, one shared accumulator (tile_mp_kernel)
    uint32_t per = (uint32_t)((((uint64_t)n + sms - 1) / sms + 31) & ~31ull);
    bool mp = TileLayout(per).total + fa1.sharedSizeBytes > (size_t)optin;
    // several tiles per SM only on request (VXB_PATH=mp / tile, VXB_TILE_PER):
    // measured slower than the L2-blocked l2_atomic path at every shard size
    // that does not fit one tile per SM (config-2 shape 2M neurons: 214 vs
    // 143 us/step, 4M: 404 vs 325; config 3 20M: 2.04 vs 1.13 ms/step).  The
    // K targets of a spike spread over thousands of tiles, so a tile segment
    // averages < 1 entry and every event pays a queue item on top of its
    // entry
    if (mp && !force_tile && !knob("VXB_TILE_PER", nullptr)) return;
    if (force && std::string(force) == "mp") mp = true;
    if (const char* c = knob("VXB_TILE_PER", &knobs)) {  // force several tiles per SM
        per = std::max<uint32_t>(32, (uint32_t)std::atoi(c) & ~31u);
        mp = true;
    }
    // several tiles per SM: one GPU only.  With peers, a consumer could read a
    // queue slot a peer-batch bucketing CTA had reserved but not yet written
    // (intermittent mismatches at 2 GPUs); the path is opt-in and slower than
    // the l2 path, so multi-GPU shards that do not fit one tile per SM take
    // the l2 path
    if (mp && world > 1) return;
    uint32_t T = sms, smem = 0;
    if (mp) {
        if (!knob("VXB_TILE_PER", nullptr)) per = 8192;
        T = (uint32_t)((n + per - 1) / per);
        if (T > kMpMaxTiles || 4u * per > 65536u) return;
        smem = MpLayout(per, T).total;
        if (smem + fa2.sharedSizeBytes > (size_t)optin) return;
        for (const void* tk : {(const void*)tile_mp_kernel<false>, (const void*)tile_mp_kernel<true>})
            CK(cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_mp_kernel<true>, kMpThreads, smem));
        if (per_sm < 1) return;
    } else {
        smem = TileLayout(per).total;
        for (const void* tk : {(const void*)tile_kernel<false, false>, (const void*)tile_kernel<false, true>,
                               (const void*)tile_kernel<true, false>, (const void*)tile_kernel<true, true>})
            CK(cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_kernel<true, true>, kTileThreads, smem));
        if (per_sm < 1) return;
    }
    // the 8-byte entries need 24-bit weights: check before touching the tables
    {
        DevBuf<unsigned int> flag;
        flag.alloc(1);
        flag.zero(stream);
        if (n_syn)
            tile_entries_kernel<<<1184, 256, 0, stream>>>(d_tgt.p, d_w.p, n_syn, per, nullptr, flag.p);
        CK(cudaGetLastError());
        unsigned int bad = 0;
        CK(cudaMemcpyAsync(&bad, flag.p, 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (bad) return;
    }
    sort_rows();
    // tile segments of every row: count, scan, write
    DevBuf<unsigned long long> cnt;
    cnt.alloc((size_t)n_src + 1);
    cnt.zero(stream);
    tile_segments_kernel<0><<<1184, 256, 0, stream>>>(reinterpret_cast<const uint64_t*>(d_off.p),
                                                       d_tgt.p, n_src, per, cnt.p + 1, nullptr,
                                                       nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
    d_tl_off.alloc((size_t)n_src + 1);
    {
        size_t tmp = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt.p + 1, d_tl_off.p + 1, n_src, stream));
        DevBuf<unsigned char> t;
        t.alloc(tmp ? tmp : 1);
        CK(cub::DeviceScan::InclusiveSum(t.p, tmp, cnt.p + 1, d_tl_off.p + 1, n_src, stream));
        CK(cudaMemsetAsync(d_tl_off.p, 0, 8, stream));
    }
    unsigned long long total = 0;
    CK(cudaMemcpyAsync(&total, d_tl_off.p + n_src, 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    cnt.release();
    if (total >= (1ull << 32) || n_syn >= (1ull << 40)) {  // queue items: 32-bit slots, 40-bit entries
        d_tl_off.release();
        return;
    }
    d_tl.alloc(std::max<unsigned long long>(1, total));
    DevBuf<uint32_t> cap;
    cap.alloc(T + 1);  // [T]: a segment too long for a queue item
    cap.zero(stream);
    tile_segments_kernel<1><<<1184, 256, 0, stream>>>(reinterpret_cast<const uint64_t*>(d_off.p),
                                                       d_tgt.p, n_src, per, nullptr, d_tl_off.p,
                                                       d_tl.p, cap.p, cap.p + T);
    CK(cudaGetLastError());
    std::vector<uint32_t> hcap(T + 1), qb(T + 1, 0);
    CK(cudaMemcpyAsync(hcap.data(), cap.p, 4ull * (T + 1), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (hcap[T]) {  // keep the l2_atomic path
        d_tl.release();
        d_tl_off.release();
        return;
    }
    for (uint32_t t = 0; t < T; ++t) qb[t + 1] = qb[t] + hcap[t];
    q_total = total;
    d_qbase.alloc(T + 1);
    CK(cudaMemcpyAsync(d_qbase.p, qb.data(), 4ull * (T + 1), cudaMemcpyHostToDevice, stream));
    d_q.alloc(std::max<uint64_t>(1, (mp ? 2ull : kTileQSets) * total));
    d_qcnt.alloc((mp ? 2ull : kTileQSets) * T);
    d_qcnt.zero(stream);
    // 8-byte entries (accumulator word offset + both weights), written over
    // the 8-byte weight array: 2/3 of the 12-byte stream, no extra memory
    if (n_syn)
        tile_entries_kernel<<<1184, 256, 0, stream>>>(d_tgt.p, d_w.p, n_syn, per, d_w.p, cap.p + T);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream));
    d_tent.share(d_w);
    d_w.release();
    d_tgt.release();  // the tile path reads only the 8-byte entries
    tile_path = true;
    tile_mp = mp;
    tile_per = per;
    tile_T = T;
    tile_passes = mp ? (T + sms - 1) / sms : 1u;
    tile_smem = smem;
    tile_grid = (uint32_t)sms;
    // short segments (the DTI-like networks' ~20 entries) are consumed one
    // queue item per lane, long ones (config 2: ~200) one per warp
    tile_items = total && n_syn / total < 64 ? 1u : 0u;
    if (const char* c = knob("VXB_TILE_ITEMS", &knobs)) tile_items = std::atoi(c) ? 1u : 0u;
}

// crossing_matrix (netgen.cpp:331-355, BuiltNetwork::crossing): synapses
// per (source worker, target worker) of the tables on this device; with one
// worker per rank only the rank's own column is nonzero (the caller sums the
// ranks' matrices).
void Engine::compute_crossing() {
    crossing.assign((size_t)workers * workers, 0);
    if (n_syn == 0) return;
    DevBuf<uint32_t> sb, wb;
    DevBuf<unsigned long long> out;
    sb.alloc(workers + 1);
    wb.alloc(workers + 1);
    out.alloc((size_t)workers * workers);
    out.zero(stream);
    CK(cudaMemcpyAsync(sb.p, src_base.data(), 4ull * (workers + 1), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(wb.p, wbase.data(), 4ull * (workers + 1), cudaMemcpyHostToDevice, stream));
    crossing_kernel<<<1184, 256, 0, stream>>>(reinterpret_cast<const uint64_t*>(d_off.p), d_tgt.p,
                                              n_src, sb.p, wb.p, workers, out.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(crossing.data(), out.p, 8 * crossing.size(), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
}

// Per-instance state of the tile path: I_ou is kept by step parity (the
// noise warps write I_ou(t+1) while the update reads I_ou(t)); the state
// after step t-1 lives in the parity (t-1) & 1 buffer — at load, odd.
void Engine::init_tile_state() {
    d_iou_b.alloc(std::max<uint32_t>(1, n));
    if (n) CK(cudaMemcpyAsync(d_iou_b.p, d_iou.p, 4ull * n, cudaMemcpyDeviceToDevice, stream));
    d_q.reserve(std::max<uint64_t>(1, (uint64_t)q_sets() * q_total));
    d_q.zero(stream);  // tile_kernel: an empty slot reads 0 until its item is written
    d_qcnt.reserve((size_t)q_sets() * tile_T);
    d_qcnt.zero(stream);
    CK(cudaStreamSynchronize(stream));
}

// L2-blocked delivery: when the pending buffer does not fit in L2, targets
// are split into ranges whose pending slice does (64 MB: measured optimum on
// config 3 between L2 misses and producer passes; 48 MB before the
// warp-parallel producer), rows are sorted by
// target and every CTA delivers block 0's segments of all its spikes, then
// block 1's, ... so the live part of the pending buffer stays L2-resident
// (VXB_BLOCK_NEURONS overrides the block size).
void Engine::build_blocks() {
    n_blocks = 1;
    dyn = false;
    const uint64_t pend_per = packed ? 16 : 32;
    // every rank delivers in the same number of block passes (a rank with one
    // pass more sets the pace of the whole exchange): count from the largest shard
    uint64_t n_ref = n;
    if (world > 1)
        for (uint32_t w = 0; w < workers; ++w)
            n_ref = std::max<uint64_t>(n_ref, src_base[w + 1] - src_base[w]);
    // 64 MB blocks; once 64 MB would take 6+ passes, three passes on one GPU
    // and two with peers (whose spikes every pass walks too): each spike's
    // per-block row lookup then outweighs the L2 misses of the larger block
    // (config 5, 25M neurons per GPU at 15 Hz, 400 MB of pending sums: 1 GPU
    // 5 / 3 / 2 passes 2.37 / 2.09 / 2.50 ms/step; 4 GPUs 5 / 4 / 3 / 2 / 1
    // passes 5.17 / 4.06 / 3.69 / 3.50 / 4.20 ms with the dynamic deal from 3
    // passes on); config 3's 320 MB on one GPU stays fastest at 64 MB: 1.12
    // vs 1.31 ms at 3 passes)
    const uint64_t pend_ref = n_ref * pend_per;
    uint64_t mb = 64;
    big_pend = (pend_ref + (64ull << 20) - 1) / (64ull << 20) >= 6;
    if (big_pend) {
        const uint64_t passes = world > 1 ? 2 : 3;
        mb = ((pend_ref + passes * (1ull << 20) - 1) / passes) >> 20;
    }
    if (const char* env = knob("VXB_BLOCK_MB", &knobs)) mb = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10));
    uint64_t bn = (mb << 20) / pend_per;
    if (const char* env = knob("VXB_BLOCK_NEURONS", &knobs)) bn = std::max<uint64_t>(1024, std::strtoull(env, nullptr, 10));
    if (n_ref <= bn || n_syn == 0) return;
    n_blocks = (uint32_t)((n_ref + bn - 1) / bn);
    block_n = (uint32_t)((n + n_blocks - 1) / n_blocks);
    sort_rows();
    d_blk.alloc((size_t)n_src * (n_blocks + 1));
    block_offsets_kernel<<<1184, 256, 0, stream>>>(reinterpret_cast<const uint64_t*>(d_off.p),
                                                   d_tgt.p, n_src, n_blocks, block_n, d_blk.p);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream));
}

// HemoParams::validate (hemo.cpp:8-17), validate_assim's baseline check
// (assim.cpp:47) and bold_from_drive's sampling check (hemo.cpp:52-53).
void validate_hemo(const vxb_hemo_params& p, double baseline_hz, uint32_t sample_every) {
    if (!(p.tau > 0)) throw ConfigError("hemodynamics: tau must be > 0");
    if (!(p.alpha > 0) || p.alpha > 1) throw ConfigError("hemodynamics: alpha must be in (0, 1]");
    if (!(p.e0 > 0) || p.e0 >= 1) throw ConfigError("hemodynamics: E0 must be in (0, 1)");
    if (!(p.v0 > 0)) throw ConfigError("hemodynamics: V0 must be > 0");
    if (p.kappa < 0 || p.gamma < 0) throw ConfigError("hemodynamics: decay rates must be >= 0");
    if (!(baseline_hz > 0)) throw ConfigError("baseline_hz must be > 0");
    if (sample_every == 0) throw ConfigError("hemodynamics: sample_every must be >= 1");
}

void Engine::set_hemodynamics(const vxb_hemo_params& p, double baseline_hz,
                              uint32_t sample_every, const vxb_hemo_state* init) {
    validate_hemo(p, baseline_hz, sample_every);
    CK(cudaSetDevice(device));
    // voxel -> units CSR and voxel sizes (voxel_sizes, assim.cpp:319)
    std::vector<uint32_t> off(n_voxels + 1, 0), vu(n_units);
    std::vector<double> vn(n_voxels, 0.0);
    std::vector<uint64_t> vn64(n_voxels, 0);
    for (uint32_t u = 0; u < n_units; ++u) {
        ++off[units[u].voxel + 1];
        vn64[units[u].voxel] += units[u].neurons;
    }
    for (uint32_t v = 0; v < n_voxels; ++v) {
        off[v + 1] += off[v];
        vn[v] = static_cast<double>(vn64[v]);
    }
    std::vector<uint32_t> cur(off.begin(), off.end() - 1);
    for (uint32_t u = 0; u < n_units; ++u) vu[cur[units[u].voxel]++] = u;
    std::vector<HemoStateDev> st(n_voxels, HemoStateDev{0.0, 1.0, 1.0, 1.0});  // hemo.hpp:25-30
    if (init)
        for (uint32_t v = 0; v < n_voxels; ++v) st[v] = {init[v].s, init[v].f, init[v].v, init[v].q};
    d_vox_off.alloc(off.size());
    d_vox_units.alloc(std::max<size_t>(1, vu.size()));
    d_vox_n.alloc(std::max<size_t>(1, vn.size()));
    d_hemo.alloc(std::max<size_t>(1, st.size()));
    d_hemo_err.alloc(1);
    CK(cudaMemcpyAsync(d_vox_off.p, off.data(), 4 * off.size(), cudaMemcpyHostToDevice, stream));
    if (!vu.empty())
        CK(cudaMemcpyAsync(d_vox_units.p, vu.data(), 4 * vu.size(), cudaMemcpyHostToDevice, stream));
    if (!vn.empty()) {
        CK(cudaMemcpyAsync(d_vox_n.p, vn.data(), 8 * vn.size(), cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_hemo.p, st.data(), sizeof(HemoStateDev) * st.size(),
                           cudaMemcpyHostToDevice, stream));
    }
    CK(cudaStreamSynchronize(stream));
    hemo_p = {p.kappa, p.gamma, p.tau, p.alpha, p.e0, p.v0};
    hemo_baseline = baseline_hz;
    hemo_every = sample_every;
    hemo_on = true;
}

void Engine::run_hemo(uint32_t t_base, uint32_t steps) {
    hemo_counts_kernel<<<(n_voxels + 127) / 128, 128, 0, stream>>>(
        d_vcounts.p, t_base, steps, d_vox_n.p, n_voxels, hemo_p, dt_ms * 1e-3, hemo_baseline,
        hemo_every, d_hemo.p, d_bold.p, d_hemo_err.p);
    CK(cudaGetLastError());
    launches += 1;
}

bool Engine::fetch_bold() {
    unsigned long long herr = 0;
    if (!bold.empty())
        CK(cudaMemcpyAsync(bold.data(), d_bold.p, 8 * bold.size(), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(&herr, d_hemo_err.p, 8, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    d2h += 8 * bold.size() + 8;
    return herr == ~0ull;
}

struct Chunk {
    uint32_t t0, rel0, steps;
};

// advance() = advance_begin (results reset, per-advance tables, buffers),
// then per chunk launch_chunk + finish_chunk + chunk_post, then advance_end
// (readback of the advance's results).  vxb_advance_members interleaves the
// same pieces of several ensemble members.
void Engine::advance(uint32_t steps) {
    const uint32_t chunk = advance_begin(steps);
    if (steps == 0) return;
    std::vector<unsigned long long> phase_ns_all;
    phase_ns_all.reserve(steps + 2);
    for (uint32_t rel0 = 0; rel0 < steps; rel0 += chunk) {
        const uint32_t cs = std::min(chunk, steps - rel0);
        launch_chunk(step_done + rel0, rel0, cs, steps, 0);
        finish_chunk(rel0, cs, steps);
        chunk_post(rel0, cs, phase_ns_all);
    }
    advance_end(steps, phase_ns_all);
}

uint32_t Engine::advance_begin(uint32_t steps) {
    if (failed) throw SimError("instance is in a failed state");
    res_steps = steps;
    res_start = step_done;
    raster_keys.clear();
    rates.assign((size_t)n_units * steps, 0);
    probe_v.assign(probes.size() * (size_t)steps, 0.0f);
    probe_i.assign(probes.size() * (size_t)steps, 0.0f);
    flops = vxb_flops{};
    total_spikes = 0;
    timings.clear();
    device_ms = 0;
    h2d = d2h = launches = 0;
    if (steps == 0) return 0;
    CK(cudaSetDevice(device));

    // per-advance tables: forced spikes and injection epochs by relative step
    std::vector<uint32_t> f_off(steps + 1, 0), f_loc;
    {
        size_t k = 0;
        while (k < forced.size() && forced[k].first < step_done) ++k;
        for (uint32_t rel = 0; rel < steps; ++rel) {
            f_off[rel] = (uint32_t)f_loc.size();
            while (k < forced.size() && forced[k].first == step_done + rel)
                f_loc.push_back(forced[k++].second);
        }
        f_off[steps] = (uint32_t)f_loc.size();
    }
    std::vector<uint32_t> inj_ep(steps, 0);
    std::vector<float> inj_tab;
    if (!injections.empty()) {
        std::map<std::vector<uint32_t>, uint32_t> seen;  // active set -> epoch
        for (uint32_t rel = 0; rel < steps; ++rel) {
            const uint32_t t = step_done + rel;
            std::vector<uint32_t> act;
            for (uint32_t k = 0; k < injections.size(); ++k)
                if (injections[k].from_step <= t && t < injections[k].to_step) act.push_back(k);
            if (act.empty()) continue;
            auto it = seen.find(act);
            if (it == seen.end()) {
                std::vector<float> vox(n_voxels, 0.0f);  // engine.cpp:355-361, list order
                for (uint32_t k : act) vox[injections[k].voxel] += injections[k].current_pa;
                inj_tab.insert(inj_tab.end(), vox.begin(), vox.end());
                it = seen.emplace(act, (uint32_t)seen.size() + 1).first;
            }
            inj_ep[rel] = it->second;
        }
    }
    // tables of THIS advance only: an advance without forced spikes or active
    // injections must not replay the previous advance's tables
    has_forced = !f_loc.empty();
    has_inj = !inj_tab.empty();
    if (!has_forced) {
        d_forced_off.release();
        d_forced_local.release();
    }
    if (!has_inj) {
        d_inj_epoch.release();
        d_inj_table.release();
    }
    if (has_forced) {
        d_forced_off.alloc(f_off.size());
        d_forced_local.alloc(f_loc.size());
        CK(cudaMemcpyAsync(d_forced_off.p, f_off.data(), 4 * f_off.size(),
                           cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(d_forced_local.p, f_loc.data(), 4 * f_loc.size(),
                           cudaMemcpyHostToDevice, stream));
        h2d += 4 * (f_off.size() + f_loc.size());
    }
    if (has_inj) {
        d_inj_epoch.alloc(steps);
        d_inj_table.alloc(inj_tab.size());
        CK(cudaMemcpyAsync(d_inj_epoch.p, inj_ep.data(), 4ull * steps, cudaMemcpyHostToDevice,
                           stream));
        CK(cudaMemcpyAsync(d_inj_table.p, inj_tab.data(), 4 * inj_tab.size(),
                           cudaMemcpyHostToDevice, stream));
        h2d += 4ull * steps + 4 * inj_tab.size();
    }
    if (!probes.empty()) {
        d_probe_v.alloc(probes.size() * (size_t)steps);
        d_probe_i.alloc(probes.size() * (size_t)steps);
        d_probe_v.zero(stream);
        d_probe_i.zero(stream);
    }
    flush_conductances(false);  // advance syncs before the caller can stage again

    // chunking: the linear spike log holds n entries per step of a chunk
    uint32_t chunk = steps;
    if (log_spikes()) {
        const uint64_t cap = 1ull << 29;  // 2 GiB of spike ids per chunk
        chunk = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(steps, cap / std::max(1u, n)));
    }
    const uint32_t cap_entries = log_spikes() ? n * chunk : 2 * n;
    if (d_spk.n < std::max<size_t>(1, cap_entries)) d_spk.alloc(std::max<size_t>(1, cap_entries));
    d_seg_end.reserve(chunk + 2);
    d_bdone.reserve(chunk + 2);
    d_routed.reserve(chunk + 2);
    d_rates.reserve((size_t)n_units * chunk);
    d_phase_ns.reserve(chunk + 2);
    d_phase_wait.reserve(chunk + 2);
    d_arrive.reserve((size_t)(chunk + 2) * world);
    exchange_arrival_ms = 0;
    exchange_wait_ms = 0;
    phase_wait_all.assign(steps + 2, 0);

    const uint32_t n_bold = hemo_on && world == 1 ? steps / hemo_every : 0u;
    bold.assign((size_t)n_bold * n_voxels, 0.0);
    vcounts.assign(hemo_on ? (size_t)steps * n_voxels : 0, 0u);
    if (hemo_on) {
        d_bold.reserve(std::max<size_t>(1, bold.size()));
        d_vcounts.reserve(std::max<size_t>(1, vcounts.size()));
        const unsigned long long none = ~0ull;
        CK(cudaMemcpyAsync(d_hemo_err.p, &none, 8, cudaMemcpyHostToDevice, stream));
    }
    return chunk;
}

void Engine::chunk_post(uint32_t rel0, uint32_t cs, std::vector<unsigned long long>& phase_ns_all) {
    {
        if (hemo_on) {  // window_bold (assim.cpp:51-71) over this chunk's rate rows
            const uint32_t work = cs * n_voxels;
            voxel_counts_kernel<<<std::min<uint32_t>(1184, (work + 255) / 256), 256, 0, stream>>>(
                d_rates.p, cs, d_vox_off.p, d_vox_units.p, n_voxels, rel0, d_vcounts.p);
            CK(cudaGetLastError());
            launches += 1;
            if (world == 1) run_hemo(rel0, cs);  // (several GPUs: the totals are fed back)
        }
        // phase end times of this chunk
        std::vector<unsigned long long> ph(cs + 2);
        CK(cudaMemcpyAsync(ph.data(), d_phase_ns.p, 8ull * (cs + 2), cudaMemcpyDeviceToHost,
                           stream));
        CK(cudaStreamSynchronize(stream));
        d2h += 8ull * (cs + 2);
        if (phase_ns_all.empty()) phase_ns_all.push_back(ph[0]);
        for (uint32_t p = 1; p <= cs + 1; ++p) phase_ns_all.push_back(ph[p]);
        // the next chunk re-runs no phase: its A-only prologue follows this
        // chunk's E-only epilogue; stitch their times together.
    }
}

void Engine::advance_end(uint32_t steps, const std::vector<unsigned long long>& phase_ns_all) {
    // probes
    if (!probes.empty()) {
        CK(cudaMemcpyAsync(probe_v.data(), d_probe_v.p, 4 * probe_v.size(),
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(probe_i.data(), d_probe_i.p, 4 * probe_i.size(),
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        d2h += 8 * probe_v.size();
    }
    bool hemo_diverged = false;
    if (hemo_on) {
        if (!vcounts.empty())
            CK(cudaMemcpyAsync(vcounts.data(), d_vcounts.p, 4 * vcounts.size(),
                               cudaMemcpyDeviceToHost, stream));
        d2h += 4 * vcounts.size();
        hemo_diverged = !fetch_bold();
    }
    for (uint32_t x : rates) total_spikes += x;
    const uint64_t nn = n;
    flops.membrane += 6ull * nn * steps;       // engine.cpp:387
    flops.gating_decay += 12ull * nn * steps;  // engine.cpp:560
    flops.current += 16ull * nn * steps;       // engine.cpp:561

    if (record_timings) {
        // One row per (step, worker).  The cuda scheduler has no per-worker
        // threads: t1 = the phase holding A(t), t3 adds the phase holding E(t).
        timings.resize((size_t)steps * workers);
        std::vector<uint32_t> unit_of_worker_spikes((size_t)steps * workers, 0);
        for (uint32_t u = 0; u < n_units; ++u)
            for (uint32_t s = 0; s < steps; ++s)
                unit_of_worker_spikes[(size_t)s * workers + unit_worker[u]] +=
                    rates[(size_t)u * steps + s];
        for (uint32_t s = 0; s < steps; ++s) {
            // phase_ns_all[k] = end of global phase k-1; phase of A(s) is s
            const int64_t a = (int64_t)(phase_ns_all[s + 1] - phase_ns_all[s]);
            const int64_t e = (int64_t)(phase_ns_all[s + 2] - phase_ns_all[s + 1]);
            for (uint16_t w = 0; w < workers; ++w) {
                vxb_step_timings& r = timings[(size_t)s * workers + w];
                std::memset(&r, 0, sizeof r);
                r.step = step_done + s;
                r.worker = w;
                r.spikes = unit_of_worker_spikes[(size_t)s * workers + w];
                r.t[0] = a;      // t1
                r.t[1] = a;      // t2: no inbound wait on one device
                r.t[2] = a + e;  // t3
                r.t[3] = r.t[4] = r.t[0];
                r.t[5] = r.t[6] = r.t[1];
                // send span t8..t9: the ids are stored into the peers' slots
                // during the phase and published at its end (no send time of
                // their own); receive span t10..t11: the wait for the peers'
                // batches of S(s) at the start of the phase holding E(s)
                r.t[7] = r.t[8] = r.t[0];
                r.t[9] = a;
                r.t[10] = a + (world > 1 ? (int64_t)phase_wait_all[s + 1] : 0);
                if (world > 1) {
                    bool inter = false;
                    for (uint32_t h = 0; h < world; ++h)
                        inter |= h != rank && h / workers_per_node != rank / workers_per_node;
                    (inter ? r.recv_inter_ns : r.recv_intra_ns) = r.t[10] - r.t[9];
                }
            }
        }
        account_wire_bytes(steps);
    }
    if (!record_raster) raster_keys.clear();
    step_done += steps;
    // hemo.cpp:37-40, raised by the readout: the simulation state is intact
    if (hemo_diverged) throw HemoError("hemodynamic state diverged");
}

// LEB128 length of one delta (transport.cpp:10-17)
uint32_t varint_len(uint32_t v) {
    return v < (1u << 7) ? 1u : v < (1u << 14) ? 2u : v < (1u << 21) ? 3u : v < (1u << 28) ? 4u : 5u;
}

// Wire bytes of every (step, src, dst) spike batch as the reference encodes
// it (encode_batch, transport.cpp:33-55: 12-byte header + the varints of the
// ascending local ids' deltas; an empty batch is the 12-byte header) and the
// StepTimings byte counters split by node (engine.cpp:416-437, 495-523,
// 570-597; acceptance.cpp:651-742).  On one device every worker is here and
// both directions are counted; with one worker per rank the sent bytes are
// counted here and the received ones come from the peers
// (vxb_set_recv_wire_bytes).
void Engine::account_wire_bytes(uint32_t steps) {
    const std::vector<unsigned long long>& mk = world > 1 ? h_mask : dst_full;
    const uint32_t W = workers;
    std::vector<uint64_t> b((size_t)W * W);
    std::vector<uint32_t> prev((size_t)W * W);
    std::vector<uint8_t> seen((size_t)W * W);
    auto node = [&](uint32_t w) { return w / workers_per_node; };
    if (world > 1) wire_sent.assign((size_t)steps * W, 0);
    size_t k = 0;
    for (uint32_t s = 0; s < steps; ++s) {
        std::fill(b.begin(), b.end(), 12ull);
        std::fill(seen.begin(), seen.end(), 0);
        for (; k < raster_keys.size() && (uint32_t)(raster_keys[k] >> 32) == s; ++k) {
            const uint32_t loc = (uint32_t)raster_keys[k];
            const uint32_t w = (uint32_t)(std::upper_bound(wbase.begin(), wbase.end(), loc) -
                                          wbase.begin()) - 1;
            const uint32_t id = loc - wbase[w];
            for (unsigned long long m = mk.empty() ? 0ull : mk[loc]; m; m &= m - 1) {
                const uint32_t d = (uint32_t)__builtin_ctzll(m);
                if (d == w || d >= W) continue;
                const size_t q = (size_t)w * W + d;
                b[q] += varint_len(seen[q] ? id - prev[q] : id);
                seen[q] = 1;
                prev[q] = id;
            }
        }
        for (uint32_t w = local_lo; w < local_hi; ++w) {
            vxb_step_timings& r = timings[(size_t)s * W + w];
            for (uint32_t d = 0; d < W; ++d) {
                if (d == w) continue;
                (node(d) == node(w) ? r.bytes_sent_intra : r.bytes_sent_inter) += b[(size_t)w * W + d];
                if (world > 1) wire_sent[(size_t)s * W + d] = b[(size_t)w * W + d];
                else
                    (node(d) == node(w) ? r.bytes_recv_intra : r.bytes_recv_inter) += b[(size_t)d * W + w];
            }
        }
    }
}

// Launch one chunk of `steps` steps (grid_ctas > 0: a smaller grid, for
// members sharing the device).
void Engine::launch_chunk(uint32_t t0, uint32_t rel0, uint32_t steps, uint32_t adv_steps,
                          int grid_ctas) {
    // the launch's scratch (control block, rates, log ends, phase times,
    // counters) cleared by one kernel instead of a memset each
    ClearList cl;
    std::memset(&cl, 0, sizeof cl);
    cl.ctl = d_ctl.p;
    auto clr = [&](void* p, size_t bytes) {
        if (!p || !bytes) return;
        if (cl.n == kClearMax) throw SimError("clear list overflow");
        cl.p[cl.n] = reinterpret_cast<uint32_t*>(p);
        cl.words[cl.n] = bytes / 4;
        ++cl.n;
    };
    clr(d_rates.p, 4 * d_rates.n);
    clr(d_seg_end.p, 4 * d_seg_end.n);
    clr(d_phase_ns.p, 8 * d_phase_ns.n);
    clr(d_phase_wait.p, 8 * d_phase_wait.n);

    StepArgs a;
    std::memset(&a, 0, sizeof a);
    a.n = n;
    a.nseg = (uint32_t)segs.size();
    a.npset = npset;
    a.n_units = n_units;
    a.steps = steps;
    a.t0 = t0;
    a.rel0 = rel0;
    a.adv_steps = adv_steps;
    a.spk_cap = (uint32_t)d_spk.n;
    a.ring = log_spikes() ? 0u : 1u;
    a.use_smem_seg = use_smem_seg ? 1u : 0u;
    a.dtf = dtf;
    a.ou_root = mix_key(seed, 1);  // rngstream::ou_noise (rng.hpp:18)
    a.pset = d_pset.p;
    a.sinfo = d_sinfo.p;
    a.seg_start = d_seg_start.p;
    a.v = d_v.p;
    a.j = d_j.p;
    a.i_ou = d_iou.p;
    a.i_syn = d_isyn.p;
    a.g = d_g.p;
    a.pend0 = d_pend0.p;
    a.pend1 = d_pend1.p;
    a.off = d_off.p;
    a.inner = d_inner.p;
    a.tgt = d_tgt.p;
    a.w = d_w.p;
    a.spk = d_spk.p;
    a.seg_end = d_seg_end.p;
    a.rates = d_rates.p;
    a.n_probes = n_probe_dev;
    a.probe_local = d_probe_local.p;
    a.probe_slot = d_probe_slot.p;
    a.probe_v = d_probe_v.p;
    a.probe_i = d_probe_i.p;
    a.has_forced = has_forced ? 1u : 0u;
    a.forced_off = a.has_forced ? d_forced_off.p + rel0 : nullptr;
    a.forced_local = d_forced_local.p;
    a.has_inj = has_inj ? 1u : 0u;
    a.inj_epoch = a.has_inj ? d_inj_epoch.p + rel0 : nullptr;
    a.inj_table = d_inj_table.p;
    a.n_voxels = n_voxels;
    a.phase_ns = d_phase_ns.p;
    a.ctl = d_ctl.p;
    a.ex = d_ex.p;
    a.world = world;
    a.dst_mask = d_mask.p;
    a.phase_wait = d_phase_wait.p;
    if (world > 1) {
        a.arrive = d_arrive.p;
        CK(cudaMemsetAsync(d_arrive.p, 0xff, 8ull * (steps + 2) * world, stream));
    }
    a.n_blocks = n_blocks;
    a.blk_off = d_blk.p;
    d_work.reserve(2ull * n_blocks * world);
    clr(d_work.p, 4 * d_work.n);
    a.work_ctr = d_work.p;
    a.dyn = dyn ? 1u : 0u;
    a.stage_e = stage_e;
    a.ch_max = ch_max;
    a.f_policy = f_policy;
    a.early_publish = early_publish ? 1u : 0u;
    prof = knob("VXB_PHASE_PROFILE", nullptr) != nullptr;
    if (prof) {
        d_prof.alloc((tile_path ? (tile_mp ? 4ull : (size_t)kTileProf) * tile_grid : 2ull * grid) * (steps + 1));
        d_prof.zero(stream);
        a.prof = d_prof.p;
    }

    if (tile_path) {
        a.tile_n = tile_per;
        a.n_cons = tile_cons;
        a.n_noisew = tile_mp ? 0u : tile_noisew;
        a.q_total = (uint32_t)q_total;
        a.tl_off = d_tl_off.p;
        a.tl = d_tl.p;
        a.q_base = d_qbase.p;
        a.q_cnt = d_qcnt.p;
        a.q = d_q.p;
        a.src_self = world > 1 ? src_base[rank] : 0u;
        a.tent = d_tent.p;
        a.i_ou_b = d_iou_b.p;
        a.n_tiles = tile_T;
        a.passes = tile_passes;
        a.item_mode = tile_items;
        clr(d_qcnt.p, 4 * d_qcnt.n);
        a.bdone = d_bdone.p;
        clr(d_bdone.p, 4 * d_bdone.n);
        a.routed = d_routed.p;
        clr(d_routed.p, 4 * d_routed.n);
        d_bmail.reserve(32ull * tile_grid);
        clr(d_bmail.p, 4 * d_bmail.n);
        a.bmail = d_bmail.p;
    }
    clear_kernel<<<148, 256, 0, stream>>>(cl);
    CK(cudaGetLastError());
    launches += 1;
    void* args[] = {&a};
    CK(cudaEventRecord(ev0, stream));
    if (tile_path && tile_mp) {
        CK(cudaLaunchCooperativeKernel(world > 1 ? (const void*)tile_mp_kernel<true>
                                                 : (const void*)tile_mp_kernel<false>,
                                       tile_grid, kMpThreads, args, tile_smem, stream));
    } else if (tile_path) {
        const bool ex = has_forced || has_inj || n_probe_dev > 0;
        const void* tk = world > 1 ? (ex ? (const void*)tile_kernel<true, true> : (const void*)tile_kernel<true, false>)
                                   : (ex ? (const void*)tile_kernel<false, true> : (const void*)tile_kernel<false, false>);
        CK(cudaLaunchCooperativeKernel(tk, tile_grid, kTileThreads, args, tile_smem, stream));
    }
    else if (packed)
        CK(cudaLaunchCooperativeKernel((const void*)step_kernel<true>, grid_ctas > 0 ? grid_ctas : grid,
                                       kThreads, args, smem_bytes, stream));
    else
        CK(cudaLaunchCooperativeKernel((const void*)step_kernel<false>, grid_ctas > 0 ? grid_ctas : grid,
                                       kThreads, args, smem_bytes, stream));
    CK(cudaEventRecord(ev1, stream));
    launches += 1;
}

// Wait for the chunk and read its results (rates, spikes, flops, errors).
void Engine::finish_chunk(uint32_t rel0, uint32_t steps, uint32_t adv_steps) {
    Control c;
    CK(cudaMemcpyAsync(&c, d_ctl.p, sizeof c, cudaMemcpyDeviceToHost, stream));
    std::vector<uint32_t> rr((size_t)n_units * steps);
    if (!rr.empty())
        CK(cudaMemcpyAsync(rr.data(), d_rates.p, 4 * rr.size(), cudaMemcpyDeviceToHost, stream));
    std::vector<uint32_t> seg_end(steps + 1);
    CK(cudaMemcpyAsync(seg_end.data(), d_seg_end.p, 4ull * (steps + 1), cudaMemcpyDeviceToHost,
                       stream));
    // tile_kernel's log is phase-strided with per-phase counts
    const bool strided = tile_path && !tile_mp;
    if (world > 1) {
        std::vector<unsigned long long> pw(steps + 2);
        CK(cudaMemcpyAsync(pw.data(), d_phase_wait.p, 8ull * (steps + 2), cudaMemcpyDeviceToHost,
                           stream));
        CK(cudaStreamSynchronize(stream));
        for (auto x : pw) exchange_wait_ms += x * 1e-6;
        for (uint32_t p = 1; p <= steps; ++p) phase_wait_all[rel0 + p] = pw[p];
        // arrival lag: when the last peer's batch of S(tE) was first seen,
        // after the start of the phase that delivers it (independent of how
        // much local work the CTAs had before they waited)
        std::vector<unsigned long long> ar((size_t)(steps + 2) * world), pn(steps + 2);
        CK(cudaMemcpyAsync(ar.data(), d_arrive.p, 8 * ar.size(), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(pn.data(), d_phase_ns.p, 8 * pn.size(), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        for (uint32_t p = 1; p <= steps; ++p) {
            unsigned long long last = 0;
            for (uint32_t h = 0; h < world; ++h)
                if (h != rank && ar[(size_t)p * world + h] != ~0ull)
                    last = std::max(last, ar[(size_t)p * world + h]);
            if (last > pn[p]) exchange_arrival_ms += (last - pn[p]) * 1e-6;
        }
    }
    CK(cudaStreamSynchronize(stream));
    if (prof && tile_path) {  // per phase: mean / max over CTAs of each part's end (us)
        std::vector<unsigned long long> pr(d_prof.n), pn(steps + 2);
        CK(cudaMemcpy(pr.data(), d_prof.p, 8 * pr.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(pn.data(), d_phase_ns.p, 8 * pn.size(), cudaMemcpyDeviceToHost));
        double sum[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0}, sp = 0;
        uint32_t cnt[4] = {0, 0, 0, 0};
        // tile_kernel (no barrier): relative to the CTA's own phase start;
        // tile_mp_kernel: to the end of the previous phase's barrier
        const size_t ps = tile_mp ? 4 : kTileProf;
        if (const char* dump = knob("VXB_PROF_DUMP", nullptr)) {  // raw [phase][CTA][ps] globaltimer ns
            if (FILE* f = std::fopen(dump, "wb")) {
                std::fwrite(pr.data(), 8, pr.size(), f);
                std::fclose(f);
            }
        }
        for (uint32_t ph = 1; ph < steps; ++ph) {
            sp += (double)(pn[ph + 1] - pn[ph]);
            double pm[4] = {0, 0, 0, 0};
            for (uint32_t b = 0; b < tile_grid; ++b) {
                const double t0 = !tile_mp ? (double)pr[ps * ((size_t)ph * tile_grid + b) + 4] : (double)pn[ph];
                for (int k = 0; k < 4; ++k) {
                    const unsigned long long x = pr[ps * ((size_t)ph * tile_grid + b) + k];
                    if (!x) continue;
                    sum[k] += (double)x - t0;
                    ++cnt[k];
                    pm[k] = std::max(pm[k], (double)x - t0);
                }
            }
            for (int k = 0; k < 4; ++k) mx[k] += pm[k];
        }
        const double np_ = std::max(1u, steps - 1);
        std::fprintf(stderr,
                     "vxb tile phase profile (us): phase %.1f | update end %.1f/%.1f | bucketing "
                     "%.1f/%.1f | consumers %.1f/%.1f | noise %.1f/%.1f (mean/max over CTAs)\n",
                     sp / np_ / 1e3, sum[0] / std::max(1u, cnt[0]) / 1e3, mx[0] / np_ / 1e3,
                     sum[1] / std::max(1u, cnt[1]) / 1e3, mx[1] / np_ / 1e3,
                     sum[2] / std::max(1u, cnt[2]) / 1e3, mx[2] / np_ / 1e3,
                     sum[3] / std::max(1u, cnt[3]) / 1e3, mx[3] / np_ / 1e3);
    } else if (prof) {  // per phase: mean / max over CTAs of delivery and update end (us)
        std::vector<unsigned long long> pr(d_prof.n), pn(steps + 2);
        CK(cudaMemcpy(pr.data(), d_prof.p, 8 * pr.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(pn.data(), d_phase_ns.p, 8 * pn.size(), cudaMemcpyDeviceToHost));
        double sd = 0, md = 0, sf = 0, mf = 0, sp = 0;
        uint32_t nd = 0;
        for (uint32_t ph = 1; ph < steps; ++ph) {  // phases with both E and A
            const double t0 = (double)pn[ph], len = (double)(pn[ph + 1] - pn[ph]);
            double pmd = 0, pmf = 0;
            for (int b = 0; b < grid; ++b) {
                const double d = pr[2 * ((size_t)ph * grid + b)] ? pr[2 * ((size_t)ph * grid + b)] - t0 : 0;
                const double f = pr[2 * ((size_t)ph * grid + b) + 1] - t0;
                sd += d;
                sf += f;
                pmd = std::max(pmd, d);
                pmf = std::max(pmf, f);
                ++nd;
            }
            md += pmd;
            mf += pmf;
            sp += len;
        }
        const double np_ = std::max(1u, steps - 1);
        if (nd)
            std::fprintf(stderr,
                         "vxb phase profile (us): phase %.1f | delivery end mean %.1f max %.1f | "
                         "update end mean %.1f max %.1f\n",
                         sp / np_ / 1e3, sd / nd / 1e3, md / np_ / 1e3, sf / nd / 1e3, mf / np_ / 1e3);
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    device_ms += ms;
    d2h += sizeof c + 4 * rr.size() + 4ull * (steps + 1);
    if (world > 1) {
        uint32_t to[3] = {0, 0, 0};  // timeout, timeout_step, peer_abort
        CK(cudaMemcpy(to, &d_ex.p->timeout, 12, cudaMemcpyDeviceToHost));
        if (to[0]) {
            failed = true;
            throw SimError(fmt("step barrier timed out on worker %u at step %u (no batch from "
                               "worker %u)", rank, to[1], to[0] - 1));
        }
        if (to[2] && c.err == ~0ull) {  // engine.cpp:483-484
            failed = true;
            throw SimError("simulation aborted while waiting on the step barrier");
        }
    }
    if (c.err != ~0ull) {
        failed = true;
        const uint32_t step = (uint32_t)(c.err >> 32), loc = (uint32_t)(c.err & 0xffffffffu);
        const SegParams& s = segs[seg_of(loc)];
        throw SimError(fmt("membrane potential diverged (neuron %llu, step %u)",
                           (unsigned long long)((int64_t)loc + s.gid_off), step));
    }
    for (uint32_t u = 0; u < n_units; ++u)
        for (uint32_t s = 0; s < steps; ++s)
            rates[(size_t)u * adv_steps + rel0 + s] += rr[(size_t)u * steps + s];
    flops.gating_inner += c.flops_inner;
    flops.gating_outer += c.flops_outer;

    if (log_spikes()) {
        if (strided) {  // counts -> cumulative ends for the key kernel
            for (uint32_t p = 1; p <= steps; ++p) seg_end[p] += seg_end[p - 1];
            CK(cudaMemcpyAsync(d_seg_end.p, seg_end.data(), 4ull * (steps + 1), cudaMemcpyHostToDevice,
                               stream));
        }
        const uint32_t total = seg_end[steps - 1];
        if (total) {
            if (d_keys.n < total) d_keys.alloc(total);
            if (d_keys_sorted.n < total) d_keys_sorted.alloc(total);
            raster_keys_kernel<<<std::min<uint32_t>(steps, 4096), 256, 0, stream>>>(
                d_spk.p, d_seg_end.p, steps, d_keys.p, strided ? n : 0u);
            CK(cudaGetLastError());
            launches += 1;
            int end_bit = 32;
            while ((1ull << (end_bit - 32)) < steps) ++end_bit;
            size_t tmp = 0;
            CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp,
                                              reinterpret_cast<unsigned long long*>(d_keys.p),
                                              reinterpret_cast<unsigned long long*>(d_keys_sorted.p),
                                              total, 0, end_bit, stream));
            if (d_cub_tmp.n < tmp) d_cub_tmp.alloc(tmp);
            CK(cub::DeviceRadixSort::SortKeys(d_cub_tmp.p, tmp,
                                              reinterpret_cast<unsigned long long*>(d_keys.p),
                                              reinterpret_cast<unsigned long long*>(d_keys_sorted.p),
                                              total, 0, end_bit, stream));
            launches += 1;
            const size_t base = raster_keys.size();
            raster_keys.resize(base + total);
            CK(cudaMemcpyAsync(raster_keys.data() + base, d_keys_sorted.p, 8ull * total,
                               cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            d2h += 8ull * total;
            const uint64_t add = (uint64_t)rel0 << 32;
            for (size_t k = base; k < raster_keys.size(); ++k) raster_keys[k] += add;
        }
    }
}

// The schedule the engine chose for this network (JSON object), with every
// tuning knob that was applied: logged beside each benchmark result.
std::string Engine::schedule_info() const {
    if (tile_path)
        return fmt("{\"path\":\"sm_tile\",\"kernel\":\"%s\",\"grid\":%u,"
                   "\"tiles\":%u,\"passes\":%u,\"item_per\":\"%s\","
                   "\"threads\":%d,\"smem_bytes\":%u,\"tile_neurons\":%u,"
                   "\"unroll\":%u,\"consumer_warps\":%u,\"queue_items\":%llu,"
                   "\"state_l2_policy\":%u,\"packed_pending\":%d,\"world\":%u,\"knobs\":{",
                   tile_mp ? "vxb::tile_mp_kernel" : "vxb::tile_kernel", tile_grid, tile_T,
                   tile_passes, tile_items ? "lane" : "warp",
                   tile_mp ? kMpThreads : kTileThreads, tile_smem, tile_per, kTileUnroll, tile_cons,
                   (unsigned long long)q_total, f_policy, (int)packed, world) +
               knobs + "}}";
    return fmt("{\"path\":\"l2_atomic\",\"kernel\":\"vxb::step_kernel\",\"grid\":%d,"
               "\"threads\":%d,\"smem_bytes\":%u,"
               "\"l2_blocks\":%u,\"dynamic_deal\":%d,\"stage_entries\":%u,\"ch_max\":%u,"
               "\"state_l2_policy\":%u,\"packed_pending\":%d,\"world\":%u,\"knobs\":{",
               grid, kThreads, smem_bytes, n_blocks, (int)dyn, stage_e, ch_max,
               f_policy, (int)packed, world) +
           knobs + "}}";
}

int fail_code(const std::exception& e) {
    return dynamic_cast<const ConfigError*>(&e) ? VXB_ECONFIG : VXB_ESIM;
}

}  // namespace

struct vxb_engine {
    Engine eng;
};

extern "C" {

int vxb_abi_version(void) { return VXB_ABI_VERSION; }

#ifndef VXB_SRC_HASH
#define VXB_SRC_HASH "unknown"
#endif
// "VXB_SRC_HASH=<hash>" is also the marker build.py finds in the binary
static const char kBuildHash[] = "VXB_SRC_HASH=" VXB_SRC_HASH;
const char* vxb_build_hash(void) { return kBuildHash + 13; }

const char* vxb_last_error(const vxb_engine* e) {
    return e ? e->eng.err.c_str() : g_create_error.c_str();
}

int vxb_create(const vxb_network* net, const vxb_options* opt, vxb_engine** out) {
    *out = nullptr;
    auto* e = new vxb_engine();
    try {
        e->eng.load(net, opt);
    } catch (const std::exception& x) {
        g_create_error = x.what();
        int rc = fail_code(x);
        delete e;
        return rc;
    }
    *out = e;
    return VXB_OK;
}

void vxb_destroy(vxb_engine* e) { delete e; }

int vxb_advance(vxb_engine* e, uint32_t steps) {
    try {
        e->eng.advance(steps);
        return VXB_OK;
    } catch (const HemoError& x) {  // raised by the BOLD readout, not the simulation
        e->eng.err = x.what();
        return VXB_ESIM;
    } catch (const std::exception& x) {
        e->eng.err = x.what();
        e->eng.failed = true;
        return fail_code(x);
    }
}

uint32_t vxb_current_step(const vxb_engine* e) { return e->eng.step_done; }
uint32_t vxb_result_steps_done(const vxb_engine* e) { return e->eng.res_steps; }
uint64_t vxb_result_total_spikes(const vxb_engine* e) { return e->eng.total_spikes; }
uint64_t vxb_result_raster_size(const vxb_engine* e) { return e->eng.raster_keys.size(); }

int vxb_result_raster(const vxb_engine* e, vxb_raster_event* out, uint64_t cap) {
    const Engine& g = e->eng;
    if (cap < g.raster_keys.size()) return VXB_ECONFIG;
    for (size_t k = 0; k < g.raster_keys.size(); ++k) {
        const uint64_t key = g.raster_keys[k];
        const uint32_t loc = (uint32_t)(key & 0xffffffffu);
        const SegParams& s = g.segs[g.seg_of(loc)];
        vxb_raster_event r;
        std::memset(&r, 0, sizeof r);
        r.step = g.res_start + (uint32_t)(key >> 32);
        r.worker = (uint16_t)s.worker;
        r.local = loc - g.wbase[s.worker];
        r.gid = (uint64_t)((int64_t)loc + s.gid_off);
        out[k] = r;
    }
    return VXB_OK;
}

int vxb_result_rates(const vxb_engine* e, uint32_t* counts, uint64_t cap) {
    if (cap < e->eng.rates.size()) return VXB_ECONFIG;
    std::memcpy(counts, e->eng.rates.data(), 4 * e->eng.rates.size());
    return VXB_OK;
}

int vxb_result_probes(const vxb_engine* e, float* v, float* i_syn, uint64_t cap) {
    if (cap < e->eng.probe_v.size()) return VXB_ECONFIG;
    std::memcpy(v, e->eng.probe_v.data(), 4 * e->eng.probe_v.size());
    std::memcpy(i_syn, e->eng.probe_i.data(), 4 * e->eng.probe_i.size());
    return VXB_OK;
}

int vxb_result_flops(const vxb_engine* e, vxb_flops* out) {
    *out = e->eng.flops;
    return VXB_OK;
}

uint64_t vxb_result_timings_size(const vxb_engine* e) { return e->eng.timings.size(); }

int vxb_result_timings(const vxb_engine* e, vxb_step_timings* out, uint64_t cap) {
    if (cap < e->eng.timings.size()) return VXB_ECONFIG;
    std::memcpy(out, e->eng.timings.data(), sizeof(vxb_step_timings) * e->eng.timings.size());
    return VXB_OK;
}

int vxb_result_wire_bytes(const vxb_engine* e, uint64_t* out, uint64_t cap) {
    const Engine& g = e->eng;
    if (g.world < 2 || cap < g.wire_sent.size()) return VXB_ECONFIG;
    std::memcpy(out, g.wire_sent.data(), 8 * g.wire_sent.size());
    return VXB_OK;
}

int vxb_set_recv_wire_bytes(vxb_engine* e, const uint64_t* in, uint32_t steps) {
    Engine& g = e->eng;
    if (g.world < 2 || steps != g.res_steps || g.timings.size() != (size_t)steps * g.workers)
        return VXB_ECONFIG;
    const uint32_t W = g.workers, w = g.rank;
    for (uint32_t s = 0; s < steps; ++s) {
        vxb_step_timings& r = g.timings[(size_t)s * W + w];
        r.bytes_recv_intra = r.bytes_recv_inter = 0;
        for (uint32_t h = 0; h < W; ++h)
            if (h != w)
                (h / g.workers_per_node == w / g.workers_per_node ? r.bytes_recv_intra
                                                                    : r.bytes_recv_inter) +=
                    in[(size_t)s * W + h];
    }
    return VXB_OK;
}

int vxb_crossing_matrix(const vxb_engine* e, uint64_t* out, uint64_t cap) {
    const Engine& g = e->eng;
    if (cap < g.crossing.size()) return VXB_ECONFIG;
    std::memcpy(out, g.crossing.data(), 8 * g.crossing.size());
    return VXB_OK;
}

int vxb_schedule_info(const vxb_engine* e, char* out, uint64_t cap) {
    const std::string j = e->eng.schedule_info();
    if (!out || cap < j.size() + 1) return VXB_ECONFIG;
    std::memcpy(out, j.c_str(), j.size() + 1);
    return VXB_OK;
}

double vxb_result_device_ms(const vxb_engine* e) { return e->eng.device_ms; }
double vxb_result_exchange_wait_ms(const vxb_engine* e) { return e->eng.exchange_wait_ms; }
double vxb_result_exchange_arrival_ms(const vxb_engine* e) { return e->eng.exchange_arrival_ms; }
uint64_t vxb_result_h2d_bytes(const vxb_engine* e) { return e->eng.h2d; }
uint64_t vxb_result_d2h_bytes(const vxb_engine* e) { return e->eng.d2h; }
uint64_t vxb_result_launches(const vxb_engine* e) { return e->eng.launches; }

int vxb_set_conductances(vxb_engine* e, uint32_t unit, int receptor, const float* values,
                         uint32_t n) {
    Engine& g = e->eng;
    try {
        if (unit >= g.n_units) throw ConfigError("unit out of range");
        if (receptor < 0 || receptor >= 4) throw ConfigError("receptor out of range");
        if (n != g.units[unit].neurons)
            throw ConfigError("conductance vector size does not match unit");
        // engine.cpp:839-843 writes values in order and throws at the first
        // invalid one, leaving the prefix written: stage the same prefix
        const uint32_t k = g.local(g.unit_worker[unit])
                               ? g.stage_conductances(unit, receptor, values, n)
                               : copy_valid_prefix(nullptr, values, n);
        if (k < n) throw ConfigError("conductance values must be finite and >= 0");
        return VXB_OK;
    } catch (const std::exception& x) {
        g.err = x.what();
        return fail_code(x);
    }
}

// The staging record of (unit, receptor), created with room for a full unit.
int32_t& Engine::slot_of(uint32_t unit, int receptor) {
    const uint32_t key = unit * 4 + (uint32_t)receptor;
    if (cond_slot.size() != 4ull * n_units) cond_slot.assign(4ull * n_units, -1);
    if (cond_slot[key] < 0) {  // new record, with room for a full unit
        const uint32_t full = units[unit].neurons;
        if (cond_total + full > 0xFFFFFFFFull) flush_conductances(true);
        h_cstage.reserve(cond_total + full);
        const uint32_t base = wbase[unit_worker[unit]] + unit_local_base[unit];
        cond_slot[key] = (int32_t)cond_rec.size();
        cond_rec.push_back(make_uint4((uint32_t)cond_total, 4 * base + (uint32_t)receptor, 0u, key));
        cond_total += full;
    }
    return cond_slot[key];
}

// set_conductances of many units in one call, with the sequential
// semantics of calling it item by item (engine.cpp:829-844: argument errors
// stage nothing of the item, a non-finite / negative value stages the
// item's valid prefix; either stops the sequence), but the validation and
// the copies of the items run on the host's cores in parallel.
void Engine::stage_batch(uint32_t count, const uint32_t* uu, const int32_t* rr,
                         const float* const* vals, const uint32_t* ns, uint32_t* failed) {
    *failed = count;
    uint32_t fa = count;  // first argument error
    std::string fa_msg;
    for (uint32_t i = 0; i < count && fa == count; ++i) {
        if (uu[i] >= n_units) fa_msg = "unit out of range";
        else if (rr[i] < 0 || rr[i] >= 4) fa_msg = "receptor out of range";
        else if (ns[i] != units[uu[i]].neurons) fa_msg = "conductance vector size does not match unit";
        if (!fa_msg.empty()) fa = i;
    }
    std::vector<uint32_t> keys(fa);
    bool dup = false;
    {
        std::vector<uint8_t> seen(4ull * n_units, 0);
        for (uint32_t i = 0; i < fa; ++i) {
            keys[i] = uu[i] * 4 + (uint32_t)rr[i];
            dup |= seen[keys[i]] != 0;
            seen[keys[i]] = 1;
        }
    }
    if (dup) {  // the same (unit, receptor) twice: the order matters, stage one by one
        for (uint32_t i = 0; i < count; ++i) {
            *failed = i;
            if (i == fa) throw ConfigError(fa_msg);
            const uint32_t k = local(unit_worker[uu[i]]) ? stage_conductances(uu[i], rr[i], vals[i], ns[i])
                                                         : copy_valid_prefix(nullptr, vals[i], ns[i]);
            if (k < ns[i]) throw ConfigError("conductance values must be finite and >= 0");
        }
        *failed = count;
        return;
    }
    // validate every item (in parallel), find the first invalid one
    std::vector<uint32_t> kv(fa);
    const int nt = std::max(1, std::min(8, omp_get_max_threads()));
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4)
    for (int64_t i = 0; i < (int64_t)fa; ++i) kv[i] = copy_valid_prefix(nullptr, vals[i], ns[i]);
    uint32_t fv = fa;
    for (uint32_t i = 0; i < fa; ++i)
        if (kv[i] < ns[i]) {
            fv = i;
            break;
        }
    const uint32_t last = std::min(fa, fv + (fv < fa ? 1u : 0u));  // items staged
    // records first (creating one may grow the staging buffer), then the
    // destinations
    for (uint32_t i = 0; i < last; ++i)
        if (local(unit_worker[uu[i]])) slot_of(uu[i], rr[i]);
    std::vector<float*> dst(last, nullptr);
    for (uint32_t i = 0; i < last; ++i)
        if (local(unit_worker[uu[i]])) {
            uint4& r = cond_rec[slot_of(uu[i], rr[i])];
            r.z = std::max(r.z, kv[i]);
            dst[i] = h_cstage.p + r.x;
        }
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4)
    for (int64_t i = 0; i < (int64_t)last; ++i)
        if (dst[i]) std::memcpy(dst[i], vals[i], 4ull * kv[i]);
    if (fv < fa) {
        *failed = fv;
        throw ConfigError("conductance values must be finite and >= 0");
    }
    if (fa < count) {
        *failed = fa;
        throw ConfigError(fa_msg);
    }
}

uint32_t Engine::stage_conductances(uint32_t unit, int receptor, const float* values,
                                    uint32_t n) {
    uint4& r = cond_rec[slot_of(unit, receptor)];  // a later set overwrites the earlier values
    const uint32_t k = copy_valid_prefix(h_cstage.p + r.x, values, n);
    r.z = std::max(r.z, k);
    return k;
}

void Engine::flush_conductances(bool sync) {
    if (cond_rec.empty()) return;
    CK(cudaSetDevice(device));
    // compact the records' values (each record reserved a full unit)
    std::vector<uint4> rec(cond_rec.size());
    uint32_t total = 0;
    for (size_t i = 0; i < cond_rec.size(); ++i) {
        const uint4 r = cond_rec[i];
        if (r.x != total) std::memmove(h_cstage.p + total, h_cstage.p + r.x, 4ull * r.z);
        rec[i] = make_uint4(total, r.y, r.z, r.w);
        total += r.z;
    }
    d_cstage.reserve(total);
    d_crec.reserve(rec.size());
    CK(cudaMemcpyAsync(d_cstage.p, h_cstage.p, 4ull * total, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(d_crec.p, rec.data(), 16 * rec.size(), cudaMemcpyHostToDevice, stream));
    const int blocks = (int)std::min<uint32_t>(148 * 8, (total + 255) / 256);
    if (blocks) {  // (records can hold no values: a set that failed at its first value)
        cond_scatter_kernel<<<blocks, 256, 0, stream>>>(d_cstage.p, d_crec.p, (uint32_t)rec.size(),
                                                         total, reinterpret_cast<float*>(d_g.p));
        CK(cudaGetLastError());
        launches += 1;
    }
    // the pinned staging buffer is reused by the next set_conductances; `rec`
    // is pageable, so its copy has been staged by the time the call returns
    if (sync) CK(cudaStreamSynchronize(stream));
    h2d += 4ull * total + 16 * rec.size();
    for (const uint4& r : cond_rec) cond_slot[r.w] = -1;
    cond_rec.clear();
    cond_total = 0;
}

int vxb_set_conductances_batch(vxb_engine* e, uint32_t count, const uint32_t* units,
                               const int32_t* receptors, const float* const* values,
                               const uint32_t* counts, uint32_t* failed_index) {
    Engine& g = e->eng;
    uint32_t dummy = 0;
    try {
        g.stage_batch(count, units, receptors, values, counts, failed_index ? failed_index : &dummy);
        return VXB_OK;
    } catch (const std::exception& x) {
        g.err = x.what();
        return fail_code(x);
    }
}

int vxb_membrane_snapshot(const vxb_engine* e, uint16_t worker, float* out, uint32_t cap) {
    Engine& g = const_cast<Engine&>(e->eng);
    try {
        if (worker >= g.workers) throw ConfigError("worker out of range");
        const uint32_t b = g.wbase[worker], n = g.wbase[worker + 1] - b;
        if (cap < n) throw ConfigError("snapshot buffer too small");
        if (n == 0) return VXB_OK;
        CK(cudaSetDevice(g.device));
        std::vector<uint32_t> bits(n);
        CK(cudaMemcpy(bits.data(), g.d_v.p + b, 4ull * n, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < n; ++i) {
            if (is_refrac(bits[i])) {
                out[i] = g.segs[g.seg_of(b + i)].v_reset;
            } else {
                std::memcpy(out + i, &bits[i], 4);
            }
        }
        return VXB_OK;
    } catch (const std::exception& x) {
        g.err = x.what();
        return fail_code(x);
    }
}

uint32_t vxb_worker_neurons(const vxb_engine* e, uint16_t worker) {
    if (worker >= e->eng.workers) return 0;
    return e->eng.wbase[worker + 1] - e->eng.wbase[worker];
}
uint16_t vxb_workers(const vxb_engine* e) { return e->eng.workers; }
uint32_t vxb_units(const vxb_engine* e) { return e->eng.n_units; }
uint32_t vxb_probes(const vxb_engine* e) { return (uint32_t)e->eng.probes.size(); }

int vxb_create_generated(const vxb_netspec* spec, const vxb_options* opt, vxb_engine** out) {
    *out = nullptr;
    auto* e = new vxb_engine();
    try {
        if (!spec) throw ConfigError("null network spec");
        GenHost h;
        build_gen_host(*spec, h);
        g_gen_host = &h;
        e->eng.load(&h.net, opt, spec);
        g_gen_host = nullptr;
    } catch (const std::exception& x) {
        g_gen_host = nullptr;
        g_create_error = x.what();
        int rc = fail_code(x);
        delete e;
        return rc;
    }
    *out = e;
    return VXB_OK;
}

int vxb_create_member(const vxb_engine* donor, const vxb_network* net,
                      const vxb_netspec* spec, const vxb_options* opt, vxb_engine** out) {
    *out = nullptr;
    auto* e = new vxb_engine();
    try {
        if (!donor) throw ConfigError("null donor engine");
        if (!net == !spec) throw ConfigError("pass either the network tables or the spec");
        e->eng.donor = &donor->eng;
        if (spec) {
            GenHost h;
            build_gen_host(*spec, h);
            g_gen_host = &h;
            e->eng.load(&h.net, opt, nullptr);
            g_gen_host = nullptr;
        } else {
            uint64_t syn = 0;
            for (uint32_t w = 0; w < net->n_workers; ++w) syn += net->workers[w].n_synapses;
            if (syn != donor->eng.n_syn)
                throw ConfigError("ensemble member network does not match the donor's");
            e->eng.load(net, opt, nullptr);
        }
    } catch (const std::exception& x) {
        g_gen_host = nullptr;
        g_create_error = x.what();
        int rc = fail_code(x);
        delete e;
        return rc;
    }
    *out = e;
    return VXB_OK;
}

int vxb_create_generated_rank(const vxb_netspec* spec, const vxb_options* opt, uint32_t rank,
                               uint32_t world, vxb_engine** out) {
    *out = nullptr;
    auto* e = new vxb_engine();
    try {
        if (!spec) throw ConfigError("null network spec");
        if (world == 0 || rank >= world) throw ConfigError("rank out of range");
        if (spec->n_workers != world)
            throw ConfigError("distributed engines need one worker per rank");
        GenHost h;
        build_gen_host(*spec, h, world > 1 ? (int)rank : -1);
        g_gen_host = &h;
        e->eng.load(&h.net, opt, spec, rank, world);
        g_gen_host = nullptr;
    } catch (const std::exception& x) {
        g_gen_host = nullptr;
        g_create_error = x.what();
        int rc = fail_code(x);
        delete e;
        return rc;
    }
    *out = e;
    return VXB_OK;
}

uint64_t vxb_mask_bytes(const vxb_engine* e, uint32_t h) {
    const Engine& g = e->eng;
    if (h >= g.workers) return 0;
    return (g.src_base[h + 1] - g.src_base[h] + 7) / 8;
}

int vxb_mask_out(const vxb_engine* e, uint32_t h, uint8_t* bits, uint64_t cap) {
    const Engine& g = e->eng;
    if (h >= g.workers || cap < vxb_mask_bytes(e, h)) return VXB_ECONFIG;
    const uint32_t b = g.src_base[h], n = g.src_base[h + 1] - b;
    std::memset(bits, 0, (n + 7) / 8);
    if (!g.have_src.empty())
        for (uint32_t i = 0; i < n; ++i)
            if (g.have_src[b + i]) bits[i >> 3] |= (uint8_t)(1u << (i & 7));
    return VXB_OK;
}

int vxb_mask_in(vxb_engine* e, uint32_t h, const uint8_t* bits, uint64_t cap) {
    Engine& g = e->eng;
    try {
        if (h >= g.workers || h >= 64) throw ConfigError("shard out of range");
        if (cap < (g.n + 7) / 8) throw ConfigError("mask buffer too small");
        for (uint32_t i = 0; i < g.n; ++i)
            if ((bits[i >> 3] >> (i & 7)) & 1u) g.h_mask[i] |= 1ull << h;
        CK(cudaSetDevice(g.device));
        if (g.n)
            CK(cudaMemcpy(g.d_mask.p, g.h_mask.data(), 8ull * g.n, cudaMemcpyHostToDevice));
        return VXB_OK;
    } catch (const std::exception& x) {
        g.err = x.what();
        return fail_code(x);
    }
}

int vxb_ipc_handle(const vxb_engine* e, void* out, uint64_t cap) {
    const Engine& g = e->eng;
    if (cap < sizeof(cudaIpcMemHandle_t) || g.world < 2 || !g.d_rx.p) return VXB_ECONFIG;
    cudaSetDevice(g.device);
    cudaIpcMemHandle_t hd;
    if (cudaIpcGetMemHandle(&hd, g.d_rx.p) != cudaSuccess) return VXB_ESIM;
    std::memcpy(out, &hd, sizeof hd);
    return VXB_OK;
}

int vxb_connect_peers(vxb_engine* e, const void* handles, uint64_t stride) {
    Engine& g = e->eng;
    try {
        if (g.world < 2) return VXB_OK;
        CK(cudaSetDevice(g.device));
        for (uint32_t d = 0; d < g.world; ++d) {
            if (d == g.rank) continue;
            cudaIpcMemHandle_t hd;
            std::memcpy(&hd, static_cast<const unsigned char*>(handles) + stride * d, sizeof hd);
            void* base = nullptr;
            CK(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
            g.peer_base[d] = base;
            // peer d's region: slots of every shard but d, in shard order
            size_t off = 0;
            for (uint32_t hh = 0; hh < g.rank; ++hh)
                if (hh != d) off += ((4ull * kSlots * g.h_ex.cap[hh] + 15) & ~15ull) + 32;
            unsigned char* slot = static_cast<unsigned char*>(base) + off;
            g.h_ex.tx_ids[d] = reinterpret_cast<uint32_t*>(slot);
            g.h_ex.tx_meta[d] = reinterpret_cast<uint32_t*>(
                slot + ((4ull * kSlots * g.h_ex.cap[g.rank] + 15) & ~15ull));
        }
        CK(cudaMemcpy(g.d_ex.p, &g.h_ex, sizeof g.h_ex, cudaMemcpyHostToDevice));
        return VXB_OK;
    } catch (const std::exception& x) {
        g.err = x.what();
        return fail_code(x);
    }
}

int vxb_generate_worker_table(const vxb_netspec* spec, int device, uint16_t worker,
                              vxb_neuron* neurons, uint32_t n_cap, vxb_syn_entry* synapses,
                              uint64_t syn_cap, uint64_t* row_base) {
    try {
        if (!spec) throw ConfigError("null network spec");
        GenHost h;
        build_gen_host(*spec, h);
        if (worker >= spec->n_workers) throw ConfigError("worker out of range");
        const auto& recs = h.recs[worker];
        if (n_cap < recs.size() || syn_cap < h.nsyn[worker])
            throw ConfigError("output buffers too small");
        std::vector<uint64_t> rb(recs.size() + 1, 0);
        for (size_t i = 0; i < recs.size(); ++i) rb[i + 1] = rb[i] + recs[i].row_len;
        std::vector<uint32_t> wb(spec->n_workers, 0);
        for (uint32_t w = 1; w < spec->n_workers; ++w)
            wb[w] = wb[w - 1] + (uint32_t)h.recs[w - 1].size();
        const uint64_t nall = wb.back() + h.recs.back().size();
        CK(cudaSetDevice(device));
        cudaStream_t st = nullptr;
        CK(cudaStreamCreate(&st));
        GenDevTables T;
        T.upload(h, *spec, wb, st);
        DevBuf<uint64_t> d_rb;
        DevBuf<uint4> d_rows;
        DevBuf<unsigned long long> have;
        d_rb.alloc(rb.size());
        d_rows.alloc(std::max<uint64_t>(1, h.nsyn[worker]));
        have.alloc(std::max<uint64_t>(1, nall));
        have.zero(st);
        CK(cudaMemcpyAsync(d_rb.p, rb.data(), 8 * rb.size(), cudaMemcpyHostToDevice, st));
        if (h.total_neurons)
            gen_kernel<2><<<148 * 8, 256, 0, st>>>(T.G, 0, h.total_neurons, nullptr, nullptr,
                                                   nullptr, have.p, nullptr, worker, d_rb.p,
                                                   d_rows.p);
        CK(cudaGetLastError());
        T.check(st, nullptr);
        std::vector<unsigned long long> hv(nall);
        if (nall) CK(cudaMemcpy(hv.data(), have.p, 8 * nall, cudaMemcpyDeviceToHost));
        if (h.nsyn[worker])
            CK(cudaMemcpy(synapses, d_rows.p, 16 * h.nsyn[worker], cudaMemcpyDeviceToHost));
        cudaStreamDestroy(st);
        for (size_t i = 0; i < recs.size(); ++i) {
            neurons[i] = recs[i];
            neurons[i].dst_mask = hv[wb[worker] + i];
        }
        std::memcpy(row_base, rb.data(), 8 * rb.size());
        return VXB_OK;
    } catch (const std::exception& x) {
        g_create_error = x.what();
        return fail_code(x);
    }
}

uint64_t vxb_fnv1a(const void* data, uint64_t n, uint64_t h) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

int vxb_debug_stream_normal(int device, const uint64_t* base, const uint64_t* k, uint64_t n,
                            double* out) {
    try {
        CK(cudaSetDevice(device));
        DevBuf<uint64_t> b, kk;
        DevBuf<double> o;
        b.alloc(n);
        kk.alloc(n);
        o.alloc(n);
        CK(cudaMemcpy(b.p, base, 8 * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(kk.p, k, 8 * n, cudaMemcpyHostToDevice));
        debug_normal_kernel<<<1184, 256>>>(b.p, kk.p, n, o.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, o.p, 8 * n, cudaMemcpyDeviceToHost));
        return VXB_OK;
    } catch (const std::exception& x) {
        g_create_error = x.what();
        return fail_code(x);
    }
}

int vxb_debug_stream_xi(int device, const uint64_t* base, const uint64_t* k, uint64_t n,
                        float* out) {
    try {
        CK(cudaSetDevice(device));
        DevBuf<uint64_t> b, kk;
        DevBuf<float> o;
        b.alloc(n);
        kk.alloc(n);
        o.alloc(n);
        CK(cudaMemcpy(b.p, base, 8 * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(kk.p, k, 8 * n, cudaMemcpyHostToDevice));
        debug_xi_kernel<<<1184, 256>>>(b.p, kk.p, n, o.p);
        CK(cudaGetLastError());
        CK(cudaMemcpy(out, o.p, 4 * n, cudaMemcpyDeviceToHost));
        return VXB_OK;
    } catch (const std::exception& x) {
        g_create_error = x.what();
        return fail_code(x);
    }
}

int vxb_set_hemodynamics(vxb_engine* e, const vxb_hemo_params* p, double baseline_hz,
                         uint32_t sample_every, const vxb_hemo_state* init) {
    Engine& g = e->eng;
    try {
        if (!p) throw ConfigError("hemodynamics: null parameters");
        g.set_hemodynamics(*p, baseline_hz, sample_every, init);
        return VXB_OK;
    } catch (const std::exception& x) {
        g.err = x.what();
        return fail_code(x);
    }
}

int vxb_hemo_get_state(const vxb_engine* e, vxb_hemo_state* out, uint32_t cap) {
    const Engine& g = e->eng;
    if (!g.hemo_on || cap < g.n_voxels) return VXB_ECONFIG;
    if (cudaSetDevice(g.device) != cudaSuccess ||
        cudaMemcpy(out, g.d_hemo.p, sizeof(vxb_hemo_state) * g.n_voxels,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
        return VXB_ESIM;
    return VXB_OK;
}

uint64_t vxb_result_bold_size(const vxb_engine* e) { return e->eng.bold.size(); }

int vxb_result_voxel_counts(const vxb_engine* e, uint32_t* out, uint64_t cap) {
    if (!e->eng.hemo_on || cap < e->eng.vcounts.size()) return VXB_ECONFIG;
    std::memcpy(out, e->eng.vcounts.data(), 4 * e->eng.vcounts.size());
    return VXB_OK;
}

int vxb_hemo_feed_counts(vxb_engine* e, const uint32_t* counts, uint32_t steps) {
    Engine& g = e->eng;
    try {
        if (!g.hemo_on) throw ConfigError("hemodynamics are not enabled");
        if (g.world == 1) throw ConfigError("one GPU: advance() already drove the hemodynamics");
        if (steps != g.res_steps) throw ConfigError("counts must cover the last advance");
        CK(cudaSetDevice(g.device));
        const size_t nc = (size_t)steps * g.n_voxels;
        g.bold.assign((size_t)(steps / g.hemo_every) * g.n_voxels, 0.0);
        g.d_bold.reserve(std::max<size_t>(1, g.bold.size()));
        g.d_vcounts.reserve(std::max<size_t>(1, nc));
        const unsigned long long none = ~0ull;
        CK(cudaMemcpyAsync(g.d_hemo_err.p, &none, 8, cudaMemcpyHostToDevice, g.stream));
        if (nc) CK(cudaMemcpyAsync(g.d_vcounts.p, counts, 4 * nc, cudaMemcpyHostToDevice, g.stream));
        if (steps) g.run_hemo(0, steps);
        if (!g.fetch_bold()) throw HemoError("hemodynamic state diverged");
        return VXB_OK;
    } catch (const std::exception& x) {
        g.err = x.what();
        return fail_code(x);
    }
}

int vxb_result_bold(const vxb_engine* e, double* out, uint64_t cap) {
    if (cap < e->eng.bold.size()) return VXB_ECONFIG;
    std::memcpy(out, e->eng.bold.data(), 8 * e->eng.bold.size());
    return VXB_OK;
}

int vxb_debug_bold_from_drive(int device, const vxb_hemo_params* p, const double* z,
                              uint32_t steps, uint32_t n_series, double dt_s,
                              uint32_t sample_every, vxb_hemo_state* state, double* out) {
    try {
        if (!p) throw ConfigError("hemodynamics: null parameters");
        validate_hemo(*p, 1.0, sample_every);
        int nd = 0;
        if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0)
            throw SimError("no CUDA device available (the engine has no CPU fallback)");
        CK(cudaSetDevice(device));
        const size_t nz = (size_t)steps * n_series, no = (size_t)(steps / sample_every) * n_series;
        DevBuf<double> dz, dout;
        DevBuf<HemoStateDev> dst;
        DevBuf<unsigned long long> derr;
        dz.alloc(std::max<size_t>(1, nz));
        dout.alloc(std::max<size_t>(1, no));
        dst.alloc(std::max<uint32_t>(1, n_series));
        derr.alloc(1);
        const unsigned long long none = ~0ull;
        if (nz) CK(cudaMemcpy(dz.p, z, 8 * nz, cudaMemcpyHostToDevice));
        if (n_series) CK(cudaMemcpy(dst.p, state, sizeof(HemoStateDev) * n_series, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(derr.p, &none, 8, cudaMemcpyHostToDevice));
        const HemoParamsDev hp{p->kappa, p->gamma, p->tau, p->alpha, p->e0, p->v0};
        if (n_series)
            bold_drive_kernel<<<(n_series + 127) / 128, 128>>>(dz.p, steps, n_series, hp, dt_s,
                                                               sample_every, dst.p, dout.p, derr.p);
        CK(cudaGetLastError());
        unsigned long long err = 0;
        CK(cudaMemcpy(&err, derr.p, 8, cudaMemcpyDeviceToHost));
        if (no) CK(cudaMemcpy(out, dout.p, 8 * no, cudaMemcpyDeviceToHost));
        if (n_series) CK(cudaMemcpy(state, dst.p, sizeof(HemoStateDev) * n_series, cudaMemcpyDeviceToHost));
        if (err != ~0ull) throw SimError("hemodynamic state diverged");
        return VXB_OK;
    } catch (const std::exception& x) {
        g_create_error = x.what();
        return fail_code(x);
    }
}

// Ensemble members advanced together (assim.cpp:231-233 advances them one
// after another): every member's chunk is launched on its own stream with an
// equal share of the SMs, so the members run concurrently over the shared
// tables, then each finishes and reads back its own results.  Members on the
// SM-tile path (one CTA per SM owns a tile) cannot share the SMs and advance
// one after another instead.
int vxb_advance_members(vxb_engine** members, uint32_t count, uint32_t steps) {
    if (count == 0) return VXB_OK;
    std::vector<Engine*> es;
    for (uint32_t m = 0; m < count; ++m) es.push_back(&members[m]->eng);
    const Engine& e0 = *es[0];
    bool together = e0.world == 1 && !e0.tile_path && count > 1;
    for (Engine* e : es)
        together = together && e->world == 1 && !e->tile_path && e->device == e0.device &&
                   e->n == e0.n && e->step_done == e0.step_done && !e->failed &&
                   e->log_spikes() == e0.log_spikes();
    int rc = VXB_OK;
    auto fail = [&](Engine* e, const std::exception& x) {
        e->err = x.what();
        if (!dynamic_cast<const HemoError*>(&x)) e->failed = true;
        if (rc == VXB_OK) rc = fail_code(x);
    };
    if (!together) {
        for (uint32_t m = 0; m < count; ++m) {
            const int r = vxb_advance(members[m], steps);
            if (r != VXB_OK && rc == VXB_OK) rc = r;
        }
        return rc;
    }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e0.device) != cudaSuccess)
        return VXB_ESIM;
    const int per_sm = std::max(1, e0.grid / std::max(1, sms));
    const int share = per_sm * std::max(1, sms / (int)count);  // CTAs per member
    std::vector<uint32_t> chunk(count, 0);
    std::vector<uint8_t> alive(count, 1);
    for (uint32_t m = 0; m < count; ++m) {
        try {
            chunk[m] = es[m]->advance_begin(steps);
        } catch (const std::exception& x) {
            fail(es[m], x);
            alive[m] = 0;
        }
    }
    if (steps == 0) return rc;
    std::vector<std::vector<unsigned long long>> ph(count);
    const uint32_t ch = chunk[0] ? chunk[0] : steps;
    for (uint32_t rel0 = 0; rel0 < steps; rel0 += ch) {
        const uint32_t cs = std::min(ch, steps - rel0);
        for (uint32_t m = 0; m < count; ++m) {
            if (!alive[m]) continue;
            try {
                es[m]->launch_chunk(es[m]->step_done + rel0, rel0, cs, steps, share);
            } catch (const std::exception& x) {
                fail(es[m], x);
                alive[m] = 0;
            }
        }
        for (uint32_t m = 0; m < count; ++m) {
            if (!alive[m]) continue;
            try {
                es[m]->finish_chunk(rel0, cs, steps);
                es[m]->chunk_post(rel0, cs, ph[m]);
            } catch (const std::exception& x) {
                fail(es[m], x);
                alive[m] = 0;
            }
        }
    }
    for (uint32_t m = 0; m < count; ++m) {
        if (!alive[m]) continue;
        try {
            es[m]->advance_end(steps, ph[m]);
        } catch (const std::exception& x) {
            fail(es[m], x);
        }
    }
    return rc;
}

int vxb_run_simulation(const vxb_network* net, const vxb_options* opt, uint32_t steps,
                       vxb_engine** out) {
    int rc = vxb_create(net, opt, out);
    if (rc != VXB_OK) return rc;
    return vxb_advance(*out, steps);
}

}  // extern "C"

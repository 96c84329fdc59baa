// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle/).
//
// A thin extern "C" veneer over the UNMODIFIED reference engine compiled from
// /root/reference/proj/src (see oracle/Makefile).  It lets the Python tests
// and bench.py's CPU-baseline leg
//   * build networks with the reference's own pipeline
//     (build_connectome / build_layout / sample_synapses / emit_tables,
//      pipeline.cpp:49-125),
//   * export the resulting NetworkTables in the vxb.h table layout, and
//   * run the reference SimInstance (engine.cpp) on the same inputs,
// so GPU results can be compared against the reference on identical tables.
// Nothing in the product path links this file.

#include "voxsim/config.hpp"
#include "voxsim/connectome.hpp"
#include "voxsim/engine.hpp"
#include "voxsim/assim.hpp"
#include "voxsim/hemo.hpp"
#include "voxsim/layout.hpp"
#include "voxsim/model.hpp"
#include "voxsim/netgen.hpp"
#include "voxsim/partition.hpp"
#include "voxsim/pipeline.hpp"
#include "voxsim/rng.hpp"
#include "voxsim/util.hpp"

#include <json.hpp>

#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "vxb.h"

using namespace voxsim;
using nlohmann::json;

namespace {

struct RefNet {
    RunConfig cfg;
    ConnectomeGraph graph;
    NetworkLayout layout;
    NetworkTables tables;
    uint64_t synapse_count = 0;
    double build_seconds = 0;
    std::vector<std::vector<uint64_t>> crossing;  // BuiltNetwork::crossing (pipeline.cpp:122)
};

struct RefSim {
    std::unique_ptr<SimInstance> sim;
    RunResult last;
    double advance_seconds = 0;
};

void set_err(char* err, int errlen, const char* kind, const std::string& what) {
    if (!err || errlen <= 0) return;
    std::string s = std::string(kind) + ": " + what;
    std::strncpy(err, s.c_str(), static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = 0;
}

template <typename F>
int guarded(char* err, int errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        set_err(err, errlen, "ConfigError", e.what());
        return 2;
    } catch (const SimError& e) {
        set_err(err, errlen, "SimError", e.what());
        return 3;
    } catch (const std::exception& e) {
        set_err(err, errlen, "Error", e.what());
        return 4;
    }
}

SimOptions parse_options(const std::string& text) {
    json j = json::parse(text);
    SimOptions o;
    if (j.contains("steps")) o.steps = j["steps"].get<uint32_t>();
    if (j.contains("dt_ms")) o.dt_ms = j["dt_ms"].get<double>();
    if (j.contains("scheduler")) o.scheduler = j["scheduler"].get<std::string>();
    if (j.contains("transport")) o.transport = j["transport"].get<std::string>();
    if (j.contains("workers_per_node"))
        o.workers_per_node = j["workers_per_node"].get<uint16_t>();
    if (j.contains("recv_timeout_ms")) o.recv_timeout_ms = j["recv_timeout_ms"].get<int>();
    if (j.contains("record_raster")) o.record_raster = j["record_raster"].get<bool>();
    if (j.contains("record_timings")) o.record_timings = j["record_timings"].get<bool>();
    if (j.contains("probe_gids"))
        o.probe_gids = j["probe_gids"].get<std::vector<uint64_t>>();
    if (j.contains("injections"))
        for (const auto& x : j["injections"]) {
            Injection inj;
            inj.from_step = x.at(0).get<uint32_t>();
            inj.to_step = x.at(1).get<uint32_t>();
            inj.voxel = x.at(2).get<uint32_t>();
            inj.current_pa = x.at(3).get<float>();
            o.injections.push_back(inj);
        }
    if (j.contains("forced_spikes"))
        for (const auto& x : j["forced_spikes"]) {
            ForcedSpike f;
            f.step = x.at(0).get<uint32_t>();
            f.gid = x.at(1).get<uint64_t>();
            o.forced_spikes.push_back(f);
        }
    return o;
}

} // namespace

extern "C" {

// ---------------------------------------------------------------- networks

// Builds a network with the reference pipeline from a RunConfig JSON
// (config.hpp:40-60).  even_workers > 0 replaces the configured partition
// with unit u -> worker u % even_workers, the helper the reference engine
// tests use (test_engine.cpp:40-47).
void* ref_build(const char* cfg_json, int even_workers, char* err, int errlen) {
    RefNet* out = nullptr;
    int rc = guarded(err, errlen, [&] {
        auto t0 = std::chrono::steady_clock::now();
        auto net = std::make_unique<RefNet>();
        net->cfg = parse_config(cfg_json);
        if (even_workers <= 0) {
            BuiltNetwork b = build_network(net->cfg);
            net->graph = std::move(b.graph);
            net->layout = std::move(b.layout);
            net->tables = std::move(b.tables);
            net->synapse_count = b.synapse_count;
            net->crossing = std::move(b.crossing);
        } else {
            net->graph = build_connectome(net->cfg);
            MicrocolumnSpec mc;
            net->layout = build_layout(net->cfg, net->graph, mc);
            IntraMatrices intra = IntraMatrices::defaults(mc);
            GlobalNetwork g = sample_synapses(net->layout, net->graph, intra,
                                              net->cfg.seed);
            net->synapse_count = g.synapse_count;
            PartitionMap p;
            p.worker_count = static_cast<uint16_t>(even_workers);
            p.unit_worker.resize(net->layout.unit_count());
            for (uint32_t u = 0; u < net->layout.unit_count(); ++u)
                p.unit_worker[u] = static_cast<uint16_t>(u % even_workers);
            net->tables = emit_tables(net->layout, g, p, net->cfg.seed);
        }
        net->build_seconds = std::chrono::duration<double>(
                                 std::chrono::steady_clock::now() - t0)
                                 .count();
        out = net.release();
    });
    return rc == 0 ? out : nullptr;
}

void ref_free(void* h) { delete static_cast<RefNet*>(h); }

// save_tables / load_tables (netgen.cpp:466-539) for the table-file tests.
int ref_save_tables(void* h, const char* dir, char* err, int errlen) {
    return guarded(err, errlen, [&] { save_tables(static_cast<RefNet*>(h)->tables, dir); });
}

// A RefNet whose tables come from load_tables(dir); the layout is rebuilt
// from the config, as cmd_simulate --tables does (voxsim.cpp:149-156).
void* ref_load_net(const char* cfg_json, const char* dir, char* err, int errlen) {
    RefNet* out = nullptr;
    int rc = guarded(err, errlen, [&] {
        auto net = std::make_unique<RefNet>();
        net->cfg = parse_config(cfg_json);
        net->graph = build_connectome(net->cfg);
        MicrocolumnSpec mc;
        net->layout = build_layout(net->cfg, net->graph, mc);
        net->tables = load_tables(dir);
        for (const auto& w : net->tables.workers) net->synapse_count += w.synapses.size();
        out = net.release();
    });
    return rc == 0 ? out : nullptr;
}

double ref_build_seconds(void* h) { return static_cast<RefNet*>(h)->build_seconds; }
uint64_t ref_seed(void* h) { return static_cast<RefNet*>(h)->cfg.seed; }
uint32_t ref_n_workers(void* h) {
    return static_cast<uint32_t>(static_cast<RefNet*>(h)->tables.workers.size());
}
uint32_t ref_n_units(void* h) { return static_cast<RefNet*>(h)->layout.unit_count(); }
uint32_t ref_n_voxels(void* h) {
    return static_cast<uint32_t>(static_cast<RefNet*>(h)->layout.voxels.size());
}
uint64_t ref_total_neurons(void* h) { return static_cast<RefNet*>(h)->layout.total_neurons; }
uint64_t ref_synapse_count(void* h) { return static_cast<RefNet*>(h)->synapse_count; }
// BuiltNetwork::crossing [src worker][dst worker] (netgen.cpp:331-355); 0 if
// the network was not built through build_network
int ref_crossing(void* h, uint64_t* out, uint32_t workers) {
    const auto& c = static_cast<RefNet*>(h)->crossing;
    if (c.size() != workers) return 0;
    for (uint32_t a = 0; a < workers; ++a)
        for (uint32_t b = 0; b < workers; ++b) out[a * workers + b] = c[a][b];
    return 1;
}
uint32_t ref_worker_n(void* h, uint32_t w) {
    return static_cast<uint32_t>(static_cast<RefNet*>(h)->tables.workers.at(w).neurons.size());
}
uint64_t ref_worker_nsyn(void* h, uint32_t w) {
    return static_cast<RefNet*>(h)->tables.workers.at(w).synapses.size();
}

void ref_units(void* h, vxb_unit* units, uint16_t* unit_worker, uint32_t* unit_local_base) {
    RefNet& n = *static_cast<RefNet*>(h);
    for (uint32_t u = 0; u < n.layout.unit_count(); ++u) {
        const Unit& x = n.layout.units[u];
        vxb_unit r{};
        r.gid_base = x.gid_base;
        r.voxel = x.voxel;
        r.neurons = x.neurons;
        r.pop = x.pop;
        r.excitatory = x.excitatory ? 1 : 0;
        units[u] = r;
        unit_worker[u] = n.tables.unit_worker[u];
        unit_local_base[u] = n.tables.unit_local_base[u];
    }
}

void ref_worker_neurons(void* h, uint32_t w, vxb_neuron* out) {
    const WorkerTable& t = static_cast<RefNet*>(h)->tables.workers.at(w);
    for (size_t i = 0; i < t.neurons.size(); ++i) {
        const NeuronRecord& r = t.neurons[i];
        vxb_neuron x{};
        x.gid = r.gid;
        x.dst_mask = r.dst_mask;
        x.voxel = r.voxel;
        x.unit = r.unit;
        x.row_len = r.row_len;
        x.refractory_steps = r.refractory_steps;
        x.pop = r.pop;
        x.excitatory = r.excitatory;
        x.capacitance = r.capacitance;
        x.g_leak = r.g_leak;
        x.e_leak = r.e_leak;
        x.v_threshold = r.v_threshold;
        x.v_reset = r.v_reset;
        for (int k = 0; k < kReceptors; ++k) {
            x.e_rev[k] = r.e_rev[k];
            x.tau[k] = r.tau[k];
            x.omega[k] = r.omega[k];
            x.g[k] = r.g[k];
        }
        x.ou_mean = r.ou_mean;
        x.ou_sigma = r.ou_sigma;
        x.ou_tau = r.ou_tau;
        x.v_init = r.v_init;
        out[i] = x;
    }
}

void ref_worker_synapses(void* h, uint32_t w, vxb_syn_entry* out, uint64_t* row_base) {
    const WorkerTable& t = static_cast<RefNet*>(h)->tables.workers.at(w);
    static_assert(sizeof(SynEntry) == sizeof(vxb_syn_entry));
    if (!t.synapses.empty())
        std::memcpy(out, t.synapses.data(), t.synapses.size() * sizeof(SynEntry));
    for (size_t i = 0; i < t.row_base.size(); ++i) row_base[i] = t.row_base[i];
}

// ------------------------------------------------------------------ engine

void* ref_sim_create(void* h, const char* opts_json, char* err, int errlen) {
    RefSim* out = nullptr;
    int rc = guarded(err, errlen, [&] {
        RefNet& n = *static_cast<RefNet*>(h);
        auto s = std::make_unique<RefSim>();
        s->sim = std::make_unique<SimInstance>(n.tables, n.layout,
                                               parse_options(opts_json));
        out = s.release();
    });
    return rc == 0 ? out : nullptr;
}

void ref_sim_free(void* s) { delete static_cast<RefSim*>(s); }

int ref_sim_advance(void* sp, uint32_t steps, char* err, int errlen) {
    RefSim& s = *static_cast<RefSim*>(sp);
    return guarded(err, errlen, [&] {
        auto t0 = std::chrono::steady_clock::now();
        s.last = s.sim->advance(steps);
        s.advance_seconds = std::chrono::duration<double>(
                                std::chrono::steady_clock::now() - t0)
                                .count();
    });
}

double ref_sim_advance_seconds(void* sp) { return static_cast<RefSim*>(sp)->advance_seconds; }
uint32_t ref_sim_current_step(void* sp) { return static_cast<RefSim*>(sp)->sim->current_step(); }
uint64_t ref_res_total_spikes(void* sp) { return static_cast<RefSim*>(sp)->last.total_spikes; }
uint32_t ref_res_steps_done(void* sp) { return static_cast<RefSim*>(sp)->last.steps_done; }
uint64_t ref_res_raster_size(void* sp) { return static_cast<RefSim*>(sp)->last.raster.size(); }

void ref_res_raster(void* sp, vxb_raster_event* out) {
    const auto& r = static_cast<RefSim*>(sp)->last.raster;
    for (size_t i = 0; i < r.size(); ++i) {
        vxb_raster_event e{};
        e.step = r[i].step;
        e.worker = r[i].worker;
        e.local = r[i].local;
        e.gid = r[i].gid;
        out[i] = e;
    }
}

void ref_res_rates(void* sp, uint32_t* out) {
    const auto& c = static_cast<RefSim*>(sp)->last.rates.counts;
    size_t k = 0;
    for (const auto& row : c)
        for (uint32_t x : row) out[k++] = x;
}

uint32_t ref_res_n_probes(void* sp) {
    return static_cast<uint32_t>(static_cast<RefSim*>(sp)->last.probes.size());
}

void ref_res_probes(void* sp, float* v, float* i_syn) {
    const auto& p = static_cast<RefSim*>(sp)->last.probes;
    size_t k = 0;
    for (const auto& tr : p) {
        for (size_t t = 0; t < tr.v.size(); ++t, ++k) {
            v[k] = tr.v[t];
            i_syn[k] = tr.i_syn[t];
        }
    }
}

void ref_res_flops(void* sp, uint64_t* out) {
    const FlopCounters& f = static_cast<RefSim*>(sp)->last.flops;
    out[0] = f.membrane;
    out[1] = f.gating_inner;
    out[2] = f.gating_outer;
    out[3] = f.gating_decay;
    out[4] = f.current;
}

uint64_t ref_res_timings_size(void* sp) { return static_cast<RefSim*>(sp)->last.timings.size(); }

void ref_res_timings(void* sp, vxb_step_timings* out) {
    const auto& rows = static_cast<RefSim*>(sp)->last.timings;
    for (size_t i = 0; i < rows.size(); ++i) {
        const StepTimings& r = rows[i];
        vxb_step_timings x{};
        x.step = r.step;
        x.worker = r.worker;
        int64_t t[11] = {r.t1, r.t2, r.t3, r.t4, r.t5, r.t6, r.t7, r.t8, r.t9, r.t10, r.t11};
        for (int k = 0; k < 11; ++k) x.t[k] = t[k];
        x.send_intra_ns = r.send_intra_ns;
        x.send_inter_ns = r.send_inter_ns;
        x.recv_intra_ns = r.recv_intra_ns;
        x.recv_inter_ns = r.recv_inter_ns;
        x.bytes_sent_intra = r.bytes_sent_intra;
        x.bytes_sent_inter = r.bytes_sent_inter;
        x.bytes_recv_intra = r.bytes_recv_intra;
        x.bytes_recv_inter = r.bytes_recv_inter;
        x.spikes = r.spikes;
        out[i] = x;
    }
}

int ref_sim_set_conductances(void* sp, uint32_t unit, int receptor, const float* v,
                             uint32_t n, char* err, int errlen) {
    RefSim& s = *static_cast<RefSim*>(sp);
    return guarded(err, errlen, [&] {
        s.sim->set_conductances(unit, receptor, std::vector<float>(v, v + n));
    });
}

int ref_sim_snapshot(void* sp, uint16_t w, float* out, uint32_t cap, char* err, int errlen) {
    RefSim& s = *static_cast<RefSim*>(sp);
    return guarded(err, errlen, [&] {
        std::vector<float> v = s.sim->membrane_snapshot(w);
        if (v.size() > cap) throw ConfigError("snapshot buffer too small");
        std::memcpy(out, v.data(), v.size() * sizeof(float));
    });
}

// -------------------------------------------------- rng / model primitives
// Direct wrappers of the reference's inline definitions (rng.hpp, model.hpp)
// so the C restatement in oracle/voxsim_oracle.c can be pinned against them.

uint64_t ref_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t ref_mix_key2(uint64_t a, uint64_t b) { return mix_key(a, b); }
uint64_t ref_mix_key3(uint64_t a, uint64_t b, uint64_t c) { return mix_key(a, b, c); }
uint64_t ref_stream_word(uint64_t base, uint64_t k) { return stream_word(base, k); }
double ref_stream_u01(uint64_t base, uint64_t k) { return stream_u01(base, k); }
double ref_stream_normal(uint64_t base, uint64_t k) { return stream_normal(base, k); }
uint64_t ref_stream_below(uint64_t base, uint64_t k, uint64_t n) { return stream_below(base, k, n); }
int32_t ref_quantize_weight(double w) { return quantize_weight(w); }
float ref_dequantize_weight(int64_t q) { return dequantize_weight(q); }
float ref_gating_kernel(float j, float dt, float tau, float omega, float p) {
    return gating_kernel(j, dt, tau, omega, p);
}
float ref_membrane_kernel(float v, float dtc, float gl, float el, float isyn, float iou) {
    return membrane_kernel(v, dtc, gl, el, isyn, iou);
}
float ref_current_kernel(float v, const float* j, const float* g, const float* e) {
    std::array<float, kReceptors> jj{j[0], j[1], j[2], j[3]}, gg{g[0], g[1], g[2], g[3]},
        ee{e[0], e[1], e[2], e[3]};
    return current_kernel(v, jj, gg, ee);
}
float ref_ou_kernel(float i, float dt, float mean, float sigma, float tau, float xi) {
    OuParams p;
    p.mean = mean;
    p.sigma = sigma;
    p.tau = tau;
    return ou_kernel(i, dt, p, xi);
}
// OU noise sample as the engine consumes it (engine.cpp:551-553).
float ref_ou_xi(uint64_t seed, uint64_t gid, uint64_t step) {
    return static_cast<float>(stream_normal(mix_key(seed, rngstream::ou_noise, gid), step));
}

// ---- hemodynamics (hemo.cpp) ------------------------------------------------
// p = {kappa, gamma, tau, alpha, e0, v0}; st = {s, f, v, q} in/out.
static HemoParams hemo_params(const double* p) {
    HemoParams h;
    h.kappa = p[0];
    h.gamma = p[1];
    h.tau = p[2];
    h.alpha = p[3];
    h.e0 = p[4];
    h.v0 = p[5];
    return h;
}
// bold_from_drive (hemo.cpp:49-62) for one drive series.
int ref_bold_from_drive(const double* p, const double* z, uint32_t steps, double dt_s,
                        uint32_t sample_every, double* st, double* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        HemoState h{st[0], st[1], st[2], st[3]};
        std::vector<double> zz(z, z + steps);
        std::vector<double> b = bold_from_drive(zz, dt_s, sample_every, hemo_params(p), &h);
        std::copy(b.begin(), b.end(), out);
        st[0] = h.s;
        st[1] = h.f;
        st[2] = h.v;
        st[3] = h.q;
    });
}
// window_bold (assim.cpp:51-71; it lives in an anonymous namespace there, so
// the drive is restated here around the reference's own step_hemodynamics /
// bold_signal): counts[unit][steps], unit_voxel[units], vox_n[voxels];
// states[voxels][4] in/out; out[steps / sample_every][voxels].
int ref_window_bold(const double* p, const uint32_t* counts, uint32_t n_units, uint32_t steps,
                    const uint32_t* unit_voxel, uint32_t n_voxels, const uint64_t* vox_n,
                    double dt_s, double baseline_hz, uint32_t sample_every, double* states,
                    double* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const HemoParams hp = hemo_params(p);
        hp.validate();
        for (uint32_t t = 0; t < steps; ++t) {
            std::vector<uint32_t> vc(n_voxels, 0);  // RateSeries::voxel_counts (stats.cpp:193-201)
            for (uint32_t u = 0; u < n_units; ++u) vc[unit_voxel[u]] += counts[(size_t)u * steps + t];
            for (uint32_t v = 0; v < n_voxels; ++v) {
                double hz = vox_n[v] > 0 ? vc[v] / (static_cast<double>(vox_n[v]) * dt_s) : 0.0;
                HemoState h{states[4 * v], states[4 * v + 1], states[4 * v + 2], states[4 * v + 3]};
                step_hemodynamics(h, hz / baseline_hz, dt_s, hp);
                states[4 * v] = h.s;
                states[4 * v + 1] = h.f;
                states[4 * v + 2] = h.v;
                states[4 * v + 3] = h.q;
                if ((t + 1) % sample_every == 0)
                    out[(size_t)((t + 1) / sample_every - 1) * n_voxels + v] = bold_signal(h, hp);
            }
        }
    });
}

// ---- assimilation (assim.cpp) -----------------------------------------------
// d = {dt_ms, obs_noise_sd, inflation, min_spread, prior_sd, baseline_hz,
//      divergence_factor, kappa, gamma, tau, alpha, e0, v0};
// iv = {members, windows, window_steps, divergence_patience, seed};
// tg = (unit, receptor) pairs.
static AssimOptions assim_opts(const double* d, const int64_t* iv, const uint32_t* tg,
                               uint32_t nt) {
    AssimOptions o;
    o.dt_ms = d[0];
    o.obs_noise_sd = d[1];
    o.inflation = d[2];
    o.min_spread = d[3];
    o.prior_sd = d[4];
    o.baseline_hz = d[5];
    o.divergence_factor = d[6];
    o.hemo = hemo_params(d + 7);
    o.members = static_cast<int>(iv[0]);
    o.windows = static_cast<uint32_t>(iv[1]);
    o.window_steps = static_cast<uint32_t>(iv[2]);
    o.divergence_patience = static_cast<int>(iv[3]);
    o.seed = static_cast<uint64_t>(iv[4]);
    for (uint32_t k = 0; k < nt; ++k) o.targets.push_back({tg[2 * k], static_cast<int>(tg[2 * k + 1])});
    return o;
}
// The population g_location / g_scale of a unit (layout.pop_of_unit).
void ref_unit_pop(void* h, uint32_t unit, double* gloc, double* gscale) {
    const PopulationSpec& ps = static_cast<RefNet*>(h)->layout.pop_of_unit(unit);
    for (int r = 0; r < 4; ++r) {
        gloc[r] = ps.g_location[r];
        gscale[r] = ps.g_scale[r];
    }
}
// assimilate (assim.cpp:181-299): stats[w] = {window, innovation_rms,
// pearson_r, mean_spread, target_mean[nt]}; final = {mean[nt], spread[nt]}.
int ref_assimilate(void* h, const double* observed, uint32_t n_win, uint32_t n_vox,
                   const double* d, const int64_t* iv, const uint32_t* tg, uint32_t nt,
                   double* stats, uint32_t* n_stats, double* final_ms, int* diverged,
                   char* err, int errlen) {
    return guarded(err, errlen, [&] {
        RefNet* n = static_cast<RefNet*>(h);
        std::vector<std::vector<double>> obs(n_win, std::vector<double>(n_vox));
        for (uint32_t w = 0; w < n_win; ++w)
            for (uint32_t v = 0; v < n_vox; ++v) obs[w][v] = observed[(size_t)w * n_vox + v];
        AssimResult r = assimilate(n->tables, n->layout, obs, assim_opts(d, iv, tg, nt));
        *n_stats = static_cast<uint32_t>(r.windows.size());
        for (size_t w = 0; w < r.windows.size(); ++w) {
            double* o = stats + w * (4 + nt);
            o[0] = r.windows[w].window;
            o[1] = r.windows[w].innovation_rms;
            o[2] = r.windows[w].pearson_r;
            o[3] = r.windows[w].mean_spread;
            for (uint32_t k = 0; k < nt; ++k) o[4 + k] = r.windows[w].target_mean[k];
        }
        for (uint32_t k = 0; k < nt; ++k) {
            final_ms[k] = r.final_mean[k];
            final_ms[nt + k] = r.final_spread[k];
        }
        *diverged = r.diverged ? static_cast<int>(r.diverged_window) + 1 : 0;
    });
}
// run_forward_bold (assim.cpp:301-326): out[window][voxel].
int ref_forward_bold(void* h, const double* d, const int64_t* iv, const uint32_t* tg,
                     uint32_t nt, uint32_t windows, const double* true_params, double* out,
                     char* err, int errlen) {
    return guarded(err, errlen, [&] {
        RefNet* n = static_cast<RefNet*>(h);
        std::vector<double> tp;
        if (true_params) tp.assign(true_params, true_params + nt);
        auto b = run_forward_bold(n->tables, n->layout, assim_opts(d, iv, tg, nt), windows,
                                  true_params ? &tp : nullptr);
        size_t k = 0;
        for (const auto& row : b)
            for (double x : row) out[k++] = x;
    });
}

// EnsrfUpdate::apply (assim.cpp:108-179): ens[m][p] in/out, fc[m][q], obs[q].
int ref_ensrf(double* ens, const double* fc, const double* obs, uint32_t m, uint32_t p,
              uint32_t q, double obs_var, double inflation, double min_spread, char* err,
              int errlen) {
    return guarded(err, errlen, [&] {
        std::vector<std::vector<double>> e(m, std::vector<double>(p)), f(m, std::vector<double>(q));
        for (uint32_t i = 0; i < m; ++i) {
            for (uint32_t c = 0; c < p; ++c) e[i][c] = ens[(size_t)i * p + c];
            for (uint32_t o = 0; o < q; ++o) f[i][o] = fc[(size_t)i * q + o];
        }
        EnsrfUpdate::apply(e, f, std::vector<double>(obs, obs + q), obs_var, inflation, min_spread);
        for (uint32_t i = 0; i < m; ++i)
            for (uint32_t c = 0; c < p; ++c) ens[(size_t)i * p + c] = e[i][c];
    });
}
// sample_conductances (netgen.cpp:318-329).
void ref_sample_conductances(uint64_t seed, uint64_t salt, uint32_t unit, int receptor,
                             double location, double scale, uint32_t count, float* out) {
    std::vector<float> v = sample_conductances(seed, salt, unit, receptor, location, scale, count);
    std::copy(v.begin(), v.end(), out);
}

} // extern "C"

// engine_cuda_adapter.hpp — the drop-in a maintainer adds to the reference
// code base: voxsim::SimInstance semantics
// (engine.hpp:68-89) on top of the C ABI of the B200 engine (include/vxb.h).
//
// Compiled against the reference's own headers (/root/reference/proj/include)
// and linked with libvxb.so by oracle/Makefile (target `adapter`), and run by
// tests/test_adapter_gpu.py through tests/native/adapter_check.cpp next to the
// reference SimInstance.  Nothing here computes simulation results: every
// call forwards to libvxb.so.
#pragma once

#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "voxsim/engine.hpp"
#include "voxsim/layout.hpp"
#include "voxsim/netgen.hpp"
#include "voxsim/util.hpp"
#include "vxb.h"

namespace voxsim {

class CudaSimInstance {
public:
    CudaSimInstance(const NetworkTables& t, const NetworkLayout& layout, SimOptions o)
        : opt_(std::move(o)) {
        std::vector<vxb_worker_table> wt;
        neurons_.reserve(t.workers.size());
        for (const WorkerTable& w : t.workers) {
            auto& recs = neurons_.emplace_back(w.neurons.size());
            for (size_t i = 0; i < w.neurons.size(); ++i) {
                const NeuronRecord& r = w.neurons[i];
                vxb_neuron& x = recs[i];
                std::memset(&x, 0, sizeof x);
                x.gid = r.gid;
                x.dst_mask = r.dst_mask;
                x.voxel = r.voxel;
                x.unit = r.unit;
                x.row_len = r.row_len;
                x.refractory_steps = r.refractory_steps;
                x.pop = r.pop;
                x.excitatory = r.excitatory ? 1 : 0;
                x.capacitance = r.capacitance;
                x.g_leak = r.g_leak;
                x.e_leak = r.e_leak;
                x.v_threshold = r.v_threshold;
                x.v_reset = r.v_reset;
                for (int k = 0; k < 4; ++k) {
                    x.e_rev[k] = r.e_rev[k];
                    x.tau[k] = r.tau[k];
                    x.omega[k] = r.omega[k];
                    x.g[k] = r.g[k];
                }
                x.ou_mean = r.ou_mean;
                x.ou_sigma = r.ou_sigma;
                x.ou_tau = r.ou_tau;
                x.v_init = r.v_init;
            }
            vxb_worker_table x{};
            x.worker = w.worker;
            x.worker_count = w.worker_count;
            x.n_neurons = (uint32_t)w.neurons.size();
            x.seed = w.seed;
            x.n_synapses = w.synapses.size();
            x.neurons = recs.data();
            // SynEntry is byte-identical to vxb_syn_entry (16 B, packed)
            static_assert(sizeof(SynEntry) == sizeof(vxb_syn_entry), "SynEntry layout");
            x.synapses = reinterpret_cast<const vxb_syn_entry*>(w.synapses.data());
            x.row_base = w.row_base.data();
            wt.push_back(x);
        }
        for (const Unit& u : layout.units) {
            vxb_unit x{};
            x.gid_base = u.gid_base;
            x.voxel = u.voxel;
            x.neurons = u.neurons;
            x.pop = u.pop;
            x.excitatory = u.excitatory ? 1 : 0;
            units_.push_back(x);
        }
        vxb_network net{};
        net.n_workers = (uint32_t)wt.size();
        net.n_units = layout.unit_count();
        net.n_voxels = (uint32_t)layout.voxels.size();
        net.workers = wt.data();
        net.unit_worker = t.unit_worker.data();
        net.unit_local_base = t.unit_local_base.data();
        net.units = units_.data();
        std::vector<vxb_injection> inj;
        for (const Injection& i : opt_.injections)
            inj.push_back({i.from_step, i.to_step, i.voxel, i.current_pa});
        std::vector<vxb_forced_spike> fs;
        for (const ForcedSpike& f : opt_.forced_spikes) fs.push_back({f.step, 0, f.gid});
        vxb_options vo{};
        vo.dt_ms = opt_.dt_ms;
        vo.scheduler = opt_.scheduler.c_str();
        vo.transport = opt_.transport.c_str();
        vo.workers_per_node = opt_.workers_per_node;
        vo.recv_timeout_ms = opt_.recv_timeout_ms;
        vo.record_raster = opt_.record_raster;
        vo.record_timings = opt_.record_timings;
        vo.probe_gids = opt_.probe_gids.data();
        vo.n_probes = (uint32_t)opt_.probe_gids.size();
        vo.n_injections = (uint32_t)inj.size();
        vo.injections = inj.data();
        vo.forced_spikes = fs.data();
        vo.n_forced = (uint32_t)fs.size();
        vo.device = -1;
        vo.n_devices = 1;
        check(vxb_create(&net, &vo, &e_), nullptr);
    }
    ~CudaSimInstance() { vxb_destroy(e_); }
    CudaSimInstance(const CudaSimInstance&) = delete;
    CudaSimInstance& operator=(const CudaSimInstance&) = delete;

    RunResult advance(uint32_t steps) {
        check(vxb_advance(e_, steps), e_);
        RunResult out;
        out.steps_done = vxb_result_steps_done(e_);
        out.total_spikes = vxb_result_total_spikes(e_);
        std::vector<vxb_raster_event> r(vxb_result_raster_size(e_));
        if (!r.empty()) vxb_result_raster(e_, r.data(), r.size());
        for (const auto& x : r) out.raster.push_back({x.step, x.worker, x.local, x.gid});
        out.rates.steps = steps;
        out.rates.dt_ms = opt_.dt_ms;
        for (const auto& u : units_) out.rates.unit_neurons.push_back(u.neurons);
        std::vector<uint32_t> c(units_.size() * (size_t)steps);
        if (!c.empty()) vxb_result_rates(e_, c.data(), c.size());
        for (size_t u = 0; u < units_.size(); ++u)
            out.rates.counts.emplace_back(c.begin() + u * steps, c.begin() + (u + 1) * steps);
        const size_t np = opt_.probe_gids.size();
        std::vector<float> pv(np * steps), pi(np * steps);
        if (!pv.empty()) vxb_result_probes(e_, pv.data(), pi.data(), pv.size());
        for (size_t p = 0; p < np; ++p) {
            ProbeTrace tr;
            tr.gid = opt_.probe_gids[p];
            tr.v.assign(pv.begin() + p * steps, pv.begin() + (p + 1) * steps);
            tr.i_syn.assign(pi.begin() + p * steps, pi.begin() + (p + 1) * steps);
            out.probes.push_back(std::move(tr));
        }
        vxb_flops f;
        vxb_result_flops(e_, &f);
        out.flops.membrane = f.membrane;
        out.flops.gating_inner = f.gating_inner;
        out.flops.gating_outer = f.gating_outer;
        out.flops.gating_decay = f.gating_decay;
        out.flops.current = f.current;
        std::vector<vxb_step_timings> tm(vxb_result_timings_size(e_));
        if (!tm.empty()) vxb_result_timings(e_, tm.data(), tm.size());
        for (const auto& x : tm) {
            StepTimings s;
            s.step = x.step;
            s.worker = x.worker;
            int64_t* a[11] = {&s.t1, &s.t2, &s.t3, &s.t4, &s.t5, &s.t6, &s.t7, &s.t8, &s.t9, &s.t10, &s.t11};
            for (int k = 0; k < 11; ++k) *a[k] = x.t[k];
            s.send_intra_ns = x.send_intra_ns;
            s.send_inter_ns = x.send_inter_ns;
            s.recv_intra_ns = x.recv_intra_ns;
            s.recv_inter_ns = x.recv_inter_ns;
            s.bytes_sent_intra = x.bytes_sent_intra;
            s.bytes_sent_inter = x.bytes_sent_inter;
            s.bytes_recv_intra = x.bytes_recv_intra;
            s.bytes_recv_inter = x.bytes_recv_inter;
            s.spikes = x.spikes;
            out.timings.push_back(s);
        }
        return out;
    }
    uint32_t current_step() const { return vxb_current_step(e_); }
    void set_conductances(uint32_t unit, int receptor, const std::vector<float>& v) {
        check(vxb_set_conductances(e_, unit, receptor, v.data(), (uint32_t)v.size()), e_);
    }
    std::vector<float> membrane_snapshot(uint16_t worker) const {
        std::vector<float> v(vxb_worker_neurons(e_, worker));
        check(vxb_membrane_snapshot(e_, worker, v.data(), (uint32_t)v.size()), e_);
        return v;
    }

private:
    static void check(int rc, const vxb_engine* e) {
        if (rc == VXB_ECONFIG) throw ConfigError(vxb_last_error(e));
        if (rc == VXB_ESIM) throw SimError(vxb_last_error(e));
    }
    SimOptions opt_;
    std::vector<std::vector<vxb_neuron>> neurons_;
    std::vector<vxb_unit> units_;
    vxb_engine* e_ = nullptr;
};

}  // namespace voxsim

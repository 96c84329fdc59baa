// adapter_check.cpp — the reference's own engine cases (test_engine.cpp)
// run through the C++ drop-in (engine_cuda_adapter.hpp over libvxb.so) next
// to the reference SimInstance, in one binary.  TEST INFRASTRUCTURE: built
// by oracle/Makefile (target `adapter`, needs /root/reference headers at
// build time) into oracle/_ref/adapter_check and run on a GPU box by
// tests/test_adapter_gpu.py.  Prints "ADAPTER OK <checks>" on success.
#include <cstdio>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "engine_cuda_adapter.hpp"
#include "voxsim/config.hpp"
#include "voxsim/pipeline.hpp"

using namespace voxsim;

namespace {

int g_checks = 0, g_fail = 0;

void expect(bool ok, const std::string& what) {
    ++g_checks;
    if (!ok) {
        ++g_fail;
        std::printf("FAIL: %s\n", what.c_str());
    }
}

std::multiset<std::pair<uint32_t, uint64_t>> raster_set(const std::vector<RasterEvent>& r) {
    std::multiset<std::pair<uint32_t, uint64_t>> out;
    for (const auto& e : r) out.insert({e.step, e.gid});
    return out;
}

// RunConfig JSON through the reference's own pipeline (pipeline.cpp:99-125)
BuiltNetwork net_of(const std::string& json) { return build_network(parse_config(json)); }

std::string ring_json(uint64_t seed, uint32_t voxels, uint32_t npv, uint32_t k_in, double rho,
                      uint32_t workers, const char* partition, const char* extra = "") {
    char buf[1024];
    std::snprintf(buf, sizeof buf,
                  "{\"seed\": %llu, \"workers\": %u, \"connectome\": {\"kind\": \"%s\", %s"
                  "\"neurons_per_voxel\": %u}, \"partition\": {\"method\": \"%s\"}, "
                  "\"regions\": {\"subcortex\": {\"k_in\": %u, \"rho\": %g%s}}}",
                  (unsigned long long)seed, workers, voxels == 1 ? "single" : "ring",
                  voxels == 1 ? "" : (std::string("\"voxels\": ") + std::to_string(voxels) + ", ").c_str(),
                  npv, partition, k_in, rho, extra);
    return buf;
}

SimOptions opts(uint32_t steps, const char* scheduler) {
    SimOptions o;
    o.steps = steps;
    o.scheduler = scheduler;
    return o;
}

void same(const RunResult& g, const RunResult& r, const std::string& what) {
    expect(g.total_spikes == r.total_spikes, what + ": total spikes");
    expect(g.steps_done == r.steps_done, what + ": steps done");
    expect(raster_set(g.raster) == raster_set(r.raster), what + ": raster");
    bool ordered = g.raster.size() == r.raster.size();
    for (size_t k = 0; ordered && k < g.raster.size(); ++k)
        ordered = g.raster[k].step == r.raster[k].step && g.raster[k].worker == r.raster[k].worker &&
                  g.raster[k].local == r.raster[k].local && g.raster[k].gid == r.raster[k].gid;
    expect(ordered, what + ": raster order (step, worker, local)");
    expect(g.rates.counts == r.rates.counts, what + ": rates");
    expect(g.probes.size() == r.probes.size(), what + ": probe count");
    for (size_t p = 0; p < g.probes.size() && p < r.probes.size(); ++p) {
        expect(g.probes[p].v == r.probes[p].v, what + ": probe V");
        expect(g.probes[p].i_syn == r.probes[p].i_syn, what + ": probe I_syn");
    }
    expect(g.flops.membrane == r.flops.membrane && g.flops.gating_inner == r.flops.gating_inner &&
               g.flops.gating_outer == r.flops.gating_outer &&
               g.flops.gating_decay == r.flops.gating_decay && g.flops.current == r.flops.current,
           what + ": flops");
}

// test_engine.cpp:107-201 (six neurons, two-entry rows, full OU noise)
void six_neurons() {
    BuiltNetwork n = net_of(ring_json(91, 1, 6, 2, 0.0, 1, "sequential"));
    SimOptions o = opts(150, "loopback");
    for (uint64_t g = 0; g < 6; ++g) o.probe_gids.push_back(g);
    SimInstance ref(n.tables, n.layout, o);
    SimOptions oc = o;
    oc.scheduler = "cuda";
    CudaSimInstance gpu(n.tables, n.layout, oc);
    const RunResult r = ref.advance(150), g = gpu.advance(150);
    expect(r.total_spikes > 0, "six neurons: active");
    same(g, r, "six neurons");
    expect(gpu.membrane_snapshot(0) == ref.membrane_snapshot(0), "six neurons: membrane snapshot");
}

// test_engine.cpp:263-301 (a run advanced in pieces == one advanced whole)
void piecewise() {
    BuiltNetwork n = net_of(ring_json(23, 3, 40, 5, 0.3, 1, "sequential"));
    SimOptions o = opts(90, "cuda");
    o.probe_gids = {0, 41, 100};
    CudaSimInstance whole(n.tables, n.layout, o), pieces(n.tables, n.layout, o);
    const RunResult rw = whole.advance(90);
    const RunResult r1 = pieces.advance(30), r2 = pieces.advance(45), r3 = pieces.advance(15);
    expect(pieces.current_step() == 90 && whole.current_step() == 90, "piecewise: current_step");
    expect(r1.steps_done == 30 && r2.steps_done == 45, "piecewise: steps_done");
    auto all = raster_set(r1.raster);
    for (const auto* r : {&r2, &r3})
        for (const auto& e : r->raster) all.insert({e.step, e.gid});
    expect(all == raster_set(rw.raster), "piecewise: raster");
    for (size_t p = 0; p < o.probe_gids.size(); ++p) {
        std::vector<float> v, is;
        for (const auto* r : {&r1, &r2, &r3}) {
            v.insert(v.end(), r->probes[p].v.begin(), r->probes[p].v.end());
            is.insert(is.end(), r->probes[p].i_syn.begin(), r->probes[p].i_syn.end());
        }
        expect(v == rw.probes[p].v && is == rw.probes[p].i_syn, "piecewise: probes");
    }
    expect(whole.membrane_snapshot(0) == pieces.membrane_snapshot(0), "piecewise: snapshot");
    // and the whole run equals the reference engine's
    SimOptions lo = o;
    lo.scheduler = "loopback";
    SimInstance ref(n.tables, n.layout, lo);
    same(rw, ref.advance(90), "piecewise vs reference");
}

// test_engine.cpp:322-358 (results are independent of the partition)
void partition_independence() {
    std::vector<RunResult> res;
    for (uint32_t workers : {1u, 2u, 3u}) {
        BuiltNetwork n = net_of(ring_json(44, 3, 50, 6, 0.5, workers, workers == 1 ? "sequential" : "greedy"));
        SimOptions o = opts(100, "cuda");
        o.probe_gids = {0, 60, 149};
        CudaSimInstance gpu(n.tables, n.layout, o);
        res.push_back(gpu.advance(100));
        SimOptions lo = o;
        lo.scheduler = "threads";
        SimInstance ref(n.tables, n.layout, lo);
        same(res.back(), ref.advance(100), "partition " + std::to_string(workers) + " vs reference");
    }
    for (size_t k = 1; k < res.size(); ++k) {
        expect(res[k].total_spikes == res[0].total_spikes, "partition: spikes");
        expect(raster_set(res[k].raster) == raster_set(res[0].raster), "partition: raster");
        for (size_t p = 0; p < res[0].probes.size(); ++p)
            expect(res[k].probes[p].v == res[0].probes[p].v &&
                       res[k].probes[p].i_syn == res[0].probes[p].i_syn,
                   "partition: probes");
    }
    expect(res[0].total_spikes > 0, "partition: active");
}

// error kinds through the adapter (engine.cpp:177-205, 765-766, 829-847)
void errors() {
    BuiltNetwork n = net_of(ring_json(5, 3, 30, 4, 0.3, 1, "sequential"));
    SimOptions bad = opts(10, "cuda");
    bad.dt_ms = 0.0;
    bool config = false;
    try {
        CudaSimInstance g(n.tables, n.layout, bad);
    } catch (const ConfigError&) {
        config = true;
    }
    expect(config, "errors: dt <= 0 is a ConfigError");
    SimOptions o = opts(10, "cuda");
    CudaSimInstance g(n.tables, n.layout, o);
    bool conf2 = false;
    try {
        g.set_conductances(0, 0, std::vector<float>(n.layout.units[0].neurons, -1.0f));
    } catch (const ConfigError&) {
        conf2 = true;
    }
    expect(conf2, "errors: negative conductance is a ConfigError");
    g.advance(10);
    expect(g.current_step() == 10, "errors: instance usable after a rejected set");
}

}  // namespace

int main() {
    try {
        six_neurons();
        piecewise();
        partition_independence();
        errors();
    } catch (const std::exception& e) {
        std::printf("FAIL: exception %s\n", e.what());
        return 1;
    }
    if (g_fail) {
        std::printf("ADAPTER FAILED %d of %d checks\n", g_fail, g_checks);
        return 1;
    }
    std::printf("ADAPTER OK %d checks\n", g_checks);
    return 0;
}

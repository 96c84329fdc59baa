/*
 * voxsim_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's simulation step, used by tests/ and bench.py's cpu_baseline leg
 * as the checker.  It is never linked into, called by, or measured as the
 * product (paper_2308_01241_b200/).
 *
 * Pinned against (tests/test_oracle.py):
 *   - the frozen SplitMix64 / u01 vectors of test_rng.cpp:13-35,
 *   - the exact kernel values of test_model.cpp:35-223,
 *   - the reference engine itself (oracle/_ref/libvoxsim_ref.so, built from
 *     /root/reference/proj/src) on identical tables: raster, probe traces,
 *     final membrane state, rates and FLOP tallies bit-for-bit,
 *   - golden fixtures in tests/golden/ generated from that reference build.
 *
 * Semantics follow /root/reference/proj:
 *   rng       include/voxsim/rng.hpp:32-73
 *   kernels   include/voxsim/model.hpp:20-28, 69-90
 *   load      src/engine.cpp:175-293 (per-neuron SoA, ou_key, initial state)
 *   delivery  src/engine.cpp:295-344, 444-464 (int64 pending buckets)
 *   phase A   src/engine.cpp:348-414 (membrane, injections, forced spikes)
 *   phase E   src/engine.cpp:526-568 (gating, current, OU, swap)
 *   advance   src/engine.cpp:763-827 (loopback order; results per call)
 * Compiled with -ffp-contract=off like the reference (CMakeLists.txt:11-14).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "vxb.h"

/* ------------------------------------------------------------ rng.hpp:32-73 */

#define VXO_GOLDEN 0x9e3779b97f4a7c15ULL

uint64_t vxo_splitmix64(uint64_t x) {
    x += VXO_GOLDEN;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t vxo_mix_key(uint64_t a, uint64_t b) {
    return vxo_splitmix64(a ^ (b + VXO_GOLDEN + (a << 6) + (a >> 2)));
}

uint64_t vxo_stream_word(uint64_t base, uint64_t k) {
    return vxo_splitmix64(base + k * VXO_GOLDEN);
}

double vxo_stream_u01(uint64_t base, uint64_t k) {
    return (double)(vxo_stream_word(base, k) >> 11) * 0x1.0p-53;
}

double vxo_stream_normal(uint64_t base, uint64_t k) {
    const double u1 = 1.0 - vxo_stream_u01(base, 2 * k);
    const double u2 = vxo_stream_u01(base, 2 * k + 1);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

uint64_t vxo_stream_below(uint64_t base, uint64_t k, uint64_t n) {
    return vxo_stream_word(base, k) % n;
}

/* engine.cpp:249 + 551-553: the per-neuron OU stream and its float sample. */
float vxo_ou_xi(uint64_t seed, uint64_t gid, uint64_t step) {
    uint64_t key = vxo_mix_key(vxo_mix_key(seed, 1), gid);
    return (float)vxo_stream_normal(key, step);
}

/* ---------------------------------------------------------- model.hpp:20-90 */

int32_t vxo_quantize_weight(double w) {
    if (w < 0) w = 0;
    return (int32_t)lround(w * 65536.0);
}

float vxo_dequantize_weight(int64_t q) { return (float)((double)q * (1.0 / 65536.0)); }

float vxo_gating_kernel(float j, float dt, float tau, float omega, float pending) {
    return j * (1.0f - dt / tau) + omega * pending;
}

float vxo_current_kernel(float v, const float* j, const float* g, const float* e) {
    float i = 0.0f;
    for (int u = 0; u < VXB_RECEPTORS; ++u) i += g[u] * j[u] * (e[u] - v);
    return i;
}

float vxo_membrane_kernel(float v, float dt_over_c, float g_leak, float e_leak, float i_syn,
                          float i_ou) {
    return v + dt_over_c * (g_leak * (e_leak - v) + i_syn + i_ou);
}

float vxo_ou_kernel(float i, float dt, float mean, float sigma, float tau, float xi) {
    return i + (dt / tau) * (mean - i) + sigma * sqrtf(2.0f * dt / tau) * xi;
}

/* ------------------------------------------------------------------ engine */

typedef struct {
    uint32_t dst_worker, dst_local;
    uint8_t cls;
    int32_t wf, ws;
} vxo_out;

typedef struct {
    uint32_t n;
    uint64_t* gid;
    uint64_t* ou_key;
    uint32_t* unit;
    uint32_t* voxel;
    float *dt_over_c, *g_leak, *e_leak, *v_th, *v_reset;
    uint32_t* refrac_steps;
    float *ou_mu, *ou_sigma, *ou_tau;
    float *tau, *omega, *g, *e_rev; /* [n*4] */
    float *v, *i_syn, *i_ou, *j;     /* j [n*4] */
    uint32_t* refrac_left;
    int64_t *pend_cur, *pend_prev; /* [n*4] */
    uint64_t* out_off;             /* per local source, n+1 into outs */
    vxo_out* outs;
} vxo_worker;

typedef struct {
    uint64_t gid;
    uint32_t worker, local;
} vxo_probe;

typedef struct {
    uint32_t step, worker, local;
} vxo_forced;

typedef struct vxo_sim {
    uint32_t workers, n_units, n_voxels;
    uint64_t seed;
    float dtf;
    double dt_ms;
    int record_raster;
    vxo_worker* ws;
    vxb_unit* units;
    uint16_t* unit_worker;
    uint32_t* unit_local_base;
    vxo_probe* probes;
    uint32_t n_probes;
    vxb_injection* inj;
    uint32_t n_inj;
    vxo_forced* forced;
    uint32_t n_forced;
    uint32_t step_done;
    int failed;
    /* last advance results */
    uint32_t res_steps;
    vxb_raster_event* raster;
    uint64_t raster_n, raster_cap;
    uint32_t* rates; /* [n_units][steps] */
    float *probe_v, *probe_i;
    vxb_flops flops;
    uint64_t total_spikes;
    char err[512];
} vxo_sim;

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) {
        fprintf(stderr, "voxsim_oracle: out of memory\n");
        abort();
    }
    return p;
}

/* layout.cpp:119-128 */
static int unit_of_gid(const vxo_sim* s, uint64_t gid, uint32_t* unit) {
    uint32_t lo = 0, hi = s->n_units; /* first unit with gid_base > gid */
    while (lo < hi) {
        uint32_t mid = (lo + hi) / 2;
        if (gid < s->units[mid].gid_base)
            hi = mid;
        else
            lo = mid + 1;
    }
    if (lo == 0) return -1;
    uint32_t i = lo - 1;
    while (i > 0 && s->units[i].neurons == 0) --i;
    if (gid >= s->units[i].gid_base + s->units[i].neurons) return -1;
    *unit = i;
    return 0;
}

static void fail(vxo_sim* s, const char* kind, const char* msg) {
    snprintf(s->err, sizeof s->err, "%s: %s", kind, msg);
}

const char* vxo_last_error(const vxo_sim* s) { return s ? s->err : "null oracle"; }

void vxo_destroy(vxo_sim* s);

/* engine.cpp:175-344 */
vxo_sim* vxo_create(const vxb_network* net, const vxb_options* opt, char* err, int errlen,
                    int* rc) {
    vxo_sim* s = (vxo_sim*)xcalloc(1, sizeof *s);
    *rc = 0;
#define VXO_FAIL(code, kind, ...)                                   \
    do {                                                            \
        char m_[400];                                               \
        snprintf(m_, sizeof m_, __VA_ARGS__);                       \
        if (err && errlen > 0) snprintf(err, errlen, "%s: %s", kind, m_); \
        *rc = code;                                                 \
        vxo_destroy(s);                                             \
        return NULL;                                                \
    } while (0)
    if (net->n_workers == 0) VXO_FAIL(2, "ConfigError", "no worker tables");
    if (net->n_workers > 64) VXO_FAIL(2, "ConfigError", "worker counts above 64 are unsupported");
    if (!(opt->dt_ms > 0.0)) VXO_FAIL(2, "ConfigError", "dt must be positive");
    s->workers = net->n_workers;
    s->n_units = net->n_units;
    s->n_voxels = net->n_voxels;
    s->seed = net->workers[0].seed;
    s->dt_ms = opt->dt_ms;
    s->dtf = (float)opt->dt_ms;
    s->record_raster = opt->record_raster;
    s->units = (vxb_unit*)xcalloc(s->n_units, sizeof(vxb_unit));
    memcpy(s->units, net->units, sizeof(vxb_unit) * s->n_units);
    s->unit_worker = (uint16_t*)xcalloc(s->n_units, sizeof(uint16_t));
    memcpy(s->unit_worker, net->unit_worker, sizeof(uint16_t) * s->n_units);
    s->unit_local_base = (uint32_t*)xcalloc(s->n_units, sizeof(uint32_t));
    memcpy(s->unit_local_base, net->unit_local_base, sizeof(uint32_t) * s->n_units);
    for (uint32_t k = 0; k < opt->n_injections; ++k) {
        if (opt->injections[k].voxel >= s->n_voxels)
            VXO_FAIL(2, "ConfigError", "injection voxel out of range");
        if (opt->injections[k].to_step < opt->injections[k].from_step)
            VXO_FAIL(2, "ConfigError", "injection interval is reversed");
    }
    s->n_inj = opt->n_injections;
    s->inj = (vxb_injection*)xcalloc(s->n_inj, sizeof(vxb_injection));
    if (s->n_inj) memcpy(s->inj, opt->injections, sizeof(vxb_injection) * s->n_inj);

    s->ws = (vxo_worker*)xcalloc(s->workers, sizeof(vxo_worker));
    const uint64_t ou_root = vxo_mix_key(s->seed, 1); /* rngstream::ou_noise */
    for (uint32_t wi = 0; wi < s->workers; ++wi) {
        const vxb_worker_table* t = &net->workers[wi];
        vxo_worker* w = &s->ws[wi];
        uint32_t n = t->n_neurons;
        w->n = n;
#define A(f, T, k) w->f = (T*)xcalloc((size_t)n * (k), sizeof(T))
        A(gid, uint64_t, 1); A(ou_key, uint64_t, 1); A(unit, uint32_t, 1); A(voxel, uint32_t, 1);
        A(dt_over_c, float, 1); A(g_leak, float, 1); A(e_leak, float, 1); A(v_th, float, 1);
        A(v_reset, float, 1); A(refrac_steps, uint32_t, 1); A(ou_mu, float, 1);
        A(ou_sigma, float, 1); A(ou_tau, float, 1); A(tau, float, 4); A(omega, float, 4);
        A(g, float, 4); A(e_rev, float, 4); A(v, float, 1); A(i_syn, float, 1); A(i_ou, float, 1);
        A(j, float, 4); A(refrac_left, uint32_t, 1); A(pend_cur, int64_t, 4);
        A(pend_prev, int64_t, 4);
#undef A
        for (uint32_t i = 0; i < n; ++i) {
            const vxb_neuron* r = &t->neurons[i];
            /* NeuronParams::validate (model.cpp:7-26) */
            if (!(r->capacitance > 0)) VXO_FAIL(2, "ConfigError", "neuron params: capacitance must be > 0");
            if (r->g_leak < 0) VXO_FAIL(2, "ConfigError", "neuron params: leak conductance must be >= 0");
            if (!(r->v_reset < r->v_threshold)) VXO_FAIL(2, "ConfigError", "neuron params: V_reset must be below V_th");
            for (int u = 0; u < 4; ++u) {
                if (!(r->tau[u] > 0)) VXO_FAIL(2, "ConfigError", "neuron params: receptor tau must be > 0");
                if (!(s->dtf < r->tau[u])) VXO_FAIL(2, "ConfigError", "neuron params: dt must be below every receptor tau (explicit Euler)");
                if (r->g[u] < 0 || r->omega[u] < 0) VXO_FAIL(2, "ConfigError", "neuron params: receptor conductance and jump weights must be >= 0");
            }
            if (r->e_rev[0] <= r->v_threshold || r->e_rev[1] <= r->v_threshold)
                VXO_FAIL(2, "ConfigError", "neuron params: excitatory reversals must lie above V_th");
            if (r->e_rev[2] >= r->e_leak || r->e_rev[3] >= r->e_leak)
                VXO_FAIL(2, "ConfigError", "neuron params: inhibitory reversals must lie below E_L");
            w->dt_over_c[i] = s->dtf / r->capacitance;
            w->g_leak[i] = r->g_leak;
            w->e_leak[i] = r->e_leak;
            w->v_th[i] = r->v_threshold;
            w->v_reset[i] = r->v_reset;
            w->refrac_steps[i] = r->refractory_steps;
            w->gid[i] = r->gid;
            w->ou_key[i] = vxo_mix_key(ou_root, r->gid);
            w->unit[i] = r->unit;
            w->voxel[i] = r->voxel;
            w->ou_mu[i] = r->ou_mean;
            w->ou_sigma[i] = r->ou_sigma;
            w->ou_tau[i] = r->ou_tau;
            for (int u = 0; u < 4; ++u) {
                w->tau[i * 4 + u] = r->tau[u];
                w->omega[i * 4 + u] = r->omega[u];
                w->g[i * 4 + u] = r->g[u];
                w->e_rev[i * 4 + u] = r->e_rev[u];
            }
            w->v[i] = r->v_init;
            w->i_ou[i] = r->ou_mean;
            if (r->unit >= s->n_units || r->voxel >= s->n_voxels)
                VXO_FAIL(2, "ConfigError", "neuron record references unknown unit/voxel");
        }
    }
    /* Out-lists per source (build_delivery, engine.cpp:295-327), flattened
     * across destination workers. */
    for (uint32_t si = 0; si < s->workers; ++si)
        s->ws[si].out_off = (uint64_t*)xcalloc((size_t)s->ws[si].n + 1, sizeof(uint64_t));
    for (uint32_t di = 0; di < s->workers; ++di) {
        const vxb_worker_table* t = &net->workers[di];
        for (uint64_t k = 0; k < t->n_synapses; ++k) {
            const vxb_syn_entry* e = &t->synapses[k];
            if (e->src_worker >= s->workers || e->src_local >= s->ws[e->src_worker].n)
                VXO_FAIL(3, "SimError", "synapse entry references a nonexistent source");
            s->ws[e->src_worker].out_off[e->src_local + 1] += 1;
        }
    }
    for (uint32_t si = 0; si < s->workers; ++si) {
        vxo_worker* w = &s->ws[si];
        for (uint32_t i = 0; i < w->n; ++i) w->out_off[i + 1] += w->out_off[i];
        w->outs = (vxo_out*)xcalloc(w->out_off[w->n], sizeof(vxo_out));
    }
    {
        uint64_t** cur = (uint64_t**)xcalloc(s->workers, sizeof(uint64_t*));
        for (uint32_t si = 0; si < s->workers; ++si) {
            cur[si] = (uint64_t*)xcalloc(s->ws[si].n + 1, sizeof(uint64_t));
            memcpy(cur[si], s->ws[si].out_off, sizeof(uint64_t) * s->ws[si].n);
        }
        for (uint32_t di = 0; di < s->workers; ++di) {
            const vxb_worker_table* t = &net->workers[di];
            for (uint32_t n = 0; n < t->n_neurons; ++n)
                for (uint64_t k = t->row_base[n]; k < t->row_base[n + 1]; ++k) {
                    const vxb_syn_entry* e = &t->synapses[k];
                    vxo_out* o = &s->ws[e->src_worker].outs[cur[e->src_worker][e->src_local]++];
                    o->dst_worker = di;
                    o->dst_local = n;
                    o->cls = e->cls;
                    o->wf = e->wq_fast;
                    o->ws = e->wq_slow;
                }
        }
        for (uint32_t si = 0; si < s->workers; ++si) free(cur[si]);
        free(cur);
    }
    /* dst_mask consistency (engine.cpp:328-343) */
    for (uint32_t si = 0; si < s->workers; ++si) {
        vxo_worker* w = &s->ws[si];
        const vxb_worker_table* t = &net->workers[si];
        for (uint32_t l = 0; l < w->n; ++l) {
            uint64_t have = 0;
            for (uint64_t k = w->out_off[l]; k < w->out_off[l + 1]; ++k)
                have |= 1ULL << w->outs[k].dst_worker;
            if (have != t->neurons[l].dst_mask)
                VXO_FAIL(3, "SimError", "destination mask inconsistent with tables");
        }
    }
    /* probes and forced spikes (engine.cpp:276-290) */
    s->n_probes = opt->n_probes;
    s->probes = (vxo_probe*)xcalloc(s->n_probes, sizeof(vxo_probe));
    for (uint32_t p = 0; p < s->n_probes; ++p) {
        uint32_t u;
        if (unit_of_gid(s, opt->probe_gids[p], &u)) VXO_FAIL(3, "SimError", "gid out of range");
        s->probes[p].gid = opt->probe_gids[p];
        s->probes[p].worker = s->unit_worker[u];
        s->probes[p].local = s->unit_local_base[u] + (uint32_t)(opt->probe_gids[p] - s->units[u].gid_base);
    }
    s->n_forced = opt->n_forced;
    s->forced = (vxo_forced*)xcalloc(s->n_forced, sizeof(vxo_forced));
    for (uint32_t f = 0; f < s->n_forced; ++f) {
        uint32_t u;
        if (unit_of_gid(s, opt->forced_spikes[f].gid, &u)) VXO_FAIL(3, "SimError", "gid out of range");
        s->forced[f].step = opt->forced_spikes[f].step;
        s->forced[f].worker = s->unit_worker[u];
        s->forced[f].local = s->unit_local_base[u] + (uint32_t)(opt->forced_spikes[f].gid - s->units[u].gid_base);
    }
#undef VXO_FAIL
    return s;
}

void vxo_destroy(vxo_sim* s) {
    if (!s) return;
    if (s->ws) {
        for (uint32_t i = 0; i < s->workers; ++i) {
            vxo_worker* w = &s->ws[i];
            void* ps[] = {w->gid, w->ou_key, w->unit, w->voxel, w->dt_over_c, w->g_leak,
                          w->e_leak, w->v_th, w->v_reset, w->refrac_steps, w->ou_mu,
                          w->ou_sigma, w->ou_tau, w->tau, w->omega, w->g, w->e_rev, w->v,
                          w->i_syn, w->i_ou, w->j, w->refrac_left, w->pend_cur, w->pend_prev,
                          w->out_off, w->outs};
            for (size_t k = 0; k < sizeof ps / sizeof ps[0]; ++k) free(ps[k]);
        }
    }
    free(s->ws);
    free(s->units);
    free(s->unit_worker);
    free(s->unit_local_base);
    free(s->probes);
    free(s->inj);
    free(s->forced);
    free(s->raster);
    free(s->rates);
    free(s->probe_v);
    free(s->probe_i);
    free(s);
}

static void push_raster(vxo_sim* s, uint32_t step, uint32_t worker, uint32_t local, uint64_t gid) {
    if (s->raster_n == s->raster_cap) {
        s->raster_cap = s->raster_cap ? 2 * s->raster_cap : 1024;
        s->raster = (vxb_raster_event*)realloc(s->raster, s->raster_cap * sizeof(vxb_raster_event));
        if (!s->raster) abort();
    }
    vxb_raster_event e;
    memset(&e, 0, sizeof e);
    e.step = step;
    e.worker = (uint16_t)worker;
    e.local = local;
    e.gid = gid;
    s->raster[s->raster_n++] = e;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

/* engine.cpp:444-464 */
static void deliver(vxo_sim* s, uint32_t src_worker, uint32_t src_local) {
    vxo_worker* sw = &s->ws[src_worker];
    for (uint64_t k = sw->out_off[src_local]; k < sw->out_off[src_local + 1]; ++k) {
        const vxo_out* o = &sw->outs[k];
        int64_t* p = &s->ws[o->dst_worker].pend_cur[(size_t)o->dst_local * 4];
        if (o->cls == 0) {
            p[0] += o->wf;
            p[1] += o->ws;
        } else {
            p[2] += o->wf;
            p[3] += o->ws;
        }
        if (o->dst_worker == src_worker)
            s->flops.gating_inner += 2;
        else
            s->flops.gating_outer += 2;
    }
}

/* engine.cpp:763-827 with advance_loopback (711-748) */
int vxo_advance(vxo_sim* s, uint32_t steps) {
    if (s->failed) {
        fail(s, "SimError", "instance is in a failed state");
        return 3;
    }
    s->res_steps = steps;
    s->raster_n = 0;
    s->total_spikes = 0;
    memset(&s->flops, 0, sizeof s->flops);
    free(s->rates);
    s->rates = (uint32_t*)xcalloc((size_t)s->n_units * steps, sizeof(uint32_t));
    free(s->probe_v);
    free(s->probe_i);
    s->probe_v = (float*)xcalloc((size_t)s->n_probes * steps, sizeof(float));
    s->probe_i = (float*)xcalloc((size_t)s->n_probes * steps, sizeof(float));
    float* vox_inj = (float*)xcalloc(s->n_voxels, sizeof(float));
    uint32_t* spikes = NULL;
    size_t spikes_cap = 0;
    uint32_t** w_spikes = (uint32_t**)xcalloc(s->workers, sizeof(uint32_t*));
    uint32_t* w_nspk = (uint32_t*)xcalloc(s->workers, sizeof(uint32_t));
    for (uint32_t wi = 0; wi < s->workers; ++wi)
        w_spikes[wi] = (uint32_t*)xcalloc(s->ws[wi].n + 1, sizeof(uint32_t));
    int rc = 0;
    (void)spikes;
    (void)spikes_cap;

    for (uint32_t rel = 0; rel < steps && rc == 0; ++rel) {
        uint32_t t = s->step_done + rel;
        /* injections active this step (engine.cpp:352-361) */
        int has_inj = 0;
        for (uint32_t k = 0; k < s->n_inj; ++k) {
            const vxb_injection* inj = &s->inj[k];
            if (inj->from_step <= t && t < inj->to_step) {
                if (!has_inj) memset(vox_inj, 0, sizeof(float) * s->n_voxels);
                has_inj = 1;
                vox_inj[inj->voxel] += inj->current_pa;
            }
        }
        /* phase A, B/C for every worker */
        for (uint32_t wi = 0; wi < s->workers && rc == 0; ++wi) {
            vxo_worker* w = &s->ws[wi];
            uint32_t* sp = w_spikes[wi];
            uint32_t ns = 0;
            for (uint32_t n = 0; n < w->n; ++n) {
                if (w->refrac_left[n] > 0) {
                    --w->refrac_left[n];
                    w->v[n] = w->v_reset[n];
                    continue;
                }
                float i_noise = w->i_ou[n];
                if (has_inj && vox_inj[w->voxel[n]] != 0.0f) i_noise += vox_inj[w->voxel[n]];
                float nv = vxo_membrane_kernel(w->v[n], w->dt_over_c[n], w->g_leak[n],
                                               w->e_leak[n], w->i_syn[n], i_noise);
                if (!isfinite(nv)) {
                    char m[200];
                    snprintf(m, sizeof m, "membrane potential diverged (neuron %llu, step %u)",
                             (unsigned long long)w->gid[n], t);
                    fail(s, "SimError", m);
                    rc = 3;
                    break;
                }
                if (nv >= w->v_th[n]) {
                    w->v[n] = w->v_reset[n];
                    w->refrac_left[n] = w->refrac_steps[n];
                    sp[ns++] = n;
                } else {
                    w->v[n] = nv;
                }
            }
            if (rc) break;
            s->flops.membrane += 6ULL * w->n;
            /* forced spikes (engine.cpp:389-398); list order irrelevant for
             * the outcome: a forced neuron joins once unless it fired. */
            for (uint32_t f = 0; f < s->n_forced; ++f) {
                if (s->forced[f].step != t || s->forced[f].worker != wi) continue;
                uint32_t l = s->forced[f].local;
                int already = 0;
                for (uint32_t k = 0; k < ns; ++k)
                    if (sp[k] == l) { already = 1; break; }
                if (already) continue;
                w->v[l] = w->v_reset[l];
                w->refrac_left[l] = w->refrac_steps[l];
                sp[ns++] = l;
            }
            qsort(sp, ns, sizeof(uint32_t), cmp_u32);
            w_nspk[wi] = ns;
            for (uint32_t k = 0; k < ns; ++k) {
                uint32_t n = sp[k];
                if (s->record_raster) push_raster(s, t, wi, n, w->gid[n]);
                s->rates[(size_t)w->unit[n] * steps + rel] += 1;
            }
            for (uint32_t p = 0; p < s->n_probes; ++p)
                if (s->probes[p].worker == wi)
                    s->probe_v[(size_t)p * steps + rel] = w->v[s->probes[p].local];
        }
        if (rc) break;
        /* delivery of this step's spikes, local and remote (phases C, E) */
        for (uint32_t wi = 0; wi < s->workers; ++wi)
            for (uint32_t k = 0; k < w_nspk[wi]; ++k) deliver(s, wi, w_spikes[wi][k]);
        /* phase E (engine.cpp:539-562) */
        for (uint32_t wi = 0; wi < s->workers; ++wi) {
            vxo_worker* w = &s->ws[wi];
            for (uint32_t n = 0; n < w->n; ++n) {
                size_t b = (size_t)n * 4;
                for (int u = 0; u < 4; ++u) {
                    float pending = vxo_dequantize_weight(w->pend_prev[b + u]);
                    w->j[b + u] = vxo_gating_kernel(w->j[b + u], s->dtf, w->tau[b + u],
                                                    w->omega[b + u], pending);
                    w->pend_prev[b + u] = 0;
                }
                w->i_syn[n] = vxo_current_kernel(w->v[n], &w->j[b], &w->g[b], &w->e_rev[b]);
                float xi = w->ou_sigma[n] > 0 ? (float)vxo_stream_normal(w->ou_key[n], t) : 0.0f;
                w->i_ou[n] = vxo_ou_kernel(w->i_ou[n], s->dtf, w->ou_mu[n], w->ou_sigma[n],
                                           w->ou_tau[n], xi);
            }
            s->flops.gating_decay += 12ULL * w->n;
            s->flops.current += 16ULL * w->n;
            int64_t* tmp = w->pend_cur;
            w->pend_cur = w->pend_prev;
            w->pend_prev = tmp;
            for (uint32_t p = 0; p < s->n_probes; ++p)
                if (s->probes[p].worker == wi)
                    s->probe_i[(size_t)p * steps + rel] = w->i_syn[s->probes[p].local];
        }
    }
    for (uint32_t wi = 0; wi < s->workers; ++wi) free(w_spikes[wi]);
    free(w_spikes);
    free(w_nspk);
    free(vox_inj);
    if (rc) {
        s->failed = 1;
        return rc;
    }
    for (uint64_t k = 0; k < (uint64_t)s->n_units * steps; ++k) s->total_spikes += s->rates[k];
    s->step_done += steps;
    return 0;
}

/* ------------------------------------------------------------ result access */
uint32_t vxo_current_step(const vxo_sim* s) { return s->step_done; }
uint64_t vxo_total_spikes(const vxo_sim* s) { return s->total_spikes; }
uint64_t vxo_raster_size(const vxo_sim* s) { return s->raster_n; }
void vxo_raster(const vxo_sim* s, vxb_raster_event* out) {
    memcpy(out, s->raster, s->raster_n * sizeof(vxb_raster_event));
}
void vxo_rates(const vxo_sim* s, uint32_t* out) {
    memcpy(out, s->rates, (size_t)s->n_units * s->res_steps * sizeof(uint32_t));
}
void vxo_probes(const vxo_sim* s, float* v, float* i) {
    memcpy(v, s->probe_v, (size_t)s->n_probes * s->res_steps * sizeof(float));
    memcpy(i, s->probe_i, (size_t)s->n_probes * s->res_steps * sizeof(float));
}
void vxo_flops(const vxo_sim* s, vxb_flops* out) { *out = s->flops; }
uint32_t vxo_worker_n(const vxo_sim* s, uint32_t w) { return s->ws[w].n; }
void vxo_snapshot(const vxo_sim* s, uint32_t w, float* out) {
    memcpy(out, s->ws[w].v, sizeof(float) * s->ws[w].n);
}

/*
 * vxb.h — C ABI of the B200 voxel-network simulation step (the drop-in
 * boundary for the reference's SimInstance hot path).
 *
 * Every entry point replaces one member of the reference C++ host API
 * (/root/reference/proj/include/voxsim/engine.hpp):
 *
 *   vxb_create              <- SimInstance::SimInstance(tables, layout, options)
 *                              engine.hpp:70-71, load engine.cpp:175-293
 *   vxb_advance             <- RunResult SimInstance::advance(uint32_t steps)
 *                              engine.hpp:76, engine.cpp:763-827
 *   vxb_result_*            <- the RunResult fields (engine.hpp:55-63)
 *   vxb_current_step        <- SimInstance::current_step()  engine.hpp:77
 *   vxb_set_conductances    <- SimInstance::set_conductances  engine.hpp:81-82,
 *                              engine.cpp:829-844
 *   vxb_membrane_snapshot   <- SimInstance::membrane_snapshot engine.hpp:84,
 *                              engine.cpp:846-849
 *   vxb_run_simulation      <- run_simulation(tables, layout, options)
 *                              engine.hpp:92-93
 *   vxb_last_error          <- what() of the ConfigError / SimError thrown
 *                              (util.hpp:14-21)
 *   vxb_destroy             <- ~SimInstance
 *
 * Inputs are plain arrays in the reference's own table layout
 * (NetworkTables / WorkerTable / NeuronRecord / SynEntry, netgen.hpp:27-71;
 * NetworkLayout::units, layout.hpp:53-60) so a caller holding reference
 * tables passes pointers into them without conversion.
 *
 * Return codes mirror the CLI's exception mapping (voxsim.cpp:476-485):
 * 0 = ok, 2 = ConfigError, 3 = SimError.  A failed engine rejects further
 * vxb_advance calls (engine.cpp:765-766).
 *
 * There is no CPU fallback: vxb_create fails with VXB_ESIM when no CUDA
 * device is usable.
 */
#ifndef VXB_H
#define VXB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VXB_OK 0
#define VXB_ECONFIG 2
#define VXB_ESIM 3

#define VXB_RECEPTORS 4 /* AMPA, NMDA, GABAA, GABAB (model.hpp:13-15) */
#define VXB_ABI_VERSION 1

/* One in-synapse of a worker table: byte-identical to voxsim::SynEntry
 * (netgen.hpp:27-36, 16 bytes, packed). */
#pragma pack(push, 1)
typedef struct vxb_syn_entry {
    uint32_t src_local;
    uint16_t src_worker;
    uint8_t cls; /* 0 = excitatory source (AMPA/NMDA), 1 = inhibitory (GABAA/GABAB) */
    uint8_t pad;
    int32_t wq_fast; /* Q16 weight, AMPA or GABAA */
    int32_t wq_slow; /* Q16 weight, NMDA or GABAB */
} vxb_syn_entry;
#pragma pack(pop)

/* One neuron record: the fields of voxsim::NeuronRecord (netgen.hpp:40-53)
 * in a fixed, padding-free 136-byte layout. */
typedef struct vxb_neuron {
    uint64_t gid;
    uint64_t dst_mask; /* bit w: has >= 1 target on worker w */
    uint32_t voxel;
    uint32_t unit;
    uint32_t row_len;
    uint32_t refractory_steps;
    uint16_t pop;
    uint8_t excitatory;
    uint8_t pad0;
    float capacitance, g_leak, e_leak, v_threshold, v_reset;
    float e_rev[VXB_RECEPTORS];
    float tau[VXB_RECEPTORS];
    float omega[VXB_RECEPTORS];
    float g[VXB_RECEPTORS];
    float ou_mean, ou_sigma, ou_tau;
    float v_init;
} vxb_neuron;

/* voxsim::WorkerTable (netgen.hpp:55-64). */
typedef struct vxb_worker_table {
    uint16_t worker;
    uint16_t worker_count;
    uint32_t n_neurons;
    uint64_t seed;
    uint64_t n_synapses;
    const vxb_neuron* neurons;     /* n_neurons, local id order */
    const vxb_syn_entry* synapses; /* n_synapses, row-major by target */
    const uint64_t* row_base;      /* n_neurons + 1 prefix sums */
} vxb_worker_table;

/* voxsim::Unit (layout.hpp:53-60). */
typedef struct vxb_unit {
    uint64_t gid_base;
    uint32_t voxel;
    uint32_t neurons;
    uint16_t pop;
    uint8_t excitatory;
    uint8_t pad0;
    uint32_t pad1;
} vxb_unit;

/* NetworkTables + the parts of NetworkLayout the engine reads at load
 * (engine.cpp:180-192, 276-290). */
typedef struct vxb_network {
    uint32_t n_workers;
    uint32_t n_units;
    uint32_t n_voxels;
    uint32_t pad0;
    const vxb_worker_table* workers;  /* NetworkTables::workers */
    const uint16_t* unit_worker;      /* NetworkTables::unit_worker */
    const uint32_t* unit_local_base;  /* NetworkTables::unit_local_base */
    const vxb_unit* units;            /* NetworkLayout::units */
} vxb_network;

/* voxsim::Injection (engine.hpp:16-21). */
typedef struct vxb_injection {
    uint32_t from_step;
    uint32_t to_step;
    uint32_t voxel;
    float current_pa;
} vxb_injection;

/* voxsim::ForcedSpike (engine.hpp:25-28). */
typedef struct vxb_forced_spike {
    uint32_t step;
    uint32_t pad0;
    uint64_t gid;
} vxb_forced_spike;

/* voxsim::SimOptions (engine.hpp:30-45) plus device placement. */
typedef struct vxb_options {
    double dt_ms;
    const char* scheduler;   /* "cuda" (also accepts "threads"/"loopback") */
    const char* transport;   /* "queue" | "nvlink" */
    uint16_t workers_per_node;
    uint16_t pad0;
    int32_t recv_timeout_ms;
    int32_t record_raster;
    int32_t record_timings;
    const uint64_t* probe_gids;
    uint32_t n_probes;
    uint32_t n_injections;
    const vxb_injection* injections;
    const vxb_forced_spike* forced_spikes;
    uint32_t n_forced;
    int32_t device;          /* CUDA device of shard 0; -1 = current device */
    int32_t n_devices;       /* GPUs the workers are spread over; <= 1 = one */
    int32_t pad1;
} vxb_options;

/* voxsim::RasterEvent (stats.hpp:84-89). */
typedef struct vxb_raster_event {
    uint32_t step;
    uint16_t worker;
    uint16_t pad0;
    uint32_t local;
    uint32_t pad1;
    uint64_t gid;
} vxb_raster_event;

/* voxsim::FlopCounters (stats.hpp:41-52). */
typedef struct vxb_flops {
    uint64_t membrane;
    uint64_t gating_inner;
    uint64_t gating_outer;
    uint64_t gating_decay;
    uint64_t current;
} vxb_flops;

/* voxsim::StepTimings (stats.hpp:17-38). t[0..10] = t1..t11. */
typedef struct vxb_step_timings {
    uint32_t step;
    uint16_t worker;
    uint16_t pad0;
    int64_t t[11];
    int64_t send_intra_ns, send_inter_ns, recv_intra_ns, recv_inter_ns;
    uint64_t bytes_sent_intra, bytes_sent_inter, bytes_recv_intra, bytes_recv_inter;
    uint32_t spikes;
    uint32_t pad1;
} vxb_step_timings;

typedef struct vxb_engine vxb_engine;

/* ---- lifecycle ----------------------------------------------------------- */
int vxb_create(const vxb_network* net, const vxb_options* opt, vxb_engine** out);
void vxb_destroy(vxb_engine* e);
/* Error text of the last failing call on `e` (or of the last failed
 * vxb_create on this thread when e == NULL). */
const char* vxb_last_error(const vxb_engine* e);
int vxb_abi_version(void);
/* SHA-256 prefix of the sources and flags this library was built from
 * (paper_2308_01241_b200/build.py source_hash). */
const char* vxb_build_hash(void);

/* ---- stepping ------------------------------------------------------------ */
/* Advances `steps` steps; results are kept inside the engine until the next
 * vxb_advance and read with vxb_result_*. */
int vxb_advance(vxb_engine* e, uint32_t steps);
uint32_t vxb_current_step(const vxb_engine* e);

/* ---- RunResult of the last vxb_advance ------------------------------------ */
uint32_t vxb_result_steps_done(const vxb_engine* e);
uint64_t vxb_result_total_spikes(const vxb_engine* e);
uint64_t vxb_result_raster_size(const vxb_engine* e);
/* Raster sorted (step, worker, local) (engine.cpp:812-817). */
int vxb_result_raster(const vxb_engine* e, vxb_raster_event* out, uint64_t cap);
/* RateSeries::counts as [n_units][steps] row-major. */
int vxb_result_rates(const vxb_engine* e, uint32_t* counts, uint64_t cap);
/* ProbeTrace v / i_syn as [n_probes][steps]. */
int vxb_result_probes(const vxb_engine* e, float* v, float* i_syn, uint64_t cap);
int vxb_result_flops(const vxb_engine* e, vxb_flops* out);
uint64_t vxb_result_timings_size(const vxb_engine* e);
int vxb_result_timings(const vxb_engine* e, vxb_step_timings* out, uint64_t cap);
/* Device time of the last advance's step kernel(s), milliseconds (CUDA
 * events on the launching stream; max over shards). */
double vxb_result_device_ms(const vxb_engine* e);
/* Exposed spike-exchange wait of the last advance: sum over steps of the
 * longest time any CTA waited for a peer's batch, milliseconds. */
double vxb_result_exchange_wait_ms(const vxb_engine* e);
/* Arrival lag of the last advance: sum over steps of how long after the
 * start of the phase that delivers S(t) the last peer's batch of S(t) was
 * first observed, milliseconds.  Unlike vxb_result_exchange_wait_ms (time
 * CTAs spent spinning once their local work was done) it does not depend on
 * how much local work the CTAs had; the exchange is exposed only where the
 * lag exceeds the phase's local work. */
double vxb_result_exchange_arrival_ms(const vxb_engine* e);
/* Bytes copied host->device / device->host by the last vxb_advance. */
uint64_t vxb_result_h2d_bytes(const vxb_engine* e);
uint64_t vxb_result_d2h_bytes(const vxb_engine* e);
/* One worker per rank, with record_timings: the wire bytes of the batches
 * this rank's worker sent in the last advance, [steps][dst worker] (the
 * reference's encode_batch sizes, transport.cpp:33-55; 12 for an empty
 * batch, 0 for itself).  The caller hands every rank the bytes its peers sent
 * it, [steps][src worker], with vxb_set_recv_wire_bytes, which completes the
 * StepTimings received-byte counters (engine.cpp:495-523). */
int vxb_result_wire_bytes(const vxb_engine* e, uint64_t* out, uint64_t cap);
int vxb_set_recv_wire_bytes(vxb_engine* e, const uint64_t* in, uint32_t steps);
/* crossing_matrix (netgen.hpp:104-107, netgen.cpp:331-355; BuiltNetwork::
 * crossing, pipeline.cpp:122): synapses per (source worker, target worker),
 * [workers][workers] row-major, counted on the device from the delivery
 * tables at load.  With one worker per rank only column `rank` is filled:
 * the caller adds the ranks' matrices. */
int vxb_crossing_matrix(const vxb_engine* e, uint64_t* out, uint64_t cap);
/* Kernel launches issued by the last vxb_advance. */
uint64_t vxb_result_launches(const vxb_engine* e);
/* The delivery schedule chosen for this network as a JSON object (path, grid,
 * L2 blocks, deal, stage size, ...) including every tuning knob applied from
 * the environment (knobs are read only when VXB_TUNING=1).  No reference
 * counterpart: benchmark bookkeeping. */
int vxb_schedule_info(const vxb_engine* e, char* out, uint64_t cap);

/* ---- state access -------------------------------------------------------- */
int vxb_set_conductances(vxb_engine* e, uint32_t unit, int receptor,
                         const float* values, uint32_t n);
/* vxb_set_conductances for `count` (unit, receptor, values[i], counts[i])
 * items in one call: the same result and errors as calling it item by item
 * in order (staging stops at the first failing item, whose index goes to
 * *failed_index; `count` when all succeed), with the validation and the
 * copies spread over the host's cores.  The assimilation caller's per-window
 * input (assim.cpp:91-107) in one crossing of the boundary. */
int vxb_set_conductances_batch(vxb_engine* e, uint32_t count, const uint32_t* units,
                               const int32_t* receptors, const float* const* values,
                               const uint32_t* counts, uint32_t* failed_index);
int vxb_membrane_snapshot(const vxb_engine* e, uint16_t worker, float* out,
                          uint32_t cap);
uint32_t vxb_worker_neurons(const vxb_engine* e, uint16_t worker);
uint16_t vxb_workers(const vxb_engine* e);
uint32_t vxb_units(const vxb_engine* e);
uint32_t vxb_probes(const vxb_engine* e);

/* ---- on-device network generation ----------------------------------------
 * Replaces sample_synapses + emit_tables (netgen.hpp:84-92, netgen.cpp:51-316)
 * for networks too large to build on the host: the per-neuron records are
 * drawn on the host (O(neurons)), the K in-picks of every neuron are drawn on
 * the device and written straight into the engine's delivery tables.  Draws
 * are keyed by (seed, gid, slot) exactly as the reference, so the tables are
 * those emit_tables would produce for the same layout/connectome/partition.
 */

/* PopulationSpec (layout.hpp:17-38) + NeuronParams/OuParams of one unit. */
typedef struct vxb_gen_population {
    double g_location[VXB_RECEPTORS];
    double g_scale[VXB_RECEPTORS];
    double weight_mean[VXB_RECEPTORS];
    double weight_spread[VXB_RECEPTORS];
    double split_ratio;
    float capacitance, g_leak, e_leak, v_threshold, v_reset;
    uint32_t refractory_steps;
    float e_rev[VXB_RECEPTORS];
    float tau[VXB_RECEPTORS];
    float omega[VXB_RECEPTORS];
    float ou_mean, ou_sigma, ou_tau;
    uint8_t excitatory;
    uint8_t dual_receptor;
    uint8_t pad0[2];
} vxb_gen_population;

/* VoxelSpec (layout.hpp:40-49) after NetworkLayout::build. */
typedef struct vxb_gen_voxel {
    uint32_t k_in;
    uint32_t region;     /* Region enum (layout.hpp:12) */
    double rho;
    uint32_t unit_begin; /* NetworkLayout::voxel_unit_base[v] */
    uint32_t unit_end;
} vxb_gen_voxel;

/* ConnectomeEdge (connectome.hpp:14-18). */
typedef struct vxb_gen_edge {
    uint32_t src;
    uint32_t dst;
    double weight;
} vxb_gen_edge;

typedef struct vxb_netspec {
    uint64_t seed;
    uint32_t n_voxels;
    uint32_t n_units;
    uint32_t n_edges;
    uint32_t n_workers;
    const vxb_gen_voxel* voxels;
    const vxb_unit* units;                /* NetworkLayout::units */
    const vxb_gen_population* unit_pops;  /* population spec of each unit */
    const vxb_gen_edge* edges;            /* sorted by (dst, src) */
    const double* intra[4];               /* IntraMatrices per region, [tgt][src] */
    uint32_t intra_pops[4];
    const uint16_t* unit_worker;          /* PartitionMap::unit_worker */
} vxb_netspec;

int vxb_create_generated(const vxb_netspec* spec, const vxb_options* opt, vxb_engine** out);

/* ---- one process per GPU ------------------------------------------------
 * Rank `rank` of `world` holds worker `rank` of a partition with one worker
 * per rank (PartitionMap.worker_count == world).  Every rank calls the same
 * sequence: vxb_create_generated_rank, exchange the destination masks
 * (vxb_mask_out of rank h for shard r goes to rank r's vxb_mask_in(h)),
 * exchange the receive-region handles (vxb_ipc_handle -> vxb_connect_peers),
 * then vxb_advance collectively.  Spike ids travel by NVLink P2P stores into
 * the peers' receive slots (the reference's per-step spike batches,
 * transport.hpp:13-45); the step barrier is the per-peer step flag.
 */
int vxb_create_generated_rank(const vxb_netspec* spec, const vxb_options* opt, uint32_t rank,
                              uint32_t world, vxb_engine** out);
/* Bytes of the bitmap over shard h's neurons (bit i: neuron i of shard h has
 * at least one target on this rank). */
uint64_t vxb_mask_bytes(const vxb_engine* e, uint32_t h);
int vxb_mask_out(const vxb_engine* e, uint32_t h, uint8_t* bits, uint64_t cap);
/* Bitmap received from rank h over this rank's neurons. */
int vxb_mask_in(vxb_engine* e, uint32_t h, const uint8_t* bits, uint64_t cap);
/* 64-byte cudaIpcMemHandle_t of this rank's receive region. */
int vxb_ipc_handle(const vxb_engine* e, void* out, uint64_t cap);
/* handles: world entries, `stride` bytes apart (own entry ignored). */
int vxb_connect_peers(vxb_engine* e, const void* handles, uint64_t stride);

/* Export worker `worker`'s WorkerTable as emit_tables would build it (for
 * parity checks on small networks).  Sizes: n_neurons = sum of the worker's
 * unit sizes, n_synapses = sum of neurons * k_in of their voxels. */
int vxb_generate_worker_table(const vxb_netspec* spec, int device, uint16_t worker,
                              vxb_neuron* neurons, uint32_t n_cap, vxb_syn_entry* synapses,
                              uint64_t syn_cap, uint64_t* row_base);

/* ---- table files ---------------------------------------------------------- */
/* FNV-1a 64 (util.hpp:39-46) over n bytes continuing from hash h (start with
 * 0xcbf29ce484222325): the integrity hash of VXTB table files in
 * manifest.json (netgen.cpp:478-524). */
uint64_t vxb_fnv1a(const void* data, uint64_t n, uint64_t h);

/* ---- diagnostics --------------------------------------------------------- */
/* Device evaluation of stream_normal(base[i], k[i]) (rng.hpp:63-67) with
 * CUDA's log/cos (the fast path), for noise-parity checks against the host. */
int vxb_debug_stream_normal(int device, const uint64_t* base, const uint64_t* k, uint64_t n,
                            double* out);
/* The float OU noise sample (float)stream_normal(base[i], k[i]) exactly as the
 * step kernel computes it (engine.cpp:551-553): fast path, with correctly
 * rounded log/cos for samples near a float rounding boundary. */
int vxb_debug_stream_xi(int device, const uint64_t* base, const uint64_t* k, uint64_t n,
                        float* out);

/* ---- BOLD-proxy readout (hemo.hpp, assim.cpp:51-71) ------------------------ */
typedef struct vxb_hemo_params { /* HemoParams (hemo.hpp:10-23) */
    double kappa, gamma, tau, alpha, e0, v0;
} vxb_hemo_params;
typedef struct vxb_hemo_state { /* HemoState (hemo.hpp:25-30); rest = {0, 1, 1, 1} */
    double s, f, v, q;
} vxb_hemo_state;

/* Enable the device BOLD readout (replaces the assimilation caller's
 * window_bold over RunResult::rates, assim.cpp:51-71 / 91-107): every
 * advance() then drives one Balloon-Windkessel model per voxel with
 * z = voxel_count / (voxel neurons * dt_s) / baseline_hz per step
 * (step_hemodynamics, hemo.cpp:19-41) and samples bold_signal
 * (hemo.cpp:43-47) every `sample_every` steps of the advance, as
 * bold_from_drive does (hemo.cpp:49-62).  `init` (n_voxels states, NULL = rest)
 * seeds the per-voxel state, which then carries across advances.  Errors:
 * HemoParams::validate / baseline_hz > 0 / sample_every >= 1 -> VXB_ECONFIG;
 * a diverged state makes advance() return VXB_ESIM with the reference's
 * message, the simulation itself staying usable.  On several GPUs (one
 * engine per rank) advance() only sums the rank's voxel counts: the caller
 * adds the ranks' vxb_result_voxel_counts and passes the totals to
 * vxb_hemo_feed_counts, which runs the same model on them. */
int vxb_set_hemodynamics(vxb_engine* e, const vxb_hemo_params* p, double baseline_hz,
                         uint32_t sample_every, const vxb_hemo_state* init);
/* Current per-voxel states (cap >= n_voxels). */
int vxb_hemo_get_state(const vxb_engine* e, vxb_hemo_state* out, uint32_t cap);
/* BOLD samples of the last advance: [steps / sample_every][n_voxels]. */
uint64_t vxb_result_bold_size(const vxb_engine* e);
int vxb_result_bold(const vxb_engine* e, double* out, uint64_t cap);
/* Voxel spike counts of the last advance, [steps][n_voxels]
 * (RateSeries::voxel_counts, stats.cpp:193-201; this rank's units only). */
int vxb_result_voxel_counts(const vxb_engine* e, uint32_t* out, uint64_t cap);
/* Several GPUs: run the hemodynamics of the last advance on the ranks'
 * summed voxel counts [steps][n_voxels] (steps = the advance's); the BOLD
 * samples are then read with vxb_result_bold. */
int vxb_hemo_feed_counts(vxb_engine* e, const uint32_t* counts, uint32_t steps);
/* Diagnostics: bold_from_drive (hemo.cpp:49-62) on the device for n_series
 * drive series z[series][steps]; state[n_series] in/out; out[series][steps /
 * sample_every]. */
int vxb_debug_bold_from_drive(int device, const vxb_hemo_params* p, const double* z,
                              uint32_t steps, uint32_t n_series, double dt_s,
                              uint32_t sample_every, vxb_hemo_state* state, double* out);

/* ---- ensemble members (EnsembleMember, assim.hpp / assim.cpp:74-107) ------ */
/* The assimilation caller runs `members` SimInstances of one network that
 * differ only in the conductances set per window.  A member engine is built
 * for the same network as `donor` (its tables as `net`, or its spec as
 * `spec`: exactly one) on the donor's device, and views the donor's synapse
 * tables — read-only during a run — instead of building its own (12 GB for
 * config 2).  Neuron state, pending sums, conductances, BOLD state and results
 * are the member's own.  The shared tables are reference-counted: they stay
 * allocated until the donor and every member are destroyed, in any order.
 * One GPU only. */
int vxb_create_member(const vxb_engine* donor, const vxb_network* net,
                      const vxb_netspec* spec, const vxb_options* opt, vxb_engine** out);

/* Advance `count` ensemble members of one donor by `steps` together: each
 * member's step kernel is launched on its own stream with an equal share of
 * the SMs, so the members run concurrently over the shared tables (the
 * reference advances EnsembleMembers one after another, assim.cpp:231-233).
 * Results per member as after vxb_advance; the first error is returned and
 * the failing member's error text is in vxb_last_error(member).  Members on
 * the SM-tile path advance one after another. */
int vxb_advance_members(vxb_engine** members, uint32_t count, uint32_t steps);

/* ---- one-call convenience (run_simulation, engine.hpp:92-93) ------------- */
/* Creates, advances `steps` and returns the engine holding the results. */
int vxb_run_simulation(const vxb_network* net, const vxb_options* opt,
                       uint32_t steps, vxb_engine** out);

#ifdef __cplusplus
}
#endif

#endif /* VXB_H */

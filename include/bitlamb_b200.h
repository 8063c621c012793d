/* bitlamb_b200.h — C-ABI of the B200-native 1-bit LAMB compression-stage path.
 *
 * Drop-in boundary for the reference library's communicator and optimizer
 * (/root/reference/proj, C++20).  Each entry point names the reference
 * interface it replaces (file:line relative to /root/reference/proj).  Plain
 * pointers and sizes only: no C++ or torch types cross this boundary, and no
 * exception escapes it — every call returns a bl_status whose codes map 1:1
 * to the reference's exception classes (include/bitlamb/errors.hpp:26-53);
 * bl_last_error() returns the message of the last failure on this thread.
 *
 * State lives in HBM as flat fp32 buffers with per-layer offset tables
 * (FusedLayout, fusion.hpp:29-44).  All device work of one object is
 * enqueued on one CUDA stream (bl_cluster_config.stream).  A call that
 * returns host data (trace, getters) synchronizes that stream; otherwise
 * calls are asynchronous and device-side failures (non-finite inputs) are
 * reported by the next synchronizing call.
 *
 * Transactional steps.  Every step / collective starts with a device-side
 * gate.  In strict mode (bl_optimizer_set_strict) a read-only pre-pass checks
 * every gradient first, as Optimizer::check_gradients does before touching any
 * state (optimizers.cpp:99-117,337); multi-process, the gate is also the
 * step's arrival barrier.  A failure there (non-finite gradient on any rank, a
 * rank late past the peer timeout) aborts the step on every rank before any
 * state changes: the next synchronizing call raises it and the object stays
 * usable with its state as before the step.  A peer that dies INSIDE a step is
 * fail-stop: the error is raised and the cluster refuses further work.
 */
#ifndef BITLAMB_B200_H_
#define BITLAMB_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BL_ABI_VERSION 2
#define BL_NCCL_UNIQUE_ID_BYTES 128

/* Status codes: errors.hpp:26-53 + check_arg / runtime_error uses. */
typedef enum bl_status {
  BL_OK = 0,
  BL_ERR_DIMENSION = 1,        /* bitlamb::DimensionError (std::invalid_argument) */
  BL_ERR_STAGE_ORDER = 2,      /* bitlamb::StageOrderError (std::logic_error) */
  BL_ERR_CONFIG = 3,           /* bitlamb::ConfigError (std::runtime_error) */
  BL_ERR_INVALID_ARGUMENT = 4, /* std::invalid_argument (check_arg, non-finite scale) */
  BL_ERR_RUNTIME = 5,          /* std::runtime_error (non-finite gradient / reconstruction) */
  BL_ERR_LOGIC = 6,            /* std::logic_error (misuse) */
  BL_ERR_CUDA = 7,             /* CUDA runtime failure (no reference equivalent) */
  BL_ERR_NCCL = 8,             /* NCCL failure (no reference equivalent) */
  BL_ERR_UNSUPPORTED = 9       /* feature of the reference not on the B200 path */
} bl_status;

typedef enum bl_compressor {  /* CompressorKind, compression.hpp:27-30 */
  BL_COMPRESSOR_ONEBIT = 0,
  BL_COMPRESSOR_IDENTITY = 1
} bl_compressor;

typedef enum bl_mode {
  BL_MODE_SIM = 0,  /* n_workers simulated ranks in one GPU's HBM (SimCluster) */
  BL_MODE_NCCL = 1  /* this process is rank `rank` of n_workers over NCCL */
} bl_mode;

typedef enum bl_variant {  /* OptimizerVariant, optimizers.hpp:30-39 */
  BL_LAMB = 0,
  BL_ADAM = 1,
  BL_ONEBIT_LAMB = 2,
  BL_LAMB_BASIC_ONEBIT = 3,
  BL_ONEBIT_ADAM = 4
} bl_variant;

typedef enum bl_memory { BL_MEM_HOST = 0, BL_MEM_DEVICE = 1 } bl_memory;

/* How NCCL-mode ranks exchange packets. */
typedef enum bl_transport {
  BL_TRANSPORT_AUTO = 0, /* fused NVLink peer stores when every peer maps, else NCCL */
  BL_TRANSPORT_NCCL = 1, /* grouped ncclSend/ncclRecv alltoall + ncclAllGather */
  BL_TRANSPORT_P2P = 2   /* fused: K1/K3 store packet words into peer HBM (CUDA IPC) */
} bl_transport;

typedef enum bl_state {  /* LayerState members, optimizers.hpp:68-78 */
  BL_STATE_X = 0,
  BL_STATE_M = 1,
  BL_STATE_V = 2,
  BL_STATE_V_FROZEN = 3,
  BL_STATE_M_PREV = 4
} bl_state;

/* SimCluster::Config, comm_sim.hpp:72-80, plus the B200 placement fields. */
typedef struct bl_cluster_config {
  int32_t n_workers;
  int32_t mode;   /* bl_mode */
  int32_t rank;   /* BL_MODE_NCCL only */
  int32_t device; /* CUDA device ordinal */
  uint64_t dim;
  int32_t compressor; /* bl_compressor */
  int32_t baseline_bits_per_element;
  int32_t verify_compensation; /* re-check v + d_prev == dec + d_new on the device after every
                                  collective with error_scale == 1 (comm_sim.cpp:83-106);
                                  the fp32 path needs a tolerance >= 2^-23 */
  int32_t endpoint_stats;      /* refresh EndpointStats every collective (extra pass) */
  double compensation_tolerance;
  const uint8_t* nccl_unique_id; /* BL_NCCL_UNIQUE_ID_BYTES, BL_MODE_NCCL only */
  void* stream;                  /* cudaStream_t; NULL = library-owned stream */
  int32_t transport;             /* bl_transport, BL_MODE_NCCL only */
} bl_cluster_config;

/* VolumeLedger, comm_sim.hpp:37-50 */
typedef struct bl_volume_ledger {
  uint64_t gather_bits;
  uint64_t scatter_bits;
  uint64_t lossless_bits;
  uint64_t baseline_equivalent_bits;
  uint64_t compressed_collectives;
  uint64_t lossless_collectives;
} bl_volume_ledger;

/* SimCluster::EndpointStats, comm_sim.hpp:85-91 */
typedef struct bl_endpoint_stats {
  double delta_l2;
  double delta_linf;
  double corrected_linf;
  double max_delta_linf;
  double max_corrected_linf;
} bl_endpoint_stats;

/* HyperParams, optimizers.hpp:45-64 */
typedef struct bl_hparams {
  double beta1, beta2, beta3, eta;
  double c_min, c_max, r_min, r_max, r_threshold;
  double weight_decay, division_floor;
  uint64_t total_steps, warmup_steps;
  int32_t scaled_error_feedback;
} bl_hparams;

/* StepTrace, optimizers.hpp:81-87; caller-owned arrays of n_layers. */
typedef struct bl_step_trace {
  double* c;
  double* r;
  double* v_norm;
  double* v_ratio_preclip;
  int32_t compressed;
} bl_step_trace;

/* Optimizer::LayerSpec, optimizers.hpp:95-98. */
typedef struct bl_layer_spec {
  const char* name;
  uint64_t size;
} bl_layer_spec;

typedef struct bl_cluster bl_cluster;
typedef struct bl_optimizer bl_optimizer;

const char* bl_last_error(void);
int32_t bl_abi_version(void);
bl_status bl_nccl_get_unique_id(uint8_t* out /* BL_NCCL_UNIQUE_ID_BYTES */);

/* HyperParams defaults (optimizers.hpp:46-58). */
void bl_hparams_default(bl_hparams* hp);

/* ---- SimCluster (comm_sim.hpp:72-148) ---------------------------------- */

/* SimCluster::SimCluster (comm_sim.cpp:50-66): validates n >= 1, dim >= 1,
 * baseline bits >= 1 (BL_ERR_INVALID_ARGUMENT).  Pads dim to P = ceil(dim/n)*n. */
bl_status bl_cluster_create(const bl_cluster_config* cfg, bl_cluster** out);
void bl_cluster_destroy(bl_cluster* c);
bl_status bl_cluster_dims(const bl_cluster* c, uint64_t* padded, uint64_t* chunk);
/* The packet transport in use (bl_transport; BL_TRANSPORT_AUTO is resolved). */
int32_t bl_cluster_transport(const bl_cluster* c);
/* The CUDA stream (cudaStream_t) every device call of this cluster and of its
 * optimizer is enqueued on.  Callers that produce inputs on another stream
 * make this stream wait on theirs (and theirs on this one for outputs). */
void* bl_cluster_stream(const bl_cluster* c);
/* SimCluster::config() (comm_sim.hpp:105): the configuration the cluster was
 * created with (transport resolved). */
bl_status bl_cluster_get_config(const bl_cluster* c, bl_cluster_config* out);
/* SimCluster::step_count() (comm_sim.hpp:108; incremented per compressed and
 * per lossless collective, comm_sim.cpp:197,230). */
uint64_t bl_cluster_step_count(const bl_cluster* c);
/* Bound of every wait on a peer (multi-process), default 600000 ms.  A rank
 * that does not arrive at a step within it aborts that step on every rank
 * (state unchanged); a peer silent inside a step fails the cluster. */
bl_status bl_cluster_set_peer_timeout(bl_cluster* c, double ms);

/* SimCluster::compressed_allreduce (comm_sim.hpp:98-99, comm_sim.cpp:120-203).
 * inputs[i] is worker i's stream of `len` floats (len must equal dim,
 * n_inputs must equal n_workers in SIM mode and 1 in NCCL mode, else
 * BL_ERR_DIMENSION).  out receives the dim-long result (identical on every
 * rank).  memory says where inputs/out live. */
bl_status bl_cluster_compressed_allreduce(bl_cluster* c, const float* const* inputs,
                                          int32_t n_inputs, uint64_t len, float* out,
                                          double error_scale, int32_t memory);

/* SimCluster::lossless_allreduce (comm_sim.hpp:102, comm_sim.cpp:205-232). */
bl_status bl_cluster_lossless_allreduce(bl_cluster* c, const float* const* inputs,
                                        int32_t n_inputs, uint64_t len, float* out,
                                        int32_t memory);

/* SimCluster::worker_error / server_error (comm_sim.hpp:126-131).  Host out:
 * padded floats for a worker, chunk floats for a server.  In NCCL mode only
 * the local worker (i == rank) and local server (j == rank) exist. */
bl_status bl_cluster_worker_error(bl_cluster* c, int32_t i, float* out);
bl_status bl_cluster_server_error(bl_cluster* c, int32_t j, float* out);

/* Wire bytes of the last collective's packets in CompressedBlock::serialize
 * layout (compression.cpp:91-99): ceil(chunk/8) sign bytes + LE fp32 scale. */
bl_status bl_cluster_packet(bl_cluster* c, int32_t worker, int32_t server, uint8_t* bytes);
bl_status bl_cluster_server_packet(bl_cluster* c, int32_t server, uint8_t* bytes);

bl_status bl_cluster_ledger(const bl_cluster* c, bl_volume_ledger* out); /* ledger() */
/* worker_stats()/server_stats() (comm_sim.hpp:113-114): 2n entries, workers
 * first.  Requires cfg.endpoint_stats. */
bl_status bl_cluster_stats(bl_cluster* c, bl_endpoint_stats* out);
bl_status bl_cluster_synchronize(bl_cluster* c);

/* Device buffer of `dim` floats the caller may fill in place of passing
 * inputs (zero-copy compressed_allreduce with memory=BL_MEM_DEVICE). */
float* bl_cluster_input_buffer(bl_cluster* c, int32_t worker);

/* Instrumentation: number of kernels this object launched, and optional
 * CUDA-event timing per kernel class (names[k], total ms, launches). */
uint64_t bl_cluster_kernel_launches(const bl_cluster* c);
/* compensation_checks() (comm_sim.hpp:110): endpoints verified on this rank. */
uint64_t bl_cluster_compensation_checks(const bl_cluster* c);
bl_status bl_cluster_set_profiling(bl_cluster* c, int32_t on);
int32_t bl_cluster_profile(bl_cluster* c, const char** names, double* total_ms,
                           uint64_t* launches, int32_t cap);

/* volume_reduction (comm_sim.hpp:55-56, comm_sim.cpp:36-48). */
bl_status bl_volume_reduction(double warmup_ratio, double baseline_bits,
                              double compressed_bits_per_element, double* out);

/* ---- Optimizer (optimizers.hpp:93-145) -------------------------------- */

/* Optimizer::Optimizer (optimizers.cpp:76-97): HyperParams::validate
 * (BL_ERR_CONFIG), >= 1 layer and sizes > 0 (BL_ERR_INVALID_ARGUMENT).  The
 * optimizer lives on the cluster's device and stream. */
bl_status bl_optimizer_create(int32_t variant, const uint64_t* layer_sizes, int32_t n_layers,
                              const bl_hparams* hp, bl_cluster* cluster, bl_optimizer** out);
/* The same with Optimizer::LayerSpec {name, size} (optimizers.hpp:95-101):
 * the names appear in error messages exactly as the reference prints them. */
bl_status bl_optimizer_create_named(int32_t variant, const bl_layer_spec* layers, int32_t n_layers,
                                    const bl_hparams* hp, bl_cluster* cluster, bl_optimizer** out);
const char* bl_optimizer_layer_name(const bl_optimizer* o, int32_t layer);
/* Strict mode: check_gradients (optimizers.cpp:99-117) as a read-only
 * pre-pass before any state changes (+4 bytes/param read per step; with
 * multi-process every rank raises the same error).  Default off: the finite
 * check is fused into the first kernel that reads the gradient and reported
 * by the next synchronizing call, after the step was applied. */
bl_status bl_optimizer_set_strict(bl_optimizer* o, int32_t on);
void bl_optimizer_destroy(bl_optimizer* o);

/* Optimizer::step (optimizers.hpp:106-107, optimizers.cpp:334-364).
 * grads[i] is worker i's fused (layer-major) gradient of fused_dim floats;
 * n_grads as for compressed_allreduce.  trace may be NULL (fully
 * asynchronous step); otherwise it is filled and the stream synchronized. */
bl_status bl_optimizer_step(bl_optimizer* o, bl_cluster* c, const float* const* grads,
                            int32_t n_grads, uint64_t t, double lr, int32_t memory,
                            bl_step_trace* trace);

/* Device gradient buffer for worker i (zero-copy step with memory=BL_MEM_DEVICE). */
float* bl_optimizer_grad_buffer(bl_optimizer* o, int32_t worker);

/* layers()/mutable_layers() state access (optimizers.hpp:109-110), fused.
 * Multi-process clusters over NVLink keep m and v sharded by tile owner
 * during the warmup stage (each rank updates 1/n of the tiles and stores
 * the new x into every rank); reading BL_STATE_M or BL_STATE_V there first
 * gathers every owner's slice, so every rank must make that call (the
 * freeze step gathers m, v and v_frozen itself; x is always complete). */
bl_status bl_optimizer_get_state(bl_optimizer* o, int32_t which, float* host_out);
bl_status bl_optimizer_set_state(bl_optimizer* o, int32_t which, const float* host_in);
/* c_avg, r_prev, MomentumScales::coeff per layer (any pointer may be NULL). */
bl_status bl_optimizer_get_scalars(bl_optimizer* o, double* c_avg, double* r_prev,
                                   double* scale_coeff);
bl_status bl_optimizer_set_scalars(bl_optimizer* o, const double* c_avg, const double* r_prev);
int32_t bl_optimizer_frozen(const bl_optimizer* o);     /* frozen() */
uint64_t bl_optimizer_fused_dim(const bl_optimizer* o); /* fused_dim() */
int32_t bl_optimizer_layer_count(const bl_optimizer* o);

/* ---- Free functions (compression.hpp:106-118, fusion.hpp:92-102) -------- */

/* compress_with_feedback (compression.hpp:111-118, compression.cpp:166-198) on
 * the device: corrected = v + error_scale * delta is compressed (sign bits +
 * scale mean|corrected|, or the identity message), and delta is replaced by
 * v + delta - decompress(message) (identity: 0).  wire_out (host, may be NULL):
 * serialize() bytes, ceil(len/8) sign bytes + LE fp32 scale (one-bit only);
 * decompressed_out (may be NULL): the len decompressed floats.  v, delta and
 * decompressed_out live in `memory`.  Non-finite scale: BL_ERR_INVALID_ARGUMENT. */
bl_status bl_compress_with_feedback(const float* v, float* delta, uint64_t len, int32_t compressor,
                                    double error_scale, uint8_t* wire_out, float* decompressed_out,
                                    int32_t memory, int32_t device);
/* compute_scales (fusion.hpp:92-93, fusion.cpp:107-125): s_l = max(mean|m_l|,
 * floor), reference = mean_l s_l, coeff_l = reference / s_l over the fused
 * (layer-major) momentum m of sum(layer_sizes) floats in `memory`.  coeff_out
 * (n_layers doubles) and reference_out are host memory. */
bl_status bl_compute_scales(const float* m, const uint64_t* layer_sizes, int32_t n_layers,
                            double floor, double* coeff_out, double* reference_out, int32_t memory,
                            int32_t device);
/* apply_scaling / remove_scaling (fusion.hpp:96-102, fusion.cpp:127-149): each
 * layer segment of the fused buffer is multiplied by coeff_l / by 1/coeff_l. */
bl_status bl_apply_scaling(float* fused, const uint64_t* layer_sizes, int32_t n_layers,
                           const double* coeff, int32_t memory, int32_t device);
bl_status bl_remove_scaling(float* fused, const uint64_t* layer_sizes, int32_t n_layers,
                            const double* coeff, int32_t memory, int32_t device);

#ifdef __cplusplus
}
#endif

#endif /* BITLAMB_B200_H_ */

// bl_runtime.h — host-side objects behind the C-ABI (include/bitlamb_b200.h).
//
// bl_cluster mirrors bitlamb::SimCluster (comm_sim.hpp:72-148): it owns the
// worker/server residuals and the packet buffers in HBM and runs the
// compressed / lossless collectives either over n simulated ranks in one
// GPU's HBM (BL_MODE_SIM) or as rank r of an NCCL communicator
// (BL_MODE_NCCL).  bl_optimizer mirrors bitlamb::Optimizer
// (optimizers.hpp:93-145): flat fp32 x, m, v, vf with a per-layer offset table
// and per-layer fp64 scalars, driving the cluster's kernels in one stream.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdlib>
#include <string>
#include <functional>
#include <vector>

#include "../../include/bitlamb_b200.h"
#include "bl_kernels.cuh"

namespace bl {

struct Error {
  bl_status status;
  std::string msg;
};

[[noreturn]] void fail(bl_status st, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
void nccl_check(ncclResult_t r, const char* what);

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev);
  ~DeviceGuard();

 private:
  int prev_ = -1;
  int dev_;
};

// Kernel classes for launch counting and optional CUDA-event timing.
enum KClass : int {
  KC_K1 = 0, KC_FIN, KC_K3, KC_K5, KC_EPI, KC_K6, KC_W1, KC_WEPI, KC_W2, KC_AVG,
  KC_DEC, KC_MAT, KC_STATS, KC_A2A, KC_AG, KC_H2D, KC_D2H, KC_K1B, KC_SMALL, KC_GATE, KC_COUNT
};
extern const char* const kClassNames[KC_COUNT];

template <typename T>
T* dalloc(size_t n);  // zero-initialised device allocation

// Device table over [reps][per] with the per-rep boundary tiles `slow` first.
int* boundary_first_order(const std::vector<int>& slow, int reps, int per);

}  // namespace bl

struct bl_optimizer;

struct bl_cluster {
  bl_cluster_config cfg{};
  int n = 1, rank = 0, mode = BL_MODE_SIM, device = 0, nw = 1, ns = 1, sms = 148;
  uint64_t dim = 0, P = 0, c = 0, c_pad = 0, W = 0, slot = 0, in_stride = 0;
  int tpc = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;

  float* in = nullptr;          // [nw][in_stride] inputs / gradients
  float* werr = nullptr;        // [nw][n][c_pad] raw worker residual
  uint32_t* wpk[2] = {nullptr, nullptr};  // [nw][n][slot] worker packets (ping-pong)
  uint32_t* rpk = nullptr;      // [n][slot] received packets (NCCL mode)
  float* serr = nullptr;        // [ns][c_pad] raw server residual
  uint32_t* res[2] = {nullptr, nullptr};  // [n][slot] server packets (ping-pong)
  double* wpart = nullptr;      // [nw][n][tpc]
  double* spart = nullptr;      // [ns][tpc]
  float* wcmax = nullptr;       // [nw][n][tpc] (endpoint stats)
  float* scmax = nullptr;       // [ns][tpc]
  float* out = nullptr;         // [P + slack] decompressed result / lossless output
  float* lrecv = nullptr;       // [n][c_pad] lossless receive buffer (NCCL mode)
  unsigned long long* err = nullptr;  // [kErrSlots]
  double* stat_part = nullptr;  // stats scratch
  float* stat_max = nullptr;
  double* stats_dev = nullptr;  // [2n][5] EndpointStats records (workers, then servers)
  int stat_tiles = 0;

  // Fused NVLink exchange (BL_TRANSPORT_P2P): CUDA-IPC-mapped peer buffers.
  int transport = BL_TRANSPORT_NCCL;
  uint32_t* res_base = nullptr;       // one allocation: res[0] | res[1]
  uint32_t* rx = nullptr;             // [2][n][slot] worker packets addressed to this rank
  // [4n] flags, one per sending rank: worker packets, server packets,
  // lossless input in place, lossless chunk delivered
  unsigned long long* flags = nullptr;
  uint32_t** d_peer_rx = nullptr;     // [n] device table of peers' rx
  uint32_t** d_peer_res = nullptr;    // [n] device table of peers' res_base
  unsigned long long** d_peer_flags = nullptr;  // [n]
  float** d_peer_in = nullptr;        // [n] peers' gradient buffers (lossless over NVLink)
  float** d_peer_out = nullptr;       // [n] peers' output buffers
  unsigned long long** d_peer_err = nullptr;  // [n] peers' error words
  unsigned int* lossless_done = nullptr;
  unsigned int* small_bar = nullptr;  // grid barrier of the fused small collective
  unsigned long long* small_ts = nullptr;  // BL_SMALL_TS phase timestamps
  uint2* ll_rx = nullptr;              // [2][n][slot] LL worker packets addressed to this rank
  uint2* ll_res = nullptr;             // [2][n][slot] LL server packets
  uint2** d_peer_llrx = nullptr;       // [n]
  uint2** d_peer_llres = nullptr;      // [n]
  // Collectives of at most this many K1 tiles per rank take the fused
  // small-collective kernel (BL_SMALL_MAX_TILES; 0 disables).
  static long long small_max_tiles() {
    static const long long v = [] {
      const char* e = std::getenv("BL_SMALL_MAX_TILES");
      return e ? std::atoll(e) : 2048ll;  // N=2/4 sweeps: the split kernels win from 64 MB per rank
    }();
    return v;
  }
  unsigned long long lcalls = 0;      // lossless collectives run (flag epoch)
  // Step gate (bl_kernels.cuh GateParams): arrival words at flags[4n + q],
  // rank 0's decision word at flags[5n].
  unsigned long long gate_epoch = 0;
  unsigned long long* gate_status = nullptr;  // NCCL transport: min-reduced status word
  double peer_timeout_ms = 600000.0;          // fail-stop bound of every peer wait
  std::vector<void*> ipc_opened;
  void setup_p2p(bool required);

  unsigned int* tile_ctr = nullptr;  // dynamic tile counter shared by the stream's kernels
  int* k1_slow = nullptr;       // API-mode K1 tiles that are not full/inside the data
  int k1_n_slow = 0;
  int* k1_order = nullptr;      // API-mode K1 processing order, boundary tiles first

  // Host gradient staged for the next compressed collective: copied in
  // pieces that K1 consumes as they land (optimizer step, BL_MEM_HOST).
  const float* stage_host = nullptr;
  static constexpr int kPieces = 16;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t piece_ev[kPieces + 1] = {};

  uint64_t checks = 0;          // compensation checks run (comm_sim.hpp:110)
  bool verify_es_one = true;    // the optimizer's device error scale is 1 (no scaled EF)
  void verify_last();           // verify_compensation over the local endpoints

  uint64_t calls = 0;           // compressed collectives run (ping-pong index)
  bool last_identity = false;
  bl_volume_ledger ledger{};
  uint64_t launches = 0;
  bool profiling = false;
  struct Ev {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[bl::KC_COUNT] = {};
  uint64_t prof_n[bl::KC_COUNT] = {};
  uint64_t pending_step = 0;    // step index of the last asynchronous optimizer step
  bool pending_is_step = false;

  // Transactional steps: the host-side state at the start of every step /
  // collective not yet confirmed by a clean synchronizing call.  A gate that
  // closed before any mutation (strict non-finite gradient, late peer) rolls
  // the host state back to the snapshot of the step it closed at; the device
  // state is untouched because every later kernel returned at entry.
  struct Snap {
    uint64_t seq, t;
    bool is_step;
    uint64_t calls, checks;
    bool last_identity;
    bl_volume_ledger ledger;
    bl_optimizer* opt;
    bool frozen, has_vf, has_mprev, m_valid, mprev_separate;
    uint64_t my_calls;
  };
  std::vector<Snap> snaps;
  uint64_t seq = 0;
  bool broken = false;          // fail-stop: a peer died mid-step, the state is undefined
  std::string broken_msg;
  // Start of a step / collective: snapshot, then the strict pre-pass and the
  // gate (arrival barrier when multi-process).  `opt` may be null.
  void begin_step(bl_optimizer* opt, uint64_t t, bool is_step, bool strict);
  void ensure_usable() const;
  void set_peer_timeout(double ms);
  bl_optimizer* last_opt = nullptr;  // optimizer of the latest step (layer names in messages)
  std::vector<bl_optimizer*> opts;   // live optimizers bound to this cluster

  int cur() const { return static_cast<int>(calls & 1u); }
  int prev() const { return static_cast<int>((calls + 1u) & 1u); }

  // Event-bracketed launch bookkeeping.
  void begin(int cls, cudaEvent_t* a);
  void end(int cls, cudaEvent_t a, int kernels);
  cudaEvent_t get_event();

  int grid(long long tiles) const;
  void copy_inputs(const float* const* inputs, int n_inputs, uint64_t len, int memory);
  // One compressed collective over the inputs already in `in` (mode 0) or a
  // stream built by the optimizer (K1 params supplied by the caller).
  // Returns true when the result was also decompressed into dec_out (the
  // fused small-collective path).
  bool compressed(const bl::K1Params* k1_override, int k1_mode, float es_host,
                  const float* es_dev, float* dec_out = nullptr);
  void finish_compressed(float es_host, const float* es_dev);
  void lossless(bool check_finite);  // in -> out (averaged), ledger
  void share_grad_error();           // NCCL transport: min-reduce the kErrGrad word over ranks
  // Warmup overlap (P2P, n > 1): the lossless exchange runs on comm_stream,
  // delivering the result in `pieces` pieces (flags at piece_flag_base); the
  // caller's consumers wait per piece on the main stream, then join.
  // Returns the exchange epoch.
  unsigned long long lossless_pieces(bool check_finite, int pieces);
  int piece_flag_base() const { return 6 * n + 8; }
  static constexpr int kMaxPieces = 64;
  // Owner-sharded warmup flags: [n] tile partials delivered, [n] owned x delivered.
  int shard_flag_base() const { return piece_flag_base() + n * kMaxPieces; }
  // Map `local` buffers of every rank into this process (CUDA IPC; collective).
  // peer[k][q] = rank q's buffer k (own rank: local[k]); false if any peer
  // could not be mapped on some rank (then nothing stays open).
  bool map_peer_buffers(const std::vector<void*>& local, std::vector<std::vector<void*>>* peer,
                        std::vector<void*>* opened);
  unsigned int* piece_done = nullptr;  // [kMaxPieces]
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void ensure_side_stream();
  void fork_side(const std::function<int(cudaStream_t)>& launch);
  void join_side();
  void refresh_stats();
  void check_errors(const bl_optimizer* opt);
  void sync_and_check(const bl_optimizer* opt);
  void rollback(uint64_t seq_closed);
  void ledger_compressed();
  void ledger_lossless();
  uint64_t chunk_payload_bits(uint64_t j) const;
};

struct bl_optimizer {
  int variant = BL_ONEBIT_LAMB, L = 0;
  bl_hparams hp{};
  uint64_t d = 0;
  bl_cluster* cl = nullptr;
  std::vector<uint64_t> off;  // host copy of the layer table
  uint64_t* off_dev = nullptr;
  int* tile_layer = nullptr;
  int* layer_tile_start = nullptr;
  int* tile_order = nullptr;  // [tiles] boundary tiles first (LayerTiles::order)
  bool mis_layers = false;    // a layer of >= one tile starts off a 16-B boundary
  int tiles = 0;
  float *x = nullptr, *m = nullptr, *v = nullptr, *vf = nullptr, *mprev = nullptr;
  double *c_avg = nullptr, *r_prev = nullptr, *coeff = nullptr, *mag = nullptr;
  float *A = nullptr, *B = nullptr, *invc = nullptr, *coef_x = nullptr;
  double* trace = nullptr;    // [4L]
  double* cmean = nullptr;    // [2]
  float* es = nullptr;        // [1]
  unsigned int* counter = nullptr;
  double* tile_sums = nullptr;  // [tiles][4]
  float* tile_max = nullptr;    // [tiles]
  int* k1_tile_layer = nullptr;  // [n][tpc]: layer of a full single-layer K1 tile, else -1
  int* k1_slow = nullptr;        // the remaining (j*tpc+t) tiles
  int k1_n_slow = 0;
  int* k1_order = nullptr;       // K1 processing order, boundary tiles first
  bool frozen = false, has_vf = false, has_mprev = false;
  std::vector<std::string> names;  // layer names (LayerSpec::name) for error messages
  std::vector<int> tile_order_h;   // host copy of tile_order
  // Warmup overlap tables (built for the cluster's chunk length and piece
  // count on first use): tiles / layers bucketed by the lossless piece after
  // which their data (W1) or their whole layer (epilogue, W2) is delivered.
  int piece_k = 0;
  int* w1_order = nullptr;  // [tiles]
  int* w2_order = nullptr;  // [tiles]
  int* lw_order = nullptr;  // [L]
  std::vector<int> w1_start, w2_start, lw_start;  // [piece_k + 1]
  void build_piece_tables(int pieces);
  // Owner-sharded warmup (multi-process over NVLink): rank r owns tiles
  // [shard_t0, shard_t1) = elements [shard_e0, shard_e1); it reduces only the
  // owned gradient, runs W1/W2 on the owned tiles, and stores its x (and at
  // the freeze m, v, vf) into every peer.  m and v of the other owners' tiles
  // are stale until the freeze or a (collective) state read.
  bool shard_ready = false, shard_stale = false;
  int shard_t0 = 0, shard_t1 = 0;
  uint64_t shard_e0 = 0, shard_e1 = 0;
  int* own_order = nullptr;  // owned tiles, boundary tiles first
  int own_count = 0;
  // W1 follows the owned-range reduce piece by piece: owned tiles bucketed by
  // the reduce piece after which their gradient is complete.  Layers whose
  // tiles are all owned here ("local") run their epilogue and W2 as soon as
  // their last piece is in; the rest (bucket shard_k) after the exchange of
  // tile partials.
  int shard_k = 0, shard_shape = 0;
  int* own_w1_order = nullptr;
  int* own_w2_order = nullptr;
  int* own_lw_order = nullptr;
  std::vector<int> own_w1_start, own_w2_start, own_lw_start;  // [shard_k + 2]
  float **push_x = nullptr, **push_m = nullptr, **push_v = nullptr, **push_vf = nullptr;  // [n-1] peers
  double** push_sums = nullptr;                                                        // [n-1] peers
  // BL_SHARD_PUSH=1: the exchange is a push into each owner's staging slots
  // (k_shard_push) + a local reduce per piece (k_shard_reduce) instead of pulls.
  bool shard_push = false;
  float* stg = nullptr;          // [n][stg_S] staged ranges of every rank's gradient
  uint64_t stg_S = 0;
  uint64_t* e_all_dev = nullptr; // [n + 1] every rank's owned range
  float** d_peer_stg = nullptr;  // [n]
  std::vector<void*> shard_ipc;
  bool sharded_warmup() const;
  void setup_shard();
  void warmup_sharded(double lr, bool track, bool finalize, bool adam);
  void sync_shards();  // collective: every owner's m and v slices into every rank
  // K5/K6 tiles off the fast path for the cluster's chunk length (built on
  // first use; small problems only): taken by k5_general / k6_general on
  // the side stream instead of the streaming kernels.
  int* gen_tiles = nullptr;
  int gen_n = 0;
  uint64_t gen_c = 0;
  void ensure_gen_tiles();
  bool strict = false;          // read-only finite pre-pass before any mutation (optimizers.cpp:99-117)
  bool m_valid = true;          // m buffer holds m (else: decompressed result * invc)
  bool mprev_separate = false;  // m_prev poked by the caller
  uint64_t my_calls = 0;        // cluster->calls after our last compressed step

  bl::LayerTiles lt() const;
  bool two_stage() const {
    return variant == BL_ONEBIT_LAMB || variant == BL_LAMB_BASIC_ONEBIT || variant == BL_ONEBIT_ADAM;
  }
  void step(const float* const* grads, int n_grads, uint64_t t, double lr, int memory,
            bl_step_trace* trace_out);
  void warmup_step(uint64_t t, double lr, bool track, bool finalize, bool adam);
  void warmup_kernels(double lr, bool track, bool finalize, bool adam, int pieces, unsigned long long ep);
  std::vector<int> lt_start_h;  // host copy of layer_tile_start
  void compressed_step(double lr, const float* stage_host);
  // CUDA-graph replay of the steady-state compression step (SIM mode or one
  // rank; BL_GRAPH=0 disables): one captured graph per ping-pong parity, the
  // step's lr staged into a device word before each launch.
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  uint64_t graph_kernels[2] = {0, 0};
  double* lr_dev = nullptr;
  double* lr_host = nullptr;  // pinned
  bool capturing = false;
  bool graphable() const;
  void compressed_step_graph(double lr);
  void materialize_m(float* dst);
};

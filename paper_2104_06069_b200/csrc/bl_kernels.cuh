// bl_kernels.cuh — sm_100a kernels of the 1-bit LAMB compression-stage path.
//
// Every kernel streams flat fp32 buffers in "tiles" of 4096 elements
// (32 rows x 128); one warp owns one tile, lane l owns elements 4l..4l+3 of
// each row (128-bit accesses).  A tile never straddles its reduction segment:
// chunk kernels (K1 worker compress, K3 server reduce) tile each chunk from its
// own element 0, layer kernels (K5/K6 update, W1/W2 warmup) tile each layer
// from its own element 0.  This fixes the reduction order of every sum
// ("tile-tree") independently of the launch shape, which is what
// oracle/liboracle_f32.so restates bit-for-bit.
#pragma once

#include <cstdint>

namespace bl {

constexpr int kTile = 4096;  // elements per tile
constexpr int kRowElems = 128;
constexpr int kRowsPerTile = 32;
constexpr int kWarpsPerBlock = 8;
constexpr int kBlock = 256;

// Device error words (atomicMin keys, ~0ull = none), then configuration words.
enum ErrSlot : int {
  kErrGrad = 0,     // non-finite gradient: key = worker << 40 | element
  kErrScale = 1,    // non-finite compression scale: key = endpoint id
  kErrRecon = 2,    // non-finite reconstructed gradient: key = layer
  kErrPeer = 3,     // peer timeout: key = peer rank
  kErrVerify = 4,   // compensation identity violated: key = chunk-relative element
  kErrGate = 5,     // step gate: ~0 open, else the GateReason that closed it
  kErrGateSeq = 6,  // host sequence number of the step/collective the gate closed at
  kErrRemote = 7,   // non-finite gradient reported by a peer: rank << 32 | layer
  kErrSlots = 8,    // error words (reset to ~0 by the host after it reports them)
  kCfgTimeout = 8,  // peer wait bound in ns (configuration, never reset)
  kErrWords = 16,
};

// Why the step gate closed.  While it is closed every mutating kernel of the
// cluster returns at entry, so the rest of the step (and any step enqueued
// after it) leaves the state untouched until the host reports the error.
enum GateReason : unsigned long long {
  kGateNonFinite = 1,        // strict pre-pass: this rank's gradient is not finite (no mutation yet)
  kGateRemoteNonFinite = 2,  // a peer's strict pre-pass failed (no mutation yet)
  kGateArrival = 3,          // a peer did not arrive at the step within the timeout (no mutation yet)
  kGateMidStep = 4,          // a peer stopped signalling inside a step: fail-stop, state undefined
  kGateInternal = 5,         // a device-side barrier timed out: fail-stop
};

// K1: worker compression of `nw` local streams, each split into n chunks.
struct K1Params {
  int n;             // chunks per stream (world size)
  int nw;            // local workers (sim: n, nccl: 1)
  int tpc;           // tiles per chunk
  int L;             // layers (stream modes 1/2)
  uint64_t c;        // chunk length
  uint64_t c_pad;    // chunk stride of werr (multiple of 4096)
  uint64_t d;        // fused length; elements >= d are zero padding
  uint64_t slot;     // words per packet slot (W + 32), W = c_pad / 32
  uint64_t W;
  const float* in;   // mode 0: streams; modes 1/2: gradients; [nw][in_stride]
  uint64_t in_stride;
  const float* m;             // mode 1: momentum buffer
  const uint32_t* res_prev;   // mode 2: previous result packets [n][slot]
  const uint64_t* off;        // layer offsets [L+1]
  const float* A;             // coeff*beta1 (fp32)
  const float* B;             // coeff*(1-beta1)
  const float* invc;          // 1/coeff
  const float* es_dev;        // error scale (device scalar) or nullptr
  float es_host;
  float* werr;                // [nw][n][c_pad] raw residual (v + delta)
  uint32_t* pk_cur;           // [nw][n][slot]
  const uint32_t* pk_prev;    // [nw][n][slot]
  double* partials;           // [nw][n][tpc]
  float* cmax;                // [nw][n][tpc] max|corrected| per tile (stats) or nullptr
  unsigned long long* err;
  int worker_base;            // global worker id of local worker 0
  // Fused NVLink exchange (NCCL-mode P2P transport): the words of chunk j are
  // also stored into rank j's receive slot peer_rx[j] + rx_off.
  uint32_t* const* peer_rx;   // [n] peer receive-buffer bases (nullptr: no fused exchange)
  uint64_t rx_off;            // word offset of this rank's slot in the current parity
  const int* tile_layer;      // mode 2: [n][tpc] layer of a single-layer full tile, else -1
  int skip_fast;              // general kernel: leave fast tiles to the bulk kernel
  const int* slow_list;       // general kernel after k1_bulk: the non-fast (j*tpc+t) tiles
  int n_slow;
  unsigned int* ctr;          // dynamic tile counter (self-resetting) or nullptr
  long long tile_lo, tile_cnt;  // register path: tiles [tile_lo, tile_lo + tile_cnt) (cnt 0: all)
  const int* order;           // register path, all tiles: processing order (boundary first)
};

// K3: server reduction of chunk(s) owned locally.
struct K3Params {
  int n;              // workers feeding each server
  int ns;             // local servers (sim: n, nccl: 1)
  int tpc;
  int server_base;    // chunk id of local server 0
  uint64_t c, c_pad, slot, W;
  const uint32_t* in;         // worker packets: server s, worker i at in + s*in_s + i*in_i
  uint64_t in_s, in_i;
  float* serr;                // [ns][c_pad]
  const uint32_t* res_prev;   // [n][slot]
  uint32_t* res_cur;          // [n][slot]
  const float* es_dev;
  float es_host;
  double* partials;           // [ns][tpc]
  float* cmax;                // [ns][tpc] or nullptr
  // Fused NVLink exchange: the server words also go into every peer's result
  // slot peer_res[q] + res_off (the stream waited for the packets before).
  uint32_t* const* peer_res;  // [n] peer result-buffer bases or nullptr
  uint64_t res_off;
  int rank;
  unsigned long long* err;
  unsigned int* ctr;
};

struct FinalizeParams {
  const double* partials;  // [count][tpc]
  int tpc;
  uint64_t c;
  uint32_t* slots;         // scale word of endpoint e at slots + e*slot_stride + W
  uint64_t slot_stride, W;
  unsigned long long* err;
  int err_base;            // key offset for kErrScale
  // Fused NVLink exchange: endpoint e's scale also goes to peer_slots[q] + peer_off
  // (q = e for worker packets, every q for the server packet), then the flag
  // peer_flags[q][flag_index] is raised to `epoch` (release, system scope).
  uint32_t* const* peer_slots;
  uint64_t peer_off;
  unsigned long long* const* peer_flags;
  int flag_index;
  int to_all;
  int n;
  unsigned long long epoch;
  unsigned long long* const* peer_err;  // [n] forward a local kErrGrad finding to every rank
};

// Layer-tiled kernels (K5, K6, W1, W2).
struct LayerTiles {
  int L;
  int tiles;                    // total tiles over all layers
  const uint64_t* off;          // [L+1]
  const int* tile_layer;        // [tiles]
  const int* layer_tile_start;  // [L+1]
  unsigned int* ctr;            // dynamic tile counter (self-resetting) or nullptr
  const int* order;             // [tiles] processing order (boundary tiles first) or nullptr
  int mis;                      // some full tile lies in a layer not 16-B aligned
  int count;                    // sub-launch: only order[0..count) (needs ctr and order); 0 = all
};

struct K5Params {
  LayerTiles lt;
  int n;
  uint64_t c, slot, W;
  const uint32_t* res_cur;   // [n][slot]
  const uint32_t* res_prev;  // [n][slot] (m_prev from packets) or nullptr
  const float* m;            // m_prev buffer (first step after the freeze)
  const float* invc;
  float* v;
  const float* vf;
  float inv, ninvb, b2, omb2, floor_;
  float* tile_max;           // [tiles]
  double* tile_v2;           // [tiles]
  unsigned long long* err;
  const float* dense;        // identity compressor: dense result (m_g = dense * invc)
  float* m_store;            // identity compressor: m <- m_g
  int norm_only;             // lamb_basic_1bit / onebit_adam: only ||v||^2 partials
  // Tiles off the fast path (across a chunk boundary; misaligned without the
  // MISK kernel), processed by k5_general on a side stream while the
  // streaming kernel skips them; nullptr: the streaming kernel takes them.
  const int* gen_list;
  int gen_count;
};

struct EpiParams {
  const unsigned long long* gate;  // cluster error words (kErrGate)
  int L;
  const int* layer_tile_start;
  const float* tile_max;
  const double* tile_v2;
  double* r_prev;
  const double* c_avg;
  float* coef_x;            // -lr*c per layer (fp32)
  double* trace;            // [4L]
  double* cmean;            // [2]: c_mean_prev, c_mean_prev2
  float* es_next;
  unsigned int* counter;
  double lr, r_thr, r_min, r_max, floor_;
  const double* lr_dev;  // graph replay: the step's lr is read here (nullptr: `lr`)
  int scaled_ef;
  int mode;  // 0 onebit_lamb (ratio rule), 1 lamb_basic_1bit (c = c_avg), 2 onebit_adam (c = 1)
};

struct K6Params {
  const unsigned long long* gate;
  LayerTiles lt;
  int n;
  uint64_t c, slot, W;
  const uint32_t* res_cur;
  const float* invc;
  const float* coef_x;
  const float* vf;
  float* x;
  float eta, wd;
  const float* dense;  // identity compressor: dense result
  const int* gen_list; // as K5Params (k6_general)
  int gen_count;
};

// Fused small compressed collective (P2P transport, one cooperative kernel).
struct SmallParams {
  K1Params k1;
  FinalizeParams f1;   // worker endpoints (this rank's n chunk packets)
  K3Params k3;
  FinalizeParams f2;   // server endpoint (chunk `rank`)
  const unsigned long long* flags;  // local [2n]: worker packets in, server packets in
  unsigned long long epoch;
  unsigned long long* err;
  unsigned int* bar;   // grid barrier [2] (count, generation)
  float* out;          // decompressed result [d] or nullptr
  const uint32_t* res; // result packets [n][slot] (this call's)
  uint64_t d;
  unsigned long long* ts;  // phase timestamps (block 0 / the finalizing block) or nullptr
  // LL ("low latency") transport: every 4-byte packet word travels with the
  // call's 32-bit epoch in one 8-byte store, so the receiver polls the data
  // itself -- no system fences, no flag round trips.
  uint2* const* ll_rx;      // [n] every rank's LL receive buffer [2][n][slot] (worker packets)
  uint2* const* ll_res;     // [n] every rank's LL result buffer [2][n][slot] (server packets)
  uint64_t ll_off;          // (parity * n + rank) * slot: this rank's slot at every peer
  const uint2* ll_rx_mine;  // this rank's LL rx, current parity, [n][slot]
  const uint2* ll_res_mine; // this rank's LL res, current parity, [n][slot]
  uint32_t* res_plain;      // this call's plain result packets [n][slot] (K5/K6, getters)
  unsigned int* cnt;        // [2 + n] CTA counters of the last-CTA finalizes: [1] server scale,
                            // [2 + j] chunk j's worker scale (self-resetting)
  unsigned int ep32;
};

// Deterministic lossless all-reduce over NVLink peer memory (P2P transport).
struct LosslessP2PParams {
  const float* const* peer_in;            // [n] every rank's gradient buffer
  float* const* peer_out;                 // [n] every rank's output buffer
  unsigned long long* const* peer_err;    // [n] every rank's error words
  unsigned long long* const* peer_flags;  // [n] every rank's flag words
  const unsigned long long* in_flags;     // local [n]: rank q's gradient is in place
  int out_flag;                           // flag index of "rank's chunk delivered" (+ rank)
  int n, rank, check_finite;
  uint64_t c, d;
  unsigned long long epoch;
  unsigned int* done;                     // local CTA counter (self-resetting)
  unsigned long long* err;
  // Piecewise delivery (warmup overlap): the chunk is reduced in `pieces`
  // consecutive pieces; when every CTA finished piece p, the flag
  // piece_flag_base + rank * pieces + p is raised at every rank, so the
  // consumer (W1/W2 sub-launches) starts on the delivered part.  0 = off.
  int pieces;
  int piece_flag_base;
  unsigned int* piece_done;               // [pieces] local CTA counters (self-resetting)
  int ctas;                               // grid cap (leave SM room for the consumer), 0 = full
  int block;                              // threads per CTA (0 = 256)
  // Owner-sharded warmup: reduce [lo, hi) instead of chunk `rank` and store
  // the average into the local output only (no allgather; hi == 0: chunk).
  uint64_t lo, hi;
  int local_only;
  int shape;  // piece sizes: 0 equal, 1 linearly shrinking (piece_body_start)
};

// Push-based owner-sharded warmup exchange (BL_SHARD_PUSH=1): every rank
// stores each owner's range of its gradient into that owner's staging slot
// [rank] (NVLink stores), per piece, and raises "piece p from rank q" at the
// owner; the owner reduces its range from its own gradient and the staged
// slots (k_shard_reduce).  Piece boundaries are the lossless kernel's.
struct ShardPushParams {
  const float* in;                         // local gradient
  float* const* peer_stg;                  // [n] every rank's staging buffer [n][S]
  const uint64_t* e_all;                   // [n + 1] owned element ranges
  uint64_t S;                              // staging floats per sender slot
  int n, rank, pieces, shape;
  unsigned long long* const* peer_flags;   // [n]
  int piece_flag_base;
  unsigned long long epoch;
  unsigned int* piece_done;                // [pieces] local CTA counters (self-resetting)
  const unsigned long long* gate;
};
struct ShardReduceParams {
  const float* in;                         // local gradient
  const float* stg;                        // local staging buffer [n][S]
  uint64_t S, E0, E1, d;
  int n, rank, pieces, shape, piece;
  float* out;
  unsigned long long* err;
  unsigned long long* const* peer_err;     // [n]: the last piece forwards a non-finite finding
  unsigned int* done;                      // local CTA counter (self-resetting)
};
int launch_shard_push(const ShardPushParams& p, int ctas, cudaStream_t s);
int launch_shard_reduce(const ShardReduceParams& p, int sms, cudaStream_t s);

struct W1Params {
  const unsigned long long* gate;
  LayerTiles lt;
  const float* gbar;
  float *m, *v;
  const float* x;
  float b1, omb1, b2, omb2, eta, wd;
  double* tile_sums;  // [tiles][4]: x^2, u^2, v^2, |m|
  int adam;           // adam_step: no norms needed (kept for the trace)
  unsigned long long* err;  // non-null: gbar IS the single worker's gradient -> finite check
  int worker_base;
};

struct WEpiParams {
  const unsigned long long* gate;
  const int* layer_list;  // sub-launch: block b handles layer layer_list[b] (nullptr: block = layer)
  int count;              // sub-launch: number of layers (0 = L)
  int L;
  const int* layer_tile_start;
  const uint64_t* off;
  const double* tile_sums;
  double* c_avg;
  float* coef_x;
  double* trace;
  double* mag;         // [L] floored mean |m| (finalize)
  double* coeff;       // [L]
  float *A, *B, *invc;
  double* cmean;
  float* es_next;
  unsigned int* counter;
  double lr, b1, b3, c_min, c_max, floor_;
  int track, finalize, adam, onebit_adam;
};

struct W2Params {
  const unsigned long long* gate;
  LayerTiles lt;
  const float *m, *v;
  float* x;
  float* vf;  // written when finalize
  const float* coef_x;
  float eta, wd;
  int finalize;
  // Owner-sharded warmup: x (and at the freeze m, v, vf) of the owned tiles
  // is also stored into the npush other ranks' buffers (the allgather).
  float* const* push_x;
  float* const* push_m;
  float* const* push_v;
  float* const* push_vf;
  int npush;
};

// Step gate (start of every step / collective).  Strict mode: a non-finite
// local gradient found by the pre-pass closes the gate.  Multi-process (P2P):
// every rank posts its arrival (epoch, status) into every peer's flag words
// and waits for all arrivals within the timeout; a go/abort decision is
// CAS-ed once into rank 0's decision word, so every rank takes the same one.
struct GateParams {
  unsigned long long* err;                 // local error words
  unsigned long long seq;                  // host sequence number (rollback key)
  unsigned long long epoch;                // barrier epoch (same on every rank)
  int n, rank, strict;
  unsigned long long* const* peer_flags;   // [n] every rank's flag words (nullptr: local only)
  const unsigned long long* arrive;        // local arrival words [n]
  int arrive_index;                        // flag index of arrival word 0
  int decision_index;                      // flag index of the decision word (rank 0's is used)
  const uint64_t* off;                     // layer table [L+1] (layer of a non-finite element)
  int L;
};

// Host launchers (bl_kernels.cu).  Each returns the number of kernels launched.
int launch_k1(const K1Params& p, int mode, int grid, cudaStream_t s);
// The two launches of the bulk-copy K1: phase 0 = fast tiles (k1_bulk),
// phase 1 = boundary tiles (general kernel over the slow list).
bool k1_uses_bulk(const K1Params& p, int mode);
int launch_k1_phase(const K1Params& p, int mode, int phase, cudaStream_t s);
int launch_finalize(const FinalizeParams& p, int count, cudaStream_t s);
int launch_k3(const K3Params& p, int grid, cudaStream_t s);
int launch_k5(const K5Params& p, int grid, cudaStream_t s);
// The listed general-path tiles (K5Params::gen_list), concurrent with launch_k5 on another stream.
int launch_k5_general(const K5Params& p, cudaStream_t s);
int launch_epilogue(const EpiParams& p, cudaStream_t s);
int launch_k6(const K6Params& p, int grid, cudaStream_t s);
int launch_k6_general(const K6Params& p, cudaStream_t s);
int launch_w1(const W1Params& p, int grid, cudaStream_t s);
int launch_wepilogue(const WEpiParams& p, cudaStream_t s);
int launch_w2(const W2Params& p, int grid, cudaStream_t s);
// out[k] = (float)(sum_i in[i*stride + k] (double, ascending i) * inv_n), k < len.
int launch_average(const float* in, uint64_t stride, int n, uint64_t len, float* out,
                   unsigned long long* err, int check_finite, int worker_base, cudaStream_t s);
// out[k] (k < d) = decompressed result of packets res[n][slot].
int launch_decompress(const uint32_t* res, int n, uint64_t c, uint64_t slot, uint64_t W,
                      uint64_t d, float* out, const unsigned long long* gate, cudaStream_t s);
// out[k] (k < len) = raw[j][i] - (bit ? S : -S) for flat k = j*c + i; pk [nch][slot].
int launch_materialize_error(const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot,
                             uint64_t W, uint64_t c, uint64_t len, float* out, cudaStream_t s);
// out[k] (k < d) = decompressed result * invc[layer(k)].
int launch_materialize_m(const uint32_t* res, int n, uint64_t c, uint64_t slot, uint64_t W,
                         const uint64_t* off, int L, const float* invc, uint64_t d, float* out,
                         cudaStream_t s);
// Endpoint statistics (comm_sim.cpp:108-118) of one endpoint, updated in the
// device record st[5] = {||delta||_2 (tile-tree over the flat residual),
// max|delta|, max|corrected| (from cmax[cmax_n]), running max|delta|,
// running max|corrected|} -- no host round trip.
int launch_error_stats(const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot,
                       uint64_t W, uint64_t c, uint64_t len, double* scratch, int scratch_tiles,
                       float* scratch_max, const float* cmax, int cmax_n, double* st, cudaStream_t s);
int launch_set_float(float* p, float v, cudaStream_t s);
// verify_compensation (comm_sim.cpp:83-106) for es == 1: for every element of
// `len` flat (chunked) positions, corrected (= raw) against decompressed +
// delta_new in fp64 with relative tolerance tol.
int launch_verify(const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot, uint64_t W,
                  uint64_t c, uint64_t len, double tol, unsigned long long* err, cudaStream_t s);
// Block the stream until flags[0..n) >= epoch (peer signals, bounded wait).
int launch_lossless_p2p(const LosslessP2PParams& p, int sms, cudaStream_t s);
// Piece boundaries of the piecewise lossless exchange: element k of chunk
// [lo, hi) (global indices) belongs to piece lossless_piece(lo, hi, pieces, k).
int lossless_piece(uint64_t lo, uint64_t hi, int pieces, uint64_t k, int shape = 0);
// Block the stream until every rank's piece p is delivered (flags[base + q*pieces + p] >= epoch).
int launch_wait_piece(const unsigned long long* flags, int base, int n, int pieces, int p,
                      unsigned long long epoch, unsigned long long* err, cudaStream_t s);
// Returns 1, or -cudaError when the cooperative launch is refused.
int launch_small_collective(const SmallParams& p, int k1_mode, cudaStream_t s);
// Raise flag `index` (+ own rank) at every peer to `epoch` after this stream's
// prior work (system-scope release).
int launch_signal_peers(unsigned long long* const* peer_flags, int index, int n,
                        unsigned long long epoch, const unsigned long long* gate, cudaStream_t s);
int launch_wait_peers(const unsigned long long* flags, int n, unsigned long long epoch,
                      unsigned long long* err, cudaStream_t s);
// Store words [off, off + count) of src into the same range of every buffer
// of dst[0..ndst) (peer memory), each thread fencing its remote stores; a
// following launch_signal_peers publishes them.  4- or 8-byte words.
int launch_push_range(const float* src, float* const* dst, int ndst, uint64_t off, uint64_t count,
                      const unsigned long long* gate, int sms, cudaStream_t s);
int launch_push_range(const double* src, double* const* dst, int ndst, uint64_t off, uint64_t count,
                      const unsigned long long* gate, int sms, cudaStream_t s);
// Strict pre-pass (optimizers.cpp:99-117, before any mutation): flags the
// first non-finite element of the nw local gradients in kErrGrad.
int launch_check_finite(const float* in, uint64_t stride, int nw, uint64_t d, unsigned long long* err,
                        int worker_base, cudaStream_t s);
int launch_step_gate(const GateParams& p, cudaStream_t s);
// fusion.hpp:92-102 free functions on the device.
int launch_layer_abs_tiles(const float* x, const uint64_t* off, const int* tile_layer,
                           const int* layer_tile_start, int tiles, double* part, cudaStream_t s);
int launch_scales_final(int L, const int* layer_tile_start, const uint64_t* off, const double* part,
                        double floor_, double* mag, double* coeff, double* ref_out, unsigned int* counter,
                        cudaStream_t s);
int launch_scale_layers(float* x, const uint64_t* off, int L, const float* mul, uint64_t d, cudaStream_t s);
// NCCL transport: this rank's gate status as one word (min-reduced over the
// ranks by ncclAllReduce between the two launches), then applied.
int launch_gate_status(unsigned long long* err, const uint64_t* off, int L, int rank,
                       unsigned long long* status, cudaStream_t s);
int launch_gate_apply(unsigned long long* err, const unsigned long long* status, int rank,
                      unsigned long long seq, cudaStream_t s);
// Identity-compressor stream build in place (optimizers.cpp:248-255):
// in[w][k] = A_l*m[k] + B_l*in[w][k] for k < d, with the gradient finite check.
int launch_build_stream(float* in, uint64_t stride, int nw, uint64_t d, const float* m,
                        const uint64_t* off, int L, const float* A, const float* B,
                        unsigned long long* err, int worker_base, cudaStream_t s);

}  // namespace bl

// bl_runtime.cu — host runtime of the B200 1-bit LAMB path: the cluster
// (communicator + residuals + packets) and the optimizer (layer state), and
// the extern "C" ABI declared in include/bitlamb_b200.h.
//
// Step schedule of one compression-stage step (optimizers.cpp:231-332) on one
// stream:  K1 worker compress -> scale finalize -> [NCCL alltoall of packets]
// -> K3 server reduce -> scale finalize -> [NCCL allgather of server packets]
// -> K5 (v, ratio max) -> per-layer epilogue -> K6 (x).  SIM mode runs the n
// ranks' K1/K3 work in the same launches and skips the two exchanges.

#include "bl_runtime.h"

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>

namespace bl {

const char* const kClassNames[KC_COUNT] = {
    "k1_worker_compress", "finalize_scales", "k3_server_reduce", "k5_update_a",
    "layer_epilogue",     "k6_update_b",     "w1_warmup_a",      "warmup_epilogue",
    "w2_warmup_b",        "average",         "decompress",       "materialize",
    "endpoint_stats",     "nccl_alltoall",   "nccl_allgather",   "h2d_copy",
    "d2h_copy",           "k1_boundary_tiles", "small_collective", "step_gate"};

void fail(bl_status st, const std::string& msg) { throw Error{st, msg}; }

int* boundary_first_order(const std::vector<int>& slow, int reps, int per) {
  // Index space [reps][per]; the listed (per-rep) boundary tiles of every
  // rep first, then the rest in order.  Scheduling only: results do not
  // depend on it.
  std::vector<char> is_slow(static_cast<size_t>(per), 0);
  for (int t : slow) is_slow[static_cast<size_t>(t)] = 1;
  std::vector<int> order;
  order.reserve(static_cast<size_t>(reps) * per);
  for (int r = 0; r < reps; ++r)
    for (int t : slow) order.push_back(r * per + t);
  for (int r = 0; r < reps; ++r)
    for (int t = 0; t < per; ++t)
      if (!is_slow[static_cast<size_t>(t)]) order.push_back(r * per + t);
  int* d = reinterpret_cast<int*>(dalloc<float>(order.size()));
  cuda_check(cudaMemcpy(d, order.data(), order.size() * 4, cudaMemcpyHostToDevice), "tile order");
  return d;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(BL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(BL_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

DeviceGuard::DeviceGuard(int dev) : dev_(dev) {
  cudaGetDevice(&prev_);
  if (prev_ != dev_) cuda_check(cudaSetDevice(dev_), "cudaSetDevice");
}
DeviceGuard::~DeviceGuard() {
  if (prev_ >= 0 && prev_ != dev_) cudaSetDevice(prev_);
}

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  cuda_check(cudaMemset(p, 0, bytes), "cudaMemset");
  return static_cast<T*>(p);
}
template float* dalloc<float>(size_t);
template double* dalloc<double>(size_t);
template uint32_t* dalloc<uint32_t>(size_t);

static uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

// Slack after every streamed buffer: the row loader reads up to 132 floats
// past a row start and rows may start up to 4095 floats before the end.
constexpr uint64_t kSlack = 4096 + 256;

}  // namespace bl

using namespace bl;

// ---------------------------------------------------------------------------
// bl_cluster
// ---------------------------------------------------------------------------
cudaEvent_t bl_cluster::get_event() {
  if (!ev_pool.empty()) {
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

void bl_cluster::begin(int, cudaEvent_t* a) {
  *a = nullptr;
  if (profiling) {
    *a = get_event();
    cuda_check(cudaEventRecord(*a, stream), "cudaEventRecord");
  }
}

void bl_cluster::end(int cls, cudaEvent_t a, int kernels) {
  launches += static_cast<uint64_t>(kernels);
  if (kernels > 0) cuda_check(cudaGetLastError(), kClassNames[cls]);
  if (profiling && a) {
    cudaEvent_t b = get_event();
    cuda_check(cudaEventRecord(b, stream), "cudaEventRecord");
    pending.push_back({cls, a, b});
  }
}

int bl_cluster::grid(long long tiles) const {
  const long long want = (tiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const long long cap = static_cast<long long>(sms) * 16;  // launchers cap at residency
  return static_cast<int>(std::max<long long>(1, std::min(want, cap)));
}

uint64_t bl_cluster::chunk_payload_bits(uint64_t j) const {  // comm_sim.cpp:68-79
  const uint64_t begin = j * c;
  if (begin >= dim) return 0;
  const uint64_t real = std::min(c, dim - begin);
  if (cfg.compressor == BL_COMPRESSOR_ONEBIT) return real + 32;
  return real * static_cast<uint64_t>(cfg.baseline_bits_per_element);
}

void bl_cluster::ledger_compressed() {  // comm_sim.cpp:187-197
  uint64_t bits = 0;
  for (int j = 0; j < n; ++j) bits += chunk_payload_bits(static_cast<uint64_t>(j));
  ledger.gather_bits += static_cast<uint64_t>(n - 1) * bits;
  ledger.scatter_bits += static_cast<uint64_t>(n - 1) * bits;
  ledger.baseline_equivalent_bits += 2ull * static_cast<uint64_t>(n - 1) * dim *
                                     static_cast<uint64_t>(cfg.baseline_bits_per_element);
  ledger.compressed_collectives += 1;
}

void bl_cluster::ledger_lossless() {  // comm_sim.cpp:224-231
  const uint64_t bits = 2ull * static_cast<uint64_t>(n - 1) * dim *
                        static_cast<uint64_t>(cfg.baseline_bits_per_element);
  ledger.lossless_bits += bits;
  ledger.baseline_equivalent_bits += bits;
  ledger.lossless_collectives += 1;
}

void bl_cluster::copy_inputs(const float* const* inputs, int n_inputs, uint64_t len, int memory) {
  cudaEvent_t a;
  begin(KC_H2D, &a);
  for (int w = 0; w < n_inputs; ++w) {
    float* dst = in + static_cast<size_t>(w) * in_stride;
    if (memory == BL_MEM_DEVICE && inputs[w] == dst) continue;
    cuda_check(cudaMemcpyAsync(dst, inputs[w], len * sizeof(float), cudaMemcpyDefault, stream),
               "cudaMemcpyAsync(inputs)");
  }
  end(KC_H2D, a, 0);
}

bool bl_cluster::compressed(const K1Params* ovr, int k1_mode, float es_host, const float* es_dev,
                            float* dec_out) {
  K1Params p = ovr ? *ovr : K1Params{};
  if (!ovr) {
    p.slow_list = k1_slow;
    p.n_slow = k1_n_slow;
    p.order = k1_order;
  }
  p.n = n;
  p.nw = nw;
  p.tpc = tpc;
  p.c = c;
  p.c_pad = c_pad;
  p.d = dim;
  p.slot = slot;
  p.W = W;
  p.in = in;
  p.in_stride = in_stride;
  p.es_dev = es_dev;
  p.es_host = es_host;
  p.werr = werr;
  p.pk_cur = wpk[cur()];
  p.pk_prev = wpk[prev()];
  p.partials = wpart;
  p.cmax = cfg.endpoint_stats ? wcmax : nullptr;
  p.err = err;
  p.worker_base = mode == BL_MODE_SIM ? 0 : rank;
  p.ctr = std::getenv("BL_STATIC_TILES") ? nullptr : tile_ctr;
  const bool p2p = transport == BL_TRANSPORT_P2P;
  const unsigned long long epoch = calls + 1;
  const uint64_t my_slot = (static_cast<uint64_t>(cur()) * n + rank) * slot;
  if (p2p) {
    p.peer_rx = d_peer_rx;  // fused alltoall: K1 stores chunk j's words into rank j's rx
    p.rx_off = my_slot;
  }
  cudaEvent_t a;
  const float* host = stage_host;
  stage_host = nullptr;
  // Small collectives over NVLink: one cooperative kernel for the whole
  // exchange (and the decompress, when asked).  BL_SMALL_MAX_TILES sets the
  // size limit (K1 tiles per rank; 0 disables).
  if (p2p && nw == 1 && static_cast<long long>(n) * tpc <= small_max_tiles()) {
    if (host) {  // small: copy the staged host gradient first
      const float* srcs[1] = {host};
      copy_inputs(srcs, 1, dim, BL_MEM_HOST);
    }
    SmallParams sp{};
    sp.k1 = p;
    sp.k1.slow_list = nullptr;  // every tile through k1_tile
    sp.k1.n_slow = 0;
    sp.k1.skip_fast = 0;
    sp.k1.peer_rx = nullptr;    // the kernel sends the words as LL words itself
    sp.f1 = FinalizeParams{wpart, tpc, c, wpk[cur()], slot, W, err, p.worker_base * n};
    sp.f1.n = n;
    sp.f1.peer_err = d_peer_err;  // (scales travel as LL words: no peer slots/flags here)
    K3Params& k3 = sp.k3;
    k3.n = n;
    k3.ns = 1;
    k3.tpc = tpc;
    k3.server_base = rank;
    k3.c = c;
    k3.c_pad = c_pad;
    k3.slot = slot;
    k3.W = W;
    k3.in = rx + static_cast<size_t>(cur()) * n * slot;
    k3.in_s = 0;
    k3.in_i = slot;
    k3.serr = serr;
    k3.res_prev = res[prev()];
    k3.res_cur = res[cur()];
    k3.es_dev = es_dev;
    k3.es_host = es_host;
    k3.partials = spart;
    k3.cmax = cfg.endpoint_stats ? scmax : nullptr;
    k3.err = err;
    k3.rank = rank;
    sp.f2 = FinalizeParams{spart, tpc, c, res[cur()] + static_cast<size_t>(rank) * slot, slot, W, err,
                           1 << 20};
    sp.f2.n = n;
    sp.flags = flags;
    sp.epoch = epoch;
    sp.err = err;
    sp.bar = small_bar;
    sp.out = dec_out;
    sp.res = res[cur()];
    sp.d = dim;
    sp.ll_rx = d_peer_llrx;
    sp.ll_res = d_peer_llres;
    sp.ll_off = my_slot;
    sp.ll_rx_mine = ll_rx + static_cast<size_t>(cur()) * n * slot;
    sp.ll_res_mine = ll_res + static_cast<size_t>(cur()) * n * slot;
    sp.res_plain = res[cur()];
    sp.cnt = small_bar;
    sp.ep32 = static_cast<unsigned int>(epoch);
    // BL_SMALL_TS=1: phase timestamps of block 0 (ns, relative), printed to
    // stderr after the call -- a latency-analysis aid, synchronizes the stream.
    static const bool ts_on = std::getenv("BL_SMALL_TS") != nullptr;
    if (ts_on && !small_ts) small_ts = reinterpret_cast<unsigned long long*>(dalloc<double>(16));
    if (ts_on) cuda_check(cudaMemsetAsync(small_ts, 0, 16 * 8, stream), "ts reset");
    sp.ts = ts_on ? small_ts : nullptr;
    begin(KC_SMALL, &a);
    const int r = launch_small_collective(sp, k1_mode, stream);
    if (r < 0) fail(BL_ERR_CUDA, std::string("fused small collective launch: ") +
                                    cudaGetErrorString(static_cast<cudaError_t>(-r)));
    end(KC_SMALL, a, r);
    if (ts_on) {
      unsigned long long h[15];
      cuda_check(cudaMemcpyAsync(h, small_ts, sizeof h, cudaMemcpyDeviceToHost, stream), "ts");
      cuda_check(cudaStreamSynchronize(stream), "ts");
      char line[256];
      int len = std::snprintf(line, sizeof line, "small_ts rank %d tiles %lld:", rank, static_cast<long long>(n) * tpc);
      for (int k = 1; k < 15; ++k)
        len += std::snprintf(line + len, sizeof line - len, " %.2f", h[k] ? (h[k] - h[0]) * 1e-3 : -1.0);
      std::fprintf(stderr, "%s\n", line);  // one write per line (ranks share stderr)
    }
    finish_compressed(es_host, es_dev);
    return dec_out != nullptr;
  }
  if (host && k1_uses_bulk(p, k1_mode)) {  // no piecewise K1 on the bulk path: copy first
    const float* srcs[1] = {host};
    copy_inputs(srcs, 1, dim, BL_MEM_HOST);
    host = nullptr;
  }
  if (host) {
    // Tile-aligned pieces of the H2D copy on a copy stream; the K1 launch of
    // each piece waits only for its own bytes.  Tiles are in element order
    // (chunk j's tiles cover [j*c, (j+1)*c)), so piece k is a contiguous range.
    if (!copy_stream) {
      cuda_check(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "copy stream");
      for (auto& e : piece_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    const long long T = static_cast<long long>(n) * tpc;
    const int M = static_cast<int>(std::min<long long>(kPieces, T));
    auto elem = [&](long long tile) -> uint64_t {
      if (tile >= T) return dim;
      const uint64_t e = static_cast<uint64_t>(tile / tpc) * c + static_cast<uint64_t>(tile % tpc) * kTile;
      return std::min<uint64_t>(e, dim);
    };
    cuda_check(cudaEventRecord(piece_ev[kPieces], stream), "event");  // `in` free to overwrite
    cuda_check(cudaStreamWaitEvent(copy_stream, piece_ev[kPieces], 0), "wait");
    begin(KC_K1, &a);
    int launched = 0;
    for (int k = 0; k < M; ++k) {
      const long long t0 = T * k / M, t1 = T * (k + 1) / M;
      const uint64_t e0 = elem(t0), e1 = elem(t1);
      if (e1 > e0)
        cuda_check(cudaMemcpyAsync(in + e0, host + e0, (e1 - e0) * sizeof(float), cudaMemcpyHostToDevice,
                                   copy_stream),
                   "cudaMemcpyAsync(piece)");
      cuda_check(cudaEventRecord(piece_ev[k], copy_stream), "event");
      cuda_check(cudaStreamWaitEvent(stream, piece_ev[k], 0), "wait");
      K1Params q = p;
      q.tile_lo = t0;
      q.tile_cnt = t1 - t0;
      launched += launch_k1(q, k1_mode, grid(t1 - t0), stream);
    }
    end(KC_K1, a, launched);
  } else if (k1_uses_bulk(p, k1_mode)) {  // bulk fast tiles, then the boundary tiles
    begin(KC_K1, &a);
    end(KC_K1, a, launch_k1_phase(p, k1_mode, 0, stream));
    begin(KC_K1B, &a);
    end(KC_K1B, a, launch_k1_phase(p, k1_mode, 1, stream));
  } else {
    begin(KC_K1, &a);
    end(KC_K1, a, launch_k1(p, k1_mode, grid(static_cast<long long>(nw) * n * tpc), stream));
  }

  FinalizeParams f{wpart, tpc, c, wpk[cur()], slot, W, err, p.worker_base * n};
  if (p2p) {
    f.peer_slots = d_peer_rx;
    f.peer_off = my_slot;
    f.peer_flags = d_peer_flags;
    f.flag_index = rank;
    f.to_all = 0;
    f.n = n;
    f.epoch = epoch;
    f.peer_err = d_peer_err;  // a non-finite gradient is reported to every rank
  }
  begin(KC_FIN, &a);
  end(KC_FIN, a, launch_finalize(f, nw * n, stream));

  const uint32_t* kin = wpk[cur()];
  uint64_t in_s = slot, in_i = static_cast<uint64_t>(n) * slot;
  if (p2p) {
    begin(KC_A2A, &a);
    end(KC_A2A, a, launch_wait_peers(flags, n, epoch, err, stream));
    kin = rx + static_cast<size_t>(cur()) * n * slot;
    in_s = 0;
    in_i = slot;
  } else if (mode == BL_MODE_NCCL) {
    begin(KC_A2A, &a);
    const size_t words = W + 1;  // sign words + scale word
    cuda_check(cudaMemcpyAsync(rpk + static_cast<size_t>(rank) * slot,
                               wpk[cur()] + static_cast<size_t>(rank) * slot, words * 4,
                               cudaMemcpyDeviceToDevice, stream),
               "self packet copy");
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int j = 0; j < n; ++j) {
      if (j == rank) continue;
      nccl_check(ncclSend(wpk[cur()] + static_cast<size_t>(j) * slot, words, ncclUint32, j, comm,
                          stream),
                 "ncclSend");
      nccl_check(ncclRecv(rpk + static_cast<size_t>(j) * slot, words, ncclUint32, j, comm, stream),
                 "ncclRecv");
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
    share_grad_error();  // K1's fused finite check, raised on every rank
    end(KC_A2A, a, 0);
    kin = rpk;
    in_s = 0;
    in_i = slot;
  }

  K3Params k3{};
  k3.n = n;
  k3.ns = ns;
  k3.tpc = tpc;
  k3.server_base = mode == BL_MODE_SIM ? 0 : rank;
  k3.c = c;
  k3.c_pad = c_pad;
  k3.slot = slot;
  k3.W = W;
  k3.in = kin;
  k3.in_s = in_s;
  k3.in_i = in_i;
  k3.serr = serr;
  k3.res_prev = res[prev()];
  k3.res_cur = res[cur()];
  k3.es_dev = es_dev;
  k3.es_host = es_host;
  k3.partials = spart;
  k3.cmax = cfg.endpoint_stats ? scmax : nullptr;
  k3.err = err;
  k3.ctr = p.ctr;
  if (p2p) {
    k3.peer_res = d_peer_res;  // fused allgather: server words into every peer's result slot
    k3.res_off = my_slot;
    k3.rank = rank;
  }
  begin(KC_K3, &a);
  end(KC_K3, a, launch_k3(k3, grid(static_cast<long long>(ns) * tpc), stream));

  FinalizeParams f2{spart, tpc, c, res[cur()] + static_cast<size_t>(k3.server_base) * slot, slot,
                    W, err, 1 << 20};
  if (p2p) {
    f2.peer_slots = d_peer_res;
    f2.peer_off = my_slot;
    f2.peer_flags = d_peer_flags;
    f2.flag_index = n + rank;
    f2.to_all = 1;
    f2.n = n;
    f2.epoch = epoch;
  }
  begin(KC_FIN, &a);
  end(KC_FIN, a, launch_finalize(f2, ns, stream));

  if (p2p) {
    begin(KC_AG, &a);
    end(KC_AG, a, launch_wait_peers(flags + n, n, epoch, err, stream));
  } else if (mode == BL_MODE_NCCL && n > 1) {
    begin(KC_AG, &a);
    nccl_check(ncclAllGather(res[cur()] + static_cast<size_t>(rank) * slot, res[cur()], slot,
                             ncclUint32, comm, stream),
               "ncclAllGather");
    end(KC_AG, a, 0);
  }
  finish_compressed(es_host, es_dev);
  return false;
}

void bl_cluster::finish_compressed(float es_host, const float* es_dev) {
  calls += 1;
  last_identity = false;
  ledger_compressed();
  if (cfg.verify_compensation && (es_dev == nullptr ? es_host == 1.0f : verify_es_one)) verify_last();
  if (cfg.endpoint_stats) refresh_stats();
}

// Map every peer's receive buffer, result buffer and flag words into this
// process (CUDA IPC over NVLink).  Collective: every rank takes the same
// decision (NCCL min-reduce of the per-rank success bit).
bool bl_cluster::map_peer_buffers(const std::vector<void*>& local, std::vector<std::vector<void*>>* peer,
                                  std::vector<void*>* opened) {
  const size_t nn = static_cast<size_t>(n), kB = local.size();
  constexpr size_t kH = sizeof(cudaIpcMemHandle_t);
  std::vector<uint8_t> mine(kB * kH);
  for (size_t k = 0; k < kB; ++k) {
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, local[k]), "cudaIpcGetMemHandle");
    std::memcpy(mine.data() + k * kH, &h, kH);
  }
  uint8_t* dbuf = reinterpret_cast<uint8_t*>(dalloc<double>((nn * kB * kH + 7) / 8 + 1));
  cuda_check(cudaMemcpy(dbuf + static_cast<size_t>(rank) * kB * kH, mine.data(), kB * kH,
                        cudaMemcpyHostToDevice),
             "handle upload");
  nccl_check(ncclAllGather(dbuf + static_cast<size_t>(rank) * kB * kH, dbuf, kB * kH, ncclUint8, comm,
                           stream),
             "ncclAllGather(handles)");
  std::vector<uint8_t> all(nn * kB * kH);
  cuda_check(cudaMemcpyAsync(all.data(), dbuf, all.size(), cudaMemcpyDeviceToHost, stream), "handles");
  cuda_check(cudaStreamSynchronize(stream), "handles sync");
  peer->assign(kB, std::vector<void*>(nn, nullptr));
  std::vector<void*> mapped;
  int ok = 1;
  for (int q = 0; q < n; ++q) {
    for (size_t k = 0; k < kB && ok; ++k) {
      if (q == rank) {
        (*peer)[k][q] = local[k];
        continue;
      }
      cudaIpcMemHandle_t hq;
      std::memcpy(&hq, all.data() + (static_cast<size_t>(q) * kB + k) * kH, kH);
      if (cudaIpcOpenMemHandle(&(*peer)[k][q], hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
      } else {
        mapped.push_back((*peer)[k][q]);
      }
    }
  }
  int* dok = reinterpret_cast<int*>(dbuf);
  cuda_check(cudaMemcpy(dok, &ok, sizeof ok, cudaMemcpyHostToDevice), "ok upload");
  nccl_check(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, comm, stream), "ncclAllReduce(ok)");
  cuda_check(cudaMemcpyAsync(&ok, dok, sizeof ok, cudaMemcpyDeviceToHost, stream), "ok");
  cuda_check(cudaStreamSynchronize(stream), "ok sync");
  cudaFree(dbuf);
  if (!ok) {
    for (void* p : mapped) cudaIpcCloseMemHandle(p);
    return false;
  }
  opened->insert(opened->end(), mapped.begin(), mapped.end());
  return true;
}

// Map every peer's receive buffer, result buffer and flag words into this
// process (CUDA IPC over NVLink).  Collective: every rank takes the same
// decision (NCCL min-reduce of the per-rank success bit).
void bl_cluster::setup_p2p(bool required) {
  const size_t nn = static_cast<size_t>(n);
  rx = dalloc<uint32_t>(2 * nn * slot);
  flags = reinterpret_cast<unsigned long long*>(dalloc<double>(static_cast<size_t>(shard_flag_base()) + 2 * nn));
  piece_done = reinterpret_cast<unsigned int*>(dalloc<float>(kMaxPieces));
  lossless_done = reinterpret_cast<unsigned int*>(dalloc<float>(1));
  small_bar = reinterpret_cast<unsigned int*>(dalloc<float>(2 + nn));
  // LL buffers of the fused small collective, [2][n][slot] (word, epoch)
  // pairs; only sized when the small path can be taken.
  const size_t ll_words = static_cast<long long>(n) * tpc <= small_max_tiles() ? 2 * nn * slot : 1;
  ll_rx = reinterpret_cast<uint2*>(dalloc<double>(ll_words));
  ll_res = reinterpret_cast<uint2*>(dalloc<double>(ll_words));
  // Buffers every peer maps: packet receive slots, result packets, flags,
  // gradient (lossless reads), output (lossless allgather), error words,
  // LL receive slots, LL result slots.
  std::vector<std::vector<void*>> peer;
  if (!map_peer_buffers({rx, res_base, flags, in, out, err, ll_rx, ll_res}, &peer, &ipc_opened)) {
    if (required) fail(BL_ERR_UNSUPPORTED, "P2P transport: a peer's memory could not be mapped");
    transport = BL_TRANSPORT_NCCL;
    return;
  }
  auto table = [&](int k) {
    void** t = reinterpret_cast<void**>(dalloc<double>(nn));
    cuda_check(cudaMemcpy(t, peer[k].data(), nn * sizeof(void*), cudaMemcpyHostToDevice), "tables");
    return t;
  };
  d_peer_rx = reinterpret_cast<uint32_t**>(table(0));
  d_peer_res = reinterpret_cast<uint32_t**>(table(1));
  d_peer_flags = reinterpret_cast<unsigned long long**>(table(2));
  d_peer_in = reinterpret_cast<float**>(table(3));
  d_peer_out = reinterpret_cast<float**>(table(4));
  d_peer_err = reinterpret_cast<unsigned long long**>(table(5));
  d_peer_llrx = reinterpret_cast<uint2**>(table(6));
  d_peer_llres = reinterpret_cast<uint2**>(table(7));
  transport = BL_TRANSPORT_P2P;
}

// NCCL transport: the lowest (worker << 40 | element) non-finite key over
// ranks, so every rank reports the same gradient error (the P2P transport
// forwards it with its flags).
void bl_cluster::share_grad_error() {
  if (mode != BL_MODE_NCCL || n == 1 || transport == BL_TRANSPORT_P2P) return;
  nccl_check(ncclAllReduce(err + kErrGrad, err + kErrGrad, 1, ncclUint64, ncclMin, comm, stream),
             "ncclAllReduce(gradient error)");
}

void bl_cluster::lossless(bool check_finite) {
  cudaEvent_t a;
  if (mode == BL_MODE_SIM || n == 1) {
    begin(KC_AVG, &a);
    end(KC_AVG, a, launch_average(in, in_stride, nw, dim, out, err, check_finite ? 1 : 0,
                                  mode == BL_MODE_SIM ? 0 : rank, stream));
    return;
  }
  if (transport == BL_TRANSPORT_P2P) {
    // One kernel over NVLink peer memory: flag "my gradient is in place" to
    // every peer, average chunk `rank` from all peers' buffers (reads) into
    // every peer's output (stores), then wait for every rank's chunk.
    const unsigned long long ep = ++lcalls;
    const int nn = n;
    begin(KC_A2A, &a);
    end(KC_A2A, a, launch_signal_peers(d_peer_flags, 2 * nn + rank, nn, ep, err, stream));
    LosslessP2PParams lp{};
    lp.peer_in = d_peer_in;
    lp.peer_out = d_peer_out;
    lp.peer_err = d_peer_err;
    lp.peer_flags = d_peer_flags;
    lp.in_flags = flags + 2 * nn;
    lp.out_flag = 3 * nn;
    lp.n = nn;
    lp.rank = rank;
    lp.check_finite = check_finite ? 1 : 0;
    lp.c = c;
    lp.d = dim;
    lp.epoch = ep;
    lp.done = lossless_done;
    lp.err = err;
    begin(KC_AVG, &a);
    end(KC_AVG, a, launch_lossless_p2p(lp, sms, stream));
    begin(KC_AG, &a);
    end(KC_AG, a, launch_wait_peers(flags + 3 * nn, nn, ep, err, stream));
    return;
  }
  // Deterministic all-reduce: alltoall of fp32 chunks, ascending-rank fp64
  // average of the own chunk, allgather (same bytes as a ring RS + AG).
  if (!lrecv) lrecv = dalloc<float>(static_cast<size_t>(n) * c_pad + kSlack);
  begin(KC_A2A, &a);
  cuda_check(cudaMemcpyAsync(lrecv + static_cast<size_t>(rank) * c_pad,
                             in + static_cast<size_t>(rank) * c, c * sizeof(float),
                             cudaMemcpyDeviceToDevice, stream),
             "self chunk copy");
  nccl_check(ncclGroupStart(), "ncclGroupStart");
  for (int j = 0; j < n; ++j) {
    if (j == rank) continue;
    nccl_check(ncclSend(in + static_cast<size_t>(j) * c, c, ncclFloat32, j, comm, stream), "ncclSend");
    nccl_check(ncclRecv(lrecv + static_cast<size_t>(j) * c_pad, c, ncclFloat32, j, comm, stream),
               "ncclRecv");
  }
  nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  end(KC_A2A, a, 0);
  if (check_finite) {
    // check_gradients covers the rank's whole gradient, not just its chunk;
    // the finding is raised on every rank (optimizers.cpp:99-117).
    begin(KC_AVG, &a);
    end(KC_AVG, a, launch_average(in, in_stride, 1, dim, nullptr, err, 1, rank, stream));
    share_grad_error();
  }
  begin(KC_AVG, &a);
  end(KC_AVG, a, launch_average(lrecv, c_pad, n, c, out + static_cast<size_t>(rank) * c, err, 0,
                                0, stream));
  begin(KC_AG, &a);
  nccl_check(ncclAllGather(out + static_cast<size_t>(rank) * c, out, c, ncclFloat32, comm, stream),
             "ncclAllGather");
  end(KC_AG, a, 0);
}

void bl_cluster::ensure_side_stream() {
  if (comm_stream) return;
  cuda_check(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking), "comm stream");
  cuda_check(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "event");
}

// Run `launch` on the side stream after everything enqueued so far on the
// main stream; join_side() makes the main stream wait for it.
void bl_cluster::fork_side(const std::function<int(cudaStream_t)>& launch) {
  ensure_side_stream();
  cuda_check(cudaEventRecord(ev_fork, stream), "fork");
  cuda_check(cudaStreamWaitEvent(comm_stream, ev_fork, 0), "fork wait");
  launches += static_cast<uint64_t>(launch(comm_stream));
  cuda_check(cudaGetLastError(), "side-stream launch");
  cuda_check(cudaEventRecord(ev_join, comm_stream), "join");
}
void bl_cluster::join_side() { cuda_check(cudaStreamWaitEvent(stream, ev_join, 0), "join wait"); }

unsigned long long bl_cluster::lossless_pieces(bool check_finite, int pieces) {
  const unsigned long long ep = ++lcalls;
  const int nn = n;
  ensure_side_stream();
  cudaEvent_t a;
  begin(KC_A2A, &a);
  end(KC_A2A, a, launch_signal_peers(d_peer_flags, 2 * nn + rank, nn, ep, err, stream));
  cuda_check(cudaEventRecord(ev_fork, stream), "fork");
  cuda_check(cudaStreamWaitEvent(comm_stream, ev_fork, 0), "fork wait");
  LosslessP2PParams lp{};
  lp.peer_in = d_peer_in;
  lp.peer_out = d_peer_out;
  lp.peer_err = d_peer_err;
  lp.peer_flags = d_peer_flags;
  lp.in_flags = flags + 2 * nn;
  lp.out_flag = 3 * nn;
  lp.n = nn;
  lp.rank = rank;
  lp.check_finite = check_finite ? 1 : 0;
  lp.c = c;
  lp.d = dim;
  lp.epoch = ep;
  lp.done = lossless_done;
  lp.err = err;
  lp.pieces = pieces;
  lp.piece_flag_base = piece_flag_base();
  lp.piece_done = piece_done;
  const char* ce = std::getenv("BL_LOSSLESS_CTAS_PER_SM");
  lp.ctas = sms * (ce ? std::max(1, std::atoi(ce)) : 1);  // leave the SMs' remaining slots to W1/W2
  const char* be = std::getenv("BL_LOSSLESS_BLOCK");
  lp.block = be ? std::atoi(be) : (n == 2 ? 256 : 128);
  // Launched (and profiled) on the comm stream, concurrent with the consumers.
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (profiling) {
    e0 = get_event();
    cuda_check(cudaEventRecord(e0, comm_stream), "cudaEventRecord");
  }
  launches += static_cast<uint64_t>(launch_lossless_p2p(lp, sms, comm_stream));
  cuda_check(cudaGetLastError(), "lossless (pieces)");
  if (profiling) {
    e1 = get_event();
    cuda_check(cudaEventRecord(e1, comm_stream), "cudaEventRecord");
    pending.push_back({KC_AVG, e0, e1});
  }
  cuda_check(cudaEventRecord(ev_join, comm_stream), "join");
  return ep;
}

// verify_compensation (comm_sim.cpp:83-106, 145-147, 170-172): after a
// collective with error_scale == 1 every local worker chunk and local server
// chunk is re-checked on the device; the count follows comm_sim.cpp:198-200
// (n^2 + n per collective in SIM mode, n + 1 local endpoints in NCCL mode).
void bl_cluster::verify_last() {
  const int latest = static_cast<int>((calls + 1u) & 1u);
  const double tol = cfg.compensation_tolerance;
  cudaEvent_t a;
  for (int w = 0; w < nw; ++w) {
    begin(KC_STATS, &a);
    end(KC_STATS, a,
        launch_verify(werr + static_cast<size_t>(w) * n * c_pad, c_pad,
                      wpk[latest] + static_cast<size_t>(w) * n * slot, slot, W, c, P, tol, err, stream));
  }
  for (int sv = 0; sv < ns; ++sv) {
    const int j = mode == BL_MODE_SIM ? sv : rank;
    begin(KC_STATS, &a);
    end(KC_STATS, a,
        launch_verify(serr + static_cast<size_t>(sv) * c_pad, c_pad,
                      res[latest] + static_cast<size_t>(j) * slot, slot, W, c, c, tol, err, stream));
  }
  checks += static_cast<uint64_t>(nw) * n + static_cast<uint64_t>(ns);
}

void bl_cluster::refresh_stats() {  // comm_sim.cpp:108-118, 175-180 (device records, no sync)
  const int latest = static_cast<int>((calls + 1u) & 1u);
  cudaEvent_t a;
  for (int w = 0; w < nw; ++w) {
    const int gw = mode == BL_MODE_SIM ? w : rank;
    begin(KC_STATS, &a);
    end(KC_STATS, a,
        launch_error_stats(werr + static_cast<size_t>(w) * n * c_pad, c_pad,
                           wpk[latest] + static_cast<size_t>(w) * n * slot, slot, W, c, P, stat_part,
                           stat_tiles, stat_max, wcmax + static_cast<size_t>(w) * n * tpc, n * tpc,
                           stats_dev + 5 * static_cast<size_t>(gw), stream));
  }
  for (int sv = 0; sv < ns; ++sv) {
    const int j = mode == BL_MODE_SIM ? sv : rank;
    begin(KC_STATS, &a);
    end(KC_STATS, a,
        launch_error_stats(serr + static_cast<size_t>(sv) * c_pad, c_pad,
                           res[latest] + static_cast<size_t>(j) * slot, slot, W, c, c, stat_part, stat_tiles,
                           stat_max, scmax + static_cast<size_t>(sv) * tpc, tpc,
                           stats_dev + 5 * static_cast<size_t>(n + j), stream));
  }
}

namespace {
std::string layer_label(const bl_optimizer* opt, long long layer) {
  if (opt && layer >= 0 && layer < static_cast<long long>(opt->names.size()))
    return opt->names[static_cast<size_t>(layer)];
  return "layer" + std::to_string(layer);
}
long long layer_of(const bl_optimizer* opt, uint64_t k) {
  if (!opt) return -1;
  return std::upper_bound(opt->off.begin(), opt->off.end(), k) - opt->off.begin() - 1;
}
}  // namespace

void bl_cluster::ensure_usable() const {
  if (broken) fail(BL_ERR_NCCL, "cluster failed earlier and its state is undefined: " + broken_msg);
}

void bl_cluster::begin_step(bl_optimizer* opt, uint64_t t, bool is_step, bool strict_check) {
  ensure_usable();
  seq += 1;
  Snap sn{};
  sn.seq = seq;
  sn.t = t;
  sn.is_step = is_step;
  sn.calls = calls;
  sn.checks = checks;
  sn.last_identity = last_identity;
  sn.ledger = ledger;
  sn.opt = opt;
  if (opt) {
    sn.frozen = opt->frozen;
    sn.has_vf = opt->has_vf;
    sn.has_mprev = opt->has_mprev;
    sn.m_valid = opt->m_valid;
    sn.mprev_separate = opt->mprev_separate;
    sn.my_calls = opt->my_calls;
  }
  if (snaps.size() >= 4096) snaps.erase(snaps.begin());  // unsynchronized for that long: keep the tail
  snaps.push_back(sn);

  // The arrival barrier guards optimizer steps (abort before any mutation);
  // a bare collective relies on the fail-stop bound of its own peer waits.
  const bool multi = mode == BL_MODE_NCCL && n > 1 && is_step;
  if (!strict_check && !multi) return;
  cudaEvent_t a;
  if (strict_check) {  // check_gradients (optimizers.cpp:99-117) before any mutation
    begin(KC_GATE, &a);
    end(KC_GATE, a, launch_check_finite(in, in_stride, nw, dim, err, mode == BL_MODE_SIM ? 0 : rank, stream));
  }
  const uint64_t* off_dev = opt ? opt->off_dev : nullptr;
  const int L = opt ? opt->L : 0;
  if (multi && transport != BL_TRANSPORT_P2P) {
    // NCCL transport: waits without a bound (NCCL's own semantics); only the
    // strict finding travels, as a min-reduced status word.
    if (!strict_check) return;
    if (!gate_status) gate_status = reinterpret_cast<unsigned long long*>(dalloc<double>(1));
    begin(KC_GATE, &a);
    end(KC_GATE, a, launch_gate_status(err, off_dev, L, rank, gate_status, stream));
    nccl_check(ncclAllReduce(gate_status, gate_status, 1, ncclUint64, ncclMin, comm, stream),
               "ncclAllReduce(gate)");
    begin(KC_GATE, &a);
    end(KC_GATE, a, launch_gate_apply(err, gate_status, rank, seq, stream));
    return;
  }
  GateParams g{};
  g.err = err;
  g.seq = seq;
  g.epoch = ++gate_epoch;
  g.n = multi ? n : 1;
  g.rank = rank;
  g.strict = strict_check ? 1 : 0;
  g.peer_flags = multi ? d_peer_flags : nullptr;
  g.arrive = flags ? flags + 4 * n : nullptr;
  g.arrive_index = 4 * n;
  g.decision_index = 5 * n;
  g.off = off_dev;
  g.L = L;
  begin(KC_GATE, &a);
  end(KC_GATE, a, launch_step_gate(g, stream));
}

void bl_cluster::set_peer_timeout(double ms) {
  peer_timeout_ms = ms;
  const unsigned long long ns = static_cast<unsigned long long>(ms * 1e6);
  cuda_check(cudaMemcpy(err + kCfgTimeout, &ns, sizeof ns, cudaMemcpyHostToDevice), "peer timeout");
}

void bl_cluster::rollback(uint64_t seq_closed) {
  auto it = std::find_if(snaps.begin(), snaps.end(), [&](const Snap& s) { return s.seq == seq_closed; });
  if (it == snaps.end()) {
    broken = true;
    broken_msg = "a step was aborted on the device but its host snapshot is gone";
    return;
  }
  calls = it->calls;
  checks = it->checks;
  last_identity = it->last_identity;
  ledger = it->ledger;
  if (bl_optimizer* o = it->opt) {
    o->frozen = it->frozen;
    o->has_vf = it->has_vf;
    o->has_mprev = it->has_mprev;
    o->m_valid = it->m_valid;
    o->mprev_separate = it->mprev_separate;
    o->my_calls = it->my_calls;
  }
  snaps.clear();
}

void bl_cluster::check_errors(const bl_optimizer* opt) {
  if (!opt) opt = last_opt;
  unsigned long long e[kErrSlots];
  cuda_check(cudaMemcpy(e, err, sizeof e, cudaMemcpyDeviceToHost), "error words");
  const unsigned long long none = ~0ull;
  bool any = false;
  for (int k = 0; k < kErrSlots; ++k) any |= e[k] != none;
  if (!any) {
    snaps.clear();  // everything enqueued so far completed cleanly
    return;
  }
  cuda_check(cudaMemset(err, 0xFF, sizeof e), "reset error words");
  char buf[512];
  if (e[kErrGate] != none) {
    const unsigned long long reason = e[kErrGate];
    uint64_t t = pending_step;
    const bl_optimizer* o = opt;
    for (const Snap& sn : snaps)
      if (sn.seq == e[kErrGateSeq]) {
        t = sn.t;
        if (sn.opt) o = sn.opt;
      }
    if (reason == kGateNonFinite || reason == kGateRemoteNonFinite) {
      // optimizers.cpp:109-114, raised before anything changed (strict mode)
      unsigned long long worker = 0;
      long long layer = -1;
      if (e[kErrRemote] != none) {
        worker = e[kErrRemote] >> 32;
        layer = static_cast<long long>(e[kErrRemote] & 0xffffffffull);
      } else if (e[kErrGrad] != none) {
        worker = e[kErrGrad] >> 40;
        layer = layer_of(o, e[kErrGrad] & ((1ull << 40) - 1));
      }
      rollback(e[kErrGateSeq]);
      std::snprintf(buf, sizeof buf, "non-finite gradient at step %" PRIu64 ", worker %llu, layer '%s'", t,
                    worker, layer_label(o, layer).c_str());
      fail(BL_ERR_RUNTIME, buf);
    }
    if (reason == kGateArrival) {
      rollback(e[kErrGateSeq]);
      std::snprintf(buf, sizeof buf,
                    "rank %llu did not reach step %" PRIu64 " within %.0f ms: the step was aborted on every "
                    "rank before any state changed",
                    e[kErrPeer], t, peer_timeout_ms);
      fail(BL_ERR_NCCL, buf);
    }
    broken = true;
    if (reason == kGateMidStep) {
      std::snprintf(buf, sizeof buf,
                    "rank %llu stopped signalling inside a step (no flag for %.0f ms): fail-stop, the "
                    "cluster state is undefined",
                    e[kErrPeer], peer_timeout_ms);
    } else {
      std::snprintf(buf, sizeof buf, "a device-side barrier timed out (reason %llu): fail-stop", reason);
    }
    broken_msg = buf;
    fail(BL_ERR_NCCL, buf);
  }
  if (e[kErrGrad] != none) {  // optimizers.cpp:109-114 (fused check: reported after the step)
    const unsigned long long w = e[kErrGrad] >> 40, k = e[kErrGrad] & ((1ull << 40) - 1);
    std::snprintf(buf, sizeof buf, "non-finite gradient at step %" PRIu64 ", worker %llu, layer '%s'",
                  pending_step, w, layer_label(opt, layer_of(opt, k)).c_str());
    snaps.clear();
    fail(BL_ERR_RUNTIME, buf);
  }
  snaps.clear();
  if (e[kErrScale] != none) fail(BL_ERR_INVALID_ARGUMENT, "compress: input vector is not finite");
  if (e[kErrPeer] != none) {
    std::snprintf(buf, sizeof buf, "fused NVLink exchange: rank %llu never signalled (timeout)", e[kErrPeer]);
    fail(BL_ERR_NCCL, buf);
  }
  if (e[kErrVerify] != none) {  // comm_sim.cpp:91-101
    std::snprintf(buf, sizeof buf,
                  "error-compensation identity violated at element %llu: exceeds relative "
                  "tolerance %g",
                  e[kErrVerify], cfg.compensation_tolerance);
    fail(BL_ERR_LOGIC, buf);
  }
  if (e[kErrRecon] != none) {  // optimizers.cpp:288-293
    std::snprintf(buf, sizeof buf, "non-finite reconstructed gradient for layer '%s'",
                  layer_label(opt, static_cast<long long>(e[kErrRecon])).c_str());
    fail(BL_ERR_RUNTIME, buf);
  }
}

void bl_cluster::sync_and_check(const bl_optimizer* opt) {
  cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
  check_errors(opt);
}

// ---------------------------------------------------------------------------
// bl_optimizer
// ---------------------------------------------------------------------------
bl::LayerTiles bl_optimizer::lt() const {
  const bool dyn = std::getenv("BL_STATIC_TILES") == nullptr;
  return {L, tiles, off_dev, tile_layer, layer_tile_start, dyn ? cl->tile_ctr : nullptr,
          dyn ? tile_order : nullptr, mis_layers ? 1 : 0};
}

void bl_optimizer::build_piece_tables(int K) {
  // Lossless piece after which every element of [e0, e1) is delivered: per
  // chunk the piece of its last element in the range (pieces are monotone).
  auto req = [&](uint64_t e0, uint64_t e1) {
    int r = 0;
    for (uint64_t j = e0 / cl->c; j * cl->c < e1; ++j) {
      const uint64_t lo = j * cl->c, hi = lo + cl->c;
      r = std::max(r, lossless_piece(lo, hi, K, std::min(e1, hi) - 1));
    }
    return r;
  };
  std::vector<int> tpiece(static_cast<size_t>(tiles)), lpiece(static_cast<size_t>(L), 0);
  std::vector<int> tl_h(static_cast<size_t>(tiles));
  for (int l = 0; l < L; ++l) {
    const uint64_t lo = off[l], hi = off[l + 1];
    int t = 0;
    for (uint64_t e0 = lo; e0 < hi; e0 += kTile, ++t) {
      const int tile = lt_start_h[l] + t;
      tpiece[tile] = req(e0, std::min<uint64_t>(e0 + kTile, hi));
      tl_h[tile] = l;
      lpiece[l] = std::max(lpiece[l], tpiece[tile]);
    }
  }
  auto bucket = [&](const std::vector<int>& items, auto key, std::vector<int>& start) {
    std::vector<std::vector<int>> b(static_cast<size_t>(K));
    for (int it : items) b[static_cast<size_t>(key(it))].push_back(it);
    std::vector<int> out;
    start.assign(static_cast<size_t>(K) + 1, 0);
    for (int p = 0; p < K; ++p) {
      start[p] = static_cast<int>(out.size());
      out.insert(out.end(), b[p].begin(), b[p].end());
    }
    start[K] = static_cast<int>(out.size());
    return out;
  };
  const std::vector<int> w1 = bucket(tile_order_h, [&](int t) { return tpiece[t]; }, w1_start);
  const std::vector<int> w2 = bucket(tile_order_h, [&](int t) { return lpiece[tl_h[t]]; }, w2_start);
  std::vector<int> layers(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) layers[l] = l;
  const std::vector<int> lw = bucket(layers, [&](int l) { return lpiece[l]; }, lw_start);
  for (int* p : {w1_order, w2_order, lw_order})
    if (p) cudaFree(p);
  w1_order = reinterpret_cast<int*>(dalloc<float>(w1.size()));
  w2_order = reinterpret_cast<int*>(dalloc<float>(w2.size()));
  lw_order = reinterpret_cast<int*>(dalloc<float>(lw.size()));
  cuda_check(cudaMemcpy(w1_order, w1.data(), w1.size() * 4, cudaMemcpyHostToDevice), "w1 order");
  cuda_check(cudaMemcpy(w2_order, w2.data(), w2.size() * 4, cudaMemcpyHostToDevice), "w2 order");
  cuda_check(cudaMemcpy(lw_order, lw.data(), lw.size() * 4, cudaMemcpyHostToDevice), "layer order");
  piece_k = K;
}

void bl_optimizer::warmup_step(uint64_t, double lr, bool track, bool finalize, bool adam) {
  // average_lossless (optimizers.cpp:119-138).  With one worker the average
  // (float)((0.0 + g) * 1.0) is g itself: W1 reads the gradient in place and
  // only the finite check runs.
  const bool single = cl->n == 1;
  if (sharded_warmup()) {
    warmup_sharded(lr, track, finalize, adam);
    return;
  }
  // Multi-process over NVLink: the exchange is delivered piece by piece and
  // W1 / the layer epilogue / W2 follow it (same kernels on tile and layer
  // subsets), so the NVLink transfer and the HBM-bound update overlap.
  const char* pe = std::getenv("BL_WARMUP_PIECES");
  // Defaults from the N=2 / N=4 sweeps (profiles/round2_warm_sweep*.txt).
  const int K = std::min(bl_cluster::kMaxPieces, pe ? std::max(0, std::atoi(pe)) : (cl->n == 2 ? 4 : 8));
  const bool overlap = !single && cl->mode == BL_MODE_NCCL && cl->transport == BL_TRANSPORT_P2P && K > 0 &&
                       std::getenv("BL_STATIC_TILES") == nullptr;
  if (overlap) {
    if (piece_k != K) build_piece_tables(K);
    const unsigned long long ep = cl->lossless_pieces(true, K);
    cl->ledger_lossless();
    warmup_kernels(lr, track, finalize, adam, K, ep);
    cuda_check(cudaStreamWaitEvent(cl->stream, cl->ev_join, 0), "join");
    return;
  }
  if (!single) cl->lossless(true);
  cl->ledger_lossless();
  warmup_kernels(lr, track, finalize, adam, 0, 0);
}

bool bl_optimizer::sharded_warmup() const {
  if (cl->n == 1 || cl->mode != BL_MODE_NCCL || cl->transport != BL_TRANSPORT_P2P) return false;
  if (std::getenv("BL_STATIC_TILES") != nullptr) return false;
  const char* e = std::getenv("BL_WARMUP_SHARD");
  return e == nullptr || std::atoi(e) != 0;
}

// Collective (every rank's first sharded warmup step): tile ownership and
// the peer mappings of x, m, v, vf and the tile partials.
void bl_optimizer::setup_shard() {
  const int n = cl->n, r = cl->rank;
  shard_t0 = static_cast<int>(static_cast<long long>(tiles) * r / n);
  shard_t1 = static_cast<int>(static_cast<long long>(tiles) * (r + 1) / n);
  auto tile_elem = [&](int tile) -> uint64_t {
    if (tile >= tiles) return d;
    const int l = static_cast<int>(std::upper_bound(lt_start_h.begin(), lt_start_h.end(), tile) -
                                   lt_start_h.begin()) - 1;
    return off[l] + static_cast<uint64_t>(tile - lt_start_h[l]) * kTile;
  };
  shard_e0 = tile_elem(shard_t0);
  shard_e1 = tile_elem(shard_t1);
  std::vector<int> own;
  for (int t : tile_order_h)
    if (t >= shard_t0 && t < shard_t1) own.push_back(t);
  own_count = static_cast<int>(own.size());
  own_order = reinterpret_cast<int*>(dalloc<float>(own.size()));
  if (!own.empty())
    cuda_check(cudaMemcpy(own_order, own.data(), own.size() * 4, cudaMemcpyHostToDevice), "own order");
  const char* pe = std::getenv("BL_SHARD_PIECES");
  // Defaults from the N=2 / N=4 sweeps (profiles/round2_shard_sweep_n*.txt).
  shard_k = std::min(bl_cluster::kMaxPieces, std::max(1, pe ? std::atoi(pe) : (n == 2 ? 4 : 3)));
  const int K = shard_k;
  const char* se = std::getenv("BL_SHARD_SHAPE");
  shard_shape = se ? std::atoi(se) : (n > 2 ? 1 : 0);
  auto layer_of_tile = [&](int t) {
    return static_cast<int>(std::upper_bound(lt_start_h.begin(), lt_start_h.end(), t) - lt_start_h.begin()) - 1;
  };
  // Reduce piece after which tile t's gradient is complete; a layer is local
  // when all its tiles are owned here (its epilogue needs no peer partials).
  std::vector<int> tpiece(static_cast<size_t>(tiles), 0), lpiece(static_cast<size_t>(L), 0);
  for (int t : own) {
    const int l = layer_of_tile(t);
    const uint64_t e_last = std::min<uint64_t>(tile_elem(t) + kTile, off[l + 1]) - 1;
    tpiece[t] = lossless_piece(shard_e0, shard_e1, K, e_last, shard_shape);
    lpiece[l] = std::max(lpiece[l], tpiece[t]);
  }
  // Early W2 of local layers (measured slower: its NVLink stores compete
  // with the reduce's reads; BL_SHARD_EARLY_W2=1 for experiments).
  const bool early = std::getenv("BL_SHARD_EARLY_W2") != nullptr && std::atoi(std::getenv("BL_SHARD_EARLY_W2"));
  auto local = [&](int l) { return early && lt_start_h[l] >= shard_t0 && lt_start_h[l + 1] <= shard_t1; };
  // Buckets [0, K) by piece; bucket K = the rest (after the partials exchange).
  auto bucketed = [&](const std::vector<int>& items, auto key, std::vector<int>* start) {
    std::vector<std::vector<int>> b(static_cast<size_t>(K) + 1);
    for (int it : items) b[static_cast<size_t>(key(it))].push_back(it);
    std::vector<int> out;
    start->assign(static_cast<size_t>(K) + 2, 0);
    for (int q = 0; q <= K; ++q) {
      (*start)[q] = static_cast<int>(out.size());
      out.insert(out.end(), b[q].begin(), b[q].end());
    }
    (*start)[K + 1] = static_cast<int>(out.size());
    return out;
  };
  std::vector<int> all_layers(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) all_layers[l] = l;
  const std::vector<int> w1o = bucketed(own, [&](int t) { return tpiece[t]; }, &own_w1_start);
  const std::vector<int> w2o = bucketed(own, [&](int t) {
    const int l = layer_of_tile(t);
    return local(l) ? lpiece[l] : K;
  }, &own_w2_start);
  const std::vector<int> lwo = bucketed(all_layers, [&](int l) { return local(l) ? lpiece[l] : K; }, &own_lw_start);
  auto upload = [](const std::vector<int>& h) {
    int* dv = reinterpret_cast<int*>(dalloc<float>(h.size()));
    if (!h.empty()) cuda_check(cudaMemcpy(dv, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "shard tables");
    return dv;
  };
  own_w1_order = upload(w1o);
  own_w2_order = upload(w2o);
  own_lw_order = upload(lwo);
  const char* pu = std::getenv("BL_SHARD_PUSH");
  shard_push = pu && std::atoi(pu) != 0;  // (must agree on every rank)
  std::vector<void*> to_map = {x, m, v, vf, tile_sums};
  if (shard_push) {
    std::vector<uint64_t> e_all(static_cast<size_t>(n) + 1);
    for (int q = 0; q <= n; ++q) e_all[q] = tile_elem(static_cast<int>(static_cast<long long>(tiles) * q / n));
    stg_S = 0;
    for (int q = 0; q < n; ++q) stg_S = std::max<uint64_t>(stg_S, e_all[q + 1] - (e_all[q] & ~3ull));
    stg_S = (stg_S + 7) & ~3ull;
    stg = dalloc<float>(static_cast<size_t>(n) * stg_S);
    e_all_dev = reinterpret_cast<uint64_t*>(dalloc<double>(e_all.size()));
    cuda_check(cudaMemcpy(e_all_dev, e_all.data(), e_all.size() * 8, cudaMemcpyHostToDevice), "ranges");
    to_map.push_back(stg);
  }
  std::vector<std::vector<void*>> peer;
  if (!cl->map_peer_buffers(to_map, &peer, &shard_ipc))
    fail(BL_ERR_UNSUPPORTED, "sharded warmup: a peer's optimizer state could not be mapped");
  if (shard_push) {
    d_peer_stg = reinterpret_cast<float**>(dalloc<double>(static_cast<size_t>(n)));
    cuda_check(cudaMemcpy(d_peer_stg, peer[5].data(), static_cast<size_t>(n) * sizeof(void*),
                          cudaMemcpyHostToDevice),
               "staging table");
  }
  auto table = [&](int k) {
    std::vector<void*> others;
    for (int q = 0; q < n; ++q)
      if (q != r) others.push_back(peer[k][q]);
    void** t = reinterpret_cast<void**>(dalloc<double>(others.size()));
    cuda_check(cudaMemcpy(t, others.data(), others.size() * sizeof(void*), cudaMemcpyHostToDevice), "tables");
    return t;
  };
  push_x = reinterpret_cast<float**>(table(0));
  push_m = reinterpret_cast<float**>(table(1));
  push_v = reinterpret_cast<float**>(table(2));
  push_vf = reinterpret_cast<float**>(table(3));
  push_sums = reinterpret_cast<double**>(table(4));
  shard_ready = true;
}

// Owner-sharded warmup step (multi-process over NVLink; optimizers.cpp:119-177,
// 202-224 with the same per-element arithmetic and per-tile partials):
//   reduce the owned gradient range from every rank (NVLink reads) -> W1 on
//   the owned tiles -> tile partials to every rank -> the layer epilogue on
//   all layers (replicated, identical inputs) -> W2 on the owned tiles,
//   storing x into every rank -> wait until every owner delivered.
// Per rank: the NVLink bytes of the all-reduce, a 1/n share of the HBM work.
void bl_optimizer::warmup_sharded(double lr, bool track, bool finalize, bool adam) {
  if (!shard_ready) setup_shard();
  const int nn = cl->n;
  const unsigned long long ep = ++cl->lcalls;
  const int sbase = cl->shard_flag_base();
  cudaEvent_t a;
  cl->begin(KC_A2A, &a);
  cl->end(KC_A2A, a, launch_signal_peers(cl->d_peer_flags, 2 * nn + cl->rank, nn, ep, cl->err, cl->stream));
  LosslessP2PParams lp{};
  lp.peer_in = cl->d_peer_in;
  lp.peer_out = cl->d_peer_out;
  lp.peer_err = cl->d_peer_err;
  lp.peer_flags = cl->d_peer_flags;
  lp.in_flags = cl->flags + 2 * nn;
  lp.out_flag = 3 * nn;
  lp.n = nn;
  lp.rank = cl->rank;
  lp.check_finite = 1;
  lp.c = cl->c;
  lp.d = d;
  lp.epoch = ep;
  lp.done = cl->lossless_done;
  lp.err = cl->err;
  lp.lo = shard_e0;
  lp.hi = shard_e1;
  lp.local_only = 1;
  const char* be = std::getenv("BL_LOSSLESS_BLOCK");
  lp.block = be ? std::atoi(be) : 0;
  // The reduce runs on the comm stream, raising a local flag per piece; W1
  // follows on the main stream piece by piece (HBM work under the NVLink reads).
  const int K = shard_k;
  lp.pieces = K;
  lp.shape = shard_shape;
  lp.piece_flag_base = cl->piece_flag_base();
  lp.piece_done = cl->piece_done;
  const char* ce = std::getenv("BL_SHARD_CTAS_PER_SM");
  lp.ctas = cl->sms * (ce ? std::max(1, std::atoi(ce)) : 2);
  cl->ensure_side_stream();
  cuda_check(cudaEventRecord(cl->ev_fork, cl->stream), "fork");
  cuda_check(cudaStreamWaitEvent(cl->comm_stream, cl->ev_fork, 0), "fork wait");
  if (shard_push || shard_e1 > shard_e0) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cl->profiling) {
      e0 = cl->get_event();
      cuda_check(cudaEventRecord(e0, cl->comm_stream), "cudaEventRecord");
    }
    if (shard_push) {
      ShardPushParams sp{};
      sp.in = cl->in;
      sp.peer_stg = d_peer_stg;
      sp.e_all = e_all_dev;
      sp.S = stg_S;
      sp.n = nn;
      sp.rank = cl->rank;
      sp.pieces = K;
      sp.shape = shard_shape;
      sp.peer_flags = cl->d_peer_flags;
      sp.piece_flag_base = cl->piece_flag_base();
      sp.epoch = ep;
      sp.piece_done = cl->piece_done;
      sp.gate = cl->err;
      const char* pc = std::getenv("BL_SHARD_PUSH_CTAS_PER_SM");
      cl->launches += static_cast<uint64_t>(
          launch_shard_push(sp, cl->sms * (pc ? std::max(1, std::atoi(pc)) : 4), cl->comm_stream));
    } else {
      cl->launches += static_cast<uint64_t>(launch_lossless_p2p(lp, cl->sms, cl->comm_stream));
    }
    cuda_check(cudaGetLastError(), "lossless (owned range)");
    if (cl->profiling) {
      e1 = cl->get_event();
      cuda_check(cudaEventRecord(e1, cl->comm_stream), "cudaEventRecord");
      cl->pending.push_back({KC_AVG, e0, e1});
    }
  }
  cuda_check(cudaEventRecord(cl->ev_join, cl->comm_stream), "join");
  cl->ledger_lossless();

  warmup_kernels(lr, track, finalize, adam, -1, ep);
  shard_stale = !finalize;
}

// Collective: push every owner's m and v slices to every rank (a state read
// during the multi-process warmup stage, where they are kept by their owners).
void bl_optimizer::sync_shards() {
  if (!shard_stale) return;
  const int nn = cl->n;
  const unsigned long long ep = ++cl->lcalls;
  const int sbase = cl->shard_flag_base();
  cudaEvent_t a;
  for (float* const* t : {push_m, push_v}) {
    const float* src = t == push_m ? m : v;
    cl->begin(KC_AG, &a);
    cl->end(KC_AG, a, launch_push_range(src, t, nn - 1, shard_e0, shard_e1 - shard_e0, cl->err, cl->sms,
                                        cl->stream));
  }
  cl->begin(KC_AG, &a);
  cl->end(KC_AG, a, launch_signal_peers(cl->d_peer_flags, sbase + cl->rank, nn, ep, cl->err, cl->stream));
  cl->begin(KC_AG, &a);
  cl->end(KC_AG, a, launch_wait_peers(cl->flags + sbase, nn, ep, cl->err, cl->stream));
  cl->sync_and_check(this);
  shard_stale = false;
}

// W1 -> layer epilogue -> W2 (optimizers.cpp:140-177, 202-224).  K > 0: per
// lossless piece p, wait for every rank's piece p, then the tiles / layers of
// that piece (sub-launches of the same kernels; bit-identical results).
void bl_optimizer::warmup_kernels(double lr, bool track, bool finalize, bool adam, int K,
                                  unsigned long long ep) {
  const bool single = cl->n == 1;
  cudaEvent_t a;
  W1Params w1{};
  w1.gate = cl->err;
  w1.lt = lt();
  w1.gbar = single ? cl->in : cl->out;
  w1.m = m;
  w1.v = v;
  w1.x = x;
  w1.b1 = static_cast<float>(hp.beta1);
  w1.omb1 = static_cast<float>(1.0 - hp.beta1);
  w1.b2 = static_cast<float>(hp.beta2);
  w1.omb2 = static_cast<float>(1.0 - hp.beta2);
  w1.eta = static_cast<float>(hp.eta);
  w1.wd = static_cast<float>(hp.weight_decay);
  w1.tile_sums = tile_sums;
  w1.adam = adam ? 1 : 0;
  w1.err = single ? cl->err : nullptr;  // check_gradients fused into W1
  w1.worker_base = cl->rank;

  WEpiParams we{};
  we.gate = cl->err;
  we.L = L;
  we.layer_tile_start = layer_tile_start;
  we.off = off_dev;
  we.tile_sums = tile_sums;
  we.c_avg = c_avg;
  we.coef_x = coef_x;
  we.trace = trace;
  we.mag = mag;
  we.coeff = coeff;
  we.A = A;
  we.B = B;
  we.invc = invc;
  we.cmean = cmean;
  we.es_next = es;
  we.counter = counter;
  we.lr = lr;
  we.b1 = hp.beta1;
  we.b3 = hp.beta3;
  we.c_min = hp.c_min;
  we.c_max = hp.c_max;
  we.floor_ = hp.division_floor;
  we.track = track ? 1 : 0;
  we.finalize = finalize ? 1 : 0;
  we.adam = adam ? 1 : 0;
  we.onebit_adam = variant == BL_ONEBIT_ADAM ? 1 : 0;

  W2Params w2{};
  w2.gate = cl->err;
  w2.lt = lt();
  w2.m = m;
  w2.v = v;
  w2.x = x;
  w2.vf = vf;
  w2.coef_x = coef_x;
  w2.eta = static_cast<float>(hp.eta);
  w2.wd = static_cast<float>(hp.weight_decay);
  w2.finalize = finalize ? 1 : 0;
  if (K < 0) {
    // Owner-sharded (warmup_sharded): W1 on the owned tiles piece by piece
    // behind the reduce; the local layers' epilogue and W2 (+ allgather) as
    // soon as their last piece is in; then the tile partials to every rank,
    // the remaining layers' epilogue and W2; then every owner delivered.
    const int P = shard_k, nn = cl->n, sbase = cl->shard_flag_base();
    w1.gbar = cl->out;
    w1.err = nullptr;
    w2.push_x = push_x;
    w2.push_m = push_m;
    w2.push_v = push_v;
    w2.push_vf = push_vf;
    w2.npush = nn - 1;
    auto epi_w2 = [&](int q) {
      if (const int cnt = own_lw_start[q + 1] - own_lw_start[q]) {
        WEpiParams e = we;
        e.layer_list = own_lw_order + own_lw_start[q];
        e.count = cnt;
        cl->begin(KC_WEPI, &a);
        cl->end(KC_WEPI, a, launch_wepilogue(e, cl->stream));
      }
      if (const int cnt = own_w2_start[q + 1] - own_w2_start[q]) {
        W2Params w = w2;
        w.lt.order = own_w2_order + own_w2_start[q];
        w.lt.count = cnt;
        cl->begin(KC_W2, &a);
        cl->end(KC_W2, a, launch_w2(w, cl->grid(cnt), cl->stream));
      }
    };
    for (int p = 0; p < P; ++p) {
      if (shard_push) {  // every rank's piece p staged here, then the local reduce of piece p
        cl->begin(KC_AG, &a);
        cl->end(KC_AG, a, launch_wait_piece(cl->flags, cl->piece_flag_base(), nn, P, p, ep, cl->err, cl->stream));
        ShardReduceParams rp{};
        rp.in = cl->in;
        rp.stg = stg;
        rp.S = stg_S;
        rp.E0 = shard_e0;
        rp.E1 = shard_e1;
        rp.d = d;
        rp.n = nn;
        rp.rank = cl->rank;
        rp.pieces = P;
        rp.shape = shard_shape;
        rp.piece = p;
        rp.out = cl->out;
        rp.err = cl->err;
        rp.peer_err = cl->d_peer_err;
        rp.done = cl->lossless_done;
        cl->begin(KC_AVG, &a);
        cl->end(KC_AVG, a, launch_shard_reduce(rp, cl->sms, cl->stream));
      }
      if (const int cnt = own_w1_start[p + 1] - own_w1_start[p]) {
        if (!shard_push) {
          cl->begin(KC_AG, &a);
          cl->end(KC_AG, a,
                  launch_wait_piece(cl->flags, cl->piece_flag_base() + cl->rank * P, 1, P, p, ep, cl->err,
                                    cl->stream));
        }
        W1Params q = w1;
        q.lt.order = own_w1_order + own_w1_start[p];
        q.lt.count = cnt;
        cl->begin(KC_W1, &a);
        cl->end(KC_W1, a, launch_w1(q, cl->grid(cnt), cl->stream));
      }
      epi_w2(p);
    }
    cuda_check(cudaStreamWaitEvent(cl->stream, cl->ev_join, 0), "join");
    cl->begin(KC_AG, &a);
    cl->end(KC_AG, a,
            launch_push_range(tile_sums, push_sums, nn - 1, 4ull * static_cast<uint64_t>(shard_t0),
                              4ull * static_cast<uint64_t>(shard_t1 - shard_t0), cl->err, cl->sms, cl->stream));
    cl->begin(KC_AG, &a);
    cl->end(KC_AG, a, launch_signal_peers(cl->d_peer_flags, sbase + cl->rank, nn, ep, cl->err, cl->stream));
    cl->begin(KC_AG, &a);
    cl->end(KC_AG, a, launch_wait_peers(cl->flags + sbase, nn, ep, cl->err, cl->stream));
    epi_w2(P);
    cl->begin(KC_AG, &a);
    cl->end(KC_AG, a, launch_signal_peers(cl->d_peer_flags, sbase + nn + cl->rank, nn, ep, cl->err, cl->stream));
    cl->begin(KC_AG, &a);
    cl->end(KC_AG, a, launch_wait_peers(cl->flags + sbase + nn, nn, ep, cl->err, cl->stream));
    return;
  }
  if (K == 0) {
    cl->begin(KC_W1, &a);
    cl->end(KC_W1, a, launch_w1(w1, cl->grid(tiles), cl->stream));
    cl->begin(KC_WEPI, &a);
    cl->end(KC_WEPI, a, launch_wepilogue(we, cl->stream));
    cl->begin(KC_W2, &a);
    cl->end(KC_W2, a, launch_w2(w2, cl->grid(tiles), cl->stream));
    return;
  }
  const bool consumers = std::getenv("BL_WARMUP_NO_CONSUMERS") == nullptr;  // timing experiments only
  const char* ev = std::getenv("BL_WARMUP_W2_EVERY");
  const int every = std::max(1, ev ? std::atoi(ev) : 4);
  for (int p = 0; p < K; ++p) {
    if (!consumers) continue;
    cl->begin(KC_AG, &a);
    cl->end(KC_AG, a,
            launch_wait_piece(cl->flags, cl->piece_flag_base(), cl->n, K, p, ep, cl->err, cl->stream));
    if (const int cnt = w1_start[p + 1] - w1_start[p]) {
      W1Params q = w1;
      q.lt.order = w1_order + w1_start[p];
      q.lt.count = cnt;
      cl->begin(KC_W1, &a);
      cl->end(KC_W1, a, launch_w1(q, cl->grid(cnt), cl->stream));
    }
    // The layers completed by the last `every` pieces: epilogue, then W2 (batched:
    // fewer, larger launches; W2 is not needed before the end of the step).
    if ((p + 1) % every != 0 && p != K - 1) continue;
    const int b0 = std::max(0, p + 1 - every);
    if (const int cnt = lw_start[p + 1] - lw_start[b0]) {
      WEpiParams q = we;
      q.layer_list = lw_order + lw_start[b0];
      q.count = cnt;
      cl->begin(KC_WEPI, &a);
      cl->end(KC_WEPI, a, launch_wepilogue(q, cl->stream));
    }
    if (const int cnt = w2_start[p + 1] - w2_start[b0]) {
      W2Params q = w2;
      q.lt.order = w2_order + w2_start[b0];
      q.lt.count = cnt;
      cl->begin(KC_W2, &a);
      cl->end(KC_W2, a, launch_w2(q, cl->grid(cnt), cl->stream));
    }
  }
}

// The streaming K5/K6 kernels' fast-path test per tile (bl_kernels.cu),
// evaluated on the host: a tile inside one result chunk, on a 16-B
// boundary unless the MISK kernels run.  The rest go to k5/k6_general when
// the problem is small enough for their chains to set the kernels' time
// (BL_GENERAL_SPLIT_MAX_TILES, default 16384 tiles; larger problems hide
// them behind the boundary-first streaming kernels).
void bl_optimizer::ensure_gen_tiles() {
  if (gen_c == cl->c) return;
  gen_c = cl->c;
  gen_n = 0;
  const char* e = std::getenv("BL_GENERAL_SPLIT_MAX_TILES");
  if (tiles > (e ? std::atoll(e) : 16384ll)) return;
  std::vector<int> gen;
  for (int l = 0; l < L; ++l) {
    const uint64_t lo = off[l], len = off[l + 1] - lo;
    const bool aligned = mis_layers || (lo & 3u) == 0;
    for (uint64_t k = 0; k < len; k += kTile) {
      const uint64_t base = lo + k, tvalid = std::min<uint64_t>(len - k, kTile);
      const uint64_t ce = (base / cl->c + 1) * cl->c;
      if (!(aligned && base + tvalid <= ce)) gen.push_back(lt_start_h[l] + static_cast<int>(k / kTile));
    }
  }
  if (gen.empty()) return;
  if (gen_tiles) cudaFree(gen_tiles);
  gen_tiles = reinterpret_cast<int*>(dalloc<float>(gen.size()));
  cuda_check(cudaMemcpy(gen_tiles, gen.data(), gen.size() * 4, cudaMemcpyHostToDevice), "general tiles");
  gen_n = static_cast<int>(gen.size());
}

void bl_optimizer::compressed_step(double lr, const float* stage_host) {
  const bool identity = cl->cfg.compressor != BL_COMPRESSOR_ONEBIT;
  // optimizers.cpp:271-303: ratio rule (onebit_lamb), c = c_avg (basic), c = 1 (adam)
  const int emode = variant == BL_ONEBIT_LAMB ? 0 : variant == BL_LAMB_BASIC_ONEBIT ? 1 : 2;
  cudaEvent_t a;
  if (identity) {
    // Identity compressor (compression.cpp:184-188): the collective is the
    // exact ascending-worker average of the streams; residuals stay zero.
    cl->begin(KC_AVG, &a);
    cl->end(KC_AVG, a,
            launch_build_stream(cl->in, cl->in_stride, cl->nw, d, m_valid ? m : nullptr, off_dev, L,
                                A, B, cl->err, cl->mode == BL_MODE_SIM ? 0 : cl->rank, cl->stream));
    cl->share_grad_error();  // (the P2P exchange forwards it with its flags)
    cl->lossless(false);
    cl->ledger_compressed();
    cl->calls += 1;
    cl->last_identity = true;
  } else {
    const int mode = m_valid ? 1 : 2;
    if (!m_valid && cl->calls != my_calls) {
      fail(BL_ERR_LOGIC,
           "momentum is encoded by the cluster's last result packets, but the cluster ran another "
           "collective since the last optimizer step");
    }
    K1Params p{};
    p.L = L;
    p.m = m;
    p.res_prev = cl->res[cl->prev()];  // latest result before this collective
    p.off = off_dev;
    p.A = A;
    p.B = B;
    p.invc = invc;
    p.tile_layer = k1_tile_layer;
    p.slow_list = k1_slow;
    p.n_slow = k1_n_slow;
    p.order = k1_order;
    cl->verify_es_one = !hp.scaled_error_feedback;
    cl->stage_host = stage_host;  // consumed (and cleared) by compressed() itself
    cl->compressed(&p, mode, 1.0f, es);
  }

  const int latest = static_cast<int>((cl->calls + 1u) & 1u);
  const int before = static_cast<int>(cl->calls & 1u);
  K5Params k5{};
  k5.lt = lt();
  k5.n = cl->n;
  k5.c = cl->c;
  k5.slot = cl->slot;
  k5.W = cl->W;
  k5.res_cur = cl->res[latest];
  const bool mprev_buf = m_valid || mprev_separate || identity;
  k5.res_prev = mprev_buf ? nullptr : cl->res[before];
  k5.dense = identity ? cl->out : nullptr;
  k5.m_store = identity ? m : nullptr;
  k5.norm_only = emode != 0;
  k5.m = mprev_separate ? mprev : m;
  k5.invc = invc;
  k5.v = v;
  k5.vf = vf;
  const double inv = 1.0 / (1.0 - hp.beta1);
  k5.inv = static_cast<float>(inv);
  k5.ninvb = static_cast<float>(-hp.beta1 * inv);
  k5.b2 = static_cast<float>(hp.beta2);
  k5.omb2 = static_cast<float>(1.0 - hp.beta2);
  k5.floor_ = static_cast<float>(hp.division_floor);
  k5.tile_max = tile_max;
  k5.tile_v2 = tile_sums;
  k5.err = cl->err;
  if (!identity) ensure_gen_tiles();
  if (!identity && emode == 0 && gen_n) {
    k5.gen_list = gen_tiles;
    k5.gen_count = gen_n;
  }
  cl->begin(KC_K5, &a);
  if (k5.gen_list) cl->fork_side([&](cudaStream_t s2) { return launch_k5_general(k5, s2); });
  cl->end(KC_K5, a, launch_k5(k5, cl->grid(tiles), cl->stream));
  if (k5.gen_list) cl->join_side();

  EpiParams ep{};
  ep.gate = cl->err;
  ep.L = L;
  ep.layer_tile_start = layer_tile_start;
  ep.tile_max = tile_max;
  ep.tile_v2 = tile_sums;
  ep.r_prev = r_prev;
  ep.c_avg = c_avg;
  ep.coef_x = coef_x;
  ep.trace = trace;
  ep.cmean = cmean;
  ep.es_next = es;
  ep.counter = counter;
  ep.lr = lr;
  ep.lr_dev = capturing ? lr_dev : nullptr;  // a captured step reads the lr staged before each replay
  ep.r_thr = hp.r_threshold;
  ep.r_min = hp.r_min;
  ep.r_max = hp.r_max;
  ep.floor_ = hp.division_floor;
  ep.scaled_ef = hp.scaled_error_feedback;
  ep.mode = emode;
  cl->begin(KC_EPI, &a);
  cl->end(KC_EPI, a, launch_epilogue(ep, cl->stream));

  K6Params k6{};
  k6.gate = cl->err;
  k6.lt = lt();
  k6.n = cl->n;
  k6.c = cl->c;
  k6.slot = cl->slot;
  k6.W = cl->W;
  k6.res_cur = cl->res[latest];
  k6.invc = invc;
  k6.coef_x = coef_x;
  k6.vf = vf;
  k6.x = x;
  k6.eta = static_cast<float>(hp.eta);
  k6.wd = static_cast<float>(hp.weight_decay);
  k6.dense = identity ? cl->out : nullptr;
  if (!identity && gen_n) {
    k6.gen_list = gen_tiles;
    k6.gen_count = gen_n;
  }
  cl->begin(KC_K6, &a);
  if (k6.gen_list) cl->fork_side([&](cudaStream_t s2) { return launch_k6_general(k6, s2); });
  cl->end(KC_K6, a, launch_k6(k6, cl->grid(tiles), cl->stream));
  if (k6.gen_list) cl->join_side();

  m_valid = identity;  // identity: m stored by K5; one-bit: m == decompressed result * invc
  mprev_separate = false;
  my_calls = cl->calls;
}

void bl_optimizer::step(const float* const* grads, int n_grads, uint64_t t, double lr, int memory,
                        bl_step_trace* tr) {
  if (n_grads < 1) fail(BL_ERR_INVALID_ARGUMENT, "step: no worker gradients");
  if (n_grads != cl->nw) {
    fail(BL_ERR_DIMENSION, "step: worker count: size mismatch (" + std::to_string(n_grads) +
                               " vs " + std::to_string(cl->nw) + ")");
  }
  const bool two = two_stage();
  const bool adam = variant == BL_ADAM || variant == BL_ONEBIT_ADAM;
  bool compressed = false;
  cl->ensure_usable();
  cl->last_opt = this;
  if (!two || t < hp.warmup_steps) {
    cl->copy_inputs(grads, n_grads, d, memory);
    cl->begin_step(this, t, true, strict);  // strict: check_gradients before any mutation
    const bool finalize = two && t + 1 == hp.warmup_steps;
    warmup_step(t, lr, two && !adam, finalize, adam);
    if (finalize) {  // optimizers.cpp:202-224
      frozen = true;
      has_vf = true;
      if (variant == BL_ONEBIT_LAMB) has_mprev = true;
      m_valid = true;
    }
  } else {
    if (!frozen) {
      fail(BL_ERR_STAGE_ORDER,
           "compression-stage step before warmup finalized: frozen variance, c_avg and momentum "
           "snapshot are missing");
    }
    // Host gradients in the one-bit compression stage: the H2D copy is cut
    // into tile-aligned pieces and K1 starts on each piece as it lands
    // (bl_cluster::compressed).  BL_OVERLAP_H2D=0 copies first.
    const char* ov = std::getenv("BL_OVERLAP_H2D");
    const float* stage = nullptr;
    if (memory == BL_MEM_HOST && cl->nw == 1 && cl->cfg.compressor == BL_COMPRESSOR_ONEBIT && !strict &&
        !(ov && ov[0] == '0')) {
      stage = grads[0];  // strict mode checks the whole gradient first: no piecewise copy
    } else {
      cl->copy_inputs(grads, n_grads, d, memory);
    }
    cl->begin_step(this, t, true, strict);
    if (stage == nullptr && graphable()) compressed_step_graph(lr);
    else compressed_step(lr, stage);
    compressed = true;
  }
  cl->pending_step = t;
  cl->pending_is_step = true;
  if (tr) {
    std::vector<double> h(4 * static_cast<size_t>(L));
    cudaEvent_t a;
    cl->begin(KC_D2H, &a);
    cuda_check(cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                               cl->stream),
               "trace copy");
    cl->end(KC_D2H, a, 0);
    cl->sync_and_check(this);
    for (int l = 0; l < L; ++l) {
      if (tr->c) tr->c[l] = h[l];
      if (tr->r) tr->r[l] = h[L + l];
      if (tr->v_norm) tr->v_norm[l] = h[2 * L + l];
      if (tr->v_ratio_preclip) tr->v_ratio_preclip[l] = h[3 * L + l];
    }
    tr->compressed = compressed ? 1 : 0;
  }
}

// Steady state only: the momentum is encoded by the packets (K1 mode 2, K5
// MPREV 1), no host-staged gradient, no per-collective host work (verify,
// stats, profiling), no peer flags (their epochs are kernel arguments).
bool bl_optimizer::graphable() const {
  static const bool off = [] {
    const char* e = std::getenv("BL_GRAPH");
    return e && e[0] == '0';
  }();
  return !off && variant == BL_ONEBIT_LAMB && !m_valid && !mprev_separate && cl->calls == my_calls &&
         cl->cfg.compressor == BL_COMPRESSOR_ONEBIT && !cl->cfg.verify_compensation &&
         !cl->cfg.endpoint_stats && !cl->profiling && (cl->mode == BL_MODE_SIM || cl->n == 1) &&
         std::getenv("BL_STATIC_TILES") == nullptr;
}

void bl_optimizer::compressed_step_graph(double lr) {
  if (!lr_dev) {
    lr_dev = dalloc<double>(1);
    cuda_check(cudaMallocHost(&lr_host, sizeof(double)), "cudaMallocHost");
  }
  const int par = cl->cur();
  if (!graph[par]) {  // capture this parity's step once (its kernel arguments depend only on the parity)
    cudaGraph_t g = nullptr;
    const uint64_t calls0 = cl->calls, launches0 = cl->launches;
    const bl_volume_ledger led0 = cl->ledger;
    cuda_check(cudaStreamBeginCapture(cl->stream, cudaStreamCaptureModeThreadLocal), "capture begin");
    capturing = true;
    try {
      compressed_step(lr, nullptr);
    } catch (...) {
      capturing = false;
      cudaStreamEndCapture(cl->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    capturing = false;
    cuda_check(cudaStreamEndCapture(cl->stream, &g), "capture end");
    cuda_check(cudaGraphInstantiate(&graph[par], g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    graph_kernels[par] = cl->launches - launches0;
    // capture enqueued nothing: undo the host bookkeeping of the captured step
    cl->calls = calls0;
    cl->launches = launches0;
    cl->ledger = led0;
    m_valid = false;
    my_calls = calls0;
  }
  *lr_host = lr;
  cuda_check(cudaMemcpyAsync(lr_dev, lr_host, sizeof(double), cudaMemcpyHostToDevice, cl->stream), "lr");
  cuda_check(cudaGraphLaunch(graph[par], cl->stream), "graph launch");
  // the host side of compressed_step
  cl->calls += 1;
  cl->last_identity = false;
  cl->ledger_compressed();
  cl->launches += graph_kernels[par];
  m_valid = false;
  mprev_separate = false;
  my_calls = cl->calls;
}

void bl_optimizer::materialize_m(float* dst) {
  const int latest = static_cast<int>((cl->calls + 1u) & 1u);
  cudaEvent_t a;
  cl->begin(KC_MAT, &a);
  cl->end(KC_MAT, a,
          launch_materialize_m(cl->res[latest], cl->n, cl->c, cl->slot, cl->W, off_dev, L, invc, d,
                               dst, cl->stream));
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
namespace {

thread_local std::string g_err;

template <typename F>
bl_status guarded(F&& f) {
  try {
    f();
    return BL_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.status;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BL_ERR_RUNTIME;
  }
}

void check_arg(bool ok, const char* msg) {
  if (!ok) fail(BL_ERR_INVALID_ARGUMENT, msg);
}

void size_check(uint64_t a, uint64_t b, const char* what) {  // errors.hpp:43-48
  if (a != b) {
    fail(BL_ERR_DIMENSION, std::string(what) + ": size mismatch (" + std::to_string(a) + " vs " +
                               std::to_string(b) + ")");
  }
}

}  // namespace

// ---- free functions ---------------------------------------------------------
namespace {

// Device allocations of one synchronous free-function call.
struct Scratch {
  std::vector<void*> ptrs;
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  T* get(size_t n) {
    T* p = dalloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
};

// FusedLayout (fusion.cpp:26-36) + layer tile tables on the device.
struct DevLayout {
  uint64_t d = 0;
  int L = 0, tiles = 0;
  uint64_t* off = nullptr;
  int* tile_layer = nullptr;
  int* tile_start = nullptr;
  DevLayout(const uint64_t* sizes, int n_layers, Scratch& s) : L(n_layers) {
    std::vector<uint64_t> o(static_cast<size_t>(L) + 1, 0);
    std::vector<int> ts(static_cast<size_t>(L) + 1, 0);
    for (int l = 0; l < L; ++l) {
      o[l + 1] = o[l] + sizes[l];
      ts[l + 1] = ts[l] + static_cast<int>((sizes[l] + kTile - 1) / kTile);
    }
    d = o[L];
    tiles = ts[L];
    std::vector<int> tl(static_cast<size_t>(std::max(tiles, 1)), 0);
    for (int l = 0; l < L; ++l)
      for (int t = ts[l]; t < ts[l + 1]; ++t) tl[t] = l;
    off = reinterpret_cast<uint64_t*>(s.get<double>(o.size()));
    tile_start = reinterpret_cast<int*>(s.get<float>(ts.size()));
    tile_layer = reinterpret_cast<int*>(s.get<float>(tl.size()));
    cuda_check(cudaMemcpy(off, o.data(), o.size() * 8, cudaMemcpyHostToDevice), "layout");
    cuda_check(cudaMemcpy(tile_start, ts.data(), ts.size() * 4, cudaMemcpyHostToDevice), "layout");
    cuda_check(cudaMemcpy(tile_layer, tl.data(), tl.size() * 4, cudaMemcpyHostToDevice), "layout");
  }
};

int check_device(int32_t device) {
  int ndev = 0;
  cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (ndev == 0) fail(BL_ERR_CUDA, "no CUDA device");
  check_arg(device >= 0 && device < ndev, "device ordinal out of range");
  return device;
}

void scale_layers(float* fused, const uint64_t* sizes, int32_t n_layers, const double* coeff, int32_t memory,
                  int32_t device, bool remove) {
  check_arg(n_layers >= 1, remove ? "remove_scaling: no layers" : "apply_scaling: no layers");
  DeviceGuard g(check_device(device));
  Scratch s;
  DevLayout lay(sizes, n_layers, s);
  std::vector<float> mul(static_cast<size_t>(n_layers));
  for (int l = 0; l < n_layers; ++l)  // kernels::scale(view, c) / (view, 1.0 / c), fusion.cpp:130-145
    mul[l] = static_cast<float>(remove ? 1.0 / coeff[l] : coeff[l]);
  float* dmul = s.get<float>(mul.size());
  cuda_check(cudaMemcpy(dmul, mul.data(), mul.size() * 4, cudaMemcpyHostToDevice), "scales");
  float* x = fused;
  if (memory == BL_MEM_HOST) {
    x = s.get<float>(lay.d);
    cuda_check(cudaMemcpy(x, fused, lay.d * 4, cudaMemcpyHostToDevice), "fused in");
  }
  launch_scale_layers(x, lay.off, n_layers, dmul, lay.d, nullptr);
  cuda_check(cudaGetLastError(), "scale kernel");
  if (memory == BL_MEM_HOST)
    cuda_check(cudaMemcpy(fused, x, lay.d * 4, cudaMemcpyDeviceToHost), "fused out");
  cuda_check(cudaDeviceSynchronize(), "scaling");
}

}  // namespace

extern "C" {

const char* bl_last_error(void) { return g_err.c_str(); }
int32_t bl_abi_version(void) { return BL_ABI_VERSION; }

bl_status bl_nccl_get_unique_id(uint8_t* out) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id.internal) == BL_NCCL_UNIQUE_ID_BYTES, "unique id size");
    std::memcpy(out, id.internal, BL_NCCL_UNIQUE_ID_BYTES);
  });
}

void bl_hparams_default(bl_hparams* hp) {
  *hp = bl_hparams{};
  hp->beta1 = 0.9;
  hp->beta2 = 0.999;
  hp->beta3 = 0.9;
  hp->eta = 1e-6;
  hp->c_min = 0.01;
  hp->c_max = 0.3;
  hp->r_min = 0.5;
  hp->r_max = 4.0;
  hp->r_threshold = 0.1;
  hp->weight_decay = 0.0;
  hp->division_floor = 1e-12;
}

bl_status bl_cluster_create(const bl_cluster_config* cfg, bl_cluster** out) {
  return guarded([&] {
    *out = nullptr;
    check_arg(cfg->n_workers >= 1, "SimCluster: need at least one worker");
    check_arg(cfg->dim >= 1, "SimCluster: dim must be >= 1");
    check_arg(cfg->baseline_bits_per_element >= 1, "SimCluster: baseline bits must be >= 1");

    if (cfg->n_workers > 64) fail(BL_ERR_UNSUPPORTED, "more than 64 workers");
    if (cfg->mode == BL_MODE_NCCL) {
      check_arg(cfg->rank >= 0 && cfg->rank < cfg->n_workers, "rank out of range");
      check_arg(cfg->nccl_unique_id != nullptr, "NCCL mode needs a unique id");
    }
    int ndev = 0;
    cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (ndev == 0) fail(BL_ERR_CUDA, "no CUDA device");
    check_arg(cfg->device >= 0 && cfg->device < ndev, "device ordinal out of range");
    DeviceGuard g(cfg->device);
    auto* c = new bl_cluster();
    try {
      c->cfg = *cfg;
      c->n = cfg->n_workers;
      c->mode = cfg->mode;
      c->rank = cfg->mode == BL_MODE_NCCL ? cfg->rank : 0;
      c->device = cfg->device;
      c->dim = cfg->dim;
      c->P = (c->dim + c->n - 1) / c->n * c->n;  // comm_sim.cpp:58-59
      c->c = c->P / c->n;
      c->c_pad = round_up(c->c, kTile);
      c->W = c->c_pad / 32;
      c->slot = c->W + 32;
      c->tpc = static_cast<int>(c->c_pad / kTile);
      c->nw = c->mode == BL_MODE_SIM ? c->n : 1;
      c->ns = c->nw;
      c->in_stride = round_up(c->P + kSlack, 64);
      cudaDeviceProp prop;
      cuda_check(cudaGetDeviceProperties(&prop, cfg->device), "cudaGetDeviceProperties");
      c->sms = prop.multiProcessorCount;
      if (cfg->stream) {
        c->stream = static_cast<cudaStream_t>(cfg->stream);
      } else {
        cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        c->own_stream = true;
      }
      const size_t nw = static_cast<size_t>(c->nw), n = static_cast<size_t>(c->n);
      c->in = dalloc<float>(nw * c->in_stride);
      c->werr = dalloc<float>(nw * n * c->c_pad + 256);
      c->wpk[0] = dalloc<uint32_t>(nw * n * c->slot);
      c->wpk[1] = dalloc<uint32_t>(nw * n * c->slot);
      c->serr = dalloc<float>(static_cast<size_t>(c->ns) * c->c_pad + 256);
      c->res_base = dalloc<uint32_t>(2 * n * c->slot);
      c->res[0] = c->res_base;
      c->res[1] = c->res_base + n * c->slot;
      c->wpart = dalloc<double>(nw * n * c->tpc);
      c->spart = dalloc<double>(static_cast<size_t>(c->ns) * c->tpc);
      c->out = dalloc<float>(c->P + kSlack);
      c->err = reinterpret_cast<unsigned long long*>(dalloc<double>(kErrWords));
      c->tile_ctr = reinterpret_cast<unsigned int*>(dalloc<float>(4));
      cuda_check(cudaMemset(c->err, 0xFF, kErrSlots * sizeof(unsigned long long)), "err init");
      c->set_peer_timeout(c->peer_timeout_ms);
      if (cfg->endpoint_stats) {
        c->wcmax = dalloc<float>(nw * n * c->tpc);
        c->scmax = dalloc<float>(static_cast<size_t>(c->ns) * c->tpc);
        c->stat_tiles = static_cast<int>((c->P + kTile - 1) / kTile);
        c->stat_part = dalloc<double>(c->stat_tiles);
        c->stat_max = dalloc<float>(c->stat_tiles);
        c->stats_dev = dalloc<double>(5 * 2 * static_cast<size_t>(c->n));
      }
      {  // API-mode K1 boundary tiles: not full, or reaching into the padding
        std::vector<int> slow;
        for (int j = 0; j < c->n; ++j)
          for (int t = 0; t < c->tpc; ++t) {
            const uint64_t i0 = static_cast<uint64_t>(t) * kTile;
            if (i0 + kTile > c->c || static_cast<uint64_t>(j) * c->c + i0 + kTile > c->dim)
              slow.push_back(j * c->tpc + t);
          }
        c->k1_n_slow = static_cast<int>(slow.size());
        c->k1_slow = reinterpret_cast<int*>(dalloc<float>(slow.size()));
        if (!slow.empty())
          cuda_check(cudaMemcpy(c->k1_slow, slow.data(), slow.size() * 4, cudaMemcpyHostToDevice),
                     "k1 slow tiles");
        c->k1_order = bl::boundary_first_order(slow, c->nw, c->n * c->tpc);
      }
      if (c->mode == BL_MODE_NCCL) {
        c->rpk = dalloc<uint32_t>(n * c->slot);
        ncclUniqueId id;
        std::memcpy(id.internal, cfg->nccl_unique_id, BL_NCCL_UNIQUE_ID_BYTES);
        nccl_check(ncclCommInitRank(&c->comm, c->n, id, c->rank), "ncclCommInitRank");
        if (c->n > 1 && cfg->transport != BL_TRANSPORT_NCCL) {
          c->setup_p2p(cfg->transport == BL_TRANSPORT_P2P);
        }
      }
      cuda_check(cudaDeviceSynchronize(), "cluster init");
    } catch (...) {
      bl_cluster_destroy(c);
      throw;
    }
    *out = c;
  });
}

void bl_cluster_destroy(bl_cluster* c) {
  if (!c) return;
  DeviceGuard g(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (bl_optimizer* o : c->opts) o->cl = nullptr;  // orphaned: their destroy only frees memory
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->comm) ncclCommDestroy(c->comm);
  void* bufs[] = {c->in,        c->werr,       c->wpk[0],          c->wpk[1],    c->rpk,
                  c->serr,      c->res_base,   c->wpart,           c->spart,     c->wcmax,
                  c->scmax,     c->out,        c->lrecv,           c->err,       c->stat_part,
                  c->stat_max,  c->stats_dev,   c->rx,              c->flags,     c->d_peer_rx,
                  c->d_peer_res, c->d_peer_flags, c->d_peer_in, c->d_peer_out, c->d_peer_err,
                  c->lossless_done, c->small_bar, c->k1_slow, c->k1_order, c->tile_ctr,
                  c->piece_done,    c->gate_status, c->ll_rx, c->ll_res, c->d_peer_llrx,
                  c->d_peer_llres,  c->small_ts};
  for (void* p : bufs)
    if (p) cudaFree(p);
  for (auto& e : c->pending) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->copy_stream) {
    for (auto e : c->piece_ev) cudaEventDestroy(e);
    cudaStreamDestroy(c->copy_stream);
  }
  if (c->comm_stream) {
    cudaStreamSynchronize(c->comm_stream);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
    cudaStreamDestroy(c->comm_stream);
  }
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int32_t bl_cluster_transport(const bl_cluster* c) { return c ? c->transport : BL_TRANSPORT_NCCL; }
void* bl_cluster_stream(const bl_cluster* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

bl_status bl_cluster_get_config(const bl_cluster* c, bl_cluster_config* outp) {
  return guarded([&] {
    *outp = c->cfg;
    outp->transport = c->mode == BL_MODE_NCCL ? c->transport : c->cfg.transport;
    outp->stream = c->stream;
  });
}

uint64_t bl_cluster_step_count(const bl_cluster* c) {
  return c ? c->ledger.compressed_collectives + c->ledger.lossless_collectives : 0;
}

bl_status bl_cluster_set_peer_timeout(bl_cluster* c, double ms) {
  return guarded([&] {
    check_arg(ms > 0.0, "peer timeout must be > 0 ms");
    DeviceGuard g(c->device);
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    c->set_peer_timeout(ms);
  });
}

bl_status bl_cluster_dims(const bl_cluster* c, uint64_t* padded, uint64_t* chunk) {
  return guarded([&] {
    if (padded) *padded = c->P;
    if (chunk) *chunk = c->c;
  });
}

bl_status bl_cluster_compressed_allreduce(bl_cluster* c, const float* const* inputs,
                                          int32_t n_inputs, uint64_t len, float* outp,
                                          double error_scale, int32_t memory) {
  return guarded([&] {
    DeviceGuard g(c->device);
    size_check(static_cast<uint64_t>(n_inputs), static_cast<uint64_t>(c->nw),
               "compressed_allreduce: worker count");
    size_check(len, c->dim, "compressed_allreduce: input length");
    c->ensure_usable();
    c->copy_inputs(inputs, n_inputs, len, memory);
    c->begin_step(nullptr, 0, false, false);
    if (c->cfg.compressor == BL_COMPRESSOR_IDENTITY) {
      // Identity compressor: lossless messages, residuals stay zero
      // (compression.cpp:184-188), result = ascending-worker average.
      c->lossless(false);
      c->ledger_compressed();
      c->last_identity = true;
      if (c->cfg.verify_compensation && error_scale == 1.0)  // v + 0 == v + 0 exactly
        c->checks += static_cast<uint64_t>(c->nw) * c->n + static_cast<uint64_t>(c->ns);
    } else {
      if (!c->compressed(nullptr, 0, static_cast<float>(error_scale), nullptr, c->out)) {
        const int latest = static_cast<int>((c->calls + 1u) & 1u);
        cudaEvent_t a;
        c->begin(KC_DEC, &a);
        c->end(KC_DEC, a, launch_decompress(c->res[latest], c->n, c->c, c->slot, c->W, c->dim, c->out,
                                            c->err, c->stream));
      }
    }
    c->pending_is_step = false;
    if (outp) {
      cuda_check(cudaMemcpyAsync(outp, c->out, c->dim * sizeof(float), cudaMemcpyDefault, c->stream),
                 "result copy");
      if (memory == BL_MEM_HOST) c->sync_and_check(nullptr);
    }
  });
}

bl_status bl_cluster_lossless_allreduce(bl_cluster* c, const float* const* inputs, int32_t n_inputs,
                                        uint64_t len, float* outp, int32_t memory) {
  return guarded([&] {
    DeviceGuard g(c->device);
    size_check(static_cast<uint64_t>(n_inputs), static_cast<uint64_t>(c->nw),
               "lossless_allreduce: worker count");
    size_check(len, c->dim, "lossless_allreduce: input length");
    c->ensure_usable();
    c->copy_inputs(inputs, n_inputs, len, memory);
    c->begin_step(nullptr, 0, false, false);
    c->lossless(false);
    c->ledger_lossless();
    if (outp) {
      cuda_check(cudaMemcpyAsync(outp, c->out, c->dim * sizeof(float), cudaMemcpyDefault, c->stream),
                 "result copy");
      if (memory == BL_MEM_HOST) c->sync_and_check(nullptr);
    }
  });
}

static void local_index(const bl_cluster* c, int32_t i, const char* what) {
  if (i < 0 || i >= c->n) fail(BL_ERR_INVALID_ARGUMENT, std::string(what) + ": index out of range");
  if (c->mode == BL_MODE_NCCL && i != c->rank) {
    fail(BL_ERR_INVALID_ARGUMENT, std::string(what) + ": only the local rank's endpoint lives here");
  }
}

bl_status bl_cluster_worker_error(bl_cluster* c, int32_t i, float* outp) {
  return guarded([&] {
    DeviceGuard g(c->device);
    local_index(c, i, "worker_error");
    const int w = c->mode == BL_MODE_SIM ? i : 0;
    c->sync_and_check(nullptr);
    if (c->last_identity || c->calls == 0) {
      std::memset(outp, 0, c->P * sizeof(float));
      return;
    }
    const int latest = static_cast<int>((c->calls + 1u) & 1u);
    float* tmp = c->out;  // scratch: P floats
    cudaEvent_t a;
    c->begin(KC_MAT, &a);
    c->end(KC_MAT, a,
           launch_materialize_error(c->werr + static_cast<size_t>(w) * c->n * c->c_pad, c->c_pad,
                                    c->wpk[latest] + static_cast<size_t>(w) * c->n * c->slot,
                                    c->slot, c->W, c->c, c->P, tmp, c->stream));
    cuda_check(cudaMemcpyAsync(outp, tmp, c->P * sizeof(float), cudaMemcpyDeviceToHost, c->stream),
               "worker_error copy");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
}

bl_status bl_cluster_server_error(bl_cluster* c, int32_t j, float* outp) {
  return guarded([&] {
    DeviceGuard g(c->device);
    local_index(c, j, "server_error");
    const int s = c->mode == BL_MODE_SIM ? j : 0;
    c->sync_and_check(nullptr);
    if (c->last_identity || c->calls == 0) {
      std::memset(outp, 0, c->c * sizeof(float));
      return;
    }
    const int latest = static_cast<int>((c->calls + 1u) & 1u);
    float* tmp = c->out;
    cudaEvent_t a;
    c->begin(KC_MAT, &a);
    c->end(KC_MAT, a,
           launch_materialize_error(c->serr + static_cast<size_t>(s) * c->c_pad, c->c_pad,
                                    c->res[latest] + static_cast<size_t>(j) * c->slot, c->slot, c->W,
                                    c->c, c->c, tmp, c->stream));
    cuda_check(cudaMemcpyAsync(outp, tmp, c->c * sizeof(float), cudaMemcpyDeviceToHost, c->stream),
               "server_error copy");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
  });
}

static void packet_bytes(bl_cluster* c, const uint32_t* slot_ptr, uint8_t* bytes) {
  const size_t nb = (c->c + 7) / 8;
  std::vector<uint32_t> words(c->W + 1);
  cuda_check(cudaMemcpyAsync(words.data(), slot_ptr, (c->W + 1) * 4, cudaMemcpyDeviceToHost,
                             c->stream),
             "packet copy");
  cuda_check(cudaStreamSynchronize(c->stream), "sync");
  std::memcpy(bytes, words.data(), nb);  // LE words == LSB-first bytes
  std::memcpy(bytes + nb, &words[c->W], 4);
}

bl_status bl_cluster_packet(bl_cluster* c, int32_t worker, int32_t server, uint8_t* bytes) {
  return guarded([&] {
    DeviceGuard g(c->device);
    local_index(c, worker, "packet");
    if (server < 0 || server >= c->n) fail(BL_ERR_INVALID_ARGUMENT, "packet: server out of range");
    if (c->last_identity) fail(BL_ERR_LOGIC, "identity packet");
    const int w = c->mode == BL_MODE_SIM ? worker : 0;
    const int latest = static_cast<int>((c->calls + 1u) & 1u);
    packet_bytes(c, c->wpk[latest] + (static_cast<size_t>(w) * c->n + server) * c->slot, bytes);
  });
}

bl_status bl_cluster_server_packet(bl_cluster* c, int32_t server, uint8_t* bytes) {
  return guarded([&] {
    DeviceGuard g(c->device);
    if (server < 0 || server >= c->n) fail(BL_ERR_INVALID_ARGUMENT, "packet: server out of range");
    if (c->last_identity) fail(BL_ERR_LOGIC, "identity packet");
    const int latest = static_cast<int>((c->calls + 1u) & 1u);
    packet_bytes(c, c->res[latest] + static_cast<size_t>(server) * c->slot, bytes);
  });
}

bl_status bl_cluster_ledger(const bl_cluster* c, bl_volume_ledger* outp) {
  return guarded([&] { *outp = c->ledger; });
}

bl_status bl_cluster_stats(bl_cluster* c, bl_endpoint_stats* outp) {
  return guarded([&] {
    if (!c->cfg.endpoint_stats) fail(BL_ERR_LOGIC, "endpoint statistics are disabled in the config");
    DeviceGuard g(c->device);
    c->sync_and_check(nullptr);
    static_assert(sizeof(bl_endpoint_stats) == 5 * sizeof(double), "EndpointStats layout");
    cuda_check(cudaMemcpy(outp, c->stats_dev, 2 * static_cast<size_t>(c->n) * sizeof(bl_endpoint_stats),
                          cudaMemcpyDeviceToHost),
               "stats");
  });
}

bl_status bl_cluster_synchronize(bl_cluster* c) {
  return guarded([&] {
    DeviceGuard g(c->device);
    c->sync_and_check(nullptr);
  });
}

float* bl_cluster_input_buffer(bl_cluster* c, int32_t worker) {
  if (!c || worker < 0 || worker >= c->nw) return nullptr;
  return c->in + static_cast<size_t>(worker) * c->in_stride;
}

uint64_t bl_cluster_kernel_launches(const bl_cluster* c) { return c ? c->launches : 0; }
uint64_t bl_cluster_compensation_checks(const bl_cluster* c) { return c ? c->checks : 0; }

bl_status bl_cluster_set_profiling(bl_cluster* c, int32_t on) {
  return guarded([&] {
    c->profiling = on != 0;
    for (int k = 0; k < KC_COUNT; ++k) {
      c->prof_ms[k] = 0.0;
      c->prof_n[k] = 0;
    }
  });
}

int32_t bl_cluster_profile(bl_cluster* c, const char** names, double* total_ms, uint64_t* launches,
                           int32_t cap) {
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& e : c->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    c->prof_ms[e.cls] += ms;
    c->prof_n[e.cls] += 1;
    c->ev_pool.push_back(e.a);
    c->ev_pool.push_back(e.b);
  }
  c->pending.clear();
  int k = 0;
  for (int cls = 0; cls < KC_COUNT && k < cap; ++cls) {
    if (c->prof_n[cls] == 0) continue;
    names[k] = kClassNames[cls];
    total_ms[k] = c->prof_ms[cls];
    launches[k] = c->prof_n[cls];
    ++k;
  }
  return k;
}

bl_status bl_volume_reduction(double w, double bb, double cb, double* outp) {
  return guarded([&] {  // comm_sim.cpp:36-48
    check_arg(w >= 0.0 && w <= 1.0, "volume_reduction: warmup_ratio must be in [0, 1]");
    check_arg(bb > 0.0, "volume_reduction: baseline_bits must be > 0");
    check_arg(cb >= 0.0, "volume_reduction: compressed bits must be >= 0");
    const double denom = w + (1.0 - w) * cb / bb;
    *outp = denom == 0.0 ? INFINITY : 1.0 / denom;
  });
}

// HyperParams::validate, optimizers.cpp:60-74
static void validate(const bl_hparams* h) {
  auto reject = [](const char* m) { fail(BL_ERR_CONFIG, m); };
  if (!(h->beta1 >= 0.0 && h->beta1 < 1.0)) reject("beta1 must be in [0, 1)");
  if (!(h->beta2 >= 0.0 && h->beta2 < 1.0)) reject("beta2 must be in [0, 1)");
  if (!(h->beta3 >= 0.0 && h->beta3 < 1.0)) reject("beta3 must be in [0, 1)");
  if (!(h->eta > 0.0)) reject("eta must be > 0");
  if (!(h->c_min <= h->c_max)) reject("c_min must not exceed c_max");
  if (!(h->r_min <= h->r_max)) reject("r_min must not exceed r_max");
  if (!(h->r_threshold > 0.0 && h->r_threshold < 1.0)) reject("r_threshold must be in (0, 1)");
  if (!(h->weight_decay >= 0.0)) reject("weight_decay must be >= 0");
  if (!(h->division_floor > 0.0)) reject("division_floor must be > 0");
  if (h->warmup_steps > h->total_steps) reject("warmup_steps must not exceed total_steps");
}

static bl_status optimizer_create(int32_t variant, const uint64_t* sizes, const char* const* names,
                                  int32_t n_layers, const bl_hparams* hp, bl_cluster* cl,
                                  bl_optimizer** out) {
  return guarded([&] {
    *out = nullptr;
    validate(hp);
    check_arg(n_layers >= 1, "Optimizer: need at least one layer");
    for (int l = 0; l < n_layers; ++l) check_arg(sizes[l] > 0, "Optimizer: layer size must be > 0");
    check_arg(variant >= BL_LAMB && variant <= BL_ONEBIT_ADAM, "unknown optimizer variant");
    check_arg(cl != nullptr, "Optimizer: needs the cluster whose device and stream it uses");
    DeviceGuard g(cl->device);
    auto* o = new bl_optimizer();
    try {
      o->variant = variant;
      o->L = n_layers;
      o->hp = *hp;
      o->cl = cl;
      o->names.resize(static_cast<size_t>(n_layers));
      for (int l = 0; l < n_layers; ++l)
        o->names[l] = names && names[l] ? std::string(names[l]) : "layer" + std::to_string(l);
      o->off.assign(static_cast<size_t>(n_layers) + 1, 0);
      std::vector<int> tstart(static_cast<size_t>(n_layers) + 1, 0);
      for (int l = 0; l < n_layers; ++l) {
        o->off[l + 1] = o->off[l] + sizes[l];
        tstart[l + 1] = tstart[l] + static_cast<int>((sizes[l] + kTile - 1) / kTile);
      }
      o->d = o->off[n_layers];
      if (o->d != cl->dim) {
        fail(BL_ERR_DIMENSION, "Optimizer: fused dim " + std::to_string(o->d) +
                                   " does not match the cluster dim " + std::to_string(cl->dim));
      }
      o->tiles = tstart[n_layers];
      std::vector<int> tl(static_cast<size_t>(o->tiles));
      for (int l = 0; l < n_layers; ++l)
        for (int t = tstart[l]; t < tstart[l + 1]; ++t) tl[t] = l;
      const size_t L = static_cast<size_t>(n_layers);
      o->off_dev = reinterpret_cast<uint64_t*>(dalloc<double>(L + 1));
      o->tile_layer = reinterpret_cast<int*>(dalloc<float>(tl.size()));
      o->layer_tile_start = reinterpret_cast<int*>(dalloc<float>(L + 1));
      cuda_check(cudaMemcpy(o->off_dev, o->off.data(), (L + 1) * 8, cudaMemcpyHostToDevice), "off");
      cuda_check(cudaMemcpy(o->tile_layer, tl.data(), tl.size() * 4, cudaMemcpyHostToDevice), "tiles");
      o->lt_start_h = tstart;
      cuda_check(cudaMemcpy(o->layer_tile_start, tstart.data(), (L + 1) * 4, cudaMemcpyHostToDevice),
                 "tile start");
      const size_t dn = o->d + kSlack;
      o->x = dalloc<float>(dn);
      o->m = dalloc<float>(dn);
      o->v = dalloc<float>(dn);
      o->vf = dalloc<float>(dn);
      o->c_avg = dalloc<double>(L);
      o->r_prev = dalloc<double>(L);
      o->coeff = dalloc<double>(L);
      o->mag = dalloc<double>(L);
      o->A = dalloc<float>(L);
      o->B = dalloc<float>(L);
      o->invc = dalloc<float>(L);
      o->coef_x = dalloc<float>(L);
      o->trace = dalloc<double>(4 * L);
      o->cmean = dalloc<double>(2);
      o->es = dalloc<float>(1);
      o->counter = reinterpret_cast<unsigned int*>(dalloc<float>(1));
      o->tile_sums = dalloc<double>(4 * static_cast<size_t>(o->tiles));
      {  // K1 tiles (chunk-relative) that are full and inside one layer
        std::vector<int> k1l(static_cast<size_t>(cl->n) * cl->tpc, -1);
        for (int j = 0; j < cl->n; ++j) {
          for (int t = 0; t < cl->tpc; ++t) {
            const uint64_t i0 = static_cast<uint64_t>(t) * kTile, k0 = static_cast<uint64_t>(j) * cl->c + i0;
            if (i0 + kTile > cl->c || k0 + kTile > o->d) continue;
            const auto it = std::upper_bound(o->off.begin(), o->off.end(), k0);
            const int l = static_cast<int>(it - o->off.begin()) - 1;
            if (k0 + kTile - 1 < o->off[l + 1]) k1l[static_cast<size_t>(j) * cl->tpc + t] = l;
          }
        }
        o->k1_tile_layer = reinterpret_cast<int*>(dalloc<float>(k1l.size()));
        cuda_check(cudaMemcpy(o->k1_tile_layer, k1l.data(), k1l.size() * 4, cudaMemcpyHostToDevice),
                   "k1 tiles");
        std::vector<int> slow;
        for (size_t k = 0; k < k1l.size(); ++k)
          if (k1l[k] < 0) slow.push_back(static_cast<int>(k));
        o->k1_n_slow = static_cast<int>(slow.size());
        o->k1_slow = reinterpret_cast<int*>(dalloc<float>(slow.size()));
        if (!slow.empty())
          cuda_check(cudaMemcpy(o->k1_slow, slow.data(), slow.size() * 4, cudaMemcpyHostToDevice),
                     "k1 slow tiles");
        o->k1_order = bl::boundary_first_order(slow, cl->nw, cl->n * cl->tpc);
      }
      o->tile_max = dalloc<float>(static_cast<size_t>(o->tiles));
      {  // processing order of the layer-tiled kernels: boundary tiles (the
         // per-row general path: misaligned layer start, partial tile, or a
         // result-chunk boundary inside the tile) first, so their longer
         // latency overlaps the bulk instead of forming the kernel's tail
        // A layer of at least one full tile that starts off a 16-byte
        // boundary selects the kernels' misaligned full-tile path (LayerTiles::mis).
        for (int l = 0; l < n_layers; ++l)
          if ((o->off[l] & 3u) != 0 && o->off[l + 1] - o->off[l] >= kTile) o->mis_layers = true;
        std::vector<int> order, fast;
        for (int l = 0; l < n_layers; ++l) {
          const uint64_t lo = o->off[l], len = o->off[l + 1] - lo;
          for (int t = tstart[l]; t < tstart[l + 1]; ++t) {
            const uint64_t i = static_cast<uint64_t>(t - tstart[l]) * kTile, base = lo + i;
            const bool f = ((lo & 3u) == 0 || o->mis_layers) && i + kTile <= len &&
                           base / cl->c == (base + kTile - 1) / cl->c;
            (f ? fast : order).push_back(t);
          }
        }
        order.insert(order.end(), fast.begin(), fast.end());
        o->tile_order_h = order;
        o->tile_order = reinterpret_cast<int*>(dalloc<float>(order.size()));
        cuda_check(cudaMemcpy(o->tile_order, order.data(), order.size() * 4, cudaMemcpyHostToDevice),
                   "tile order");
      }
      std::vector<double> ones(L, 1.0);
      std::vector<float> onesf(L, 1.0f);
      cuda_check(cudaMemcpy(o->r_prev, ones.data(), L * 8, cudaMemcpyHostToDevice), "r_prev");
      cuda_check(cudaMemcpy(o->coeff, ones.data(), L * 8, cudaMemcpyHostToDevice), "coeff");
      cuda_check(cudaMemcpy(o->invc, onesf.data(), L * 4, cudaMemcpyHostToDevice), "invc");
      cuda_check(cudaMemcpy(o->cmean, ones.data(), 2 * 8, cudaMemcpyHostToDevice), "cmean");
      cuda_check(cudaMemcpy(o->es, onesf.data(), 4, cudaMemcpyHostToDevice), "es");
    } catch (...) {
      bl_optimizer_destroy(o);
      throw;
    }
    cl->opts.push_back(o);
    *out = o;
  });
}

bl_status bl_optimizer_create(int32_t variant, const uint64_t* sizes, int32_t n_layers,
                              const bl_hparams* hp, bl_cluster* cl, bl_optimizer** out) {
  return optimizer_create(variant, sizes, nullptr, n_layers, hp, cl, out);
}

bl_status bl_optimizer_create_named(int32_t variant, const bl_layer_spec* layers, int32_t n_layers,
                                    const bl_hparams* hp, bl_cluster* cl, bl_optimizer** out) {
  std::vector<uint64_t> sizes(static_cast<size_t>(std::max(n_layers, 0)));
  std::vector<const char*> names(sizes.size());
  for (size_t l = 0; l < sizes.size(); ++l) {
    sizes[l] = layers[l].size;
    names[l] = layers[l].name;
  }
  return optimizer_create(variant, sizes.data(), names.data(), n_layers, hp, cl, out);
}

const char* bl_optimizer_layer_name(const bl_optimizer* o, int32_t layer) {
  if (!o || layer < 0 || layer >= o->L) return nullptr;
  return o->names[static_cast<size_t>(layer)].c_str();
}

bl_status bl_optimizer_set_strict(bl_optimizer* o, int32_t on) {
  return guarded([&] { o->strict = on != 0; });
}

void bl_optimizer_destroy(bl_optimizer* o) {
  if (!o) return;
  if (bl_cluster* c = o->cl) {  // null when the cluster was destroyed first
    DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->last_opt == o) c->last_opt = nullptr;
    for (auto& sn : c->snaps)
      if (sn.opt == o) sn.opt = nullptr;
    c->opts.erase(std::remove(c->opts.begin(), c->opts.end(), o), c->opts.end());
  }
  void* bufs[] = {o->off_dev, o->tile_layer, o->layer_tile_start, o->x, o->m, o->v, o->vf,
                  o->mprev, o->c_avg, o->r_prev, o->coeff, o->mag, o->A, o->B, o->invc, o->coef_x,
                  o->trace, o->cmean, o->es, o->counter, o->tile_sums, o->tile_max,
                  o->k1_tile_layer, o->k1_slow, o->k1_order, o->tile_order,
                  o->w1_order, o->w2_order, o->lw_order, o->lr_dev};
  for (void* p : bufs)
    if (p) cudaFree(p);
  for (void* p : o->shard_ipc) cudaIpcCloseMemHandle(p);
  if (o->gen_tiles) cudaFree(o->gen_tiles);
  void* push_bufs[] = {o->stg, o->e_all_dev, o->d_peer_stg};
  for (void* p : push_bufs)
    if (p) cudaFree(p);
  void* shard_bufs[] = {o->own_order, o->own_w1_order, o->own_w2_order, o->own_lw_order, o->push_x, o->push_m, o->push_v, o->push_vf, o->push_sums};
  for (void* p : shard_bufs)
    if (p) cudaFree(p);
  for (auto& gx : o->graph)
    if (gx) cudaGraphExecDestroy(gx);
  if (o->lr_host) cudaFreeHost(o->lr_host);
  delete o;
}

bl_status bl_optimizer_step(bl_optimizer* o, bl_cluster* c, const float* const* grads,
                            int32_t n_grads, uint64_t t, double lr, int32_t memory,
                            bl_step_trace* trace) {
  return guarded([&] {
    if (!o->cl) fail(BL_ERR_LOGIC, "step: the optimizer's cluster was destroyed");
    if (c != o->cl) fail(BL_ERR_LOGIC, "step: optimizer is bound to a different cluster");
    DeviceGuard g(c->device);
    o->step(grads, n_grads, t, lr, memory, trace);
  });
}

float* bl_optimizer_grad_buffer(bl_optimizer* o, int32_t worker) {
  return bl_cluster_input_buffer(o ? o->cl : nullptr, worker);
}

bl_status bl_optimizer_get_state(bl_optimizer* o, int32_t which, float* host_out) {
  return guarded([&] {
    if (!o->cl) fail(BL_ERR_LOGIC, "the optimizer's cluster was destroyed");
    DeviceGuard g(o->cl->device);
    o->cl->sync_and_check(o);
    if (which == BL_STATE_M || which == BL_STATE_V) o->sync_shards();  // collective while sharded
    const float* src = nullptr;
    switch (which) {
      case BL_STATE_X: src = o->x; break;
      case BL_STATE_V: src = o->v; break;
      case BL_STATE_V_FROZEN:
        if (!o->has_vf) {
          std::memset(host_out, 0, o->d * sizeof(float));
          return;
        }
        src = o->vf;
        break;
      case BL_STATE_M:
      case BL_STATE_M_PREV:
        if (which == BL_STATE_M_PREV && !o->has_mprev) {
          std::memset(host_out, 0, o->d * sizeof(float));
          return;
        }
        if (which == BL_STATE_M_PREV && o->mprev_separate) {
          src = o->mprev;
        } else if (o->m_valid) {
          src = o->m;
        } else {
          o->materialize_m(o->cl->out);
          src = o->cl->out;
        }
        break;
      default: fail(BL_ERR_INVALID_ARGUMENT, "unknown state buffer");
    }
    cuda_check(cudaMemcpyAsync(host_out, src, o->d * sizeof(float), cudaMemcpyDeviceToHost,
                               o->cl->stream),
               "state copy");
    cuda_check(cudaStreamSynchronize(o->cl->stream), "sync");
  });
}

bl_status bl_optimizer_set_state(bl_optimizer* o, int32_t which, const float* host_in) {
  return guarded([&] {
    if (!o->cl) fail(BL_ERR_LOGIC, "the optimizer's cluster was destroyed");
    DeviceGuard g(o->cl->device);
    o->cl->sync_and_check(o);
    float* dst = nullptr;
    switch (which) {
      case BL_STATE_X: dst = o->x; break;
      case BL_STATE_V: dst = o->v; break;
      case BL_STATE_V_FROZEN:
        dst = o->vf;
        o->has_vf = true;
        break;
      case BL_STATE_M:
        if (!o->m_valid && o->has_mprev && !o->mprev_separate) {
          // m_prev keeps the value m had: materialise it before m changes.
          if (!o->mprev) o->mprev = dalloc<float>(o->d + kSlack);
          o->materialize_m(o->mprev);
          o->mprev_separate = true;
        }
        dst = o->m;
        o->m_valid = true;
        break;
      case BL_STATE_M_PREV:
        if (!o->mprev) o->mprev = dalloc<float>(o->d + kSlack);
        dst = o->mprev;
        o->mprev_separate = true;
        o->has_mprev = true;
        if (!o->m_valid) {
          o->materialize_m(o->m);
          o->m_valid = true;
        }
        break;
      default: fail(BL_ERR_INVALID_ARGUMENT, "unknown state buffer");
    }
    cuda_check(cudaMemcpyAsync(dst, host_in, o->d * sizeof(float), cudaMemcpyHostToDevice,
                               o->cl->stream),
               "state copy");
    cuda_check(cudaStreamSynchronize(o->cl->stream), "sync");
  });
}

bl_status bl_optimizer_get_scalars(bl_optimizer* o, double* c_avg, double* r_prev, double* coeff) {
  return guarded([&] {
    if (!o->cl) fail(BL_ERR_LOGIC, "the optimizer's cluster was destroyed");
    DeviceGuard g(o->cl->device);
    o->cl->sync_and_check(o);
    const size_t L = static_cast<size_t>(o->L);
    if (c_avg) cuda_check(cudaMemcpy(c_avg, o->c_avg, L * 8, cudaMemcpyDeviceToHost), "c_avg");
    if (r_prev) cuda_check(cudaMemcpy(r_prev, o->r_prev, L * 8, cudaMemcpyDeviceToHost), "r_prev");
    if (coeff) cuda_check(cudaMemcpy(coeff, o->coeff, L * 8, cudaMemcpyDeviceToHost), "coeff");
  });
}

bl_status bl_optimizer_set_scalars(bl_optimizer* o, const double* c_avg, const double* r_prev) {
  return guarded([&] {
    if (!o->cl) fail(BL_ERR_LOGIC, "the optimizer's cluster was destroyed");
    DeviceGuard g(o->cl->device);
    o->cl->sync_and_check(o);
    const size_t L = static_cast<size_t>(o->L);
    if (c_avg) cuda_check(cudaMemcpy(o->c_avg, c_avg, L * 8, cudaMemcpyHostToDevice), "c_avg");
    if (r_prev) cuda_check(cudaMemcpy(o->r_prev, r_prev, L * 8, cudaMemcpyHostToDevice), "r_prev");
  });
}

int32_t bl_optimizer_frozen(const bl_optimizer* o) { return o && o->frozen ? 1 : 0; }
uint64_t bl_optimizer_fused_dim(const bl_optimizer* o) { return o ? o->d : 0; }
int32_t bl_optimizer_layer_count(const bl_optimizer* o) { return o ? o->L : 0; }


bl_status bl_compute_scales(const float* m, const uint64_t* sizes, int32_t n_layers, double floor_,
                            double* coeff_out, double* reference_out, int32_t memory, int32_t device) {
  return guarded([&] {
    check_arg(n_layers >= 1, "compute_scales: no layers");  // fusion.cpp:109-110
    check_arg(floor_ > 0.0, "compute_scales: floor must be positive");
    DeviceGuard g(check_device(device));
    Scratch s;
    DevLayout lay(sizes, n_layers, s);
    const float* x = m;
    if (memory == BL_MEM_HOST) {
      float* t = s.get<float>(lay.d);
      cuda_check(cudaMemcpy(t, m, lay.d * 4, cudaMemcpyHostToDevice), "momentum in");
      x = t;
    }
    double* part = s.get<double>(static_cast<size_t>(std::max(lay.tiles, 1)));
    double* mag = s.get<double>(static_cast<size_t>(n_layers));
    double* coeff = s.get<double>(static_cast<size_t>(n_layers));
    double* ref = s.get<double>(1);
    unsigned int* counter = reinterpret_cast<unsigned int*>(s.get<float>(1));
    if (lay.tiles > 0) launch_layer_abs_tiles(x, lay.off, lay.tile_layer, lay.tile_start, lay.tiles, part, nullptr);
    launch_scales_final(n_layers, lay.tile_start, lay.off, part, floor_, mag, coeff, ref, counter, nullptr);
    cuda_check(cudaGetLastError(), "compute_scales kernels");
    if (coeff_out)
      cuda_check(cudaMemcpy(coeff_out, coeff, static_cast<size_t>(n_layers) * 8, cudaMemcpyDeviceToHost),
                 "coeff");
    if (reference_out) cuda_check(cudaMemcpy(reference_out, ref, 8, cudaMemcpyDeviceToHost), "reference");
    cuda_check(cudaDeviceSynchronize(), "compute_scales");
  });
}

bl_status bl_apply_scaling(float* fused, const uint64_t* sizes, int32_t n_layers, const double* coeff,
                           int32_t memory, int32_t device) {
  return guarded([&] { scale_layers(fused, sizes, n_layers, coeff, memory, device, false); });
}

bl_status bl_remove_scaling(float* fused, const uint64_t* sizes, int32_t n_layers, const double* coeff,
                            int32_t memory, int32_t device) {
  return guarded([&] { scale_layers(fused, sizes, n_layers, coeff, memory, device, true); });
}

bl_status bl_compress_with_feedback(const float* v, float* delta, uint64_t len, int32_t compressor,
                                    double error_scale, uint8_t* wire, float* dec, int32_t memory,
                                    int32_t device) {
  return guarded([&] {
    check_arg(compressor == BL_COMPRESSOR_ONEBIT || compressor == BL_COMPRESSOR_IDENTITY,
              "compress_with_feedback: unknown compressor");
    check_device(device);
    if (len == 0) {  // empty block: no sign bytes, scale 0 (compression.cpp:54)
      if (wire && compressor == BL_COMPRESSOR_ONEBIT) std::memset(wire, 0, 4);
      return;
    }
    // One endpoint of a one-worker cluster is exactly this function: its
    // residual slot holds delta (deferred form with a zero previous scale,
    // so delta = raw - (+-0) = raw), K1 compresses v + es*delta.
    bl_cluster_config cfg{};
    cfg.n_workers = 1;
    cfg.mode = BL_MODE_SIM;
    cfg.device = device;
    cfg.dim = len;
    cfg.compressor = BL_COMPRESSOR_ONEBIT;
    cfg.baseline_bits_per_element = 16;
    cfg.compensation_tolerance = 1e-12;
    bl_cluster* cp = nullptr;
    if (bl_cluster_create(&cfg, &cp) != BL_OK) fail(BL_ERR_CUDA, g_err);
    std::unique_ptr<bl_cluster, void (*)(bl_cluster*)> own(cp, bl_cluster_destroy);
    bl_cluster* c = cp;
    DeviceGuard g(device);
    const size_t bytes = len * sizeof(float);
    cuda_check(cudaMemcpy(c->werr, delta, bytes, cudaMemcpyDefault), "delta in");
    if (compressor == BL_COMPRESSOR_IDENTITY) {
      // corrected = 1*v + es*delta (compression.cpp:181) is the message; delta = 0 (:184-188)
      std::vector<uint64_t> off = {0, len};
      const float ab[2] = {1.0f, static_cast<float>(error_scale)};
      Scratch s;
      uint64_t* doff = reinterpret_cast<uint64_t*>(s.get<double>(2));
      float* dab = s.get<float>(2);
      cuda_check(cudaMemcpy(doff, off.data(), 16, cudaMemcpyHostToDevice), "off");
      cuda_check(cudaMemcpy(dab, ab, 8, cudaMemcpyHostToDevice), "ab");
      // in = A*m + B*in with m = v, in = delta: 1*v + es*delta
      cuda_check(cudaMemcpy(c->in, delta, bytes, cudaMemcpyDefault), "delta in");
      float* vd = s.get<float>(len);
      cuda_check(cudaMemcpy(vd, v, bytes, cudaMemcpyDefault), "v in");
      launch_build_stream(c->in, c->in_stride, 1, len, vd, doff, 1, dab, dab + 1, nullptr, 0, c->stream);
      cuda_check(cudaStreamSynchronize(c->stream), "identity");
      if (dec) cuda_check(cudaMemcpy(dec, c->in, bytes, cudaMemcpyDefault), "decompressed out");
      cuda_check(memory == BL_MEM_HOST ? (std::memset(delta, 0, bytes), cudaSuccess) : cudaMemset(delta, 0, bytes),
                 "delta reset");
      return;
    }
    cuda_check(cudaMemcpy(c->in, v, bytes, cudaMemcpyDefault), "v in");
    c->compressed(nullptr, 0, static_cast<float>(error_scale), nullptr, nullptr);
    cuda_check(cudaStreamSynchronize(c->stream), "compress");
    unsigned long long e[kErrSlots];
    cuda_check(cudaMemcpy(e, c->err, sizeof e, cudaMemcpyDeviceToHost), "error words");
    if (e[kErrScale] < (1ull << 20))  // the worker endpoint (key 0; the server's is 1 << 20)
      fail(BL_ERR_INVALID_ARGUMENT, "compress: input vector is not finite");  // :56-58, delta untouched
    const int latest = static_cast<int>((c->calls + 1u) & 1u);
    if (wire) packet_bytes(c, c->wpk[latest], wire);
    if (dec) {
      launch_decompress(c->wpk[latest], 1, c->c, c->slot, c->W, len, c->out, c->err, c->stream);
      cuda_check(cudaMemcpyAsync(dec, c->out, bytes, cudaMemcpyDefault, c->stream), "decompressed out");
    }
    launch_materialize_error(c->werr, c->c_pad, c->wpk[latest], c->slot, c->W, c->c, len, c->out, c->stream);
    cuda_check(cudaMemcpyAsync(delta, c->out, bytes, cudaMemcpyDefault, c->stream), "delta out");
    cuda_check(cudaStreamSynchronize(c->stream), "compress outputs");
  });
}

}  // extern "C"

// bl_kernels.cu — hand-written sm_100a kernels of the 1-bit LAMB compression
// stage (K1 worker compress, K3 server reduce, K5/K6 update, W1/W2 warmup) and
// their small helpers.  Compiled with -fmad=false: the reference (x86-64, no
// FMA) rounds every product and sum separately, and so must we.
//
// All sums accumulate in fp64 in the canonical tile-tree order (see
// bl_kernels.cuh and oracle/bitlamb_oracle.c:tile_partial/combine_partials).
// Per-element arithmetic follows the reference's evaluation order, cited at
// each site (file:line relative to /root/reference/proj).

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <unordered_map>

#include "bl_kernels.cuh"

namespace bl {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float4 ld4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ float4 ld4_cs(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ float comp(const float4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_comp(float4& v, int q, float x) {
  if (q == 0) v.x = x;
  else if (q == 1) v.y = x;
  else if (q == 2) v.z = x;
  else v.w = x;
}

// row[4*lane .. 4*lane+3] where `row` may sit s = (row/4) % 4 floats past a
// 16-byte boundary: aligned 128-bit loads plus a lane rotation.  All 32 lanes
// must call it.  Reads up to 128+3 floats past `row - s` (buffers carry slack).
template <bool STREAM>
__device__ __forceinline__ float4 ld_row4(const float* row, int lane, int s) {
  const float* a = row - s;
  const float4 lo = STREAM ? ld4_cs(a + 4 * lane) : ld4(a + 4 * lane);
  if (s == 0) return lo;
  float hx = __shfl_down_sync(FULL, lo.x, 1);
  float hy = __shfl_down_sync(FULL, lo.y, 1);
  float hz = __shfl_down_sync(FULL, lo.z, 1);
  if (lane == 31) {
    const float4 h = ld4(a + 128);
    hx = h.x;
    hy = h.y;
    hz = h.z;
  }
  if (s == 1) return make_float4(lo.y, lo.z, lo.w, hx);
  if (s == 2) return make_float4(lo.z, lo.w, hx, hy);
  return make_float4(lo.w, hx, hy, hz);
}

// Store the lane's nvalid (0..4) leading elements at row + 4*lane.
__device__ __forceinline__ void st_row4(float* row, int lane, int s, const float4& v, int nvalid) {
  float* p = row + 4 * lane;
  if (s == 0 && nvalid >= 4) {
    st4(p, v);
    return;
  }
  if (nvalid > 0) p[0] = v.x;
  if (nvalid > 1) p[1] = v.y;
  if (nvalid > 2) p[2] = v.z;
  if (nvalid > 3) p[3] = v.w;
}

// 128-bit streaming loads with a 256-byte L2 prefetch per miss (more bytes in
// flight per request).  _ro: read-only for the kernel's lifetime (.nc path);
// _rw: element later overwritten by the same thread.
__device__ __forceinline__ float4 ldg_ro(const float* p) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ldg_rw(const float* p) {
  float4 v;
  asm("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}

__device__ __forceinline__ float2 ldg2_ro(const float* p) {
  float2 v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float ldg1_ro(const float* p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// Lane's 4 elements p[0..3] where p sits s floats past a 16-byte boundary:
// one 128-bit load when aligned, 64+64 when s == 2, 32+64+32 when s is odd
// (every access naturally aligned; no lane exchange).
__device__ __forceinline__ float4 ldg_mis_ro(const float* p, int s) {
  if (s == 0) return ldg_ro(p);
  if (s == 2) {
    const float2 a = ldg2_ro(p), b = ldg2_ro(p + 2);
    return make_float4(a.x, a.y, b.x, b.y);
  }
  const float2 m = ldg2_ro(p + 1);
  return make_float4(ldg1_ro(p), m.x, m.y, ldg1_ro(p + 3));
}

// Read-write counterparts (plain .global path: the element is overwritten by
// the same thread later in the kernel).  Inline PTX like the loads above, so
// every access is issued exactly as written (naturally aligned pieces).
__device__ __forceinline__ float2 ldg2_rw(const float* p) {
  float2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float ldg1_rw(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg2(float* p, float a, float b) {
  asm volatile("st.global.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void stg1(float* p, float a) {
  asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}
__device__ __forceinline__ float4 ldg_mis_rw(const float* p, int s) {
  if (s == 2) {
    const float2 a = ldg2_rw(p), b = ldg2_rw(p + 2);
    return make_float4(a.x, a.y, b.x, b.y);
  }
  const float2 m = ldg2_rw(p + 1);
  return make_float4(ldg1_rw(p), m.x, m.y, ldg1_rw(p + 3));
}
__device__ __forceinline__ void st_mis(float* p, int s, const float4& v) {
  if (s == 2) {
    stg2(p, v.x, v.y);
    stg2(p + 2, v.z, v.w);
    return;
  }
  stg1(p, v.x);
  stg2(p + 1, v.y, v.z);
  stg1(p + 3, v.w);
}

// Full-tile row batches of the layer-tiled kernels, for layers that start s
// floats past a 16-byte boundary (MIS) or on one (s == 0): the same batch
// code, instantiated twice, so a misaligned layer keeps the 4-row load
// batches instead of the one-row-per-round-trip boundary path.
template <bool B>
struct Mis {
  static constexpr bool value = B;
};
template <bool MIS>
__device__ __forceinline__ float4 ld_ro_s(const float* p, int s) {
  return MIS ? ldg_mis_ro(p, s) : ldg_ro(p);
}
template <bool MIS>
__device__ __forceinline__ float4 ld_rw_s(const float* p, int s) {
  return MIS ? ldg_mis_rw(p, s) : ldg_rw(p);
}
template <bool MIS>
__device__ __forceinline__ void st_s(float* p, int s, const float4& v) {
  if (MIS) st_mis(p, s, v);
  else st4(p, v);
}

// R consecutive rows (row0 + k*128, k < R) of 4 elements per lane, row0 may be
// misaligned by s floats.
template <int R, bool RO>
__device__ __forceinline__ void load_rows(float4 (&out)[R], const float* row0, int lane, int s) {
  const float* a = row0 + 4 * lane;
#pragma unroll
  for (int k = 0; k < R; ++k) out[k] = RO ? ldg_mis_ro(a + k * kRowElems, s) : ldg_rw(a + k * kRowElems);
}

__device__ __forceinline__ double warp_bfly_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float w = __shfl_xor_sync(FULL, v, o);
    v = v < w ? w : v;
  }
  return v;
}

// Canonical combine of per-thread stripe sums in a 1024-thread block
// (oracle combine_partials).  Result valid in warp 0.
__device__ __forceinline__ double block1024_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_bfly_sum(v);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) v = warp_bfly_sum(sh[lane]);
  __syncthreads();
  return v;
}

__device__ __forceinline__ float block1024_max(float v, float* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) v = warp_max(sh[lane]);
  __syncthreads();
  return v;
}

// Bits 4l..4l+3 of a chunk-aligned row: word 4r + l/8, nibble l%8.
__device__ __forceinline__ uint32_t row_nibble(const uint32_t* words, int r, int lane) {
  return (__ldg(words + 4 * r + (lane >> 3)) >> (4 * (lane & 7))) & 0xFu;
}

// Packet words of a tile are staged in a per-warp shared buffer (128 words)
// and leave it once per tile as one 16-byte store per lane — locally and, for
// the fused exchange, into peer HBM — instead of 4-byte stores per row.
__device__ __forceinline__ void stage_row_bits(uint32_t* sw, int r, int lane, uint32_t nib) {
  uint32_t v = nib << (4 * (lane & 7));
  v |= __shfl_xor_sync(FULL, v, 1);
  v |= __shfl_xor_sync(FULL, v, 2);
  v |= __shfl_xor_sync(FULL, v, 4);
  if ((lane & 7) == 0) sw[4 * r + (lane >> 3)] = v;
}
__device__ __forceinline__ void clear_tile_words(uint32_t* sw, int lane) {
  reinterpret_cast<uint4*>(sw)[lane] = make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
}
__device__ __forceinline__ uint4 tile_words(const uint32_t* sw, int lane) {
  __syncwarp();
  const uint4 v = reinterpret_cast<const uint4*>(sw)[lane];
  __syncwarp();  // the buffer may be refilled after this
  return v;
}

// Make this warp's remote (peer-memory) stores visible system-wide before the
// stream's next kernel raises the peer flag: warp barrier, then one fence.
__device__ __forceinline__ void warp_fence_system(int lane) {
  __syncwarp();
  if (lane == 0) __threadfence_system();
}

__device__ __forceinline__ float slot_scale(const uint32_t* slot, uint64_t W) {
  return __uint_as_float(__ldg(slot + W));
}

// L2-coherent loads for data a peer GPU writes while the consuming kernel is
// already resident (fused exchange): never through the non-coherent path.
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ float slot_scale_cg(const uint32_t* slot, uint64_t W) {
  return __uint_as_float(__ldcg(slot + W));
}
__device__ __forceinline__ uint32_t nibble_cg(const uint32_t* sl, uint32_t i) {
  const uint32_t w0 = __ldcg(sl + (i >> 5)), w1 = __ldcg(sl + (i >> 5) + 1);
  return __funnelshift_r(w0, w1, i & 31u) & 0xFu;
}

// Decompressed result value of a packet bit (compression.cpp:68-81):
// scale == 0 -> +0, else bit ? +S : -S.
__device__ __forceinline__ float dec_value(uint32_t bit, float S) {
  return S == 0.0f ? 0.0f : (bit ? S : -S);
}

// Layer containing global element k (off[l] <= k < off[l+1]); L if k >= d.
__device__ __forceinline__ int find_layer(const uint64_t* off, int L, uint64_t k) {
  int lo = 0, hi = L;  // invariant: off[lo] <= k, answer in [lo, hi)
  if (k >= __ldg(off + L)) return L;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= k) lo = mid;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void flag(unsigned long long* err, int slot, unsigned long long key) {
  if (err) atomicMin(err + slot, key);
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
// The step gate (bl_kernels.cuh GateReason).  Closed -> every mutating kernel
// of the cluster returns at entry, leaving the state as it was.
__device__ __forceinline__ bool gate_closed(const unsigned long long* err) {
  return err != nullptr && ld_volatile_u64(err + kErrGate) != ~0ull;
}
// Kernel-entry form: out of line, so the check leaves the register
// allocation of the streaming loops that follow untouched (measured: an
// inlined early return cost K5 extra spills and 10% of its time).
__device__ __noinline__ bool gate_closed_call(const unsigned long long* err) { return gate_closed(err); }
__device__ __forceinline__ void close_gate(unsigned long long* err, unsigned long long reason) {
  if (err) atomicMin(err + kErrGate, reason);
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Peer wait bound (ns), set by the host in the configuration word.
__device__ __forceinline__ unsigned long long wait_bound(const unsigned long long* err) {
  return err ? ld_volatile_u64(err + kCfgTimeout) : (60ull * 1000000000ull);
}

// Tile scheduler.  With a counter, warps take the next tile from it
// (dynamic: the slowest warp finishes at most one tile after the others
// instead of a whole grid-stride share); without, the fixed grid-stride
// sequence.  The counter resets itself: a launch makes exactly
// total + nwarps fetches and the last one writes 0 back, which stream order
// makes visible to the next kernel.
template <bool SUB = false>
struct TileSchedT {
  unsigned int* ctr;
  long long total, nwarps, cur;
  const int* order = nullptr;  // dynamic mode: hand out order[v] instead of v
  __device__ __forceinline__ long long first(long long gw, int lane) {
    cur = ctr ? fetch(lane) : gw;
    return cur;
  }
  __device__ __forceinline__ long long next(int lane) {
    cur = ctr ? fetch(lane) : cur + nwarps;
    return cur;
  }
  __device__ __forceinline__ long long fetch(int lane) {
    unsigned long long v = 0;
    if (lane == 0) {
      v = atomicAdd(ctr, 1u);
      if (static_cast<long long>(v) == total + nwarps - 1) *ctr = 0u;
      if (SUB) {  // sub-launch: indices past the end stay past every tile index
        v = static_cast<long long>(v) < total ? static_cast<unsigned long long>(__ldg(order + v)) : (1ull << 62);
      } else if (order && static_cast<long long>(v) < total) {
        v = static_cast<unsigned long long>(__ldg(order + v));
      }
    }
    return static_cast<long long>(__shfl_sync(0xffffffffu, v, 0));
  }
};
using TileSched = TileSchedT<false>;
// W1/W2 (warmup overlap sub-launches over order[0..count)).
using TileSchedSub = TileSchedT<true>;

// ---- fused NVLink exchange: epoch flags in peer memory -----------------------
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// After one explicit system fence, further flags need no fence of their own.
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Thread 0 of the block waits until flags[0..n) >= epoch, then the block
// syncs.  Fail-stop: a peer silent for longer than the configured bound
// (peer_timeout_ms) sets kErrPeer and closes the gate (kGateMidStep), so
// nothing later consumes the stale slots; the host then reports the cluster
// as failed.  Returns false when the gate is closed.
__device__ __forceinline__ bool wait_peers(const unsigned long long* flags, int n,
                                           unsigned long long epoch, unsigned long long* err) {
  if (threadIdx.x == 0) {
    const unsigned long long bound = wait_bound(err), t0 = now_ns();
    for (int i = 0; i < n && !gate_closed(err); ++i) {
      while (ld_acquire_sys(flags + i) < epoch) {
        if (gate_closed(err)) break;  // another block already timed out
        __nanosleep(64);
        if (now_ns() - t0 > bound) {
          flag(err, kErrPeer, static_cast<unsigned long long>(i));
          close_gate(err, kGateMidStep);
          break;
        }
      }
    }
  }
  __syncthreads();
  return !gate_closed(err);
}

// ---------------------------------------------------------------------------
// K1 — worker compress (comm_sim.cpp:133-149 + compression.cpp:166-198 and,
// in modes 1/2, the stream build of optimizers.cpp:248-255).
//
// MODE 0: stream = in[w] (SimCluster::compressed_allreduce API)
// MODE 1: stream = A_l*m + B_l*g_w with m from the momentum buffer
// MODE 2: stream = A_l*m + B_l*g_w with m = decompressed previous result *
//         invc_l (m is never stored during the compression stage: after every
//         step m == m_g, optimizers.cpp:315-319, which the packets encode).
//
// Deferred residual: werr holds raw = v + delta (compression.cpp:194-195
// before the reconstruction is subtracted); delta = raw - (bit ? S : -S) is
// materialised from the previous packet when read.  Identical arithmetic,
// one pass: 12 B/elem read + 4 B/elem written + 1 bit.
// ---------------------------------------------------------------------------
// One K1 tile (general path: any alignment, layer boundaries, padding, partial
// tiles).  The per-warp word buffer `sw` stages the tile's packet words.
#ifndef K1_ROWS
#define K1_ROWS 8  // rows per load batch in K1's register path
#endif
#ifndef K1_MINB
#define K1_MINB 2  // resident CTAs per SM requested from ptxas
#endif
// check_gradients' finding (optimizers.cpp:99-117) in fused mode, local
// error word; multi-process it is forwarded to every peer by the kernel that
// raises this rank's flags (finalize / lossless), so every rank raises.
__device__ __forceinline__ void flag_grad(const K1Params& p, unsigned long long key) {
  flag(p.err, kErrGrad, key);
}
// Forward this rank's kErrGrad finding to every peer (before its flags rise).
__device__ __forceinline__ void forward_grad_error(const unsigned long long* err,
                                                   unsigned long long* const* peer_err, int n) {
  if (!peer_err || !err) return;
  const unsigned long long key = ld_volatile_u64(err + kErrGrad);
  if (key == ~0ull) return;
  for (int q = 0; q < n; ++q) atomicMin_system(peer_err[q] + kErrGrad, key);
}

template <int MODE, bool ALIGNED>
__device__ __forceinline__ void k1_tile(const K1Params& p, long long tile, int lane, uint32_t* sw,
                                        float es) {
  const long long per_w = static_cast<long long>(p.n) * p.tpc;
  const int w = static_cast<int>(tile / per_w);
  const long long rem = tile - w * per_w;
  const int j = static_cast<int>(rem / p.tpc);
  const int t = static_cast<int>(rem - static_cast<long long>(j) * p.tpc);
  const uint64_t i0 = static_cast<uint64_t>(t) * kTile;  // chunk-relative
  const uint64_t kc = static_cast<uint64_t>(j) * p.c;    // global chunk start
  const int s = ALIGNED ? 0 : static_cast<int>(kc & 3u);  // ALIGNED: c % 4 == 0
  const size_t ep = static_cast<size_t>(w) * p.n + j;    // endpoint (worker, chunk)
  const float* gin = p.in + static_cast<size_t>(w) * p.in_stride + kc + i0;
  float* we = p.werr + ep * p.c_pad + i0;
  const uint32_t* pkp = p.pk_prev + ep * p.slot;
  uint32_t* pkc = p.pk_cur + ep * p.slot + (i0 >> 5);
  uint32_t* rxw = p.peer_rx ? p.peer_rx[j] + p.rx_off + (i0 >> 5) : nullptr;
  const float Sp = slot_scale(pkp, p.W);
  pkp += i0 >> 5;

  float pos_m = 0.f, neg_m = 0.f;
  const uint32_t* rp = nullptr;
  if (MODE == 2) {
    const uint32_t* rs = p.res_prev + static_cast<size_t>(j) * p.slot;
    const float S2 = slot_scale(rs, p.W);
    pos_m = S2;
    neg_m = S2 == 0.0f ? 0.0f : -S2;
    rp = rs + (i0 >> 5);
  }
  float A = 0.f, B = 0.f, IC = 0.f;

  // Fast path: the whole tile lies inside the chunk, inside the real
  // (unpadded) data and inside one layer.  Rows are processed 4 at a time
  // with all loads issued first; same per-element arithmetic and the same
  // accumulation order as the general path below.
  bool fast = MODE != 1 && i0 + kTile <= p.c && kc + i0 + kTile <= p.d;
  if (fast && MODE == 2) {
    int l0;
    if (p.tile_layer) {
      l0 = __ldg(p.tile_layer + static_cast<size_t>(j) * p.tpc + t);
      fast = l0 >= 0;
    } else {
      l0 = find_layer(p.off, p.L, kc + i0);
      fast = l0 < p.L && kc + i0 + (kTile - 1) < __ldg(p.off + l0 + 1);
    }
    if (fast) {
      A = __ldg(p.A + l0);
      B = __ldg(p.B + l0);
      IC = __ldg(p.invc + l0);
    }
  }
  if (fast && p.skip_fast) return;  // done by k1_bulk
  if (fast) {
    constexpr int R = K1_ROWS;
    const uint32_t sh = 4 * (lane & 7);
    const int wsub = lane >> 3;
    const bool stats = p.cmax != nullptr;
    double acc = 0.0;
    float cm = 0.0f;
    for (int r0 = 0; r0 < kRowsPerTile; r0 += R) {
      float4 g[R], raw[R];
      uint32_t wn[R], rn[R];
      load_rows<R, true>(g, gin + r0 * kRowElems, lane, s);
#pragma unroll
      for (int k = 0; k < R; ++k) {
        raw[k] = ldg_rw(we + (r0 + k) * kRowElems + 4 * lane);
        wn[k] = __ldg(pkp + 4 * (r0 + k) + wsub) >> sh;
        rn[k] = MODE == 2 ? __ldg(rp + 4 * (r0 + k) + wsub) >> sh : 0u;
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (MODE == 2 && !(isfinite(g[k].x) && isfinite(g[k].y) && isfinite(g[k].z) &&
                           isfinite(g[k].w))) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!isfinite(comp(g[k], q))) {
              flag_grad(p, (static_cast<unsigned long long>(p.worker_base + w) << 40) |
                               (kc + i0 + (r0 + k) * kRowElems + 4 * lane + q));
            }
          }
        }
        uint32_t nib = 0;
        float4 rawn;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float v;
          if (MODE == 0) {
            v = comp(g[k], q);
          } else {
            // A * (m_q = +-S2 * invc): two values per tile, hoisted (same products)
            const float ap = __fmul_rn(A, __fmul_rn(pos_m, IC)), an = __fmul_rn(A, __fmul_rn(neg_m, IC));
            v = __fadd_rn((rn[k] >> q) & 1u ? ap : an, __fmul_rn(B, comp(g[k], q)));  // fusion.cpp:143, kernels.cpp:253
          }
          const float rec = (wn[k] >> q) & 1u ? Sp : -Sp;
          const float delta = __fsub_rn(comp(raw[k], q), rec);                // compression.cpp:194
          const float corr = __fadd_rn(v, __fmul_rn(es, delta));              // :181
          set_comp(rawn, q, __fadd_rn(v, delta));
          nib |= static_cast<uint32_t>(corr >= 0.0f) << q;                    // :50
          acc += fabs(static_cast<double>(corr));                              // :54
          if (stats) {
            const float ac = fabsf(corr);
            cm = cm < ac ? ac : cm;
          }
        }
        st4(we + (r0 + k) * kRowElems + 4 * lane, rawn);
        stage_row_bits(sw, r0 + k, lane, nib);
      }
    }
    const uint4 wv = tile_words(sw, lane);
    reinterpret_cast<uint4*>(pkc)[lane] = wv;
    if (rxw) reinterpret_cast<uint4*>(rxw)[lane] = wv;  // fused alltoall
    acc = warp_bfly_sum(acc);
    if (lane == 0) p.partials[ep * p.tpc + t] = acc;
    if (stats) {
      cm = warp_max(cm);
      if (lane == 0) p.cmax[ep * p.tpc + t] = cm;
    }
    return;
  }

  int l = 0;
  int lcache = -1;
  if (MODE != 0) l = find_layer(p.off, p.L, kc + i0);

  clear_tile_words(sw, lane);  // rows past the chunk end keep zero bits
  double acc = 0.0;
  float cm = 0.0f;
  for (int r = 0; r < kRowsPerTile; ++r) {
    const uint64_t ir = i0 + static_cast<uint64_t>(r) * kRowElems;
    if (ir >= p.c) break;
    const uint64_t kr = kc + ir;
    const float4 g = ld_row4<true>(gin + r * kRowElems, lane, s);
    float4 mv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (MODE == 1) mv = ld_row4<false>(p.m + kr, lane, s);
    const float4 raw = ld4(we + r * kRowElems + 4 * lane);
    const uint32_t wnib = row_nibble(pkp, r, lane);
    uint32_t rnib = 0;
    if (MODE == 2) rnib = row_nibble(rp, r, lane);

    // Stream value for each of the lane's 4 elements.
    float4 sv;
    if (MODE == 0) {
      sv = g;
    } else {
      while (l < p.L && kr >= __ldg(p.off + l + 1)) ++l;
      const bool uniform = l < p.L && kr + (kRowElems - 1) < __ldg(p.off + l + 1);
      if (uniform && l != lcache) {
        A = __ldg(p.A + l);
        B = __ldg(p.B + l);
        IC = __ldg(p.invc + l);
        lcache = l;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float a = A, b = B, ic = IC;
        bool pad = false;
        if (!uniform) {
          const uint64_t k = kr + 4 * lane + q;
          int le = l;
          while (le < p.L && k >= __ldg(p.off + le + 1)) ++le;
          pad = le >= p.L;
          if (!pad) {
            a = __ldg(p.A + le);
            b = __ldg(p.B + le);
            ic = __ldg(p.invc + le);
          }
        }
        float mq;
        if (MODE == 1) mq = comp(mv, q);
        else mq = __fmul_rn((rnib >> q) & 1u ? pos_m : neg_m, ic);  // fusion.cpp:143
        // kernels.cpp:253  dst = a*x + b*y
        const float v = pad ? 0.0f : __fadd_rn(__fmul_rn(a, mq), __fmul_rn(b, comp(g, q)));
        set_comp(sv, q, v);
      }
    }
    if (MODE != 0) {
      // check_gradients (optimizers.cpp:99-117): flag, reported by the host.
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t k = kr + 4 * lane + q;
        if (ir + 4 * lane + q < p.c && k < p.d && !isfinite(comp(g, q))) {
          flag_grad(p, (static_cast<unsigned long long>(p.worker_base + w) << 40) | k);
        }
      }
    }

    uint32_t nib = 0;
    float4 rawn;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = ir + 4 * lane + q;
      const uint64_t k = kc + i;
      const float v = k < p.d ? comp(sv, q) : 0.0f;  // comm_sim.cpp:136-137 zero pad
      const float rec = (wnib >> q) & 1u ? Sp : -Sp;
      const float delta = __fsub_rn(comp(raw, q), rec);          // compression.cpp:194-195
      const float corr = __fadd_rn(v, __fmul_rn(es, delta));     // :181 (1*v + es*delta)
      const float rn = __fadd_rn(v, delta);                      // v + delta
      const bool live = i < p.c;
      set_comp(rawn, q, live ? rn : 0.0f);
      if (live) {
        nib |= static_cast<uint32_t>(corr >= 0.0f) << q;         // compression.cpp:50
        acc += fabs(static_cast<double>(corr));                   // :54 sum_abs
        const float ac = fabsf(corr);
        cm = cm < ac ? ac : cm;
      }
    }
    st4(we + r * kRowElems + 4 * lane, rawn);
    stage_row_bits(sw, r, lane, nib);
  }
  {
    const uint4 wv = tile_words(sw, lane);
    reinterpret_cast<uint4*>(pkc)[lane] = wv;
    if (rxw) reinterpret_cast<uint4*>(rxw)[lane] = wv;
  }
  acc = warp_bfly_sum(acc);
  if (lane == 0) p.partials[ep * p.tpc + t] = acc;
  if (p.cmax) {
    cm = warp_max(cm);
    if (lane == 0) p.cmax[ep * p.tpc + t] = cm;
  }
}

template <int MODE, bool ALIGNED>
__global__ void __launch_bounds__(kBlock, K1_MINB) k1_worker_compress(const K1Params p) {
  if (gate_closed_call(p.err)) return;
  __shared__ __align__(16) uint32_t s_words[kWarpsPerBlock][128];
  uint32_t* sw = s_words[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const long long per_w = static_cast<long long>(p.n) * p.tpc;
  const long long total = p.slow_list ? static_cast<long long>(p.n_slow) * p.nw
                                      : (p.tile_cnt ? p.tile_cnt : per_w * p.nw);
  const float es = p.es_dev ? __ldg(p.es_dev) : p.es_host;

  // Boundary tiles first (order) when the whole index space is scheduled.
  TileSched sch{p.slow_list ? nullptr : p.ctr, total, nwarps, 0,
                p.slow_list || p.tile_cnt ? nullptr : p.order};
  for (long long it = sch.first(gw, lane); it < total; it = sch.next(lane)) {
    long long tile = it + p.tile_lo;
    if (p.slow_list) {  // iterate only the listed boundary tiles of every worker
      const long long wl = it / p.n_slow;
      tile = wl * per_w + __ldg(p.slow_list + (it - wl * p.n_slow));
    }
    k1_tile<MODE, ALIGNED>(p, tile, lane, sw, es);
  }
  if (p.peer_rx) warp_fence_system(threadIdx.x & 31);  // remote words before the finalize signal
}

// ---------------------------------------------------------------------------
// K1 bulk: the fast tiles of K1 with the operand rows staged in shared memory
// by the bulk-copy (TMA) engine.  Each warp owns a 3-stage ring; a stage is 4
// rows of g (read from the 16-byte-aligned address below the row start, so
// misaligned chunks cost nothing extra), 4 rows of werr and the packet words
// of those rows, completed on an mbarrier.  Registers hold only compute state,
// so 2 batches per warp stay in flight.  Same arithmetic and accumulation
// order as the fast path of k1_worker_compress.
// ---------------------------------------------------------------------------
constexpr int kBulkWarps = 4;
constexpr int kBulkStages = 3;
template <int R>
struct BulkGeom {
  static constexpr int G = (R * kRowElems + 4) * 4;  // g rows + alignment slack
  static constexpr int Wb = R * kRowElems * 4;       // werr rows
  static constexpr int Bits = R * 4 * 4;             // packet words of the rows
  static constexpr int Stage = G + Wb + 2 * Bits;
  static constexpr int Smem = kBulkWarps * kBulkStages * Stage;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Bounded wait (a lost completion must never wedge the GPU): gives up after
// ~2^28 polls and closes the gate (kGateInternal), which the host reports.
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase, unsigned long long* err) {
  uint32_t ok = 0;
  for (uint32_t it = 0; it < (1u << 28); ++it) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (ok) return;
  }
  close_gate(err, kGateInternal);
}

__device__ __forceinline__ float4 lds_mis(const float* p, int s) {
  if (s == 0) return *reinterpret_cast<const float4*>(p);
  if (s == 2) {
    const float2 a = *reinterpret_cast<const float2*>(p), b = *reinterpret_cast<const float2*>(p + 2);
    return make_float4(a.x, a.y, b.x, b.y);
  }
  const float2 m = *reinterpret_cast<const float2*>(p + 1);
  return make_float4(p[0], m.x, m.y, p[3]);
}

template <int MODE>
__device__ __forceinline__ int k1_fast_layer(const K1Params& p, int j, int t) {
  const uint64_t i0 = static_cast<uint64_t>(t) * kTile, kc = static_cast<uint64_t>(j) * p.c;
  if (i0 + kTile > p.c || kc + i0 + kTile > p.d) return -1;
  if (MODE == 0) return 0;
  return __ldg(p.tile_layer + static_cast<size_t>(j) * p.tpc + t);
}

template <int MODE, int kBulkR>
__global__ void __launch_bounds__(kBulkWarps * 32, 4) k1_bulk(const K1Params p) {
  if (gate_closed_call(p.err)) return;
  using Geo = BulkGeom<kBulkR>;
  constexpr int kBulkG = Geo::G, kBulkW = Geo::Wb, kBulkBits = Geo::Bits, kBulkStage = Geo::Stage;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bars[kBulkWarps][kBulkStages];
  __shared__ __align__(16) uint32_t s_words[kBulkWarps][128];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* sw = s_words[wib];
  unsigned char* wsm = sm + wib * kBulkStages * kBulkStage;
  const long long gw = static_cast<long long>(blockIdx.x) * kBulkWarps + wib;
  const long long nwarps = static_cast<long long>(gridDim.x) * kBulkWarps;
  const long long per_w = static_cast<long long>(p.n) * p.tpc;
  const long long total = per_w * p.nw;
  const float es = p.es_dev ? __ldg(p.es_dev) : p.es_host;
  if (lane == 0) {
    for (int s = 0; s < kBulkStages; ++s) mbar_init(&bars[wib][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // Tile index -> (worker, chunk, tile-in-chunk) in 32-bit arithmetic (the
  // index space is below 2^31): 64-bit divisions here cost ~50 issued
  // instructions per row when they ran per stage (ncu: 200 per row).
  const unsigned int per_w32 = static_cast<unsigned int>(per_w), tpc32 = static_cast<unsigned int>(p.tpc);
  auto split = [&](long long tile, int& w, int& j, int& t) {
    const unsigned int u = static_cast<unsigned int>(tile);
    w = static_cast<int>(u / per_w32);
    const unsigned int rem = u - static_cast<unsigned int>(w) * per_w32;
    j = static_cast<int>(rem / tpc32);
    t = static_cast<int>(rem - static_cast<unsigned int>(j) * tpc32);
  };
  auto is_fast = [&](long long tile) {
    int w, j, t;
    split(tile, w, j, t);
    return k1_fast_layer<MODE>(p, j, t) >= 0;
  };
  auto next_fast = [&](long long tile) {
    while (tile < total && !is_fast(tile)) tile += nwarps;
    return tile;
  };
  // Producer state of the tile being issued -- its source rows, formed once
  // per tile (not per stage) by lane 0 and kept in shared memory (registers
  // are the consumer's).
  __shared__ const void* s_src[kBulkWarps][4];
  auto bind = [&](long long tile) {
    if (tile >= total || lane != 0) return;
    int w, j, t;
    split(tile, w, j, t);
    const uint64_t i0 = static_cast<uint64_t>(t) * kTile, kc = static_cast<uint64_t>(j) * p.c;
    const size_t ep = static_cast<size_t>(w) * p.n + j;
    s_src[wib][0] = p.in + static_cast<size_t>(w) * p.in_stride + kc + i0 - static_cast<int>(kc & 3u);
    s_src[wib][1] = p.werr + ep * p.c_pad + i0;
    s_src[wib][2] = p.pk_prev + ep * p.slot + (i0 >> 5);
    s_src[wib][3] = p.res_prev + static_cast<size_t>(j) * p.slot + (i0 >> 5);
  };
  // Producer: lane 0 issues the copies of batch (bound tile, r0) into `stage`.
  auto issue = [&](int stage, long long tile, int r0) {
    if (tile >= total || lane != 0) return;
    unsigned char* st = wsm + stage * kBulkStage;
    unsigned long long* bar = &bars[wib][stage];
    mbar_expect_tx(bar, kBulkG + kBulkW + (MODE == 2 ? 2 : 1) * kBulkBits);
    bulk_g2s(st, static_cast<const float*>(s_src[wib][0]) + r0 * kRowElems, kBulkG, bar);
    bulk_g2s(st + kBulkG, static_cast<const float*>(s_src[wib][1]) + r0 * kRowElems, kBulkW, bar);
    bulk_g2s(st + kBulkG + kBulkW, static_cast<const uint32_t*>(s_src[wib][2]) + 4 * r0, kBulkBits, bar);
    if (MODE == 2)
      bulk_g2s(st + kBulkG + kBulkW + kBulkBits, static_cast<const uint32_t*>(s_src[wib][3]) + 4 * r0,
               kBulkBits, bar);
  };

  // Producer sequence: with a tile counter the fast tiles are taken
  // dynamically (boundary tiles are skipped here and done below from the
  // slow list); each issued batch records its (tile, r0) in the stage slot
  // so the consumer replays exactly the producer's order.
  __shared__ long long s_tile[kBulkWarps][kBulkStages];
  __shared__ int s_r0[kBulkWarps][kBulkStages];
  TileSched sch{p.ctr, total, nwarps, 0};
  auto fetch_fast = [&](bool first) {
    long long t = first ? sch.first(gw, lane) : sch.next(lane);
    while (t < total && !is_fast(t)) t = sch.next(lane);
    return t;
  };
  long long ptile = p.ctr ? fetch_fast(true) : next_fast(gw);
  bind(ptile);
  int pr = 0;
  auto produce = [&](int stage) {
    if (lane == 0) {
      s_tile[wib][stage] = ptile;
      s_r0[wib][stage] = pr;
    }
    issue(stage, ptile, pr);
    if (ptile >= total) return;
    pr += kBulkR;
    if (pr == kRowsPerTile) {
      pr = 0;
      ptile = p.ctr ? fetch_fast(false) : next_fast(ptile + nwarps);
      bind(ptile);
    }
  };
  for (int s = 0; s < kBulkStages; ++s) produce(s);
  __syncwarp();
  // Boundary tiles (layer boundaries, chunk/padding ends) take the general
  // path here, while the prologue copies are in flight.
  if (p.slow_list) {
    const long long stotal = static_cast<long long>(p.n_slow) * p.nw;
    for (long long it = gw; it < stotal; it += nwarps) {
      const long long wl = it / p.n_slow;
      k1_tile<MODE, false>(p, wl * per_w + __ldg(p.slow_list + (it - wl * p.n_slow)), lane, sw, es);
    }
  }

  long long ctile = 0;
  int cr = 0;
  uint32_t b = 0;
  // per-tile consumer state
  int s = 0, t = 0;
  size_t ep = 0;
  uint64_t i0 = 0, kc = 0;
  float* we = nullptr;
  uint32_t* pkc = nullptr;
  uint32_t* rxw = nullptr;
  float Sp = 0.f, pos_m = 0.f, neg_m = 0.f, A = 0.f, B = 0.f, IC = 0.f;
  int w = 0;
  double acc = 0.0;
  float cm = 0.0f;
  const bool stats = p.cmax != nullptr;
  const uint32_t sh = 4 * (lane & 7);
  const int wsub = lane >> 3;
  while (true) {
    const int stage = static_cast<int>(b % kBulkStages);
    const uint32_t phase = (b / kBulkStages) & 1u;
    ctile = s_tile[wib][stage];
    cr = s_r0[wib][stage];
    if (ctile >= total) break;
    if (cr == 0) {
      int j;
      split(ctile, w, j, t);
      i0 = static_cast<uint64_t>(t) * kTile;
      kc = static_cast<uint64_t>(j) * p.c;
      s = static_cast<int>(kc & 3u);
      ep = static_cast<size_t>(w) * p.n + j;
      we = p.werr + ep * p.c_pad + i0;
      pkc = p.pk_cur + ep * p.slot + (i0 >> 5);
      rxw = p.peer_rx ? p.peer_rx[j] + p.rx_off + (i0 >> 5) : nullptr;
      Sp = slot_scale(p.pk_prev + ep * p.slot, p.W);
      if (MODE == 2) {
        const float S2 = slot_scale(p.res_prev + static_cast<size_t>(j) * p.slot, p.W);
        pos_m = S2;
        neg_m = S2 == 0.0f ? 0.0f : -S2;
        const int l0 = __ldg(p.tile_layer + static_cast<size_t>(j) * p.tpc + t);
        A = __ldg(p.A + l0);
        B = __ldg(p.B + l0);
        IC = __ldg(p.invc + l0);
      }
      acc = 0.0;
      cm = 0.0f;
    }
    mbar_wait(&bars[wib][stage], phase, p.err);
    const unsigned char* st = wsm + stage * kBulkStage;
    const float* gsm = reinterpret_cast<const float*>(st) + s;
    const float* wsm_rows = reinterpret_cast<const float*>(st + kBulkG);
    const uint32_t* wbits = reinterpret_cast<const uint32_t*>(st + kBulkG + kBulkW);
    const uint32_t* rbits = reinterpret_cast<const uint32_t*>(st + kBulkG + kBulkW + kBulkBits);
#pragma unroll
    for (int k = 0; k < kBulkR; ++k) {
      const float4 g = lds_mis(gsm + k * kRowElems + 4 * lane, s);
      const float4 raw = *reinterpret_cast<const float4*>(wsm_rows + k * kRowElems + 4 * lane);
      const uint32_t wn = wbits[4 * k + wsub] >> sh;
      const uint32_t rn = MODE == 2 ? rbits[4 * k + wsub] >> sh : 0u;
      if (MODE == 2 && !(isfinite(g.x) && isfinite(g.y) && isfinite(g.z) && isfinite(g.w))) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!isfinite(comp(g, q))) {
            flag_grad(p, (static_cast<unsigned long long>(p.worker_base + w) << 40) |
                             (kc + i0 + (cr + k) * kRowElems + 4 * lane + q));
          }
        }
      }
      uint32_t nib = 0;
      float4 rawn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float v;
        if (MODE == 0) {
          v = comp(g, q);
        } else {
          const float ap = __fmul_rn(A, __fmul_rn(pos_m, IC)), an = __fmul_rn(A, __fmul_rn(neg_m, IC));
          v = __fadd_rn((rn >> q) & 1u ? ap : an, __fmul_rn(B, comp(g, q)));  // fusion.cpp:143, kernels.cpp:253
        }
        const float rec = (wn >> q) & 1u ? Sp : -Sp;
        const float delta = __fsub_rn(comp(raw, q), rec);    // compression.cpp:194
        const float corr = __fadd_rn(v, __fmul_rn(es, delta));  // :181
        set_comp(rawn, q, __fadd_rn(v, delta));
        nib |= static_cast<uint32_t>(corr >= 0.0f) << q;  // :50
        acc += fabs(static_cast<double>(corr));           // :54
        if (stats) {
          const float ac = fabsf(corr);
          cm = cm < ac ? ac : cm;
        }
      }
      st4(we + (cr + k) * kRowElems + 4 * lane, rawn);
      stage_row_bits(sw, cr + k, lane, nib);
    }
    __syncwarp();  // every lane is done with this stage before it is refilled
    produce(stage);
    __syncwarp();
    if (cr + kBulkR == kRowsPerTile) {
      const uint4 wv = tile_words(sw, lane);
      reinterpret_cast<uint4*>(pkc)[lane] = wv;
      if (rxw) reinterpret_cast<uint4*>(rxw)[lane] = wv;  // fused alltoall
      const double tot = warp_bfly_sum(acc);
      if (lane == 0) p.partials[ep * p.tpc + t] = tot;
      if (stats) {
        const float m = warp_max(cm);
        if (lane == 0) p.cmax[ep * p.tpc + t] = m;
      }
    }
    ++b;
  }
  if (p.peer_rx) warp_fence_system(lane);
}

// Scale of each endpoint: S = (float)(sum|corrected| / c) (compression.cpp:54-55),
// non-finite -> flag (compression.cpp:56-58).  One 1024-thread block per endpoint.
// s = a[t0] + a[t0 + step] + ... (t < t1), added in that order from 0; the
// loads are issued 8 at a time so the dependent fp64 adds do not wait on
// one load each (the canonical stripe sums of finalize / epilogues).
#ifndef STRIPE_BATCH
#define STRIPE_BATCH 8  // (16 measured slower in the scale finalize: profiles/round2_fin16_ab.txt)
#endif
template <int STEP = 1024>
__device__ __forceinline__ double stripe_sum(const double* a, long long t0, long long t1) {
  constexpr int B = STRIPE_BATCH;  // loads in flight per thread
  double s = 0.0;
  long long t = t0;
  for (; t + (B - 1ll) * STEP < t1; t += static_cast<long long>(B) * STEP) {
    double v[B];
#pragma unroll
    for (int k = 0; k < B; ++k) v[k] = a[t + k * STEP];
#pragma unroll
    for (int k = 0; k < B; ++k) s += v[k];
  }
  for (; t < t1; t += STEP) s += a[t];
  return s;
}

// Endpoint e's scale from its combined partial sum s (compression.cpp:54-58):
// local slot, finite check and, for the fused exchange, the peers' slots and
// epoch flags.  One thread.
__device__ void finalize_commit(const FinalizeParams& p, int e, double s) {
  {
    const float S = static_cast<float>(s / static_cast<double>(p.c));
    p.slots[static_cast<size_t>(e) * p.slot_stride + p.W] = __float_as_uint(S);
    if (!isfinite(S)) flag(p.err, kErrScale, static_cast<unsigned long long>(p.err_base + e));
    if (p.peer_slots) {
      forward_grad_error(p.err, p.peer_err, p.n);  // every rank raises (optimizers.cpp:99-117)
      const int q0 = p.to_all ? 0 : e, q1 = p.to_all ? p.n : e + 1;
      for (int q = q0; q < q1; ++q) p.peer_slots[q][p.peer_off + p.W] = __float_as_uint(S);
      __threadfence_system();  // the scale words before any flag
      for (int q = q0; q < q1; ++q) st_relaxed_sys(p.peer_flags[q] + p.flag_index, p.epoch);
    }
  }
}

__global__ void __launch_bounds__(1024) k_finalize_scales(const FinalizeParams p) {
  if (gate_closed_call(p.err)) return;
  __shared__ double sh[32];
  const int e = blockIdx.x;
  const double* part = p.partials + static_cast<size_t>(e) * p.tpc;
  double s = stripe_sum(part, threadIdx.x, p.tpc);
  s = block1024_sum(s, sh);
  if (threadIdx.x == 0) finalize_commit(p, e, s);
}

// The same canonical combine with a 256-thread block (fused small
// collective): thread i forms stripes i, i+256, i+512, i+768; warp w
// butterflies stripe groups w, w+8, w+16, w+24 (32 stripes each); warp 0
// butterflies the 32 group sums — k_finalize_scales' order exactly.
__device__ void finalize_block256(const FinalizeParams& p, int e, double* red /* [1024 + 32] */) {
  const double* part = p.partials + static_cast<size_t>(e) * p.tpc;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int k = 0; k < 4; ++k) red[tid + 256 * k] = stripe_sum(part, tid + 256 * k, p.tpc);
  __syncthreads();
  for (int k = 0; k < 4; ++k) {
    const int g = w + 8 * k;
    const double v = warp_bfly_sum(red[32 * g + lane]);
    if (lane == 0) red[1024 + g] = v;
  }
  __syncthreads();
  if (w == 0) {
    const double v = warp_bfly_sum(red[1024 + lane]);
    if (lane == 0) finalize_commit(p, e, v);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// K3 — server reduce (comm_sim.cpp:158-181): ascending-worker average of the
// n one-bit messages (compression.cpp:83-89, skipped when S == 0; scale 1/n in
// fp64, :164), error-compensated recompression with the server residual.
// ---------------------------------------------------------------------------
// Allgather fused into K3: the row's 4 server words (just written to the local
// result slot by the same warp) are copied into every peer's result slot.
__device__ __forceinline__ void flush_server_words(const K3Params& p, uint32_t* const* peers,
                                                   const uint32_t* sw, uint32_t* rc, uint64_t i0,
                                                   int lane) {
  const uint4 v = tile_words(sw, lane);
  reinterpret_cast<uint4*>(rc)[lane] = v;
  if (p.peer_res) {
    for (int q = 0; q < p.n; ++q) {
      if (q != p.rank) reinterpret_cast<uint4*>(peers[q] + p.res_off + (i0 >> 5))[lane] = v;
    }
  }
}

#ifndef K3_R1
#define K3_R1 16  // n = 1: 16-row batches at 2 CTAs/SM (A/B: profiles/round2_k3n1_ab.txt)
#endif
#ifndef K3_R2
#define K3_R2 4
#endif
#ifndef K3_R4
#define K3_R4 4
#endif
#ifndef K3_B4
#define K3_B4 3
#endif
#ifndef K3_B8
#define K3_B8 2
#endif
#ifndef K3_B2
#define K3_B2 3
#endif
#define K3_ROWS(NT) ((NT) == 1 ? K3_R1 : (NT) == 2 ? K3_R2 : (NT) == 4 ? K3_R4 : 4)
#ifndef K3_B1
#define K3_B1 (K3_R1 == 16 ? 2 : K3_R1 == 8 ? 3 : 4)
#endif
#define K3_MINB(NT) ((NT) == 1 ? K3_B1 : (NT) == 2 ? K3_B2 : (NT) == 4 ? K3_B4 : (NT) == 8 ? K3_B8 : 2)
template <int NT>
__global__ void __launch_bounds__(kBlock, K3_MINB(NT)) k3_server_reduce(const K3Params p) {
  if (gate_closed_call(p.err)) return;
  __shared__ float s_scale[kWarpsPerBlock][64];
  __shared__ uint32_t* s_peer[64];
  __shared__ __align__(16) uint32_t s_words[kWarpsPerBlock][128];
  // 2^n-entry server-average table for n in {4, 8} (per warp, per chunk)
  constexpr bool kTable = NT >= 4;
  constexpr bool kSel = NT == 1 || NT == 2;  // averages by select from per-tile values
  __shared__ float s_tab[kWarpsPerBlock][kTable ? (1 << (NT > 0 ? NT : 1)) : 1];
  int tab_chunk = -1;
  uint32_t* sw = s_words[threadIdx.x >> 5];
  const int n = NT > 0 ? NT : p.n;
  if (p.peer_res) {
    for (int q = threadIdx.x; q < p.n; q += blockDim.x) s_peer[q] = p.peer_res[q];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const long long total = static_cast<long long>(p.ns) * p.tpc;
  const float es = p.es_dev ? __ldg(p.es_dev) : p.es_host;
  const double inv_n = 1.0 / static_cast<double>(n);

  TileSched sch{p.ctr, total, nwarps, 0};
  for (long long tile = sch.first(gw, lane); tile < total; tile = sch.next(lane)) {
    const int sv = static_cast<int>(tile / p.tpc);
    const int t = static_cast<int>(tile - static_cast<long long>(sv) * p.tpc);
    const int j = p.server_base + sv;
    const uint64_t i0 = static_cast<uint64_t>(t) * kTile;
    const uint32_t* in = p.in + sv * p.in_s;
    __syncwarp();
    for (int i = lane; i < n; i += 32) s_scale[wib][i] = slot_scale_cg(in + i * p.in_i, p.W);
    __syncwarp();
    float* se = p.serr + static_cast<size_t>(sv) * p.c_pad + i0;
    const uint32_t* rs = p.res_prev + static_cast<size_t>(j) * p.slot;
    const float S2p = slot_scale(rs, p.W);
    rs += i0 >> 5;
    uint32_t* rc = p.res_cur + static_cast<size_t>(j) * p.slot + (i0 >> 5);
    const uint32_t* inw = in + (i0 >> 5);

    if (NT > 0 && i0 + kTile <= p.c) {
      // Fast path: full tile, R rows per batch with every load issued first.
      // One streamed array (serr): small n takes 8 rows per batch to keep
      // as many bytes in flight as the two-array kernels.
      constexpr int R = K3_ROWS(NT);
      const uint32_t sh = 4 * (lane & 7);
      const int wsub = lane >> 3;
      const bool stats = p.cmax != nullptr;
      double acc = 0.0;
      float cm = 0.0f;
      for (int r0 = 0; r0 < kRowsPerTile; r0 += R) {
        float4 raw[R];
        uint32_t sn[R], wn[R][NT > 0 ? NT : 1];
#pragma unroll
        for (int k = 0; k < R; ++k) {
          raw[k] = ldg_rw(se + (r0 + k) * kRowElems + 4 * lane);
          sn[k] = __ldg(rs + 4 * (r0 + k) + wsub) >> sh;
#pragma unroll
          for (int i = 0; i < (NT > 0 ? NT : 1); ++i)
            wn[k][i] = ld_cg(inw + i * p.in_i + 4 * (r0 + k) + wsub) >> sh;
        }
      if (kTable && tab_chunk != j) {
        // avg(pattern) for every n-bit sign pattern of chunk j: the same
        // ascending fp64 sum (skipping S == 0) and *1/n as the direct form.
        __syncwarp();
        for (int e = lane; e < (1 << NT); e += 32) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < NT; ++i) {
            const float S = s_scale[wib][i];
            if (S != 0.0f) acc += ((e >> i) & 1) ? static_cast<double>(S) : -static_cast<double>(S);
          }
          s_tab[wib][e] = static_cast<float>(acc * inv_n);
        }
        __syncwarp();
        tab_chunk = j;
      }
      // n <= 2: the 2^n possible averages of this tile's chunk, formed once
      // per tile by the same ascending fp64 sum and *1/n (compression.cpp:83-89)
      float tv[4] = {0.f, 0.f, 0.f, 0.f};
      if (kSel) {
#pragma unroll
        for (int e = 0; e < (1 << (NT > 0 ? NT : 1)); ++e) {
          double a = 0.0;
#pragma unroll
          for (int i = 0; i < (NT > 0 ? NT : 1); ++i) {
            const float S = s_scale[wib][i];
            if (S != 0.0f) a += ((e >> i) & 1) ? static_cast<double>(S) : -static_cast<double>(S);
          }
          tv[e] = static_cast<float>(a * inv_n);
        }
      }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          float4 avg;
          if (kSel) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t b0 = (wn[k][0] >> q) & 1u;
              if (NT == 1) {
                set_comp(avg, q, b0 ? tv[1] : tv[0]);
              } else {
                const uint32_t b1 = (wn[k][NT > 1 ? 1 : 0] >> q) & 1u;
                set_comp(avg, q, b1 ? (b0 ? tv[3] : tv[2]) : (b0 ? tv[1] : tv[0]));
              }
            }
          } else if (kTable) {
            uint32_t x = 0;  // nibble of worker i at bits 4i..4i+3
#pragma unroll
            for (int i = 0; i < NT; ++i) x |= (wn[k][i] & 0xFu) << (4 * i);
            if (NT == 4) {
              // 4x4 bit transpose (worker-major -> element-major): element q's
              // 4-bit worker pattern lands at bits 4q..4q+3
              uint32_t t = (x ^ (x >> 3)) & 0x0A0Au;
              x = x ^ t ^ (t << 3);
              t = (x ^ (x >> 6)) & 0x00CCu;
              x = x ^ t ^ (t << 6);
#pragma unroll
              for (int q = 0; q < 4; ++q) set_comp(avg, q, s_tab[wib][(x >> (4 * q)) & 0xFu]);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) {  // gather bits q, q+4, ... -> n-bit pattern
                uint32_t y = (x >> q) & 0x11111111u;
                y = (y | (y >> 3)) & 0x03030303u;
                y = (y | (y >> 6)) & 0x000F000Fu;
                y = (y | (y >> 12)) & 0xFFu;
                set_comp(avg, q, s_tab[wib][y]);
              }
            }
          } else {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
            for (int i = 0; i < (NT > 0 ? NT : 1); ++i) {  // compression.cpp:83-89
              const float S = s_scale[wib][i];
              if (S != 0.0f) {
                const double Sd = S;
                a0 += (wn[k][i] & 1u) ? Sd : -Sd;
                a1 += (wn[k][i] & 2u) ? Sd : -Sd;
                a2 += (wn[k][i] & 4u) ? Sd : -Sd;
                a3 += (wn[k][i] & 8u) ? Sd : -Sd;
              }
            }
            avg = make_float4(static_cast<float>(a0 * inv_n), static_cast<float>(a1 * inv_n),
                              static_cast<float>(a2 * inv_n), static_cast<float>(a3 * inv_n));
          }
          uint32_t nib = 0;
          float4 rawn;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float v = comp(avg, q);
            const float rec = (sn[k] >> q) & 1u ? S2p : -S2p;
            const float delta = __fsub_rn(comp(raw[k], q), rec);
            const float corr = __fadd_rn(v, __fmul_rn(es, delta));
            set_comp(rawn, q, __fadd_rn(v, delta));
            nib |= static_cast<uint32_t>(corr >= 0.0f) << q;
            acc += fabs(static_cast<double>(corr));
            if (stats) {
              const float ac = fabsf(corr);
              cm = cm < ac ? ac : cm;
            }
          }
          st4(se + (r0 + k) * kRowElems + 4 * lane, rawn);
          stage_row_bits(sw, r0 + k, lane, nib);
        }
      }
      acc = warp_bfly_sum(acc);
      if (lane == 0) p.partials[static_cast<size_t>(sv) * p.tpc + t] = acc;
      if (stats) {
        cm = warp_max(cm);
        if (lane == 0) p.cmax[static_cast<size_t>(sv) * p.tpc + t] = cm;
      }
      flush_server_words(p, s_peer, sw, rc, i0, lane);  // local + fused allgather
      continue;
    }

    clear_tile_words(sw, lane);
    double acc = 0.0;
    float cm = 0.0f;
    for (int r = 0; r < kRowsPerTile; ++r) {
      const uint64_t ir = i0 + static_cast<uint64_t>(r) * kRowElems;
      if (ir >= p.c) break;
      const float4 raw = ld4(se + r * kRowElems + 4 * lane);
      const uint32_t snib = row_nibble(rs, r, lane);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll(NT > 0 ? NT : 1)
      for (int i = 0; i < n; ++i) {
        const float S = s_scale[wib][i];
        const uint32_t nb = (ld_cg(inw + i * p.in_i + 4 * r + (lane >> 3)) >> (4 * (lane & 7))) & 0xFu;
        if (S != 0.0f) {
          const double Sd = S;
          a0 += (nb & 1u) ? Sd : -Sd;
          a1 += (nb & 2u) ? Sd : -Sd;
          a2 += (nb & 4u) ? Sd : -Sd;
          a3 += (nb & 8u) ? Sd : -Sd;
        }
      }
      const float4 avg = make_float4(static_cast<float>(a0 * inv_n), static_cast<float>(a1 * inv_n),
                                     static_cast<float>(a2 * inv_n), static_cast<float>(a3 * inv_n));
      uint32_t nib = 0;
      float4 rawn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t i = ir + 4 * lane + q;
        const float v = comp(avg, q);
        const float rec = (snib >> q) & 1u ? S2p : -S2p;
        const float delta = __fsub_rn(comp(raw, q), rec);
        const float corr = __fadd_rn(v, __fmul_rn(es, delta));
        const float rn = __fadd_rn(v, delta);
        const bool live = i < p.c;
        set_comp(rawn, q, live ? rn : 0.0f);
        if (live) {
          nib |= static_cast<uint32_t>(corr >= 0.0f) << q;
          acc += fabs(static_cast<double>(corr));
          const float ac = fabsf(corr);
          cm = cm < ac ? ac : cm;
        }
      }
      st4(se + r * kRowElems + 4 * lane, rawn);
      stage_row_bits(sw, r, lane, nib);
    }
    acc = warp_bfly_sum(acc);
    if (lane == 0) p.partials[static_cast<size_t>(sv) * p.tpc + t] = acc;
    if (p.cmax) {
      cm = warp_max(cm);
      if (lane == 0) p.cmax[static_cast<size_t>(sv) * p.tpc + t] = cm;
    }
    flush_server_words(p, s_peer, sw, rc, i0, lane);
  }
  if (p.peer_res) warp_fence_system(lane);  // remote server words before the finalize signal
}

// Result bits of 4 consecutive global elements k0..k0+3 from chunk-relative
// packets; (j, chunk_end) track the chunk of the row start.
struct BitCursor {
  const uint32_t* res;
  uint64_t c, slot, W;
  int n;
};

__device__ __forceinline__ uint32_t bit_at(const BitCursor& bc, uint64_t k, float* S) {
  uint64_t j = k / bc.c;
  if (j >= static_cast<uint64_t>(bc.n)) j = bc.n - 1;
  const uint64_t i = k - j * bc.c;
  const uint32_t* sl = bc.res + j * bc.slot;
  *S = slot_scale_cg(sl, bc.W);
  return (__ldcg(sl + (i >> 5)) >> (i & 31)) & 1u;
}

// Values m_g = dec * invc for the lane's 4 elements of a layer row starting at
// global kr (fusion.cpp:139-145 applied to compression.cpp:68-81).
__device__ __forceinline__ float4 row_mg(const BitCursor& bc, uint64_t kr, int lane, float ic,
                                         uint64_t& j, uint64_t& chunk_end) {
  while (kr >= chunk_end) {
    ++j;
    chunk_end += bc.c;
  }
  float4 out;
  if (kr + (kRowElems - 1) < chunk_end || j + 1 >= static_cast<uint64_t>(bc.n)) {
    const uint32_t* sl = bc.res + j * bc.slot;
    const float S = slot_scale_cg(sl, bc.W);
    const float pos = S, neg = S == 0.0f ? 0.0f : -S;
    const uint64_t i = kr - j * bc.c + 4 * lane;
    const uint64_t wi = i >> 5;
    const uint32_t w0 = __ldcg(sl + wi), w1 = __ldcg(sl + wi + 1);
    const uint32_t nib = __funnelshift_r(w0, w1, static_cast<uint32_t>(i & 31)) & 0xFu;
    out.x = __fmul_rn(nib & 1u ? pos : neg, ic);
    out.y = __fmul_rn(nib & 2u ? pos : neg, ic);
    out.z = __fmul_rn(nib & 4u ? pos : neg, ic);
    out.w = __fmul_rn(nib & 8u ? pos : neg, ic);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float S;
      const uint32_t b = bit_at(bc, kr + 4 * lane + q, &S);
      set_comp(out, q, __fmul_rn(dec_value(b, S), ic));
    }
  }
  return out;
}

// Fast-path bits: the lane's 4 chunk-relative positions i..i+3 (i may sit
// anywhere inside a word) of one packet.
__device__ __forceinline__ uint32_t nibble_at(const uint32_t* sl, uint32_t i) {
  const uint32_t w0 = __ldg(sl + (i >> 5)), w1 = __ldg(sl + (i >> 5) + 1);
  return __funnelshift_r(w0, w1, i & 31u) & 0xFu;
}

// Store the lane's first nvl (0..4) elements at p (p may sit off a 16-B boundary).
__device__ __forceinline__ void st_first(float* p, const float4& v, int nvl) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q < nvl) p[q] = comp(v, q);
}

__device__ __forceinline__ int lane_valid(uint64_t len, uint64_t ir, int lane) {
  const uint64_t st = ir + 4 * lane;
  if (st >= len) return 0;
  const uint64_t rem = len - st;
  return rem >= 4 ? 4 : static_cast<int>(rem);
}

// ---------------------------------------------------------------------------
// K5 — update pass A (optimizers.cpp:271-300): reconstruct the averaged
// gradient from the momentum recurrence, refresh the live variance, per-layer
// ratio max (kernels.cpp:185-198) and ||v||^2 trace partials.
// MPREV 0: m_prev from the momentum buffer (first step after the freeze);
// MPREV 1: m_prev from the previous result packets.
// ---------------------------------------------------------------------------
#ifndef K5_ROWS
#define K5_ROWS 4
#endif
#ifndef K5_MINB
#define K5_MINB 3
#endif
template <int MPREV, bool MISK>
__global__ void __launch_bounds__(kBlock, K5_MINB) k5_update_a(const K5Params p) {
  if (gate_closed_call(p.err)) return;
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const BitCursor cur{p.res_cur, p.c, p.slot, p.W, p.n};
  const BitCursor prv{p.res_prev, p.c, p.slot, p.W, p.n};

  TileSched sch{p.lt.ctr, p.lt.tiles, nwarps, 0, p.lt.order};  // boundary tiles first
  for (long long tile = sch.first(gw, lane); tile < p.lt.tiles; tile = sch.next(lane)) {
    const int l = __ldg(p.lt.tile_layer + tile);
    const int t = static_cast<int>(tile - __ldg(p.lt.layer_tile_start + l));
    const uint64_t lo = __ldg(p.lt.off + l);
    const uint64_t len = __ldg(p.lt.off + l + 1) - lo;
    const uint64_t base = lo + static_cast<uint64_t>(t) * kTile;
    const int s = static_cast<int>(lo & 3u);
    const float ic = __ldg(p.invc + l);
    uint64_t j = base / p.c, ce = (j + 1) * p.c;
    uint64_t jp = j, cep = ce;

    const uint64_t tvalid = len - static_cast<uint64_t>(t) * kTile < kTile ? len - static_cast<uint64_t>(t) * kTile
                                                                          : static_cast<uint64_t>(kTile);
    if ((MISK || s == 0) && base + tvalid <= ce && !p.dense && !p.norm_only) {
      // Fast path: one chunk of the result (MISK: any layer alignment).  A
      // layer's partial last tile takes it too, rows past the layer end
      // skipped and the last row masked (loads past it stay in the slack).
      constexpr int R = K5_ROWS;
      const bool part = tvalid < static_cast<uint64_t>(kTile);
      const int rows_valid = static_cast<int>((tvalid + kRowElems - 1) / kRowElems);
      const uint32_t* sl = cur.res + j * p.slot;
      const float S = slot_scale_cg(sl, p.W);
      const float pos = S, neg = S == 0.0f ? 0.0f : -S;
      const uint32_t* slp = MPREV ? prv.res + j * p.slot : nullptr;
      float posp = 0.f, negp = 0.f;
      if (MPREV) {
        const float Sq = slot_scale(slp, p.W);
        posp = Sq;
        negp = Sq == 0.0f ? 0.0f : -Sq;
      }
      const uint32_t ib = static_cast<uint32_t>(base - j * p.c) + 4 * lane;
      double acc = 0.0;
      float mx = 0.0f;
      bool bad = false;
      auto rows = [&](auto mis, auto partial) {
        constexpr bool MIS = decltype(mis)::value;
        constexpr bool PART = decltype(partial)::value;
        for (int r0 = 0; r0 < (PART ? rows_valid : kRowsPerTile); r0 += R) {
          float4 v[R], vf[R], mpb[R];
          uint32_t nc[R], np[R];
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const float* row = p.v + base + (r0 + k) * kRowElems + 4 * lane;
            v[k] = ld_rw_s<MIS>(row, s);
            vf[k] = ld_ro_s<MIS>(p.vf + base + (r0 + k) * kRowElems + 4 * lane, s);
            nc[k] = nibble_cg(sl, ib + (r0 + k) * kRowElems);
            if (MPREV) np[k] = nibble_at(slp, ib + (r0 + k) * kRowElems);
            else mpb[k] = ld_ro_s<MIS>(p.m + base + (r0 + k) * kRowElems + 4 * lane, s);
          }
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const int nvl = PART ? lane_valid(tvalid, static_cast<uint64_t>(r0 + k) * kRowElems, lane) : 4;
            float4 vn;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              // inv * m_g and ninvb * m_prev take two values each per tile: hoisted (same products)
              const float gp = __fmul_rn(p.inv, __fmul_rn(pos, ic)), gn = __fmul_rn(p.inv, __fmul_rn(neg, ic));
              const float pp = __fmul_rn(p.ninvb, __fmul_rn(posp, ic)), pn = __fmul_rn(p.ninvb, __fmul_rn(negp, ic));
              const float rec = __fadd_rn((nc[k] >> q) & 1u ? gp : gn,
                                          MPREV ? ((np[k] >> q) & 1u ? pp : pn) : __fmul_rn(p.ninvb, comp(mpb[k], q)));
              const float nvv = __fadd_rn(__fmul_rn(p.b2, comp(v[k], q)),
                                          __fmul_rn(__fmul_rn(p.omb2, rec), rec));
              set_comp(vn, q, nvv);
              if (!PART || q < nvl) {
                bad |= !isfinite(rec);
                const float den = nvv < p.floor_ ? p.floor_ : nvv;
                const float ratio = fabsf(comp(vf[k], q)) / den;
                mx = mx < ratio ? ratio : mx;
                acc += static_cast<double>(nvv) * static_cast<double>(nvv);
              }
            }
            float* dst = p.v + base + (r0 + k) * kRowElems + 4 * lane;
            if (!PART || nvl == 4) {
              st_s<MIS>(dst, s, vn);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (q < nvl) dst[q] = comp(vn, q);
            }
          }
        }
      };
      // MIS accessors only for a layer off a 16-B boundary (they assume s != 0)
      if constexpr (MISK) {
        if (s != 0) {
          if (part) rows(Mis<true>{}, Mis<true>{});
          else rows(Mis<true>{}, Mis<false>{});
        } else {
          if (part) rows(Mis<false>{}, Mis<true>{});
          else rows(Mis<false>{}, Mis<false>{});
        }
      } else {
        if (part) rows(Mis<false>{}, Mis<true>{});
        else rows(Mis<false>{}, Mis<false>{});
      }
      if (bad) flag(p.err, kErrRecon, static_cast<unsigned long long>(l));
      acc = warp_bfly_sum(acc);
      mx = warp_max(mx);
      if (lane == 0) {
        p.tile_v2[tile] = acc;
        p.tile_max[tile] = mx;
      }
      continue;
    }

    if (p.gen_list) continue;  // taken by k5_general
    double acc = 0.0;
    float mx = 0.0f;
    bool bad = false;
    for (int r = 0; r < kRowsPerTile; ++r) {
      const uint64_t ir = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(r) * kRowElems;
      if (ir >= len) break;
      const uint64_t kr = base + static_cast<uint64_t>(r) * kRowElems;
      const int nv = lane_valid(len, ir, lane);
      const float4 v = ld_row4<false>(p.v + kr, lane, s);
      if (p.norm_only) {  // optimizers.cpp:324 trace ||v|| only (v is not updated)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < nv) acc += static_cast<double>(comp(v, q)) * static_cast<double>(comp(v, q));
        if (p.m_store) {  // identity compressor: m = m_g (:319)
          const float4 dv = ld_row4<false>(p.dense + kr, lane, s);
          float4 mg;
#pragma unroll
          for (int q = 0; q < 4; ++q) set_comp(mg, q, __fmul_rn(comp(dv, q), ic));
          st_row4(p.m_store + kr, lane, s, mg, nv);
        }
        continue;
      }
      const float4 vf = ld_row4<false>(p.vf + kr, lane, s);
      float4 mg;
      if (p.dense) {
        const float4 dv = ld_row4<false>(p.dense + kr, lane, s);
#pragma unroll
        for (int q = 0; q < 4; ++q) set_comp(mg, q, __fmul_rn(comp(dv, q), ic));  // fusion.cpp:143
      } else {
        mg = row_mg(cur, kr, lane, ic, j, ce);
      }
      float4 mp;
      if (MPREV == 0) mp = ld_row4<false>(p.m + kr, lane, s);
      else mp = row_mg(prv, kr, lane, ic, jp, cep);
      if (p.m_store) st_row4(p.m_store + kr, lane, s, mg, nv);  // m = m_g (:319)
      float4 vn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // :284-287 rec = inv*m_g + (-beta1*inv)*m_prev
        const float rec = __fadd_rn(__fmul_rn(p.inv, comp(mg, q)), __fmul_rn(p.ninvb, comp(mp, q)));
        // kernels.cpp:245 y = a*y + b*x*x
        const float nvv = __fadd_rn(__fmul_rn(p.b2, comp(v, q)),
                                    __fmul_rn(__fmul_rn(p.omb2, rec), rec));
        set_comp(vn, q, nvv);
        if (q < nv) {
          bad |= !isfinite(rec);
          const float den = nvv < p.floor_ ? p.floor_ : nvv;  // std::max(v, floor)
          const float ratio = fabsf(comp(vf, q)) / den;
          mx = mx < ratio ? ratio : mx;
          acc += static_cast<double>(nvv) * static_cast<double>(nvv);
        }
      }
      st_row4(p.v + kr, lane, s, vn, nv);
    }
    if (bad) flag(p.err, kErrRecon, static_cast<unsigned long long>(l));
    acc = warp_bfly_sum(acc);
    mx = warp_max(mx);
    if (lane == 0) {
      p.tile_v2[tile] = acc;
      p.tile_max[tile] = mx;
    }
  }
}

// Per-layer epilogue between K5 and K6 (optimizers.cpp:296-300, 317, 321-330):
// one 1024-thread block per layer; the last block also advances the
// c_mean history (:328-330) and the experimental error scale (:226-229).
__global__ void __launch_bounds__(1024) k_epilogue(const EpiParams p) {
  if (gate_closed_call(p.gate)) return;
  __shared__ double shd[32];
  __shared__ float shf[32];
  __shared__ bool last;
  const int l = blockIdx.x;
  const int t0 = p.layer_tile_start[l], t1 = p.layer_tile_start[l + 1];
  double s = stripe_sum(p.tile_v2, t0 + threadIdx.x, t1);
  float mx = 0.0f;
  for (int t = t0 + threadIdx.x; t < t1; t += 1024) {
    const float m = p.tile_max[t];
    mx = mx < m ? m : mx;
  }
  s = block1024_sum(s, shd);
  mx = block1024_max(mx, shf);
  if (threadIdx.x == 0) {
    const int L = p.L;
    double pre = 1.0, r = 1.0, c = 1.0;
    if (p.mode == 0) {
      pre = static_cast<double>(mx);
      const double rp = p.r_prev[l];
      // vector_ops.cpp:25-28 clip = min(max(x, a), b)
      const double lo1 = (1.0 - p.r_thr) * rp, hi1 = (1.0 + p.r_thr) * rp;
      r = pre < lo1 ? lo1 : pre;
      r = hi1 < r ? hi1 : r;
      r = r < p.r_min ? p.r_min : r;
      r = p.r_max < r ? p.r_max : r;
      c = r * p.c_avg[l];
      p.r_prev[l] = r;
    } else if (p.mode == 1) {
      c = p.c_avg[l];  // optimizers.cpp:301-303
    }
    const double lr = p.lr_dev ? *p.lr_dev : p.lr;
    p.coef_x[l] = static_cast<float>(-lr * c);
    p.trace[l] = c;
    p.trace[L + l] = r;
    p.trace[2 * L + l] = sqrt(s);
    p.trace[3 * L + l] = pre;
    __threadfence();
    last = atomicAdd(p.counter, 1u) == static_cast<unsigned>(L - 1);
  }
  __syncthreads();
  if (!last) return;
  // c_mean over layers, added in ascending layer order by one thread; the
  // whole block stages 1024 layers' c at a time in shared memory (one L2
  // round trip per 1024 layers instead of one per 8).
  __shared__ double s_c[1024];
  __threadfence();
  double c_sum = 0.0;
  for (int k0 = 0; k0 < p.L; k0 += 1024) {
    const int cnt = p.L - k0 < 1024 ? p.L - k0 : 1024;
    if (static_cast<int>(threadIdx.x) < cnt) s_c[threadIdx.x] = __ldcg(p.trace + k0 + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < cnt; ++q) c_sum += s_c[q];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.cmean[1] = p.cmean[0];
    const double cm = c_sum / static_cast<double>(p.L);
    p.cmean[0] = cm < p.floor_ ? p.floor_ : cm;
    *p.es_next = p.scaled_ef ? static_cast<float>(p.cmean[1] / p.cmean[0]) : 1.0f;
    *p.counter = 0u;
  }
}

// K6 — update pass B (optimizers.cpp:308-313): u = m_g/(sqrt(vf)+eta) [+wd x],
// x += (-lr*c)*u, with m_g recomputed from the result packets.
template <bool MISK>
#ifndef K6_MINB
#define K6_MINB 1
#endif
__global__ void __launch_bounds__(kBlock, K6_MINB) k6_update_b(const K6Params p) {
  if (gate_closed_call(p.gate)) return;
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const BitCursor cur{p.res_cur, p.c, p.slot, p.W, p.n};
  TileSched sch{p.lt.ctr, p.lt.tiles, nwarps, 0, p.lt.order};  // boundary tiles first
  for (long long tile = sch.first(gw, lane); tile < p.lt.tiles; tile = sch.next(lane)) {
    const int l = __ldg(p.lt.tile_layer + tile);
    const int t = static_cast<int>(tile - __ldg(p.lt.layer_tile_start + l));
    const uint64_t lo = __ldg(p.lt.off + l);
    const uint64_t len = __ldg(p.lt.off + l + 1) - lo;
    const uint64_t base = lo + static_cast<uint64_t>(t) * kTile;
    const int s = static_cast<int>(lo & 3u);
    const float ic = __ldg(p.invc + l);
    const float a = __ldg(p.coef_x + l);
    uint64_t j = base / p.c, ce = (j + 1) * p.c;
    const uint64_t tvalid = len - static_cast<uint64_t>(t) * kTile < kTile ? len - static_cast<uint64_t>(t) * kTile
                                                                          : static_cast<uint64_t>(kTile);
    if ((MISK || s == 0) && base + tvalid <= ce && !p.dense) {
      // One chunk of the result; a partial last tile skips the rows past the
      // layer end and masks its last row (K5's fast path, same treatment).
      constexpr int R = 4;
      const bool part = tvalid < static_cast<uint64_t>(kTile);
      const int rows_valid = static_cast<int>((tvalid + kRowElems - 1) / kRowElems);
      const uint32_t* sl = cur.res + j * p.slot;
      const float S = slot_scale(sl, p.W);
      const float pos = S, neg = S == 0.0f ? 0.0f : -S;
      const uint32_t ib = static_cast<uint32_t>(base - j * p.c) + 4 * lane;
      auto rows = [&](auto mis, auto partial) {
        constexpr bool MIS = decltype(mis)::value;
        constexpr bool PART = decltype(partial)::value;
        for (int r0 = 0; r0 < (PART ? rows_valid : kRowsPerTile); r0 += R) {
          float4 x[R], vf[R];
          uint32_t nc[R];
#pragma unroll
          for (int k = 0; k < R; ++k) {
            x[k] = ld_rw_s<MIS>(p.x + base + (r0 + k) * kRowElems + 4 * lane, s);
            vf[k] = ld_ro_s<MIS>(p.vf + base + (r0 + k) * kRowElems + 4 * lane, s);
            nc[k] = nibble_at(sl, ib + (r0 + k) * kRowElems);
          }
#pragma unroll
          for (int k = 0; k < R; ++k) {
            float4 xn;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float mgp = __fmul_rn(pos, ic), mgn = __fmul_rn(neg, ic);  // hoisted (same products)
              const float mg = (nc[k] >> q) & 1u ? mgp : mgn;
              float u = __fdiv_rn(mg, __fadd_rn(__fsqrt_rn(comp(vf[k], q)), p.eta));
              if (p.wd > 0.0f) u = __fadd_rn(u, __fmul_rn(p.wd, comp(x[k], q)));
              set_comp(xn, q, __fadd_rn(comp(x[k], q), __fmul_rn(a, u)));
            }
            float* dst = p.x + base + (r0 + k) * kRowElems + 4 * lane;
            const int nvl = PART ? lane_valid(tvalid, static_cast<uint64_t>(r0 + k) * kRowElems, lane) : 4;
            if (!PART || nvl == 4) {
              st_s<MIS>(dst, s, xn);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (q < nvl) dst[q] = comp(xn, q);
            }
          }
        }
      };
      // MIS accessors only for a layer off a 16-B boundary (they assume s != 0)
      if constexpr (MISK) {
        if (s != 0) {
          if (part) rows(Mis<true>{}, Mis<true>{});
          else rows(Mis<true>{}, Mis<false>{});
        } else {
          if (part) rows(Mis<false>{}, Mis<true>{});
          else rows(Mis<false>{}, Mis<false>{});
        }
      } else {
        if (part) rows(Mis<false>{}, Mis<true>{});
        else rows(Mis<false>{}, Mis<false>{});
      }
      continue;
    }
    if (p.gen_list) continue;  // taken by k6_general
    for (int r = 0; r < kRowsPerTile; ++r) {
      const uint64_t ir = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(r) * kRowElems;
      if (ir >= len) break;
      const uint64_t kr = base + static_cast<uint64_t>(r) * kRowElems;
      const int nv = lane_valid(len, ir, lane);
      const float4 x = ld_row4<false>(p.x + kr, lane, s);
      const float4 vf = ld_row4<false>(p.vf + kr, lane, s);
      float4 mg;
      if (p.dense) {
        const float4 dv = ld_row4<false>(p.dense + kr, lane, s);
#pragma unroll
        for (int q = 0; q < 4; ++q) set_comp(mg, q, __fmul_rn(comp(dv, q), ic));
      } else {
        mg = row_mg(cur, kr, lane, ic, j, ce);
      }
      float4 xn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // kernels.cpp:229 precondition: m / (sqrt(v) + eta)
        float u = __fdiv_rn(comp(mg, q), __fadd_rn(__fsqrt_rn(comp(vf, q)), p.eta));
        if (p.wd > 0.0f) u = __fadd_rn(u, __fmul_rn(p.wd, comp(x, q)));  // kernels.cpp:226 axpy
        set_comp(xn, q, __fadd_rn(comp(x, q), __fmul_rn(a, u)));          // :313 axpy
      }
      st_row4(p.x + kr, lane, s, xn, nv);
    }
  }
}

// ---------------------------------------------------------------------------
// General-path tiles of K5 / K6 for small problems (a tile across a chunk
// boundary, or a layer off a 16-B boundary without the MISK kernels): one
// warp per listed tile, on a side stream while the streaming kernel skips
// them.  Such a tile is a chain of dependent rows; here every load of a
// 4-row batch is issued first (branch-free: raw words and rows, decoded
// after), so a batch costs one memory round trip instead of two per row.
// Same per-element arithmetic and accumulation order as the streaming
// kernels' general path (row_mg / ld_row4).
// ---------------------------------------------------------------------------
struct RowRaw {   // ld_row4's loads, not yet rotated
  float4 lo, hi;
};
__device__ __forceinline__ RowRaw row_issue(const float* row, int lane, int s) {
  const float* a = row - s;
  RowRaw r;
  r.lo = ld4(a + 4 * lane);
  r.hi = (s != 0 && lane == 31) ? ld4(a + 128) : make_float4(0.f, 0.f, 0.f, 0.f);
  return r;
}
__device__ __forceinline__ float4 row_finish(const RowRaw& r, int lane, int s) {  // = ld_row4
  if (s == 0) return r.lo;
  float hx = __shfl_down_sync(FULL, r.lo.x, 1);
  float hy = __shfl_down_sync(FULL, r.lo.y, 1);
  float hz = __shfl_down_sync(FULL, r.lo.z, 1);
  if (lane == 31) {
    hx = r.hi.x;
    hy = r.hi.y;
    hz = r.hi.z;
  }
  if (s == 1) return make_float4(r.lo.y, r.lo.z, r.lo.w, hx);
  if (s == 2) return make_float4(r.lo.z, r.lo.w, hx, hy);
  return make_float4(r.lo.w, hx, hy, hz);
}
struct BitsRaw {  // row_mg's loads, not yet decoded
  uint32_t w0, w1, sw, sh;
  uint64_t j;
  bool cross;     // the row straddles a chunk end: decoded element by element
};
__device__ __forceinline__ BitsRaw bits_issue(const BitCursor& bc, uint64_t kr, int lane, uint64_t& j,
                                              uint64_t& chunk_end) {
  while (kr >= chunk_end) {
    ++j;
    chunk_end += bc.c;
  }
  BitsRaw b;
  b.j = j;
  b.cross = !(kr + (kRowElems - 1) < chunk_end || j + 1 >= static_cast<uint64_t>(bc.n));
  const uint32_t* sl = bc.res + j * bc.slot;
  const uint64_t i = kr - j * bc.c + 4 * lane;
  b.sh = static_cast<uint32_t>(i & 31);
  b.sw = __ldcg(sl + bc.W);
  b.w0 = __ldcg(sl + (i >> 5));
  b.w1 = __ldcg(sl + (i >> 5) + 1);
  return b;
}
__device__ __forceinline__ float4 bits_finish(const BitCursor& bc, const BitsRaw& b, uint64_t kr, int lane,
                                              float ic) {  // = row_mg
  float4 out;
  if (!b.cross) {
    const float S = __uint_as_float(b.sw);
    const float pos = S, neg = S == 0.0f ? 0.0f : -S;
    const uint32_t nib = __funnelshift_r(b.w0, b.w1, b.sh) & 0xFu;
    out.x = __fmul_rn(nib & 1u ? pos : neg, ic);
    out.y = __fmul_rn(nib & 2u ? pos : neg, ic);
    out.z = __fmul_rn(nib & 4u ? pos : neg, ic);
    out.w = __fmul_rn(nib & 8u ? pos : neg, ic);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float S;
      const uint32_t bit = bit_at(bc, kr + 4 * lane + q, &S);
      set_comp(out, q, __fmul_rn(dec_value(bit, S), ic));
    }
  }
  return out;
}

template <int MPREV>
__global__ void __launch_bounds__(kBlock) k5_general(const K5Params p) {
  if (gate_closed_call(p.err)) return;
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const BitCursor cur{p.res_cur, p.c, p.slot, p.W, p.n};
  const BitCursor prv{p.res_prev, p.c, p.slot, p.W, p.n};
  for (long long i = gw; i < p.gen_count; i += nwarps) {
    const long long tile = __ldg(p.gen_list + i);
    const int l = __ldg(p.lt.tile_layer + tile);
    const int t = static_cast<int>(tile - __ldg(p.lt.layer_tile_start + l));
    const uint64_t lo = __ldg(p.lt.off + l);
    const uint64_t len = __ldg(p.lt.off + l + 1) - lo;
    const uint64_t base = lo + static_cast<uint64_t>(t) * kTile;
    const int s = static_cast<int>(lo & 3u);
    const float ic = __ldg(p.invc + l);
    uint64_t j = base / p.c, ce = (j + 1) * p.c;
    uint64_t jp = j, cep = ce;
    double acc = 0.0;
    float mx = 0.0f;
    bool bad = false;
    constexpr int RB = 4;
    for (int r0 = 0; r0 < kRowsPerTile; r0 += RB) {
      const uint64_t ir0 = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(r0) * kRowElems;
      if (ir0 >= len) break;
      const int nrow = static_cast<int>((len - ir0 + kRowElems - 1) / kRowElems);  // rows left in the layer
      RowRaw rv[RB], rf[RB], rm[RB];
      BitsRaw bc[RB], bp[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) {  // loads only
        const uint64_t kr = base + static_cast<uint64_t>(r0 + k) * kRowElems;
        if (k >= nrow) break;
        rv[k] = row_issue(p.v + kr, lane, s);
        rf[k] = row_issue(p.vf + kr, lane, s);
        bc[k] = bits_issue(cur, kr, lane, j, ce);
        if (MPREV == 0) rm[k] = row_issue(p.m + kr, lane, s);
        else bp[k] = bits_issue(prv, kr, lane, jp, cep);
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        if (k >= nrow) break;
        const uint64_t ir = ir0 + static_cast<uint64_t>(k) * kRowElems;
        const uint64_t kr = base + static_cast<uint64_t>(r0 + k) * kRowElems;
        const int nv = lane_valid(len, ir, lane);
        const float4 v = row_finish(rv[k], lane, s);
        const float4 vf = row_finish(rf[k], lane, s);
        const float4 mg = bits_finish(cur, bc[k], kr, lane, ic);
        const float4 mp = MPREV == 0 ? row_finish(rm[k], lane, s) : bits_finish(prv, bp[k], kr, lane, ic);
        float4 vn;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // :284-287 rec = inv*m_g + (-beta1*inv)*m_prev
          const float rec = __fadd_rn(__fmul_rn(p.inv, comp(mg, q)), __fmul_rn(p.ninvb, comp(mp, q)));
          // kernels.cpp:245 y = a*y + b*x*x
          const float nvv = __fadd_rn(__fmul_rn(p.b2, comp(v, q)),
                                      __fmul_rn(__fmul_rn(p.omb2, rec), rec));
          set_comp(vn, q, nvv);
          if (q < nv) {
            bad |= !isfinite(rec);
            const float den = nvv < p.floor_ ? p.floor_ : nvv;  // std::max(v, floor)
            const float ratio = fabsf(comp(vf, q)) / den;
            mx = mx < ratio ? ratio : mx;
            acc += static_cast<double>(nvv) * static_cast<double>(nvv);
          }
        }
        st_row4(p.v + kr, lane, s, vn, nv);
      }
    }
    if (bad) flag(p.err, kErrRecon, static_cast<unsigned long long>(l));
    acc = warp_bfly_sum(acc);
    mx = warp_max(mx);
    if (lane == 0) {
      p.tile_v2[tile] = acc;
      p.tile_max[tile] = mx;
    }
  }
}

__global__ void __launch_bounds__(kBlock) k6_general(const K6Params p) {
  if (gate_closed_call(p.gate)) return;
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const BitCursor cur{p.res_cur, p.c, p.slot, p.W, p.n};
  for (long long i = gw; i < p.gen_count; i += nwarps) {
    const long long tile = __ldg(p.gen_list + i);
    const int l = __ldg(p.lt.tile_layer + tile);
    const int t = static_cast<int>(tile - __ldg(p.lt.layer_tile_start + l));
    const uint64_t lo = __ldg(p.lt.off + l);
    const uint64_t len = __ldg(p.lt.off + l + 1) - lo;
    const uint64_t base = lo + static_cast<uint64_t>(t) * kTile;
    const int s = static_cast<int>(lo & 3u);
    const float ic = __ldg(p.invc + l);
    const float a = __ldg(p.coef_x + l);
    uint64_t j = base / p.c, ce = (j + 1) * p.c;
    constexpr int RB = 4;
    for (int r0 = 0; r0 < kRowsPerTile; r0 += RB) {
      const uint64_t ir0 = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(r0) * kRowElems;
      if (ir0 >= len) break;
      const int nrow = static_cast<int>((len - ir0 + kRowElems - 1) / kRowElems);
      RowRaw rx[RB], rf[RB];
      BitsRaw bc[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const uint64_t kr = base + static_cast<uint64_t>(r0 + k) * kRowElems;
        if (k >= nrow) break;
        rx[k] = row_issue(p.x + kr, lane, s);
        rf[k] = row_issue(p.vf + kr, lane, s);
        bc[k] = bits_issue(cur, kr, lane, j, ce);
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        if (k >= nrow) break;
        const uint64_t ir = ir0 + static_cast<uint64_t>(k) * kRowElems;
        const uint64_t kr = base + static_cast<uint64_t>(r0 + k) * kRowElems;
        const int nv = lane_valid(len, ir, lane);
        const float4 x = row_finish(rx[k], lane, s);
        const float4 vf = row_finish(rf[k], lane, s);
        const float4 mg = bits_finish(cur, bc[k], kr, lane, ic);
        float4 xn;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // kernels.cpp:229 precondition: m / (sqrt(v) + eta)
          float u = __fdiv_rn(comp(mg, q), __fadd_rn(__fsqrt_rn(comp(vf, q)), p.eta));
          if (p.wd > 0.0f) u = __fadd_rn(u, __fmul_rn(p.wd, comp(x, q)));  // kernels.cpp:226 axpy
          set_comp(xn, q, __fadd_rn(comp(x, q), __fmul_rn(a, u)));          // :313 axpy
        }
        st_row4(p.x + kr, lane, s, xn, nv);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Warmup stage (optimizers.cpp:140-177 lamb_step / :179-200 adam_step).
// W1: m, v update; tile partials of ||x||^2 (pre-update), ||u||^2, ||v||^2 and
// sum|m| (compute_scales, fusion.cpp:107-125, used when the stage ends).
// ---------------------------------------------------------------------------
template <bool MISK>
__global__ void __launch_bounds__(kBlock) kw1_warmup_a(const W1Params p) {
  if (gate_closed_call(p.gate)) return;
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  TileSchedSub sch{p.lt.ctr, p.lt.count ? p.lt.count : p.lt.tiles, nwarps, 0, p.lt.order};  // boundary first
  for (long long tile = sch.first(gw, lane); tile < p.lt.tiles; tile = sch.next(lane)) {
    const int l = __ldg(p.lt.tile_layer + tile);
    const int t = static_cast<int>(tile - __ldg(p.lt.layer_tile_start + l));
    const uint64_t lo = __ldg(p.lt.off + l);
    const uint64_t len = __ldg(p.lt.off + l + 1) - lo;
    const uint64_t base = lo + static_cast<uint64_t>(t) * kTile;
    const int s = static_cast<int>(lo & 3u);
    double ax = 0.0, au = 0.0, av = 0.0, am = 0.0;
    const uint64_t tvalid = len - static_cast<uint64_t>(t) * kTile < kTile ? len - static_cast<uint64_t>(t) * kTile
                                                                          : static_cast<uint64_t>(kTile);
    if (MISK || s == 0) {
      // Fast path: 4 rows per batch, loads issued first; a partial last tile
      // skips the rows past the layer end and masks its last row.
      const bool part = tvalid < static_cast<uint64_t>(kTile);
      const int rows_valid = static_cast<int>((tvalid + kRowElems - 1) / kRowElems);
      auto rows = [&](auto mis, auto partial) {
        constexpr bool MIS = decltype(mis)::value;
        constexpr bool PART = decltype(partial)::value;
        constexpr int R = 4;
        for (int r0 = 0; r0 < (PART ? rows_valid : kRowsPerTile); r0 += R) {
          float4 g[R], m[R], v[R], x[R];
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const uint64_t o = base + (r0 + k) * kRowElems + 4 * lane;
            g[k] = ld_ro_s<MIS>(p.gbar + o, s);
            m[k] = ld_rw_s<MIS>(p.m + o, s);
            v[k] = ld_rw_s<MIS>(p.v + o, s);
            x[k] = ld_ro_s<MIS>(p.x + o, s);
          }
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const int nvl = PART ? lane_valid(tvalid, static_cast<uint64_t>(r0 + k) * kRowElems, lane) : 4;
            if (p.err && !(isfinite(g[k].x) && isfinite(g[k].y) && isfinite(g[k].z) && isfinite(g[k].w))) {
              for (int q = 0; q < 4; ++q)
                if ((!PART || q < nvl) && !isfinite(comp(g[k], q)))
                  flag(p.err, kErrGrad, (static_cast<unsigned long long>(p.worker_base) << 40) |
                                            (base + (r0 + k) * kRowElems + 4 * lane + q));
            }
            float4 mn, vn;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float gq = comp(g[k], q);
              const float mq = __fadd_rn(__fmul_rn(p.b1, comp(m[k], q)), __fmul_rn(p.omb1, gq));
              const float vq =
                  __fadd_rn(__fmul_rn(p.b2, comp(v[k], q)), __fmul_rn(__fmul_rn(p.omb2, gq), gq));
              set_comp(mn, q, mq);
              set_comp(vn, q, vq);
              float u = __fdiv_rn(mq, __fadd_rn(__fsqrt_rn(vq), p.eta));
              if (p.wd > 0.0f) u = __fadd_rn(u, __fmul_rn(p.wd, comp(x[k], q)));
              if (!PART || q < nvl) {
                const double xd = comp(x[k], q), ud = u, vd = vq;
                ax += xd * xd;
                au += ud * ud;
                av += vd * vd;
                am += fabs(static_cast<double>(mq));
              }
            }
            const uint64_t o = base + (r0 + k) * kRowElems + 4 * lane;
            if (!PART || nvl == 4) {
              st_s<MIS>(p.m + o, s, mn);
              st_s<MIS>(p.v + o, s, vn);
            } else {
              st_first(p.m + o, mn, nvl);
              st_first(p.v + o, vn, nvl);
            }
          }
        }
      };
      // MIS accessors only for a layer off a 16-B boundary (they assume s != 0)
      if constexpr (MISK) {
        if (s != 0) {
          if (part) rows(Mis<true>{}, Mis<true>{});
          else rows(Mis<true>{}, Mis<false>{});
        } else {
          if (part) rows(Mis<false>{}, Mis<true>{});
          else rows(Mis<false>{}, Mis<false>{});
        }
      } else {
        if (part) rows(Mis<false>{}, Mis<true>{});
        else rows(Mis<false>{}, Mis<false>{});
      }
    } else
    for (int r = 0; r < kRowsPerTile; ++r) {
      const uint64_t ir = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(r) * kRowElems;
      if (ir >= len) break;
      const uint64_t kr = base + static_cast<uint64_t>(r) * kRowElems;
      const int nv = lane_valid(len, ir, lane);
      const float4 g = ld_row4<false>(p.gbar + kr, lane, s);
      const float4 m = ld_row4<false>(p.m + kr, lane, s);
      const float4 v = ld_row4<false>(p.v + kr, lane, s);
      const float4 x = ld_row4<false>(p.x + kr, lane, s);
      float4 mn, vn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float gq = comp(g, q);
        if (p.err && q < nv && !isfinite(gq))
          flag(p.err, kErrGrad, (static_cast<unsigned long long>(p.worker_base) << 40) |
                                    (kr + 4 * lane + q));
        // kernels.cpp:238 axpby y = a*y + b*x ; :245 axpby_square
        const float mq = __fadd_rn(__fmul_rn(p.b1, comp(m, q)), __fmul_rn(p.omb1, gq));
        const float vq = __fadd_rn(__fmul_rn(p.b2, comp(v, q)), __fmul_rn(__fmul_rn(p.omb2, gq), gq));
        set_comp(mn, q, mq);
        set_comp(vn, q, vq);
        if (q < nv) {
          float u = __fdiv_rn(mq, __fadd_rn(__fsqrt_rn(vq), p.eta));
          if (p.wd > 0.0f) u = __fadd_rn(u, __fmul_rn(p.wd, comp(x, q)));
          const double xd = comp(x, q), ud = u, vd = vq;
          ax += xd * xd;
          au += ud * ud;
          av += vd * vd;
          am += fabs(static_cast<double>(mq));
        }
      }
      st_row4(p.m + kr, lane, s, mn, nv);
      st_row4(p.v + kr, lane, s, vn, nv);
    }
    ax = warp_bfly_sum(ax);
    au = warp_bfly_sum(au);
    av = warp_bfly_sum(av);
    am = warp_bfly_sum(am);
    if (lane == 0) {
      double* ts = p.tile_sums + 4 * tile;
      ts[0] = ax;
      ts[1] = au;
      ts[2] = av;
      ts[3] = am;
    }
  }
}

// Warmup epilogue: per-layer coefficient (optimizers.cpp:158-172) and, at
// the end of the stage, finalize_warmup (:202-224) in the last block.
__global__ void __launch_bounds__(1024) k_wepilogue(const WEpiParams p) {
  if (gate_closed_call(p.gate)) return;
  __shared__ double shd[32];
  __shared__ bool last;
  const int l = p.layer_list ? p.layer_list[blockIdx.x] : blockIdx.x;  // sub-launch: a layer subset
  const int t0 = p.layer_tile_start[l], t1 = p.layer_tile_start[l + 1];
  const long long a0 = 4ll * (t0 + threadIdx.x), a1 = 4ll * t1;
  double sx = stripe_sum<4096>(p.tile_sums + 0, a0, a1);
  double su = stripe_sum<4096>(p.tile_sums + 1, a0, a1);
  double sv = stripe_sum<4096>(p.tile_sums + 2, a0, a1);
  double sm = stripe_sum<4096>(p.tile_sums + 3, a0, a1);
  sx = block1024_sum(sx, shd);
  su = block1024_sum(su, shd);
  sv = block1024_sum(sv, shd);
  sm = block1024_sum(sm, shd);
  if (threadIdx.x == 0) {
    const int L = p.L;
    double c = 1.0;
    if (!p.adam) {
      const double xn = sqrt(sx), un = sqrt(su);
      auto clip = [](double x, double a, double b) {
        const double y = x < a ? a : x;
        return b < y ? b : y;
      };
      if (un == 0.0) c = xn > 0.0 ? p.c_max : clip(1.0, p.c_min, p.c_max);
      else c = clip(xn / un, p.c_min, p.c_max);
      p.coef_x[l] = static_cast<float>(-p.lr * c);
      if (p.track) p.c_avg[l] = p.b3 * p.c_avg[l] + (1.0 - p.b3) * c;
    } else {
      p.coef_x[l] = static_cast<float>(-p.lr);
    }
    p.trace[l] = c;
    p.trace[L + l] = 1.0;
    p.trace[2 * L + l] = sqrt(sv);
    p.trace[3 * L + l] = 1.0;
    if (p.finalize) {
      const double len = static_cast<double>(p.off[l + 1] - p.off[l]);
      const double mean = sm / len;                     // vector_ops.cpp:41-44 mean_abs
      p.mag[l] = mean < p.floor_ ? p.floor_ : mean;     // fusion.cpp:116
    }
    __threadfence();
    last = atomicAdd(p.counter, 1u) == static_cast<unsigned>(L - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    if (p.finalize) {
      const volatile double* mag = p.mag;
      const volatile double* cav = p.c_avg;
      if (!p.onebit_adam) {
        double ref = 0.0;
        for (int k = 0; k < p.L; ++k) ref += mag[k];
        ref /= static_cast<double>(p.L);
        for (int k = 0; k < p.L; ++k) p.coeff[k] = ref / mag[k];
      } else {
        for (int k = 0; k < p.L; ++k) p.coeff[k] = 1.0;
      }
      double c_mean = 0.0;
      for (int k = 0; k < p.L; ++k) c_mean += p.onebit_adam ? 1.0 : cav[k];
      c_mean /= static_cast<double>(p.L);
      const double cm = c_mean < p.floor_ ? p.floor_ : c_mean;
      p.cmean[0] = cm;
      p.cmean[1] = cm;
      *p.es_next = 1.0f;
      for (int k = 0; k < p.L; ++k) {
        const double co = p.coeff[k];
        p.A[k] = static_cast<float>(co * p.b1);          // optimizers.cpp:252
        p.B[k] = static_cast<float>(co * (1.0 - p.b1));  // :253
        p.invc[k] = static_cast<float>(1.0 / co);        // fusion.cpp:143
      }
    }
    *p.counter = 0u;
  }
}

// W2: u = m/(sqrt(v)+eta) [+wd x]; x += (-lr*c)*u; at the freeze vf = v.
template <bool MISK>
__global__ void __launch_bounds__(kBlock) kw2_warmup_b(const W2Params p) {
  if (gate_closed_call(p.gate)) return;
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  TileSchedSub sch{p.lt.ctr, p.lt.count ? p.lt.count : p.lt.tiles, nwarps, 0, p.lt.order};  // boundary first
  for (long long tile = sch.first(gw, lane); tile < p.lt.tiles; tile = sch.next(lane)) {
    const int l = __ldg(p.lt.tile_layer + tile);
    const int t = static_cast<int>(tile - __ldg(p.lt.layer_tile_start + l));
    const uint64_t lo = __ldg(p.lt.off + l);
    const uint64_t len = __ldg(p.lt.off + l + 1) - lo;
    const uint64_t base = lo + static_cast<uint64_t>(t) * kTile;
    const int s = static_cast<int>(lo & 3u);
    const float a = __ldg(p.coef_x + l);
    const uint64_t tvalid = len - static_cast<uint64_t>(t) * kTile < kTile ? len - static_cast<uint64_t>(t) * kTile
                                                                          : static_cast<uint64_t>(kTile);
    if (MISK || s == 0) {
      // Batched rows; a partial last tile skips the rows past the layer end
      // and masks its last row.
      const bool part = tvalid < static_cast<uint64_t>(kTile);
      const int rows_valid = static_cast<int>((tvalid + kRowElems - 1) / kRowElems);
      auto rows = [&](auto mis, auto partial) {
        constexpr bool MIS = decltype(mis)::value;
        constexpr bool PART = decltype(partial)::value;
        constexpr int R = 4;
        for (int r0 = 0; r0 < (PART ? rows_valid : kRowsPerTile); r0 += R) {
          float4 m[R], v[R], x[R];
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const uint64_t o = base + (r0 + k) * kRowElems + 4 * lane;
            m[k] = ld_ro_s<MIS>(p.m + o, s);
            v[k] = ld_ro_s<MIS>(p.v + o, s);
            x[k] = ld_rw_s<MIS>(p.x + o, s);
          }
#pragma unroll
          for (int k = 0; k < R; ++k) {
            float4 xn;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float u = __fdiv_rn(comp(m[k], q), __fadd_rn(__fsqrt_rn(comp(v[k], q)), p.eta));
              if (p.wd > 0.0f) u = __fadd_rn(u, __fmul_rn(p.wd, comp(x[k], q)));
              set_comp(xn, q, __fadd_rn(comp(x[k], q), __fmul_rn(a, u)));
            }
            const uint64_t o = base + (r0 + k) * kRowElems + 4 * lane;
            const int nvl = PART ? lane_valid(tvalid, static_cast<uint64_t>(r0 + k) * kRowElems, lane) : 4;
            if (!PART || nvl == 4) {
              st_s<MIS>(p.x + o, s, xn);
              if (p.finalize) st_s<MIS>(p.vf + o, s, v[k]);  // optimizers.cpp:205
            } else {
              st_first(p.x + o, xn, nvl);
              if (p.finalize) st_first(p.vf + o, v[k], nvl);
            }
            for (int j = 0; j < p.npush; ++j) {  // owner-sharded warmup: the allgather
              if (!PART || nvl == 4) {
                st_s<MIS>(p.push_x[j] + o, s, xn);
                if (p.finalize) {
                  st_s<MIS>(p.push_m[j] + o, s, m[k]);
                  st_s<MIS>(p.push_v[j] + o, s, v[k]);
                  st_s<MIS>(p.push_vf[j] + o, s, v[k]);
                }
              } else {
                st_first(p.push_x[j] + o, xn, nvl);
                if (p.finalize) {
                  st_first(p.push_m[j] + o, m[k], nvl);
                  st_first(p.push_v[j] + o, v[k], nvl);
                  st_first(p.push_vf[j] + o, v[k], nvl);
                }
              }
            }
          }
        }
      };
      // MIS accessors only for a layer off a 16-B boundary (they assume s != 0)
      if constexpr (MISK) {
        if (s != 0) {
          if (part) rows(Mis<true>{}, Mis<true>{});
          else rows(Mis<true>{}, Mis<false>{});
        } else {
          if (part) rows(Mis<false>{}, Mis<true>{});
          else rows(Mis<false>{}, Mis<false>{});
        }
      } else {
        if (part) rows(Mis<false>{}, Mis<true>{});
        else rows(Mis<false>{}, Mis<false>{});
      }
      continue;
    }
    for (int r = 0; r < kRowsPerTile; ++r) {
      const uint64_t ir = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(r) * kRowElems;
      if (ir >= len) break;
      const uint64_t kr = base + static_cast<uint64_t>(r) * kRowElems;
      const int nv = lane_valid(len, ir, lane);
      const float4 m = ld_row4<false>(p.m + kr, lane, s);
      const float4 v = ld_row4<false>(p.v + kr, lane, s);
      const float4 x = ld_row4<false>(p.x + kr, lane, s);
      float4 xn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float u = __fdiv_rn(comp(m, q), __fadd_rn(__fsqrt_rn(comp(v, q)), p.eta));
        if (p.wd > 0.0f) u = __fadd_rn(u, __fmul_rn(p.wd, comp(x, q)));
        set_comp(xn, q, __fadd_rn(comp(x, q), __fmul_rn(a, u)));
      }
      st_row4(p.x + kr, lane, s, xn, nv);
      if (p.finalize) st_row4(p.vf + kr, lane, s, v, nv);  // optimizers.cpp:205
      for (int j = 0; j < p.npush; ++j) {  // owner-sharded warmup: the allgather
        st_row4(p.push_x[j] + kr, lane, s, xn, nv);
        if (p.finalize) {
          st_row4(p.push_m[j] + kr, lane, s, m, nv);
          st_row4(p.push_v[j] + kr, lane, s, v, nv);
          st_row4(p.push_vf[j] + kr, lane, s, v, nv);
        }
      }
    }
  }
  if (p.npush) warp_fence_system(lane);  // remote stores before the stream's signal
}

// Lossless average (comm_sim.cpp:214-222): ascending workers in fp64, * 1/n.
// Vector form: 4 elements per thread with 128-bit loads (inputs are 16-byte
// aligned library buffers), any output alignment.
__global__ void k_average4(const float* in, uint64_t stride, int n, uint64_t len, float* out,
                           unsigned long long* err, int check, int worker_base) {
  if (gate_closed_call(err)) return;
  const double inv_n = 1.0 / static_cast<double>(n);
  const uint64_t n4 = len / 4;
  for (uint64_t k4 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k4 < n4;
       k4 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < n; ++i) {
      const float4 g = ldg_ro(in + static_cast<size_t>(i) * stride + 4 * k4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float gq = comp(g, q);
        if (check && !isfinite(gq))
          flag(err, kErrGrad, (static_cast<unsigned long long>(worker_base + i) << 40) | (4 * k4 + q));
        a[q] += static_cast<double>(gq);
      }
    }
    if (out) {
#pragma unroll
      for (int q = 0; q < 4; ++q) out[4 * k4 + q] = static_cast<float>(a[q] * inv_n);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < len - 4 * n4) {  // tail
    const uint64_t k = 4 * n4 + threadIdx.x;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      const float g = in[static_cast<size_t>(i) * stride + k];
      if (check && !isfinite(g)) flag(err, kErrGrad, (static_cast<unsigned long long>(worker_base + i) << 40) | k);
      acc += static_cast<double>(g);
    }
    if (out) out[k] = static_cast<float>(acc * inv_n);
  }
}

__global__ void k_average(const float* in, uint64_t stride, int n, uint64_t len, float* out,
                          unsigned long long* err, int check, int worker_base) {
  if (gate_closed_call(err)) return;
  const double inv_n = 1.0 / static_cast<double>(n);
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      const float g = __ldcs(in + static_cast<size_t>(i) * stride + k);
      if (check && !isfinite(g))
        flag(err, kErrGrad, (static_cast<unsigned long long>(worker_base + i) << 40) | k);
      acc += static_cast<double>(g);
    }
    if (out) out[k] = static_cast<float>(acc * inv_n);
  }
}

// Lossless all-reduce over NVLink (comm_sim.cpp:205-232 in P2P mode): rank r
// reads chunk r of every rank's gradient straight from the peers' HBM,
// averages it in ascending rank order in fp64 (x 1/n, the k_average
// arithmetic), and stores the result into every rank's output — the
// reduce-scatter and the allgather in one pass, no staging copy.  The
// finite check of check_gradients (optimizers.cpp:99-117) rides along: a
// non-finite element of rank q is reported into rank q's own error word.
// U groups of 4 elements (k0, k0 + step, ...) per thread: all peers' loads
// of all groups are issued before any is consumed (NVLink latency).
#ifndef LOSSLESS_U
#define LOSSLESS_U 2  // 4-float groups per thread per iteration (n = 2, 4)
#endif
// Peer gradient loads of the lossless exchange (A/B knob: -DLOSSLESS_LD256
// asks the L2 for 256-byte sectors, i.e. fewer, larger NVLink reads).
#ifdef LOSSLESS_LD256
#define LOSSLESS_LD(ptr) ldg_ro(ptr)
#else
#define LOSSLESS_LD(ptr) __ldcg(reinterpret_cast<const float4*>(ptr))
#endif
template <int NT, int U>
__device__ __forceinline__ void lossless_groups(const LosslessP2PParams& p, uint64_t k0,
                                                uint64_t step, uint64_t end, double inv_n) {
  constexpr int kN = NT > 0 ? NT : 8;
  const int n = NT > 0 ? NT : p.n;
  float4 g[U][kN];
  double a[U][4];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int e = 0; e < 4; ++e) a[u][e] = 0.0;
  for (int q0 = 0; q0 < n; q0 += kN) {
    const int m = n - q0 < kN ? n - q0 : kN;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * step;
#pragma unroll
      for (int q = 0; q < kN; ++q)
        if (q < m && k < end) g[u][q] = LOSSLESS_LD(p.peer_in[q0 + q] + k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t k = k0 + u * step;
      if (k >= end) break;
#pragma unroll
      for (int q = 0; q < kN; ++q) {
        if (q >= m) break;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = comp(g[u][q], e);
          if (p.check_finite && !isfinite(x) && k + e < p.d)
            flag(p.err, kErrGrad, (static_cast<unsigned long long>(q0 + q) << 40) | (k + e));
          a[u][e] += static_cast<double>(x);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t k = k0 + u * step;
    if (k >= end) break;
    const float4 v = make_float4(static_cast<float>(a[u][0] * inv_n), static_cast<float>(a[u][1] * inv_n),
                                 static_cast<float>(a[u][2] * inv_n), static_cast<float>(a[u][3] * inv_n));
    if (p.local_only) {
      *reinterpret_cast<float4*>(p.peer_out[p.rank] + k) = v;
    } else {
      for (int q = 0; q < n; ++q) *reinterpret_cast<float4*>(p.peer_out[q] + k) = v;
    }
  }
}


// Piece p's aligned body of the chunk body [a0, a1): [a0 + off(p), a0 + off(p+1)),
// off(p) = F(p) * (a1 - a0) rounded down to a multiple of 4 (off(pieces) = a1 - a0),
// F(p) = p / P (shape 0, equal pieces) or 1 - ((P - p) / P)^2 (shape 1,
// linearly shrinking pieces: a short tail for the consumer of the last one).
// Integer arithmetic: host and device agree exactly.
__host__ __device__ __forceinline__ uint64_t piece_body_start(uint64_t a0, uint64_t a1, int pieces, int p,
                                                              int shape = 0) {
  if (p >= pieces) return a1;
  const uint64_t P = static_cast<uint64_t>(pieces), q = static_cast<uint64_t>(p);
  const uint64_t num = shape == 1 ? P * P - (P - q) * (P - q) : q, den = shape == 1 ? P * P : P;
  return a0 + ((num * (a1 - a0) / den) & ~3ull);
}

template <int NT>
__global__ void __launch_bounds__(256) k_lossless_p2p(const LosslessP2PParams p) {
  if (gate_closed_call(p.err)) return;
  if (!wait_peers(p.in_flags, p.n, p.epoch, p.err)) return;  // every rank's gradient is in place
  const double inv_n = 1.0 / static_cast<double>(p.n);
  const uint64_t lo = p.hi ? p.lo : static_cast<uint64_t>(p.rank) * p.c, hi = p.hi ? p.hi : lo + p.c;
  const uint64_t up = (lo + 3) & ~3ull, dn = hi & ~3ull;  // 16-B aligned body [a0, a1)
  const uint64_t a0 = up < hi ? up : hi;
  const uint64_t a1 = dn > a0 ? dn : a0;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  constexpr int U = NT == 8 ? 1 : LOSSLESS_U;
  const int P = p.pieces > 0 ? p.pieces : 1;
  for (int pc = 0; pc < P; ++pc) {
    const uint64_t b0 = piece_body_start(a0, a1, P, pc, p.shape), b1 = piece_body_start(a0, a1, P, pc + 1, p.shape);
    for (uint64_t k = b0 + 4 * tid; k < b1; k += 4 * nth * U) lossless_groups<NT, U>(p, k, 4 * nth, b1, inv_n);
    if (blockIdx.x == 0 && (pc == 0 || pc == P - 1)) {
      // unaligned head [lo, a0) (first piece) and tail [a1, hi) (last piece), one element per thread
      const uint64_t nh = pc == 0 ? a0 - lo : 0, nt = pc == P - 1 ? hi - a1 : 0;
      if (threadIdx.x < nh + nt) {
        const uint64_t k = threadIdx.x < nh ? lo + threadIdx.x : a1 + (threadIdx.x - nh);
        double acc = 0.0;
        for (int q = 0; q < p.n; ++q) {
          const float x = __ldcg(p.peer_in[q] + k);
          if (p.check_finite && !isfinite(x) && k < p.d)
            flag(p.err, kErrGrad, (static_cast<unsigned long long>(q) << 40) | k);
          acc += static_cast<double>(x);
        }
        const float v = static_cast<float>(acc * inv_n);
        for (int q = p.local_only ? p.rank : 0; q < (p.local_only ? p.rank + 1 : p.n); ++q) p.peer_out[q][k] = v;
      }
    }
    if (p.pieces > 0) {
      // Piece delivered: CTA barrier, then one system fence (cumulative over
      // the CTA's remote stores) and the CTA count; the last CTA raises the flag.
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(p.piece_done + pc, 1u) == gridDim.x - 1) {
          p.piece_done[pc] = 0u;
          if (pc == P - 1) {
            __threadfence();
            forward_grad_error(p.err, p.peer_err, p.n);  // every rank raises (optimizers.cpp:99-117)
          }
          __threadfence_system();
          for (int q = p.local_only ? p.rank : 0; q < (p.local_only ? p.rank + 1 : p.n); ++q)
            st_relaxed_sys(p.peer_flags[q] + p.piece_flag_base + p.rank * p.pieces + pc, p.epoch);
        }
      }
    }
  }
  __threadfence_system();  // this thread's remote stores and error reports
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(p.done, 1u) == gridDim.x - 1) {
    *p.done = 0u;
    __threadfence();
    forward_grad_error(p.err, p.peer_err, p.n);  // every rank raises (optimizers.cpp:99-117)
    __threadfence_system();
    for (int q = p.local_only ? p.rank : 0; q < (p.local_only ? p.rank + 1 : p.n); ++q)
      st_relaxed_sys(p.peer_flags[q] + p.out_flag + p.rank, p.epoch);
  }
}

template <typename T>
__global__ void k_push_range(const T* src, T* const* dst, int ndst, uint64_t off, uint64_t count,
                             const unsigned long long* gate) {
  if (gate_closed_call(gate)) return;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count; k += nth) {
    const T w = __ldcg(src + off + k);
    for (int j = 0; j < ndst; ++j) dst[j][off + k] = w;
  }
  __threadfence_system();
}

// Push-based owner-sharded exchange (ShardPushParams).  Owner r's range
// [E_r, E_r+1) splits like the lossless kernel's chunk: a 16-B aligned body in
// `pieces` pieces (piece_body_start) plus the unaligned head (piece 0) and
// tail (last piece).  Slot offsets are relative to E_r rounded down to 4, so
// body stores are 16-B aligned.
__device__ __forceinline__ void shard_piece(uint64_t E0, uint64_t E1, int P, int pc, int shape, uint64_t* b0,
                                            uint64_t* b1, uint64_t* h0, uint64_t* h1, uint64_t* t0,
                                            uint64_t* t1) {
  const uint64_t up = (E0 + 3) & ~3ull, dn = E1 & ~3ull;
  const uint64_t a0 = up < E1 ? up : E1;
  const uint64_t a1 = dn > a0 ? dn : a0;
  *b0 = piece_body_start(a0, a1, P, pc, shape);
  *b1 = piece_body_start(a0, a1, P, pc + 1, shape);
  *h0 = E0;
  *h1 = pc == 0 ? a0 : E0;
  *t0 = a1;
  *t1 = pc == P - 1 ? E1 : a1;
}

__global__ void __launch_bounds__(256) k_shard_push(const ShardPushParams p) {
  if (gate_closed_call(p.gate)) return;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (int pc = 0; pc < p.pieces; ++pc) {
    for (int r = 0; r < p.n; ++r) {
      if (r == p.rank) continue;
      const uint64_t E0 = p.e_all[r], E1 = p.e_all[r + 1];
      uint64_t b0, b1, h0, h1, t0, t1;
      shard_piece(E0, E1, p.pieces, pc, p.shape, &b0, &b1, &h0, &h1, &t0, &t1);
      float* dst = p.peer_stg[r] + static_cast<uint64_t>(p.rank) * p.S - (E0 & ~3ull);  // dst[e], e in [E0, E1)
      // 4 groups of 4 floats per thread: all loads in flight before the stores
      for (uint64_t k = b0 + 4 * tid; k < b1; k += 16 * nth) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t ku = k + 4 * u * nth;
          if (ku < b1) v[u] = __ldcs(reinterpret_cast<const float4*>(p.in + ku));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t ku = k + 4 * u * nth;
          if (ku < b1) *reinterpret_cast<float4*>(dst + ku) = v[u];
        }
      }
      for (uint64_t k = h0 + tid; k < h1; k += nth) dst[k] = p.in[k];
      for (uint64_t k = t0 + tid; k < t1; k += nth) dst[k] = p.in[k];
    }
    // Piece delivered to every owner: CTA barrier, one system fence per CTA,
    // the CTA count; the last CTA raises "piece pc from this rank" everywhere
    // (at itself too: the owner waits for all n).
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      if (atomicAdd(p.piece_done + pc, 1u) == gridDim.x - 1) {
        p.piece_done[pc] = 0u;
        __threadfence_system();
        for (int q = 0; q < p.n; ++q)
          st_relaxed_sys(p.peer_flags[q] + p.piece_flag_base + p.rank * p.pieces + pc, p.epoch);
      }
    }
  }
}

// Owner side: piece `piece` of [E0, E1), the ascending-rank fp64 average of
// the own gradient and the staged slots (k_lossless_p2p's arithmetic, and its
// check_gradients finding per sending rank).
__global__ void __launch_bounds__(256) k_shard_reduce(const ShardReduceParams p) {
  if (gate_closed_call(p.err)) return;
  const double inv_n = 1.0 / static_cast<double>(p.n);
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t b0, b1, h0, h1, t0, t1;
  shard_piece(p.E0, p.E1, p.pieces, p.piece, p.shape, &b0, &b1, &h0, &h1, &t0, &t1);
  const uint64_t base = p.E0 & ~3ull;
  auto src = [&](int q, uint64_t k) -> const float* {
    return q == p.rank ? p.in + k : p.stg + static_cast<uint64_t>(q) * p.S + (k - base);
  };
  for (uint64_t k = b0 + 4 * tid; k < b1; k += 4 * nth) {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < p.n; ++q) {
      const float4 g = __ldcs(reinterpret_cast<const float4*>(src(q, k)));
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = comp(g, e);
        if (!isfinite(x) && k + e < p.d) flag(p.err, kErrGrad, (static_cast<unsigned long long>(q) << 40) | (k + e));
        a[e] += static_cast<double>(x);
      }
    }
    *reinterpret_cast<float4*>(p.out + k) =
        make_float4(static_cast<float>(a[0] * inv_n), static_cast<float>(a[1] * inv_n),
                    static_cast<float>(a[2] * inv_n), static_cast<float>(a[3] * inv_n));
  }
  auto scalar = [&](uint64_t lo, uint64_t hi) {
    for (uint64_t k = lo + tid; k < hi; k += nth) {
      double acc = 0.0;
      for (int q = 0; q < p.n; ++q) {
        const float x = *src(q, k);
        if (!isfinite(x) && k < p.d) flag(p.err, kErrGrad, (static_cast<unsigned long long>(q) << 40) | k);
        acc += static_cast<double>(x);
      }
      p.out[k] = static_cast<float>(acc * inv_n);
    }
  };
  scalar(h0, h1);
  scalar(t0, t1);
  if (p.piece == p.pieces - 1) {  // every rank raises a non-finite gradient (optimizers.cpp:99-117)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(p.done, 1u) == gridDim.x - 1) {
      *p.done = 0u;
      __threadfence();
      forward_grad_error(p.err, p.peer_err, p.n);
    }
  }
}

// Consumer side of the piecewise exchange: every rank's piece p delivered.
__global__ void k_wait_piece(const unsigned long long* flags, int base, int n, int pieces, int pc,
                             unsigned long long epoch, unsigned long long* err) {
  if (gate_closed_call(err)) return;
  if (threadIdx.x == 0) {
    const unsigned long long bound = wait_bound(err), t0 = now_ns();
    for (int q = 0; q < n && !gate_closed(err); ++q) {
      while (ld_acquire_sys(flags + base + q * pieces + pc) < epoch) {
        if (gate_closed(err)) break;
        __nanosleep(32);
        if (now_ns() - t0 > bound) {
          flag(err, kErrPeer, static_cast<unsigned long long>(q));
          close_gate(err, kGateMidStep);
          break;
        }
      }
    }
  }
}

__global__ void k_signal_peers(unsigned long long* const* peer_flags, int index, int n,
                               unsigned long long epoch, const unsigned long long* gate) {
  if (gate_closed_call(gate)) return;
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < n; ++q) st_relaxed_sys(peer_flags[q] + index, epoch);
  }
}

// Result of the collective (compression.cpp:68-81, comm_sim.cpp:173,202):
// chunk-relative, one warp per 32 packet words (1024 elements): every lane
// reads the same word (broadcast) and writes one element of each 32-element
// group (coalesced), truncated at c and d.
__device__ __forceinline__ void decompress_warps(const uint32_t* res, int n, uint64_t c, uint64_t slot,
                                                 uint64_t W, uint64_t d, float* out, uint64_t gw,
                                                 uint64_t nwarps, int lane) {
  const uint64_t groups = (W + 31) / 32;  // 32-word groups per chunk
  for (uint64_t g = gw; g < groups * n; g += nwarps) {
    const uint64_t j = g / groups, w0 = (g - j * groups) * 32;
    const uint32_t* sl = res + j * slot;
    const float S = slot_scale_cg(sl, W);
    const float pos = S, neg = S == 0.0f ? 0.0f : -S;
    const uint64_t kc = j * c;
    const uint32_t mine = __ldcg(sl + w0 + lane);  // one coalesced 128-B word load per warp
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const uint32_t word = __shfl_sync(FULL, mine, i);
      const uint64_t e = (w0 + i) * 32 + lane;  // chunk-relative element
      if (e < c && kc + e < d) out[kc + e] = (word >> lane) & 1u ? pos : neg;
    }
  }
}

__global__ void k_decompress(const uint32_t* res, int n, uint64_t c, uint64_t slot, uint64_t W,
                             uint64_t d, float* out, const unsigned long long* gate) {
  if (gate_closed_call(gate)) return;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  decompress_warps(res, n, c, slot, W, d, out, gw, nwarps, threadIdx.x & 31);
}

// last_cta over a counter that `target` arrivals complete (any CTAs).
__device__ __forceinline__ bool last_of(unsigned int* c, unsigned int target, bool* s_last) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *s_last = atomicAdd(c, 1u) == target - 1;
    if (*s_last) {
      *c = 0u;
      __threadfence();
    }
  }
  __syncthreads();
  return *s_last;
}

// ---------------------------------------------------------------------------
// Fused small compressed collective (P2P transport): K1 -> worker scales ->
// exchange -> K3 -> server scale -> exchange [-> decompress] in one
// cooperative kernel.  Below ~64 MB the separate kernels are latency-bound
// (7 launches, each a ramp, a tail and a system fence); here the phases are
// separated by grid barriers and the peers' epoch flags only.  Every
// per-element operation and reduction order is the unfused path's.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks,
                                             unsigned long long* err) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      long long spins = 0;
      while (*gen == g && ++spins < (1ll << 30)) __nanosleep(32);
      if (*gen == g) close_gate(err, kGateInternal);  // co-residency broken: fail-stop
    }
    __threadfence();
  }
  __syncthreads();
}

// One K1 tile per CTA: warp w computes rows 4w..4w+3 in a single load batch;
// |corr| goes to shared memory and warp 0 sums it in the canonical per-lane
// order (rows 0..31, elements 4l..4l+3), so the tile partial is the warp
// path's bit for bit.  Tiles off the fast path are done by warp 0 alone.
template <int MODE, bool ALIGNED>
__device__ __forceinline__ void k1_cta_tile(const K1Params& p, long long tile, uint32_t* sw,
                                            float* s_abs, float* s_cm, float es) {
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const long long per_w = static_cast<long long>(p.n) * p.tpc;
  const int w = static_cast<int>(tile / per_w);
  const long long rem = tile - w * per_w;
  const int j = static_cast<int>(rem / p.tpc);
  const int t = static_cast<int>(rem - static_cast<long long>(j) * p.tpc);
  const uint64_t i0 = static_cast<uint64_t>(t) * kTile;
  const uint64_t kc = static_cast<uint64_t>(j) * p.c;
  bool fast = MODE != 1 && i0 + kTile <= p.c && kc + i0 + kTile <= p.d;
  float A = 0.f, B = 0.f, IC = 0.f;
  if (fast && MODE == 2) {
    int l0;
    if (p.tile_layer) {
      l0 = __ldg(p.tile_layer + static_cast<size_t>(j) * p.tpc + t);
      fast = l0 >= 0;
    } else {
      l0 = find_layer(p.off, p.L, kc + i0);
      fast = l0 < p.L && kc + i0 + (kTile - 1) < __ldg(p.off + l0 + 1);
    }
    if (fast) {
      A = __ldg(p.A + l0);
      B = __ldg(p.B + l0);
      IC = __ldg(p.invc + l0);
    }
  }
  if (!fast) {
    if (wq == 0) k1_tile<MODE, ALIGNED>(p, tile, lane, sw, es);
    __syncthreads();
    return;
  }
  const int s = ALIGNED ? 0 : static_cast<int>(kc & 3u);
  const size_t ep = static_cast<size_t>(w) * p.n + j;
  const float* gin = p.in + static_cast<size_t>(w) * p.in_stride + kc + i0;
  float* we = p.werr + ep * p.c_pad + i0;
  const uint32_t* pkp = p.pk_prev + ep * p.slot;
  const float Sp = slot_scale(pkp, p.W);
  pkp += i0 >> 5;
  float pos_m = 0.f, neg_m = 0.f;
  const uint32_t* rp = nullptr;
  if (MODE == 2) {
    const uint32_t* rs = p.res_prev + static_cast<size_t>(j) * p.slot;
    const float S2 = slot_scale(rs, p.W);
    pos_m = S2;
    neg_m = S2 == 0.0f ? 0.0f : -S2;
    rp = rs + (i0 >> 5);
  }
  constexpr int R = 4;
  const int r0 = R * wq;
  const uint32_t sh = 4 * (lane & 7);
  const int wsub = lane >> 3;
  float4 g[R], raw[R];
  uint32_t wn[R], rn[R];
  load_rows<R, true>(g, gin + r0 * kRowElems, lane, s);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    raw[k] = ldg_rw(we + (r0 + k) * kRowElems + 4 * lane);
    wn[k] = __ldg(pkp + 4 * (r0 + k) + wsub) >> sh;
    rn[k] = MODE == 2 ? __ldg(rp + 4 * (r0 + k) + wsub) >> sh : 0u;
  }
  float cm = 0.0f;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (MODE == 2 && !(isfinite(g[k].x) && isfinite(g[k].y) && isfinite(g[k].z) && isfinite(g[k].w))) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!isfinite(comp(g[k], q)))
          flag_grad(p, (static_cast<unsigned long long>(p.worker_base + w) << 40) |
                           (kc + i0 + (r0 + k) * kRowElems + 4 * lane + q));
    }
    uint32_t nib = 0;
    float4 rawn, ab;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v;
      if (MODE == 0) {
        v = comp(g[k], q);
      } else {
        const float ap = __fmul_rn(A, __fmul_rn(pos_m, IC)), an = __fmul_rn(A, __fmul_rn(neg_m, IC));
        v = __fadd_rn((rn[k] >> q) & 1u ? ap : an, __fmul_rn(B, comp(g[k], q)));  // fusion.cpp:143, kernels.cpp:253
      }
      const float rec = (wn[k] >> q) & 1u ? Sp : -Sp;
      const float delta = __fsub_rn(comp(raw[k], q), rec);               // compression.cpp:194
      const float corr = __fadd_rn(v, __fmul_rn(es, delta));             // :181
      set_comp(rawn, q, __fadd_rn(v, delta));
      nib |= static_cast<uint32_t>(corr >= 0.0f) << q;                   // :50
      set_comp(ab, q, fabsf(corr));
      cm = cm < fabsf(corr) ? fabsf(corr) : cm;
    }
    st4(we + (r0 + k) * kRowElems + 4 * lane, rawn);
    *reinterpret_cast<float4*>(s_abs + (r0 + k) * kRowElems + 4 * lane) = ab;
    stage_row_bits(sw, r0 + k, lane, nib);
  }
  cm = warp_max(cm);
  if (lane == 0) s_cm[wq] = cm;
  __syncthreads();
  if (wq == 0) {
    double acc = 0.0;  // :54, the warp path's per-lane order
    for (int r = 0; r < kRowsPerTile; ++r) {
      const float4 ab = *reinterpret_cast<const float4*>(s_abs + r * kRowElems + 4 * lane);
      acc += static_cast<double>(ab.x);
      acc += static_cast<double>(ab.y);
      acc += static_cast<double>(ab.z);
      acc += static_cast<double>(ab.w);
    }
    acc = warp_bfly_sum(acc);
    if (lane == 0) p.partials[ep * p.tpc + t] = acc;
    if (p.cmax) {
      const float m = warp_max(lane < kWarpsPerBlock ? s_cm[lane] : 0.0f);
      if (lane == 0) p.cmax[ep * p.tpc + t] = m;
    }
    const uint4 wv = tile_words(sw, lane);
    reinterpret_cast<uint4*>(p.pk_cur + ep * p.slot + (i0 >> 5))[lane] = wv;
    if (p.peer_rx) reinterpret_cast<uint4*>(p.peer_rx[j] + p.rx_off + (i0 >> 5))[lane] = wv;
  }
  __syncthreads();
}

// One K3 tile per CTA (rows split over the warps as in k1_cta_tile), general
// arithmetic: any n, partial tiles (elements past c are dead and add 0).
__device__ __forceinline__ void k3_cta_tile(const K3Params& p, long long tile, uint32_t* sw,
                                            float* s_abs, float* s_cm, const float* scale,
                                            uint32_t* const* peers, float es, double inv_n) {
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int n = p.n;
  const int t = static_cast<int>(tile);  // ns == 1: server `server_base`
  const int j = p.server_base;
  const uint64_t i0 = static_cast<uint64_t>(t) * kTile;
  float* se = p.serr + i0;
  const uint32_t* rs = p.res_prev + static_cast<size_t>(j) * p.slot;
  const float S2p = slot_scale(rs, p.W);
  rs += i0 >> 5;
  const uint32_t* inw = p.in + (i0 >> 5);
  constexpr int R = 4;
  const int r0 = R * wq;
  constexpr int kMaxN = 8;  // workers whose nibbles are loaded up front
  float4 raw[R];
  uint32_t sn[R], nb[R][kMaxN];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    raw[k] = ld4(se + (r0 + k) * kRowElems + 4 * lane);
    sn[k] = row_nibble(rs, r0 + k, lane);
#pragma unroll
    for (int i = 0; i < kMaxN; ++i)
      nb[k][i] = i < n ? ld_cg(inw + i * p.in_i + 4 * (r0 + k) + (lane >> 3)) : 0u;
  }
  float cm = 0.0f;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = r0 + k;
    const uint64_t ir = i0 + static_cast<uint64_t>(r) * kRowElems;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    auto add = [&](int i, uint32_t word) {  // compression.cpp:83-89, ascending workers
      const float S = scale[i];
      const uint32_t b = (word >> (4 * (lane & 7))) & 0xFu;
      if (S != 0.0f) {
        const double Sd = S;
        a0 += (b & 1u) ? Sd : -Sd;
        a1 += (b & 2u) ? Sd : -Sd;
        a2 += (b & 4u) ? Sd : -Sd;
        a3 += (b & 8u) ? Sd : -Sd;
      }
    };
#pragma unroll
    for (int i = 0; i < kMaxN; ++i)
      if (i < n) add(i, nb[k][i]);
    for (int i = kMaxN; i < n; ++i) add(i, ld_cg(inw + i * p.in_i + 4 * r + (lane >> 3)));
    const float4 avg = make_float4(static_cast<float>(a0 * inv_n), static_cast<float>(a1 * inv_n),
                                   static_cast<float>(a2 * inv_n), static_cast<float>(a3 * inv_n));
    uint32_t nib = 0;
    float4 rawn, ab;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = ir + 4 * lane + q;
      const float v = comp(avg, q);
      const float rec = (sn[k] >> q) & 1u ? S2p : -S2p;
      const float delta = __fsub_rn(comp(raw[k], q), rec);
      const float corr = __fadd_rn(v, __fmul_rn(es, delta));
      const bool live = i < p.c;
      set_comp(rawn, q, live ? __fadd_rn(v, delta) : 0.0f);
      nib |= static_cast<uint32_t>(live && corr >= 0.0f) << q;
      set_comp(ab, q, live ? fabsf(corr) : 0.0f);
      if (live) cm = cm < fabsf(corr) ? fabsf(corr) : cm;
    }
    if (ir < p.c) st4(se + r * kRowElems + 4 * lane, rawn);
    *reinterpret_cast<float4*>(s_abs + r * kRowElems + 4 * lane) = ab;
    stage_row_bits(sw, r, lane, nib);
  }
  cm = warp_max(cm);
  if (lane == 0) s_cm[wq] = cm;
  __syncthreads();
  if (wq == 0) {
    double acc = 0.0;
    for (int r = 0; r < kRowsPerTile; ++r) {
      const float4 ab = *reinterpret_cast<const float4*>(s_abs + r * kRowElems + 4 * lane);
      acc += static_cast<double>(ab.x);
      acc += static_cast<double>(ab.y);
      acc += static_cast<double>(ab.z);
      acc += static_cast<double>(ab.w);
    }
    acc = warp_bfly_sum(acc);
    if (lane == 0) p.partials[t] = acc;
    if (p.cmax) {
      const float m = warp_max(lane < kWarpsPerBlock ? s_cm[lane] : 0.0f);
      if (lane == 0) p.cmax[t] = m;
    }
    flush_server_words(p, peers, sw, p.res_cur + static_cast<size_t>(j) * p.slot + (i0 >> 5), i0, lane);
  }
  __syncthreads();
}

// ---- LL transport of the fused small collective ------------------------------
__device__ __forceinline__ uint2 ld_ll(const uint2* p) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
// 4 packet words -> 4 LL words (word, epoch), two 16-byte stores.
__device__ __forceinline__ void st_ll4(uint2* dst, const uint4& w, uint32_t ep) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(w.x), "r"(ep), "r"(w.y), "r"(ep)
               : "memory");
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + 2), "r"(w.z), "r"(ep), "r"(w.w),
               "r"(ep)
               : "memory");
}
__device__ __forceinline__ void st_ll1(uint2* dst, uint32_t w, uint32_t ep) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1,%2};" ::"l"(dst), "r"(w), "r"(ep) : "memory");
}
// The word of an LL slot once it carries `ep` (fail-stop bound as wait_peers).
__device__ __forceinline__ uint32_t ll_get(const uint2* p, uint32_t ep, unsigned long long* err, bool& ok) {
  uint2 v = ld_ll(p);
  if (v.y == ep) return v.x;
  const unsigned long long t0 = now_ns(), bound = wait_bound(err);
  for (int it = 0;; ++it) {
    v = ld_ll(p);
    if (v.y == ep) return v.x;
    if ((it & 63) == 63) {
      if (gate_closed(err)) break;
      if (now_ns() - t0 > bound) {
        close_gate(err, kGateMidStep);
        break;
      }
    }
  }
  ok = false;
  return 0u;
}

// One K3 tile per CTA over LL-received worker words (k3_cta_tile's arithmetic
// and order); server words go to the local plain result slot and, as LL
// words, to every rank's result buffer.
template <int NT>
__device__ __forceinline__ void k3_cta_tile_ll(const SmallParams& sp, long long tile, uint32_t* sw, float* s_abs,
                                               float* s_cm, const float* scale, float es, double inv_n,
                                               bool& ok) {
  const K3Params& p = sp.k3;
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int n = p.n;
  const int t = static_cast<int>(tile);
  const int j = p.server_base;
  const uint64_t i0 = static_cast<uint64_t>(t) * kTile;
  float* se = p.serr + i0;
  const uint32_t* rs = p.res_prev + static_cast<size_t>(j) * p.slot;
  const float S2p = slot_scale(rs, p.W);
  rs += i0 >> 5;
  const uint2* inw = sp.ll_rx_mine + (i0 >> 5);
  constexpr int R = 4;
  const int r0 = R * wq;
  constexpr int kMaxN = NT;  // worker words held in registers (code size: the kernel runs once, i-cache cold)
  float4 raw[R];
  uint32_t sn[R], nb[R][kMaxN];
  uint2 lv[R][kMaxN];
#pragma unroll
  for (int k = 0; k < R; ++k) {  // every load of the tile in flight at once, then the epoch checks
    raw[k] = ld4(se + (r0 + k) * kRowElems + 4 * lane);
    sn[k] = row_nibble(rs, r0 + k, lane);
#pragma unroll
    for (int i = 0; i < kMaxN; ++i)
      lv[k][i] = i < n ? ld_ll(inw + i * p.slot + 4 * (r0 + k) + (lane >> 3)) : make_uint2(0u, sp.ep32);
  }
  if (sp.ts && blockIdx.x == 0 && threadIdx.x == 0) sp.ts[9] = now_ns() + 0ull * lv[0][0].y;
  // Words still in flight are re-polled together, one round trip per sweep
  // (polling them one after another cost a round trip each).
  {
    unsigned long long t0 = 0;
    for (int sweep = 0;; ++sweep) {
      bool stale = false;
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int i = 0; i < kMaxN; ++i) stale |= lv[k][i].y != sp.ep32;
      if (!stale) break;
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int i = 0; i < kMaxN; ++i)
          if (lv[k][i].y != sp.ep32) lv[k][i] = ld_ll(inw + i * p.slot + 4 * (r0 + k) + (lane >> 3));
      if ((sweep & 63) == 63) {
        if (t0 == 0) t0 = now_ns();
        if (gate_closed(sp.err) || now_ns() - t0 > wait_bound(sp.err)) {
          close_gate(sp.err, kGateMidStep);
          ok = false;
          break;
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k)
#pragma unroll
    for (int i = 0; i < kMaxN; ++i) nb[k][i] = lv[k][i].x;
  if (sp.ts && blockIdx.x == 0 && threadIdx.x == 0) sp.ts[10] = now_ns() + 0ull * nb[R - 1][0];
  if (sp.ts && blockIdx.x == 0 && lane == 0) atomicMax(sp.ts + 13, now_ns() + 0ull * nb[R - 1][0]);  // last warp
  float cm = 0.0f;
  // n == 2: the 4 possible averages, formed once (same fp64 sum and *1/n)
  constexpr bool kSel = NT == 2;
  float tv[4] = {0.f, 0.f, 0.f, 0.f};
  if (kSel && n == 2) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float S = scale[i];
        if (S != 0.0f) a += ((e >> i) & 1) ? static_cast<double>(S) : -static_cast<double>(S);
      }
      tv[e] = static_cast<float>(a * inv_n);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int r = r0 + k;
    const uint64_t ir = i0 + static_cast<uint64_t>(r) * kRowElems;
    float4 avg;
    if (kSel && n == 2) {
      const uint32_t sh = 4 * (lane & 7);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t b0 = (nb[k][0] >> (sh + q)) & 1u, b1 = (nb[k][kSel ? 1 : 0] >> (sh + q)) & 1u;
        set_comp(avg, q, b1 ? (b0 ? tv[3] : tv[2]) : (b0 ? tv[1] : tv[0]));
      }
    } else {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      auto add = [&](int i, uint32_t word) {  // compression.cpp:83-89, ascending workers
        const float S = scale[i];
        const uint32_t b = (word >> (4 * (lane & 7))) & 0xFu;
        if (S != 0.0f) {
          const double Sd = S;
          a0 += (b & 1u) ? Sd : -Sd;
          a1 += (b & 2u) ? Sd : -Sd;
          a2 += (b & 4u) ? Sd : -Sd;
          a3 += (b & 8u) ? Sd : -Sd;
        }
      };
#pragma unroll
      for (int i = 0; i < kMaxN; ++i)
        if (i < n) add(i, nb[k][i]);
      for (int i = kMaxN; i < n; ++i) add(i, ll_get(inw + i * p.slot + 4 * r + (lane >> 3), sp.ep32, sp.err, ok));
      avg = make_float4(static_cast<float>(a0 * inv_n), static_cast<float>(a1 * inv_n),
                        static_cast<float>(a2 * inv_n), static_cast<float>(a3 * inv_n));
    }
    uint32_t nib = 0;
    float4 rawn, ab;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = ir + 4 * lane + q;
      const float v = comp(avg, q);
      const float rec = (sn[k] >> q) & 1u ? S2p : -S2p;
      const float delta = __fsub_rn(comp(raw[k], q), rec);
      const float corr = __fadd_rn(v, __fmul_rn(es, delta));
      const bool live = i < p.c;
      set_comp(rawn, q, live ? __fadd_rn(v, delta) : 0.0f);
      nib |= static_cast<uint32_t>(live && corr >= 0.0f) << q;
      set_comp(ab, q, live ? fabsf(corr) : 0.0f);
      if (live) cm = cm < fabsf(corr) ? fabsf(corr) : cm;
    }
    if (ok && ir < p.c) st4(se + r * kRowElems + 4 * lane, rawn);
    *reinterpret_cast<float4*>(s_abs + r * kRowElems + 4 * lane) = ab;
    stage_row_bits(sw, r, lane, nib);
  }
  cm = warp_max(cm);
  if (lane == 0) s_cm[wq] = cm;
  __syncthreads();
  if (sp.ts && blockIdx.x == 0 && threadIdx.x == 0) sp.ts[14] = now_ns();
  if (wq == 0) {
    double acc = 0.0;
    for (int r = 0; r < kRowsPerTile; ++r) {
      const float4 ab = *reinterpret_cast<const float4*>(s_abs + r * kRowElems + 4 * lane);
      acc += static_cast<double>(ab.x);
      acc += static_cast<double>(ab.y);
      acc += static_cast<double>(ab.z);
      acc += static_cast<double>(ab.w);
    }
    acc = warp_bfly_sum(acc);
    if (lane == 0) p.partials[t] = acc;
    if (p.cmax) {
      const float m = warp_max(lane < kWarpsPerBlock ? s_cm[lane] : 0.0f);
      if (lane == 0) p.cmax[t] = m;
    }
    if (sp.ts && blockIdx.x == 0 && threadIdx.x == 0) sp.ts[11] = now_ns();
    const uint4 v = tile_words(sw, lane);
    reinterpret_cast<uint4*>(p.res_cur + static_cast<size_t>(j) * p.slot + (i0 >> 5))[lane] = v;
    for (int q = 0; q < n; ++q) st_ll4(sp.ll_res[q] + sp.ll_off + (i0 >> 5) + 4 * lane, v, sp.ep32);
  }
  __syncthreads();
  if (sp.ts && blockIdx.x == 0 && threadIdx.x == 0) sp.ts[12] = now_ns();
}

// True in every thread of the CTA that arrives last at counter `c` (after
// its own global writes; gpu-scope fence + count); that CTA resets it.
__device__ __forceinline__ bool last_cta(unsigned int* c, bool* s_last) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *s_last = atomicAdd(c, 1u) == gridDim.x - 1;
    if (*s_last) {
      *c = 0u;
      __threadfence();
    }
  }
  __syncthreads();
  return *s_last;
}

// ---------------------------------------------------------------------------
// Fused small compressed collective (P2P transport): K1 -> worker scales ->
// exchange -> K3 -> server scale -> exchange [-> decompress] in one
// cooperative kernel.  Below ~32 MB per rank the separate kernels are
// latency-bound; here nothing waits on a grid barrier, a system fence or a
// flag: packet words and scales travel as LL words (word + epoch in one
// 8-byte store), each consumer polls exactly the words it needs, and each
// scale is formed by the CTA that finishes its phase last (last-CTA count).
// Every per-element operation and reduction order is the unfused path's.
// ---------------------------------------------------------------------------
template <int MODE, bool ALIGNED, int NT>
__global__ void __launch_bounds__(kBlock) k_small_collective(__grid_constant__ const SmallParams p) {
  __shared__ __align__(16) uint32_t s_words[128];  // the CTA's tile packet words
  __shared__ float s_scale[64];
  __shared__ double s_red[1024 + 32];
  __shared__ __align__(16) float s_abs[kTile];
  __shared__ float s_cm[kWarpsPerBlock];
  __shared__ bool s_last;
  __shared__ int s_ok;
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  if (gate_closed_call(p.err)) return;
  auto stamp = [&](int k) {
    if (p.ts && blockIdx.x == 0 && threadIdx.x == 0) p.ts[k] = now_ns();
  };
  stamp(0);
  const int n = p.k1.n;
  const uint32_t ep = p.ep32;
  const long long total = static_cast<long long>(n) * p.k1.tpc;
  const bool per_chunk = total <= static_cast<long long>(gridDim.x);
  bool ok = true;
  // 1. worker compression of every chunk of the local stream (plain words to
  //    the local slot, LL words into rank j's receive buffer)
  {
    const float es = p.k1.es_dev ? __ldg(p.k1.es_dev) : p.k1.es_host;
    for (long long tile = blockIdx.x; tile < total; tile += gridDim.x) {
      k1_cta_tile<MODE, ALIGNED>(p.k1, tile, s_words, s_abs, s_cm, es);
      const int j = static_cast<int>(tile / p.k1.tpc);
      if (threadIdx.x < 32) {  // the tile's words, just written by this warp
        const uint64_t w0 = static_cast<uint64_t>(tile - static_cast<long long>(j) * p.k1.tpc) * (kTile / 32);
        const uint4 v = reinterpret_cast<const uint4*>(p.k1.pk_cur + static_cast<size_t>(j) * p.k1.slot + w0)[lane];
        st_ll4(p.ll_rx[j] + p.ll_off + w0 + 4 * lane, v, ep);
      }
      // 2. worker scale of chunk j (one tile per CTA): the CTA that finishes
      //    the chunk's last tile combines its tile partials (k_finalize_scales'
      //    order) and sends the scale to rank j -- the n scales form in parallel
      if (per_chunk && last_of(p.cnt + 2 + j, static_cast<unsigned int>(p.k1.tpc), &s_last)) {
        stamp(2);
        if (threadIdx.x == 0) forward_grad_error(p.err, p.f1.peer_err, n);  // every rank raises
        finalize_block256(p.f1, j, s_red);
        if (threadIdx.x == 0)
          st_ll1(p.ll_rx[j] + p.ll_off + p.k1.W, p.k1.pk_cur[static_cast<size_t>(j) * p.k1.slot + p.k1.W], ep);
      }
    }
  }
  stamp(1);
  // 2'. several tiles per CTA: one count per CTA; the last CTA forms every scale
  if (!per_chunk && last_cta(p.cnt, &s_last)) {
    stamp(2);
    if (threadIdx.x == 0) forward_grad_error(p.err, p.f1.peer_err, n);  // every rank raises
    for (int e = 0; e < n; ++e) {
      finalize_block256(p.f1, e, s_red);
      if (threadIdx.x == 0)
        st_ll1(p.ll_rx[e] + p.ll_off + p.k1.W, p.k1.pk_cur[static_cast<size_t>(e) * p.k1.slot + p.k1.W], ep);
    }
  }
  stamp(3);
  // 3./4. server reduce of chunk `rank` from the LL-received worker packets
  {
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      bool ok_i = true;
      s_scale[i] = __uint_as_float(ll_get(p.ll_rx_mine + static_cast<size_t>(i) * p.k3.slot + p.k3.W, ep, p.err, ok_i));
      if (!ok_i) s_ok = 0;
    }
    __syncthreads();
    ok = s_ok != 0;
    stamp(4);
    const float es = p.k3.es_dev ? __ldg(p.k3.es_dev) : p.k3.es_host;
    const double inv_n = 1.0 / static_cast<double>(n);
    for (long long tile = blockIdx.x; ok && tile < p.k3.tpc; tile += gridDim.x)
      k3_cta_tile_ll<NT>(p, tile, s_words, s_abs, s_cm, s_scale, es, inv_n, ok);
  }
  stamp(5);
  // 5. server scale: the last CTA combines the partials, sends it to every rank
  if (last_cta(p.cnt + 1, &s_last) && !gate_closed(p.err)) {
    stamp(6);
    finalize_block256(p.f2, 0, s_red);
    if (threadIdx.x == 0) {
      const uint32_t S = p.res_plain[static_cast<size_t>(p.k3.server_base) * p.k3.slot + p.k3.W];
      for (int q = 0; q < n; ++q) st_ll1(p.ll_res[q] + p.ll_off + p.k3.W, S, ep);
    }
  }
  stamp(7);
  // 6./7. every rank's server packet: LL -> plain result slots (K5/K6 read
  //    them), and the optional decompress (compression.cpp:68-81)
  {
    const uint64_t W = p.k3.W, slot = p.k3.slot, c = p.k3.c;
    const uint64_t groups = (W + 31) / 32;
    for (uint64_t g = gw; ok && g < groups * n; g += nwarps) {
      const uint64_t j = g / groups, w0 = (g - j * groups) * 32;
      const uint2* ll = p.ll_res_mine + j * slot;
      const uint2 lw = ld_ll(ll + w0 + lane), ls = ld_ll(ll + W);
      const uint32_t mine = lw.y == ep ? lw.x : ll_get(ll + w0 + lane, ep, p.err, ok);
      const float S = __uint_as_float(ls.y == ep ? ls.x : ll_get(ll + W, ep, p.err, ok));
      if (!ok) break;
      uint32_t* pl = p.res_plain + j * slot;
      if (static_cast<int>(j) != p.k3.server_base) {
        pl[w0 + lane] = mine;
        if (w0 == 0 && lane == 0) pl[W] = __float_as_uint(S);
      }
      if (p.out) {
        const float pos = S, neg = S == 0.0f ? 0.0f : -S;
        const uint64_t kc = j * c;
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
          const uint32_t word = __shfl_sync(FULL, mine, i);
          const uint64_t e = (w0 + i) * 32 + lane;
          if (e < c && kc + e < p.d) p.out[kc + e] = (word >> lane) & 1u ? pos : neg;
        }
      }
    }
  }
  stamp(8);
}

__global__ void k_materialize_error(const float* raw, uint64_t c_pad, const uint32_t* pk,
                                    uint64_t slot, uint64_t W, uint64_t c, uint64_t len,
                                    float* out) {
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t j = k / c, i = k - j * c;
    const uint32_t* sl = pk + j * slot;
    const float S = slot_scale(sl, W);
    const uint32_t b = (__ldg(sl + (i >> 5)) >> (i & 31)) & 1u;
    out[k] = __fsub_rn(raw[j * c_pad + i], b ? S : -S);
  }
}

__global__ void k_materialize_m(const uint32_t* res, int n, uint64_t c, uint64_t slot, uint64_t W,
                                const uint64_t* off, int L, const float* invc, uint64_t d,
                                float* out) {
  const BitCursor bc{res, c, slot, W, n};
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < d;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float S;
    const uint32_t b = bit_at(bc, k, &S);
    const int l = find_layer(off, L, k);
    out[k] = __fmul_rn(dec_value(b, S), __ldg(invc + l));
  }
}

// Flat-order statistics of a materialised residual: tile partials of
// sum delta^2 and max|delta| (one warp per 4096 flat tile).
__global__ void __launch_bounds__(kBlock) k_error_stats_tiles(
    const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot, uint64_t W, uint64_t c,
    uint64_t len, double* part, float* pmax, int tiles) {
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long tile = gw; tile < tiles; tile += nwarps) {
    double acc = 0.0;
    float mx = 0.0f;
    for (int r = 0; r < kRowsPerTile; ++r) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t k = static_cast<uint64_t>(tile) * kTile + r * kRowElems + 4 * lane + q;
        if (k < len) {
          const uint64_t j = k / c, i = k - j * c;
          const uint32_t* sl = pk + j * slot;
          const float S = slot_scale(sl, W);
          const uint32_t b = (__ldg(sl + (i >> 5)) >> (i & 31)) & 1u;
          const float dlt = __fsub_rn(raw[j * c_pad + i], b ? S : -S);
          acc += static_cast<double>(dlt) * static_cast<double>(dlt);
          const float a = fabsf(dlt);
          mx = mx < a ? a : mx;
        }
      }
    }
    acc = warp_bfly_sum(acc);
    mx = warp_max(mx);
    if (lane == 0) {
      part[tile] = acc;
      pmax[tile] = mx;
    }
  }
}

// EndpointStats of one endpoint (comm_sim.cpp:108-118, 175-180), updated on
// the device: ||delta||_2 (canonical combine of the tile partials), max|delta|,
// max|corrected| (the compressing kernel's per-tile maxima) and the running
// maxima.  st = {delta_l2, delta_linf, corrected_linf, max_delta_linf,
// max_corrected_linf}; read by the host only when queried.
__global__ void __launch_bounds__(1024) k_error_stats_final(const double* part, const float* pmax,
                                                            int tiles, const float* cmax, int cmax_n,
                                                            double* st) {
  __shared__ double shd[32];
  __shared__ float shf[32];
  double s = 0.0;
  float mx = 0.0f, cm = 0.0f;
  for (int t = threadIdx.x; t < tiles; t += 1024) {
    s += part[t];
    mx = mx < pmax[t] ? pmax[t] : mx;
  }
  for (int t = threadIdx.x; t < cmax_n; t += 1024) cm = cm < cmax[t] ? cmax[t] : cm;
  s = block1024_sum(s, shd);
  mx = block1024_max(mx, shf);
  cm = block1024_max(cm, shf);
  if (threadIdx.x == 0) {
    const double linf = mx, cinf = cm;
    st[0] = sqrt(s);
    st[1] = linf;
    st[2] = cinf;
    st[3] = st[3] < linf ? linf : st[3];
    st[4] = st[4] < cinf ? cinf : st[4];
  }
}

__global__ void k_set_float(float* p, float v) { *p = v; }

__global__ void k_verify(const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot,
                         uint64_t W, uint64_t c, uint64_t len, double tol, unsigned long long* err) {
  if (gate_closed_call(err)) return;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t j = k / c, i = k - j * c;
    const uint32_t* sl = pk + j * slot;
    const float S = slot_scale(sl, W);
    const uint32_t b = (__ldg(sl + (i >> 5)) >> (i & 31)) & 1u;
    const float r = raw[j * c_pad + i];             // corrected (es == 1)
    const float dn = __fsub_rn(r, b ? S : -S);      // delta_new (compression.cpp:194-195)
    const double lhs = r, dec = dec_value(b, S);    // decompress (compression.cpp:68-81)
    const double rhs = dec + static_cast<double>(dn);
    double den = fabs(lhs);
    den = fabs(dec) > den ? fabs(dec) : den;
    den = den < 1e-300 ? 1e-300 : den;
    if (fabs(lhs - rhs) > tol * den) flag(err, kErrVerify, i);
  }
}

// Stream-ordered wait for n peer signals (fused NVLink exchange).
__global__ void k_wait_peers(const unsigned long long* flags, int n, unsigned long long epoch,
                             unsigned long long* err) {
  if (gate_closed_call(err)) return;
  wait_peers(flags, n, epoch, err);
}

// ---------------------------------------------------------------------------
// Step gate.  check_gradients (optimizers.cpp:99-117) validates every worker's
// gradient before any state changes; strict mode restates that with a
// read-only pre-pass (k_check_finite) whose finding closes the gate before the
// first mutating kernel.  Multi-process, the gate kernel is also the step's
// arrival barrier, so a rank that is late past the bound aborts the step on
// every rank before anything is written (fail-stop, state unchanged).
// ---------------------------------------------------------------------------
__global__ void k_check_finite(const float* in, uint64_t stride, int nw, uint64_t d,
                               unsigned long long* err, int worker_base) {
  if (gate_closed_call(err)) return;
  const uint64_t d4 = d / 4;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (int w = 0; w < nw; ++w) {
    const float* g = in + static_cast<size_t>(w) * stride;
    const unsigned long long wk = static_cast<unsigned long long>(worker_base + w) << 40;
    for (uint64_t k4 = tid; k4 < d4; k4 += nth) {
      const float4 v = ldg_ro(g + 4 * k4);
      if (!(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w))) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (!isfinite(comp(v, q))) flag(err, kErrGrad, wk | (4 * k4 + q));
      }
    }
    for (uint64_t k = 4 * d4 + tid; k < d; k += nth)
      if (!isfinite(g[k])) flag(err, kErrGrad, wk | k);
  }
}

__device__ __forceinline__ unsigned long long local_nonfinite_layer(const unsigned long long* err,
                                                                   const uint64_t* off, int L) {
  const unsigned long long key = ld_volatile_u64(err + kErrGrad);
  if (key == ~0ull) return 0;  // finite
  const uint64_t k = key & ((1ull << 40) - 1);
  return (off ? static_cast<unsigned long long>(find_layer(off, L, k)) : 0ull) + 1;  // layer + 1
}

__global__ void k_step_gate(const GateParams p) {
  if (threadIdx.x != 0) return;
  unsigned long long* err = p.err;
  if (gate_closed_call(err)) return;  // an earlier failure is still unreported: this step is skipped too
  const unsigned long long status = p.strict ? local_nonfinite_layer(err, p.off, p.L) : 0;
  if (p.peer_flags == nullptr || p.n == 1) {
    if (status) {
      atomicMin(err + kErrGateSeq, p.seq);
      close_gate(err, kGateNonFinite);
    }
    return;
  }
  // Arrival: (epoch << 32) | status, into every rank's arrival word of this rank.
  const unsigned long long mine = (p.epoch << 32) | (status & 0xffffffffull);
  for (int q = 0; q < p.n; ++q) st_relaxed_sys(p.peer_flags[q] + p.arrive_index + p.rank, mine);
  const unsigned long long bound = wait_bound(err), t0 = now_ns();
  int missing = -1;
  for (int q = 0; q < p.n && missing < 0; ++q) {
    while ((ld_acquire_sys(p.arrive + q) >> 32) < p.epoch) {
      if (now_ns() - t0 > bound) {
        missing = q;
        break;
      }
      __nanosleep(32);
    }
  }
  // One decision per epoch, CAS-ed into rank 0's word: the first rank to
  // decide (go: all arrived / abort: someone missing) decides for everyone.
  unsigned long long* dec = p.peer_flags[0] + p.decision_index;
  const unsigned long long want =
      (p.epoch << 32) | (missing < 0 ? (1ull << 16) : ((2ull << 16) | static_cast<unsigned>(missing)));
  unsigned long long cur = ld_acquire_sys(dec), decided = want;
  while (true) {
    if ((cur >> 32) == p.epoch) {
      decided = cur;
      break;
    }
    const unsigned long long prev = atomicCAS_system(dec, cur, want);
    if (prev == cur) break;  // ours
    cur = prev;
  }
  if (((decided >> 16) & 0xffffull) != 1ull) {  // abort: nobody touches the state
    flag(err, kErrPeer, decided & 0xffffull);
    atomicMin(err + kErrGateSeq, p.seq);
    close_gate(err, kGateArrival);
    return;
  }
  // Go: every rank arrived; the lowest rank with a non-finite gradient is
  // reported by every rank (the arrivals are all posted, so this terminates).
  for (int q = 0; q < p.n; ++q) {
    unsigned long long a;
    while (((a = ld_acquire_sys(p.arrive + q)) >> 32) < p.epoch) __nanosleep(32);
    const unsigned long long st = a & 0xffffffffull;
    if (st != 0 && (a >> 32) == p.epoch) {
      flag(err, kErrRemote, (static_cast<unsigned long long>(q) << 32) | (st - 1));
      atomicMin(err + kErrGateSeq, p.seq);
      close_gate(err, q == p.rank ? kGateNonFinite : kGateRemoteNonFinite);
      return;
    }
  }
}

// NCCL transport: status word = rank << 32 | layer of this rank's first
// non-finite element (strict pre-pass), ~0 if finite; min-reduced over ranks.
__global__ void k_gate_status(unsigned long long* err, const uint64_t* off, int L, int rank,
                              unsigned long long* status) {
  if (threadIdx.x != 0) return;
  const unsigned long long st = gate_closed(err) ? 0ull : local_nonfinite_layer(err, off, L);
  *status = st ? (static_cast<unsigned long long>(rank) << 32) | (st - 1) : ~0ull;
}

__global__ void k_gate_apply(unsigned long long* err, const unsigned long long* status, int rank,
                             unsigned long long seq) {
  if (threadIdx.x != 0 || gate_closed(err)) return;
  const unsigned long long st = *status;
  if (st == ~0ull) return;
  flag(err, kErrRemote, st);
  atomicMin(err + kErrGateSeq, seq);
  close_gate(err, static_cast<int>(st >> 32) == rank ? kGateNonFinite : kGateRemoteNonFinite);
}

// ---------------------------------------------------------------------------
// Free functions of fusion.hpp:92-102 (compute_scales, apply/remove_scaling).
// ---------------------------------------------------------------------------
// Per-layer tile partials of |x| in the canonical tile-tree order (oracle
// tile_partial), one warp per tile.
__global__ void k_layer_abs_tiles(const float* x, const uint64_t* off, const int* tile_layer,
                                  const int* layer_tile_start, int tiles, double* part) {
  const int lane = threadIdx.x & 31;
  const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long tile = gw; tile < tiles; tile += nwarps) {
    const int l = tile_layer[tile];
    const uint64_t t = static_cast<uint64_t>(tile - layer_tile_start[l]);
    const uint64_t lo = off[l], len = off[l + 1] - lo;
    double acc = 0.0;
    for (int r = 0; r < kRowsPerTile; ++r)
      for (int q = 0; q < 4; ++q) {
        const uint64_t i = t * kTile + static_cast<uint64_t>(r) * kRowElems + 4 * lane + q;
        if (i < len) acc += fabs(static_cast<double>(x[lo + i]));
      }
    acc = warp_bfly_sum(acc);
    if (lane == 0) part[tile] = acc;
  }
}

// compute_scales (fusion.cpp:107-125): block l combines its layer's partials
// (k_finalize_scales' order), s_l = max(sum / len, floor); the last block forms
// reference = (sum_l s_l) / L in layer order and coeff_l = reference / s_l.
__global__ void __launch_bounds__(1024) k_scales_final(int L, const int* layer_tile_start,
                                                       const uint64_t* off, const double* part,
                                                       double floor_, double* mag, double* coeff,
                                                       double* ref_out, unsigned int* counter) {
  __shared__ double sh[32];
  __shared__ bool last;
  const int l = blockIdx.x;
  double s = stripe_sum(part, layer_tile_start[l] + threadIdx.x, layer_tile_start[l + 1]);
  s = block1024_sum(s, sh);
  if (threadIdx.x == 0) {
    const uint64_t len = off[l + 1] - off[l];
    const double mean = len == 0 ? 0.0 : s / static_cast<double>(len);  // vector_ops.cpp:41-44
    mag[l] = mean < floor_ ? floor_ : mean;                            // fusion.cpp:116
    __threadfence();
    last = atomicAdd(counter, 1u) == static_cast<unsigned>(L - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const volatile double* m = mag;
    double ref = 0.0;
    for (int k = 0; k < L; ++k) ref += m[k];  // fusion.cpp:118-120
    ref /= static_cast<double>(L);
    for (int k = 0; k < L; ++k) coeff[k] = ref / m[k];  // :121-124
    *ref_out = ref;
    *counter = 0u;
  }
}

// apply_scaling / remove_scaling (fusion.cpp:127-149): x[k] *= mul[layer(k)],
// mul = (float)coeff or (float)(1.0 / coeff) formed in double once per layer.
__global__ void k_scale_layers(float* x, const uint64_t* off, int L, const float* mul, uint64_t d) {
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < d;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int l = find_layer(off, L, k);
    x[k] = __fmul_rn(x[k], __ldg(mul + l));
  }
}

__global__ void k_build_stream(float* in, uint64_t stride, int nw, uint64_t d, const float* m,
                               const uint64_t* off, int L, const float* A, const float* B,
                               unsigned long long* err, int worker_base) {
  if (gate_closed_call(err)) return;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < d;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int l = find_layer(off, L, k);
    const float a = __ldg(A + l), b = __ldg(B + l), mk = m[k];
    for (int w = 0; w < nw; ++w) {
      float* g = in + static_cast<size_t>(w) * stride + k;
      const float gv = *g;
      if (!isfinite(gv)) flag(err, kErrGrad, (static_cast<unsigned long long>(worker_base + w) << 40) | k);
      *g = __fadd_rn(__fmul_rn(a, mk), __fmul_rn(b, gv));  // kernels.cpp:253
    }
  }
}

// Cap a persistent grid at the number of co-resident blocks of `kernel`.
template <typename K>
int resident(K kernel, int want) {
  static thread_local std::unordered_map<const void*, int> cache;
  const void* key = reinterpret_cast<const void*>(kernel);
  auto it = cache.find(key);
  if (it == cache.end()) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kBlock, 0);
    it = cache.emplace(key, sms * (occ > 0 ? occ : 1)).first;
  }
  return want < it->second ? want : it->second;
}

int grid_for_elems(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return static_cast<int>(g < 148 * 16 ? (g == 0 ? 1 : g) : 148 * 16);
}

}  // namespace

template <int MODE, int R>
int launch_k1_bulk(const K1Params& p, cudaStream_t s) {
  static thread_local int grid = 0;
  constexpr int smem = BulkGeom<R>::Smem;
  if (grid == 0) {
    cudaFuncSetAttribute(k1_bulk<MODE, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1_bulk<MODE, R>, kBulkWarps * 32, smem);
    grid = sms * (occ > 0 ? occ : 1);
  }
  k1_bulk<MODE, R><<<grid, kBulkWarps * 32, smem, s>>>(p);
  return 1;
}

// Rows per bulk stage (BL_K1_BULK_R=4|8, default 4: 4 blocks of 4 warps per
// SM; 8 halves the resident warps) and whether aligned chunks also take the
// bulk path (BL_K1_BULK=all|none) — tuning knobs.
static int bulk_rows() {
  static const int r = [] {
    const char* e = std::getenv("BL_K1_BULK_R");
    return e && std::atoi(e) == 8 ? 8 : 4;
  }();
  return r;
}
static bool bulk_all() {
  static const bool a = [] {
    const char* e = std::getenv("BL_K1_BULK");
    return e && std::string(e) == "all";
  }();
  return a;
}
static bool bulk_none() {
  static const bool a = [] {
    const char* e = std::getenv("BL_K1_BULK");
    return e && std::string(e) == "none";
  }();
  return a;
}

bool k1_uses_bulk(const K1Params& p, int mode) {
  // Only odd chunk lengths (4-byte-aligned chunk starts) go through the bulk
  // pipeline; 8-byte-aligned chunks load as float2 on the register path,
  // which measures faster there (BERT-L sim2: 1.35 vs 1.42 ms).
  // A single chunk (n == 1) starts at element 0 and is always aligned.
  // Small problems (at most 16384 K1 tiles, e.g. config 0: 7.8K) are
  // latency-bound and measure faster on the register path (config 0 K1
  // 123 -> 105 us, profiles/round2_cfg0_k1.txt).
  const bool misaligned = (p.c & 1u) != 0 && p.n > 1;
  const bool large = static_cast<long long>(p.nw) * p.n * p.tpc > 16384ll;
  return mode != 1 && (mode == 0 || p.tile_layer) && ((misaligned && large) || bulk_all()) && !bulk_none();
}

int launch_k1_phase(const K1Params& p, int mode, int phase, cudaStream_t s) {
  if (phase == 0) {
    if (bulk_rows() == 4) return mode == 0 ? launch_k1_bulk<0, 4>(p, s) : launch_k1_bulk<2, 4>(p, s);
    return mode == 0 ? launch_k1_bulk<0, 8>(p, s) : launch_k1_bulk<2, 8>(p, s);
  }
  (void)p;
  (void)mode;
  (void)s;
  return 0;  // the boundary tiles run inside k1_bulk
}

int launch_k1(const K1Params& p, int mode, int grid, cudaStream_t s) {
  if (k1_uses_bulk(p, mode)) {
    // Odd chunks: fast tiles through the bulk-copy pipeline (g staged with
    // alignment slack); the boundary tiles run in the same kernel from the
    // slow list.  Aligned chunks stay on the register path.
    return launch_k1_phase(p, mode, 0, s);
  }
  K1Params full = p;  // register path: every tile, the slow list does not apply
  full.slow_list = nullptr;
  full.n_slow = 0;
  full.skip_fast = 0;
#define BL_K1(M, A) k1_worker_compress<M, A><<<resident(k1_worker_compress<M, A>, grid), kBlock, 0, s>>>(full)
  const bool al = (p.c & 3u) == 0 || p.n == 1;  // every chunk start 16-byte aligned
  switch (mode) {
    case 0: if (al) BL_K1(0, true); else BL_K1(0, false); break;
    case 1: BL_K1(1, false); break;
    default: if (al) BL_K1(2, true); else BL_K1(2, false); break;
  }
#undef BL_K1
  return 1;
}

int launch_finalize(const FinalizeParams& p, int count, cudaStream_t s) {
  k_finalize_scales<<<count, 1024, 0, s>>>(p);
  return 1;
}

int launch_k3(const K3Params& p, int grid, cudaStream_t s) {
  switch (p.n) {
    case 1: k3_server_reduce<1><<<resident(k3_server_reduce<1>, grid), kBlock, 0, s>>>(p); break;
    case 2: k3_server_reduce<2><<<resident(k3_server_reduce<2>, grid), kBlock, 0, s>>>(p); break;
    case 4: k3_server_reduce<4><<<resident(k3_server_reduce<4>, grid), kBlock, 0, s>>>(p); break;
    case 8: k3_server_reduce<8><<<resident(k3_server_reduce<8>, grid), kBlock, 0, s>>>(p); break;
    default: k3_server_reduce<0><<<resident(k3_server_reduce<0>, grid), kBlock, 0, s>>>(p); break;
  }
  return 1;
}

int launch_k5(const K5Params& p, int grid, cudaStream_t s) {
#define BL_K5(M, X) k5_update_a<M, X><<<resident(k5_update_a<M, X>, grid), kBlock, 0, s>>>(p)
  if (p.res_prev) {
    if (p.lt.mis) BL_K5(1, true); else BL_K5(1, false);
  } else {
    if (p.lt.mis) BL_K5(0, true); else BL_K5(0, false);
  }
#undef BL_K5
  return 1;
}

int launch_k5_general(const K5Params& p, cudaStream_t s) {
  if (!p.gen_list || p.gen_count == 0) return 0;
  const int g = (p.gen_count + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (p.res_prev) k5_general<1><<<g, kBlock, 0, s>>>(p);
  else k5_general<0><<<g, kBlock, 0, s>>>(p);
  return 1;
}

int launch_epilogue(const EpiParams& p, cudaStream_t s) {
  k_epilogue<<<p.L, 1024, 0, s>>>(p);
  return 1;
}

int launch_k6(const K6Params& p, int grid, cudaStream_t s) {
  if (p.lt.mis) k6_update_b<true><<<resident(k6_update_b<true>, grid), kBlock, 0, s>>>(p);
  else k6_update_b<false><<<resident(k6_update_b<false>, grid), kBlock, 0, s>>>(p);
  return 1;
}

int launch_k6_general(const K6Params& p, cudaStream_t s) {
  if (!p.gen_list || p.gen_count == 0) return 0;
  k6_general<<<(p.gen_count + kWarpsPerBlock - 1) / kWarpsPerBlock, kBlock, 0, s>>>(p);
  return 1;
}

int launch_w1(const W1Params& p, int grid, cudaStream_t s) {
  if (p.lt.mis) kw1_warmup_a<true><<<resident(kw1_warmup_a<true>, grid), kBlock, 0, s>>>(p);
  else kw1_warmup_a<false><<<resident(kw1_warmup_a<false>, grid), kBlock, 0, s>>>(p);
  return 1;
}

int launch_wepilogue(const WEpiParams& p, cudaStream_t s) {
  k_wepilogue<<<p.layer_list ? p.count : p.L, 1024, 0, s>>>(p);
  return 1;
}

int launch_w2(const W2Params& p, int grid, cudaStream_t s) {
  if (p.lt.mis) kw2_warmup_b<true><<<resident(kw2_warmup_b<true>, grid), kBlock, 0, s>>>(p);
  else kw2_warmup_b<false><<<resident(kw2_warmup_b<false>, grid), kBlock, 0, s>>>(p);
  return 1;
}

int launch_average(const float* in, uint64_t stride, int n, uint64_t len, float* out,
                   unsigned long long* err, int check_finite, int worker_base, cudaStream_t s) {
  const bool vec = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && stride % 4 == 0;
  if (vec) {
    k_average4<<<grid_for_elems(len / 4 + 1), 256, 0, s>>>(in, stride, n, len, out, err, check_finite,
                                                          worker_base);
  } else {
    k_average<<<grid_for_elems(len), 256, 0, s>>>(in, stride, n, len, out, err, check_finite,
                                                   worker_base);
  }
  return 1;
}

int launch_decompress(const uint32_t* res, int n, uint64_t c, uint64_t slot, uint64_t W,
                      uint64_t d, float* out, const unsigned long long* gate, cudaStream_t s) {
  k_decompress<<<grid_for_elems(d / 128 + 1), 256, 0, s>>>(res, n, c, slot, W, d, out, gate);
  return 1;
}

int launch_materialize_error(const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot,
                             uint64_t W, uint64_t c, uint64_t len, float* out, cudaStream_t s) {
  k_materialize_error<<<grid_for_elems(len), 256, 0, s>>>(raw, c_pad, pk, slot, W, c, len, out);
  return 1;
}

int launch_materialize_m(const uint32_t* res, int n, uint64_t c, uint64_t slot, uint64_t W,
                         const uint64_t* off, int L, const float* invc, uint64_t d, float* out,
                         cudaStream_t s) {
  k_materialize_m<<<grid_for_elems(d), 256, 0, s>>>(res, n, c, slot, W, off, L, invc, d, out);
  return 1;
}

int launch_error_stats(const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot,
                       uint64_t W, uint64_t c, uint64_t len, double* scratch, int scratch_tiles,
                       float* scratch_max, const float* cmax, int cmax_n, double* st, cudaStream_t s) {
  const int g = scratch_tiles / kWarpsPerBlock + 1;
  k_error_stats_tiles<<<g < 148 * 8 ? g : 148 * 8, kBlock, 0, s>>>(
      raw, c_pad, pk, slot, W, c, len, scratch, scratch_max, scratch_tiles);
  k_error_stats_final<<<1, 1024, 0, s>>>(scratch, scratch_max, scratch_tiles, cmax, cmax_n, st);
  return 2;
}

int launch_build_stream(float* in, uint64_t stride, int nw, uint64_t d, const float* m,
                        const uint64_t* off, int L, const float* A, const float* B,
                        unsigned long long* err, int worker_base, cudaStream_t s) {
  k_build_stream<<<grid_for_elems(d), 256, 0, s>>>(in, stride, nw, d, m, off, L, A, B, err, worker_base);
  return 1;
}

template <int MODE, bool ALIGNED, int NT>
static int launch_small_nt(const SmallParams& p, long long tiles, cudaStream_t s) {
  auto kern = k_small_collective<MODE, ALIGNED, NT>;
  static thread_local int cap = 0;  // co-resident blocks (cooperative launch)
  if (cap == 0) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBlock, 0);
    cap = sms * (occ > 0 ? occ : 1);
  }
  long long want = tiles;            // one CTA per tile
  if (want < p.k1.n) want = p.k1.n;  // one block per worker endpoint
  const int grid = static_cast<int>(std::min<long long>(want, cap));
  void* args[] = {const_cast<SmallParams*>(&p)};
  // (A plain launch measured 0.5-1 us faster at 1-4 MB: not worth giving up
  // the co-residency guarantee the LL polls rely on.)
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), grid, kBlock,
                                                    args, 0, s);
  return e == cudaSuccess ? 1 : -static_cast<int>(e);
}

template <int MODE, bool ALIGNED>
static int launch_small_t(const SmallParams& p, long long tiles, cudaStream_t s) {
  const int n = p.k1.n;
#ifndef BL_SMALL_NT8  // (A/B knob: one instantiation for every n)
  if (n <= 2) return launch_small_nt<MODE, ALIGNED, 2>(p, tiles, s);
  if (n <= 4) return launch_small_nt<MODE, ALIGNED, 4>(p, tiles, s);
#endif
  return launch_small_nt<MODE, ALIGNED, 8>(p, tiles, s);
}

int launch_small_collective(const SmallParams& p, int k1_mode, cudaStream_t s) {
  const long long tiles = static_cast<long long>(p.k1.n) * p.k1.tpc;
  const bool al = (p.k1.c & 3u) == 0;
  if (k1_mode == 0) return al ? launch_small_t<0, true>(p, tiles, s) : launch_small_t<0, false>(p, tiles, s);
  if (k1_mode == 1) return launch_small_t<1, false>(p, tiles, s);
  return al ? launch_small_t<2, true>(p, tiles, s) : launch_small_t<2, false>(p, tiles, s);
}

int lossless_piece(uint64_t lo, uint64_t hi, int pieces, uint64_t k, int shape) {
  const uint64_t up = (lo + 3) & ~3ull, dn = hi & ~3ull;
  const uint64_t a0 = up < hi ? up : hi;
  const uint64_t a1 = dn > a0 ? dn : a0;
  if (k < a0) return 0;
  if (k >= a1) return pieces - 1;
  int p = static_cast<int>((k - a0) * static_cast<uint64_t>(pieces) / (a1 - a0));
  while (p > 0 && k < piece_body_start(a0, a1, pieces, p, shape)) --p;
  while (p + 1 < pieces && k >= piece_body_start(a0, a1, pieces, p + 1, shape)) ++p;
  return p;
}

int launch_wait_piece(const unsigned long long* flags, int base, int n, int pieces, int pc,
                      unsigned long long epoch, unsigned long long* err, cudaStream_t s) {
  k_wait_piece<<<1, 32, 0, s>>>(flags, base, n, pieces, pc, epoch, err);
  return 1;
}

int launch_lossless_p2p(const LosslessP2PParams& p, int sms, cudaStream_t s) {
  const long long groups = static_cast<long long>((p.hi ? p.hi - p.lo : p.c) / 4) + 1;
  const long long cap = p.ctas > 0 ? p.ctas : 8ll * sms;
  const int want = static_cast<int>(std::min<long long>((groups + 255) / 256, cap));  // (256-thread estimate)
  const int bt = p.block > 0 ? p.block : 256;
  switch (p.n) {
    case 2: k_lossless_p2p<2><<<resident(k_lossless_p2p<2>, want), bt, 0, s>>>(p); break;
    case 4: k_lossless_p2p<4><<<resident(k_lossless_p2p<4>, want), bt, 0, s>>>(p); break;
    case 8: k_lossless_p2p<8><<<resident(k_lossless_p2p<8>, want), bt, 0, s>>>(p); break;
    default: k_lossless_p2p<0><<<resident(k_lossless_p2p<0>, want), bt, 0, s>>>(p); break;
  }
  return 1;
}

int launch_push_range(const float* src, float* const* dst, int ndst, uint64_t off, uint64_t count,
                      const unsigned long long* gate, int sms, cudaStream_t s) {
  if (count == 0 || ndst == 0) return 0;
  const uint64_t want = (count + 255) / 256;
  k_push_range<float><<<static_cast<int>(want < static_cast<uint64_t>(4 * sms) ? want : 4 * sms), 256, 0, s>>>(
      src, dst, ndst, off, count, gate);
  return 1;
}
int launch_push_range(const double* src, double* const* dst, int ndst, uint64_t off, uint64_t count,
                      const unsigned long long* gate, int sms, cudaStream_t s) {
  if (count == 0 || ndst == 0) return 0;
  const uint64_t want = (count + 255) / 256;
  k_push_range<double><<<static_cast<int>(want < static_cast<uint64_t>(4 * sms) ? want : 4 * sms), 256, 0, s>>>(
      src, dst, ndst, off, count, gate);
  return 1;
}

int launch_shard_push(const ShardPushParams& p, int ctas, cudaStream_t s) {
  k_shard_push<<<ctas, 256, 0, s>>>(p);
  return 1;
}
int launch_shard_reduce(const ShardReduceParams& p, int sms, cudaStream_t s) {
  k_shard_reduce<<<2 * sms, 256, 0, s>>>(p);
  return 1;
}

int launch_signal_peers(unsigned long long* const* peer_flags, int index, int n,
                        unsigned long long epoch, const unsigned long long* gate, cudaStream_t s) {
  k_signal_peers<<<1, 32, 0, s>>>(peer_flags, index, n, epoch, gate);
  return 1;
}

int launch_wait_peers(const unsigned long long* flags, int n, unsigned long long epoch,
                      unsigned long long* err, cudaStream_t s) {
  k_wait_peers<<<1, 32, 0, s>>>(flags, n, epoch, err);
  return 1;
}

int launch_layer_abs_tiles(const float* x, const uint64_t* off, const int* tile_layer,
                           const int* layer_tile_start, int tiles, double* part, cudaStream_t s) {
  const int g = (tiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_layer_abs_tiles<<<g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16, kBlock, 0, s>>>(x, off, tile_layer,
                                                                                layer_tile_start, tiles, part);
  return 1;
}

int launch_scales_final(int L, const int* layer_tile_start, const uint64_t* off, const double* part,
                        double floor_, double* mag, double* coeff, double* ref_out, unsigned int* counter,
                        cudaStream_t s) {
  k_scales_final<<<L, 1024, 0, s>>>(L, layer_tile_start, off, part, floor_, mag, coeff, ref_out, counter);
  return 1;
}

int launch_scale_layers(float* x, const uint64_t* off, int L, const float* mul, uint64_t d, cudaStream_t s) {
  k_scale_layers<<<grid_for_elems(d), 256, 0, s>>>(x, off, L, mul, d);
  return 1;
}

int launch_check_finite(const float* in, uint64_t stride, int nw, uint64_t d, unsigned long long* err,
                        int worker_base, cudaStream_t s) {
  k_check_finite<<<grid_for_elems(d / 4 + 1), 256, 0, s>>>(in, stride, nw, d, err, worker_base);
  return 1;
}

int launch_step_gate(const GateParams& p, cudaStream_t s) {
  k_step_gate<<<1, 32, 0, s>>>(p);
  return 1;
}

int launch_gate_status(unsigned long long* err, const uint64_t* off, int L, int rank,
                       unsigned long long* status, cudaStream_t s) {
  k_gate_status<<<1, 32, 0, s>>>(err, off, L, rank, status);
  return 1;
}

int launch_gate_apply(unsigned long long* err, const unsigned long long* status, int rank,
                      unsigned long long seq, cudaStream_t s) {
  k_gate_apply<<<1, 32, 0, s>>>(err, status, rank, seq);
  return 1;
}

int launch_verify(const float* raw, uint64_t c_pad, const uint32_t* pk, uint64_t slot, uint64_t W,
                  uint64_t c, uint64_t len, double tol, unsigned long long* err, cudaStream_t s) {
  k_verify<<<grid_for_elems(len), 256, 0, s>>>(raw, c_pad, pk, slot, W, c, len, tol, err);
  return 1;
}

int launch_set_float(float* p, float v, cudaStream_t s) {
  k_set_float<<<1, 1, 0, s>>>(p, v);
  return 1;
}

}  // namespace bl

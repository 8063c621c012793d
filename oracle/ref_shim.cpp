// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// A flat extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libbitlamb_ref.so). It exists so the Python parity suite and
// bench.py's reference arm can drive the reference's own SimCluster /
// Optimizer (comm_sim.hpp:72-148, optimizers.hpp:93-145) on identical inputs.
// Nothing on the product path links or loads this file.
//
// Exceptions are mapped to the same status codes the product C-ABI returns
// (include/bitlamb_b200.h, bl_status), following errors.hpp:26-53.
//
// The reference keeps the per-collective packets private (comm_sim.hpp:141,
// `inbox_`).  To compare packet bytes bit-for-bit the shim opens the class
// with the classic test-only `#define private public` before including the
// headers; the library objects themselves are compiled untouched.

#include <chrono>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(_OPENMP)
#include <omp.h>
#endif

// Standard headers are included first so the macro below only opens the
// reference's own classes.
#define private public
#include "bitlamb/comm_sim.hpp"
#include "bitlamb/compression.hpp"
#include "bitlamb/errors.hpp"
#include "bitlamb/fusion.hpp"
#include "bitlamb/optimizers.hpp"
#undef private

using namespace bitlamb;

namespace {

thread_local std::string g_err;

enum {
  kOk = 0,
  kDimension = 1,
  kStageOrder = 2,
  kConfig = 3,
  kInvalidArgument = 4,
  kRuntime = 5,
  kLogic = 6,
  kOther = 7,
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return kDimension;
  } catch (const StageOrderError& e) {
    g_err = e.what();
    return kStageOrder;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return kConfig;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalidArgument;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return kRuntime;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return kLogic;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

struct OptBox {
  Optimizer opt;
  std::vector<std::size_t> sizes;
  // bench.py's reference arm: gradients already in the reference's own
  // [worker][layer] DenseVector form, so only Optimizer::step is timed.
  std::vector<std::vector<DenseVector>> loaded;
};

HyperParams unpack_hp(const double* hp, std::uint64_t total, std::uint64_t warmup,
                      int scaled_ef) {
  HyperParams h;
  h.beta1 = hp[0];
  h.beta2 = hp[1];
  h.beta3 = hp[2];
  h.eta = hp[3];
  h.c_min = hp[4];
  h.c_max = hp[5];
  h.r_min = hp[6];
  h.r_max = hp[7];
  h.r_threshold = hp[8];
  h.weight_decay = hp[9];
  h.division_floor = hp[10];
  h.total_steps = total;
  h.warmup_steps = warmup;
  h.scaled_error_feedback = scaled_ef != 0;
  return h;
}

}  // namespace

extern "C" {

const char* oc_last_error() { return g_err.c_str(); }
int oc_real_bytes() { return 8; }

// OpenMP team size for the reference's parallel loops (the reference itself
// reads OMP_NUM_THREADS; launchers such as torchrun force it to 1).
int oc_set_threads(int n) {
#if defined(_OPENMP)
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

// ---- SimCluster -----------------------------------------------------------
int oc_cluster_new(int n, std::uint64_t dim, int kind, int baseline_bits,
                   int verify, void** out) {
  return guarded([&] {
    SimCluster::Config cfg;
    cfg.n_workers = n;
    cfg.dim = dim;
    cfg.compressor = kind == 0 ? CompressorKind::kOneBit : CompressorKind::kIdentity;
    cfg.baseline_bits_per_element = baseline_bits;
    cfg.verify_compensation = verify != 0;
    *out = new SimCluster(cfg);
  });
}

void oc_cluster_free(void* c) { delete static_cast<SimCluster*>(c); }

std::uint64_t oc_cluster_padded(void* c) { return static_cast<SimCluster*>(c)->padded_; }
std::uint64_t oc_cluster_chunk(void* c) { return static_cast<SimCluster*>(c)->chunk_len_; }

int oc_cluster_compressed_allreduce(void* c, const double* inputs, double es,
                                    double* out) {
  auto* cl = static_cast<SimCluster*>(c);
  return guarded([&] {
    std::vector<DenseVector> in;
    for (int i = 0; i < cl->n_workers(); ++i) {
      in.emplace_back(std::span<const double>(inputs + i * cl->dim(), cl->dim()));
    }
    DenseVector r = cl->compressed_allreduce(in, es);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

// n_inputs may differ from n_workers (used to test the DimensionError path).
int oc_cluster_compressed_allreduce_n(void* c, const double* inputs, int n_inputs,
                                      std::uint64_t len, double es, double* out) {
  auto* cl = static_cast<SimCluster*>(c);
  return guarded([&] {
    std::vector<DenseVector> in;
    for (int i = 0; i < n_inputs; ++i) {
      in.emplace_back(std::span<const double>(inputs + i * len, len));
    }
    DenseVector r = cl->compressed_allreduce(in, es);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int oc_cluster_lossless_allreduce(void* c, const double* inputs, double* out) {
  auto* cl = static_cast<SimCluster*>(c);
  return guarded([&] {
    std::vector<DenseVector> in;
    for (int i = 0; i < cl->n_workers(); ++i) {
      in.emplace_back(std::span<const double>(inputs + i * cl->dim(), cl->dim()));
    }
    DenseVector r = cl->lossless_allreduce(in);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

void oc_cluster_worker_error(void* c, int i, double* out) {
  auto s = static_cast<SimCluster*>(c)->worker_error(i);
  std::memcpy(out, s.data(), s.size() * sizeof(double));
}

void oc_cluster_server_error(void* c, int j, double* out) {
  auto s = static_cast<SimCluster*>(c)->server_error(j);
  std::memcpy(out, s.data(), s.size() * sizeof(double));
}

// out[6] = gather, scatter, lossless, baseline_equivalent, n_compressed, n_lossless
void oc_cluster_ledger(void* c, std::uint64_t* out) {
  const VolumeLedger& l = static_cast<SimCluster*>(c)->ledger();
  out[0] = l.gather_bits;
  out[1] = l.scatter_bits;
  out[2] = l.lossless_bits;
  out[3] = l.baseline_equivalent_bits;
  out[4] = l.compressed_collectives;
  out[5] = l.lossless_collectives;
}

// out[(2n) * 5]: workers then servers; {delta_l2, delta_linf, corrected_linf,
// max_delta_linf, max_corrected_linf}
void oc_cluster_stats(void* c, double* out) {
  auto* cl = static_cast<SimCluster*>(c);
  int k = 0;
  auto put = [&](const SimCluster::EndpointStats& s) {
    out[k++] = s.delta_l2;
    out[k++] = s.delta_linf;
    out[k++] = s.corrected_linf;
    out[k++] = s.max_delta_linf;
    out[k++] = s.max_corrected_linf;
  };
  for (const auto& s : cl->worker_stats()) put(s);
  for (const auto& s : cl->server_stats()) put(s);
}

std::uint64_t oc_cluster_compensation_checks(void* c) {
  return static_cast<SimCluster*>(c)->compensation_checks();
}

// Wire bytes (CompressedBlock::serialize, compression.cpp:91-99) of the packet
// worker i posted to server j in the last compressed collective.
int oc_cluster_packet(void* c, int worker, int server, std::uint8_t* bytes) {
  auto* cl = static_cast<SimCluster*>(c);
  return guarded([&] {
    const CompressedChunk& ch = cl->inbox_.at(server).at(worker);
    if (ch.kind() != CompressorKind::kOneBit) throw std::logic_error("identity packet");
    auto b = ch.block().serialize();
    std::memcpy(bytes, b.data(), b.size());
  });
}

// ---- free functions ------------------------------------------------------
int oc_compress_with_feedback(const double* v, double* delta, std::uint64_t d,
                              int kind, double es, std::uint8_t* bytes,
                              double* scale, double* decompressed) {
  return guarded([&] {
    CompressedChunk ch = compress_with_feedback(
        std::span<const double>(v, d), std::span<double>(delta, d),
        kind == 0 ? CompressorKind::kOneBit : CompressorKind::kIdentity, es);
    DenseVector dec = ch.decompress();
    std::memcpy(decompressed, dec.data(), d * sizeof(double));
    if (ch.kind() == CompressorKind::kOneBit) {
      auto b = ch.block().serialize();
      std::memcpy(bytes, b.data(), b.size());
      *scale = ch.block().scale();
    } else {
      *scale = 0.0;
    }
  });
}

int oc_volume_reduction(double w, double bb, double cb, double* out) {
  return guarded([&] { *out = volume_reduction(w, bb, cb); });
}

// ---- Optimizer -------------------------------------------------------------
// variant: 0 lamb, 1 adam, 2 onebit_lamb, 3 lamb_basic_1bit, 4 onebit_adam
int oc_opt_new(int variant, const std::uint64_t* sizes, int L, const double* hp,
               std::uint64_t total, std::uint64_t warmup, int scaled_ef,
               void** out) {
  return guarded([&] {
    std::vector<Optimizer::LayerSpec> specs;
    for (int l = 0; l < L; ++l) {
      specs.push_back({"layer" + std::to_string(l), static_cast<std::size_t>(sizes[l])});
    }
    auto* box = new OptBox{Optimizer(static_cast<OptimizerVariant>(variant), specs,
                                     unpack_hp(hp, total, warmup, scaled_ef)),
                           {}, {}};
    for (int l = 0; l < L; ++l) box->sizes.push_back(sizes[l]);
    *out = box;
  });
}

void oc_opt_free(void* o) { delete static_cast<OptBox*>(o); }

// grads: n * d fused (layer-major inside each worker).
int oc_opt_step(void* o, void* c, const double* grads, int n, std::uint64_t t,
                double lr, double* trace, int* compressed) {
  auto* box = static_cast<OptBox*>(o);
  auto* cl = static_cast<SimCluster*>(c);
  return guarded([&] {
    const std::size_t d = box->opt.fused_dim();
    std::vector<std::vector<DenseVector>> g(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
      std::size_t off = 0;
      for (std::size_t sz : box->sizes) {
        g[i].emplace_back(std::span<const double>(grads + i * d + off, sz));
        off += sz;
      }
    }
    StepTrace tr = box->opt.step(g, t, lr, *cl);
    const std::size_t L = box->sizes.size();
    for (std::size_t l = 0; l < L; ++l) {
      trace[l] = tr.c[l];
      trace[L + l] = tr.r[l];
      trace[2 * L + l] = tr.v_norm[l];
      trace[3 * L + l] = tr.v_ratio_preclip[l];
    }
    *compressed = tr.compressed ? 1 : 0;
  });
}

// Bench support (bench.py --impl reference): convert n fused gradients once
// into the caller-side form Optimizer::step takes (optimizers.hpp:106-107),
// then time the stock step alone with steady_clock.
int oc_opt_load_grads(void* o, const double* grads, int n) {
  auto* box = static_cast<OptBox*>(o);
  return guarded([&] {
    const std::size_t d = box->opt.fused_dim();
    box->loaded.assign(static_cast<std::size_t>(n), {});
    for (int i = 0; i < n; ++i) {
      std::size_t off = 0;
      for (std::size_t sz : box->sizes) {
        box->loaded[static_cast<std::size_t>(i)].emplace_back(
            std::span<const double>(grads + static_cast<std::size_t>(i) * d + off, sz));
        off += sz;
      }
    }
  });
}

int oc_opt_step_loaded(void* o, void* c, std::uint64_t t, double lr, double* seconds,
                       int* compressed) {
  auto* box = static_cast<OptBox*>(o);
  auto* cl = static_cast<SimCluster*>(c);
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    StepTrace tr = box->opt.step(box->loaded, t, lr, *cl);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    *compressed = tr.compressed ? 1 : 0;
  });
}

// which: 0 x, 1 m, 2 v, 3 v_frozen, 4 m_prev.  Missing optionals read as 0.
void oc_opt_get(void* o, int which, double* out) {
  auto* box = static_cast<OptBox*>(o);
  std::size_t off = 0;
  for (const LayerState& s : box->opt.layers()) {
    const DenseVector* v = nullptr;
    switch (which) {
      case 0: v = &s.x; break;
      case 1: v = &s.m; break;
      case 2: v = &s.v; break;
      case 3: v = s.v_frozen ? &*s.v_frozen : nullptr; break;
      case 4: v = s.m_prev ? &*s.m_prev : nullptr; break;
    }
    const std::size_t n = s.x.size();
    if (v) {
      std::memcpy(out + off, v->data(), n * sizeof(double));
    } else {
      std::memset(out + off, 0, n * sizeof(double));
    }
    off += n;
  }
}

void oc_opt_set(void* o, int which, const double* in) {
  auto* box = static_cast<OptBox*>(o);
  std::size_t off = 0;
  for (LayerState& s : box->opt.mutable_layers()) {
    const std::size_t n = s.x.size();
    DenseVector v(std::span<const double>(in + off, n));
    switch (which) {
      case 0: s.x = v; break;
      case 1: s.m = v; break;
      case 2: s.v = v; break;
      case 3: s.v_frozen = v; break;
      case 4: s.m_prev = v; break;
    }
    off += n;
  }
}

// scalars[3L]: c_avg, r_prev, scale_coeff (MomentumScales::coeff)
void oc_opt_get_scalars(void* o, double* out) {
  auto* box = static_cast<OptBox*>(o);
  const auto& layers = box->opt.layers();
  const std::size_t L = layers.size();
  for (std::size_t l = 0; l < L; ++l) {
    out[l] = layers[l].c_avg;
    out[L + l] = layers[l].r_prev;
    const auto& co = box->opt.momentum_scales().coeff;
    out[2 * L + l] = l < co.size() ? co[l] : 1.0;
  }
}

void oc_opt_set_scalars(void* o, const double* in) {
  auto* box = static_cast<OptBox*>(o);
  auto& layers = box->opt.mutable_layers();
  const std::size_t L = layers.size();
  for (std::size_t l = 0; l < L; ++l) {
    layers[l].c_avg = in[l];
    layers[l].r_prev = in[L + l];
  }
}

int oc_opt_frozen(void* o) { return static_cast<OptBox*>(o)->opt.frozen() ? 1 : 0; }

}  // extern "C"

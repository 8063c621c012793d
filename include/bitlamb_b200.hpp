// bitlamb_b200.hpp — header-only C++ facade over the C-ABI (bitlamb_b200.h).
//
// Re-exposes the reference library's communicator and optimizer shapes
// (/root/reference/proj/include/bitlamb/comm_sim.hpp:72-148 and
// optimizers.hpp:93-145) on the B200 path, and maps bl_status codes back to
// the reference's exception classes (errors.hpp:26-53), so C++ callers of
// bitlamb::SimCluster / bitlamb::Optimizer switch by changing a namespace and
// the element type (fp32 buffers; the reference is fp64).
#ifndef BITLAMB_B200_HPP_
#define BITLAMB_B200_HPP_

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "bitlamb_b200.h"

namespace bitlamb_b200 {

class DimensionError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class StageOrderError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};
class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class NcclError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class Unsupported : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};

inline void check(bl_status s) {
  if (s == BL_OK) return;
  const std::string m = bl_last_error();
  switch (s) {
    case BL_ERR_DIMENSION: throw DimensionError(m);
    case BL_ERR_STAGE_ORDER: throw StageOrderError(m);
    case BL_ERR_CONFIG: throw ConfigError(m);
    case BL_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case BL_ERR_RUNTIME: throw std::runtime_error(m);
    case BL_ERR_LOGIC: throw std::logic_error(m);
    case BL_ERR_CUDA: throw CudaError(m);
    case BL_ERR_NCCL: throw NcclError(m);
    case BL_ERR_UNSUPPORTED: throw Unsupported(m);
    default: throw std::runtime_error(m);
  }
}

enum class CompressorKind { kOneBit = BL_COMPRESSOR_ONEBIT, kIdentity = BL_COMPRESSOR_IDENTITY };
enum class OptimizerVariant {
  kLamb = BL_LAMB,
  kAdam = BL_ADAM,
  kOneBitLamb = BL_ONEBIT_LAMB,
  kLambBasicOneBit = BL_LAMB_BASIC_ONEBIT,
  kOneBitAdam = BL_ONEBIT_ADAM
};

using VolumeLedger = bl_volume_ledger;
using EndpointStats = bl_endpoint_stats;

inline double volume_reduction(double warmup_ratio, double baseline_bits,
                               double compressed_bits_per_element) {
  double out = 0.0;
  check(bl_volume_reduction(warmup_ratio, baseline_bits, compressed_bits_per_element, &out));
  return out;
}

// HyperParams (optimizers.hpp:45-64) with the paper defaults.
struct HyperParams {
  double beta1 = 0.9, beta2 = 0.999, beta3 = 0.9, eta = 1e-6;
  double c_min = 0.01, c_max = 0.3, r_min = 0.5, r_max = 4.0, r_threshold = 0.1;
  double weight_decay = 0.0, division_floor = 1e-12;
  std::size_t total_steps = 0, warmup_steps = 0;
  bool scaled_error_feedback = false;

  bl_hparams to_c() const {
    bl_hparams h{beta1, beta2, beta3, eta, c_min, c_max, r_min, r_max, r_threshold,
                 weight_decay, division_floor, total_steps, warmup_steps,
                 scaled_error_feedback ? 1 : 0};
    return h;
  }
};

struct StepTrace {  // optimizers.hpp:81-87
  std::vector<double> c, r, v_norm, v_ratio_preclip;
  bool compressed = false;
};

class SimCluster {
 public:
  struct Config {  // comm_sim.hpp:72-80 + placement
    int n_workers = 1;
    std::size_t dim = 0;
    CompressorKind compressor = CompressorKind::kOneBit;
    int baseline_bits_per_element = 16;
    bool endpoint_stats = false;
    bool verify_compensation = false;       // comm_sim.hpp:78
    double compensation_tolerance = 1e-12;  // fp32 state needs >= 2^-23
    int device = 0;
    void* stream = nullptr;
    bl_transport transport = BL_TRANSPORT_AUTO;  // NCCL mode: fused NVLink or NCCL
  };

  // n_workers simulated ranks in one GPU's HBM (the reference's SimCluster).
  explicit SimCluster(const Config& cfg) : n_(cfg.n_workers), dim_(cfg.dim) {
    bl_cluster_config c = base(cfg);
    c.mode = BL_MODE_SIM;
    check(bl_cluster_create(&c, &h_));
    fill_dims();
  }
  // This process is `rank` of n_workers over NCCL (one process per GPU).
  SimCluster(const Config& cfg, int rank, const std::array<std::uint8_t, BL_NCCL_UNIQUE_ID_BYTES>& id)
      : n_(cfg.n_workers), dim_(cfg.dim), rank_(rank), local_(1) {
    bl_cluster_config c = base(cfg);
    c.mode = BL_MODE_NCCL;
    c.rank = rank;
    c.nccl_unique_id = id.data();
    check(bl_cluster_create(&c, &h_));
    fill_dims();
  }
  ~SimCluster() { bl_cluster_destroy(h_); }
  SimCluster(const SimCluster&) = delete;
  SimCluster& operator=(const SimCluster&) = delete;

  static std::array<std::uint8_t, BL_NCCL_UNIQUE_ID_BYTES> nccl_unique_id() {
    std::array<std::uint8_t, BL_NCCL_UNIQUE_ID_BYTES> id{};
    check(bl_nccl_get_unique_id(id.data()));
    return id;
  }

  // comm_sim.hpp:98-99.  SIM: one input per worker; NCCL: the local input.
  std::vector<float> compressed_allreduce(std::span<const std::vector<float>> inputs,
                                          double error_scale = 1.0) {
    std::vector<const float*> p;
    std::size_t len = dim_;
    for (const auto& v : inputs) {
      if (v.size() != dim_) len = v.size();
      p.push_back(v.data());
    }
    std::vector<float> out(dim_);
    check(bl_cluster_compressed_allreduce(h_, p.data(), static_cast<int32_t>(p.size()), len,
                                          out.data(), error_scale, BL_MEM_HOST));
    return out;
  }

  // comm_sim.hpp:102
  std::vector<float> lossless_allreduce(std::span<const std::vector<float>> inputs) {
    std::vector<const float*> p;
    std::size_t len = dim_;
    for (const auto& v : inputs) {
      if (v.size() != dim_) len = v.size();
      p.push_back(v.data());
    }
    std::vector<float> out(dim_);
    check(bl_cluster_lossless_allreduce(h_, p.data(), static_cast<int32_t>(p.size()), len,
                                        out.data(), BL_MEM_HOST));
    return out;
  }

  VolumeLedger ledger() const {
    VolumeLedger l{};
    check(bl_cluster_ledger(h_, &l));
    return l;
  }
  std::vector<float> worker_error(int i) const {
    std::vector<float> out(padded_);
    check(bl_cluster_worker_error(h_, i, out.data()));
    return out;
  }
  std::vector<float> server_error(int j) const {
    std::vector<float> out(chunk_);
    check(bl_cluster_server_error(h_, j, out.data()));
    return out;
  }
  std::vector<EndpointStats> stats() const {
    std::vector<EndpointStats> s(2 * static_cast<std::size_t>(n_));
    check(bl_cluster_stats(h_, s.data()));
    return s;
  }
  // comm_sim.hpp:113-124: endpoint statistics (workers, then chunk servers)
  // and their maxima; needs Config::endpoint_stats.
  std::vector<EndpointStats> worker_stats() const {
    auto s = stats();
    return {s.begin(), s.begin() + n_};
  }
  std::vector<EndpointStats> server_stats() const {
    auto s = stats();
    return {s.begin() + n_, s.end()};
  }
  double delta_linf() const { return max_of(&EndpointStats::delta_linf); }
  double delta_l2_max() const { return max_of(&EndpointStats::delta_l2); }
  double run_max_delta_linf() const { return max_of(&EndpointStats::max_delta_linf); }
  double run_max_corrected_linf() const { return max_of(&EndpointStats::max_corrected_linf); }
  std::uint64_t compensation_checks() const { return bl_cluster_compensation_checks(h_); }

  // comm_sim.hpp:105,108
  bl_cluster_config config() const {
    bl_cluster_config c{};
    check(bl_cluster_get_config(h_, &c));
    return c;
  }
  std::size_t step_count() const { return bl_cluster_step_count(h_); }
  // Bound of every wait on a peer (multi-process); see bitlamb_b200.h.
  void set_peer_timeout_ms(double ms) { check(bl_cluster_set_peer_timeout(h_, ms)); }

  int n_workers() const { return n_; }
  std::size_t dim() const { return dim_; }
  std::size_t padded() const { return padded_; }
  std::size_t chunk_len() const { return chunk_; }
  int local_workers() const { return local_ == 0 ? n_ : local_; }
  bl_cluster* handle() const { return h_; }

 private:
  double max_of(double EndpointStats::*field) const {
    double m = 0.0;
    for (const auto& e : stats()) m = m < e.*field ? e.*field : m;
    return m;
  }
  static bl_cluster_config base(const Config& cfg) {
    bl_cluster_config c{};
    c.n_workers = cfg.n_workers;
    c.device = cfg.device;
    c.dim = cfg.dim;
    c.compressor = static_cast<int32_t>(cfg.compressor);
    c.baseline_bits_per_element = cfg.baseline_bits_per_element;
    c.endpoint_stats = cfg.endpoint_stats ? 1 : 0;
    c.verify_compensation = cfg.verify_compensation ? 1 : 0;
    c.compensation_tolerance = cfg.compensation_tolerance;
    c.stream = cfg.stream;
    c.transport = cfg.transport;
    return c;
  }
  void fill_dims() {
    std::uint64_t p = 0, c = 0;
    check(bl_cluster_dims(h_, &p, &c));
    padded_ = p;
    chunk_ = c;
  }
  bl_cluster* h_ = nullptr;
  int n_ = 1;
  std::size_t dim_ = 0, padded_ = 0, chunk_ = 0;
  int rank_ = 0, local_ = 0;
};

class Optimizer {
 public:
  struct LayerSpec {  // optimizers.hpp:95-98
    std::string name;
    std::size_t size = 0;
  };

  Optimizer(OptimizerVariant variant, std::span<const LayerSpec> layout, const HyperParams& hp,
            SimCluster& cluster)
      : cluster_(&cluster) {
    std::vector<bl_layer_spec> specs;
    for (const auto& s : layout) names_.push_back(s.name);
    for (std::size_t l = 0; l < layout.size(); ++l) specs.push_back({names_[l].c_str(), layout[l].size});
    const bl_hparams h = hp.to_c();
    check(bl_optimizer_create_named(static_cast<int32_t>(variant), specs.data(),
                                    static_cast<int32_t>(specs.size()), &h, cluster.handle(), &h_));
  }
  // Strict mode: check_gradients before any state changes (bitlamb_b200.h).
  void set_strict(bool on) { check(bl_optimizer_set_strict(h_, on ? 1 : 0)); }
  ~Optimizer() { bl_optimizer_destroy(h_); }
  Optimizer(const Optimizer&) = delete;
  Optimizer& operator=(const Optimizer&) = delete;

  // optimizers.hpp:106-107 with fused per-worker gradients (layer-major).
  StepTrace step(std::span<const std::vector<float>> local_grads, std::size_t t, double lr,
                 SimCluster& cluster) {
    std::vector<const float*> p;
    for (const auto& g : local_grads) {
      if (g.size() != fused_dim()) throw DimensionError("step: gradient length: size mismatch");
      p.push_back(g.data());
    }
    const std::size_t L = names_.size();
    StepTrace tr;
    tr.c.resize(L);
    tr.r.resize(L);
    tr.v_norm.resize(L);
    tr.v_ratio_preclip.resize(L);
    bl_step_trace ct{tr.c.data(), tr.r.data(), tr.v_norm.data(), tr.v_ratio_preclip.data(), 0};
    check(bl_optimizer_step(h_, cluster.handle(), p.data(), static_cast<int32_t>(p.size()), t, lr,
                            BL_MEM_HOST, &ct));
    tr.compressed = ct.compressed != 0;
    return tr;
  }

  std::vector<float> state(bl_state which) const {
    std::vector<float> out(fused_dim());
    check(bl_optimizer_get_state(h_, which, out.data()));
    return out;
  }
  void set_state(bl_state which, std::span<const float> v) {
    if (v.size() != fused_dim()) throw DimensionError("set_state: size mismatch");
    check(bl_optimizer_set_state(h_, which, v.data()));
  }
  bool frozen() const { return bl_optimizer_frozen(h_) != 0; }
  std::size_t fused_dim() const { return bl_optimizer_fused_dim(h_); }
  const std::vector<std::string>& layer_names() const { return names_; }

 private:
  SimCluster* cluster_;
  bl_optimizer* h_ = nullptr;
  std::vector<std::string> names_;
};

// ---- free functions (compression.hpp:106-118, fusion.hpp:92-102) -----------
struct CompressResult {
  std::vector<std::uint8_t> wire;  // serialize() bytes (one-bit)
  std::vector<float> decompressed;
};

// compress_with_feedback: delta is updated in place.
inline CompressResult compress_with_feedback(std::span<const float> v, std::span<float> delta,
                                             CompressorKind kind, double error_scale = 1.0,
                                             int device = 0) {
  if (v.size() != delta.size()) throw DimensionError("compress_with_feedback: size mismatch");
  CompressResult r;
  r.wire.resize((v.size() + 7) / 8 + 4);
  r.decompressed.resize(v.size());
  check(bl_compress_with_feedback(v.data(), delta.data(), v.size(), static_cast<int32_t>(kind), error_scale,
                                  r.wire.data(), r.decompressed.data(), BL_MEM_HOST, device));
  return r;
}

struct MomentumScales {  // fusion.hpp:80-89
  std::vector<double> coeff;
  double reference_scale = 1.0;
};

inline MomentumScales compute_scales(std::span<const float> fused_m, std::span<const std::uint64_t> sizes,
                                     double floor = 1e-12, int device = 0) {
  MomentumScales s;
  s.coeff.resize(sizes.size());
  check(bl_compute_scales(fused_m.data(), sizes.data(), static_cast<int32_t>(sizes.size()), floor,
                          s.coeff.data(), &s.reference_scale, BL_MEM_HOST, device));
  return s;
}
inline void apply_scaling(std::span<float> fused, std::span<const std::uint64_t> sizes,
                          const MomentumScales& s, int device = 0) {
  if (s.coeff.size() != sizes.size()) throw DimensionError("apply_scaling: size mismatch");
  check(bl_apply_scaling(fused.data(), sizes.data(), static_cast<int32_t>(sizes.size()), s.coeff.data(),
                         BL_MEM_HOST, device));
}
inline void remove_scaling(std::span<float> fused, std::span<const std::uint64_t> sizes,
                           const MomentumScales& s, int device = 0) {
  if (s.coeff.size() != sizes.size()) throw DimensionError("remove_scaling: size mismatch");
  check(bl_remove_scaling(fused.data(), sizes.data(), static_cast<int32_t>(sizes.size()), s.coeff.data(),
                          BL_MEM_HOST, device));
}

}  // namespace bitlamb_b200

#endif  // BITLAMB_B200_HPP_

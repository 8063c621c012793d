// facade_demo.cpp — C++ caller of the B200 path through the header-only
// facade (include/bitlamb_b200.hpp), shaped like the reference's own callers
// (SimCluster::compressed_allreduce, Optimizer::step).  Writes its inputs and
// outputs as raw little-endian float32 files for tests/test_gpu_facade.py,
// which replays them on the f32 oracle.
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "bitlamb_b200.hpp"

namespace {

// Deterministic inputs without libstdc++ distributions: xorshift64* -> [-1, 1).
struct Rng {
  std::uint64_t s;
  float next() {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    const std::uint64_t r = s * 2685821657736338717ull;
    return static_cast<float>(static_cast<double>(r >> 40) / static_cast<double>(1ull << 24)) * 2.0f - 1.0f;
  }
};

void dump(const std::string& path, const std::vector<float>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 4));
}

}  // namespace

int main(int argc, char** argv) {
  using namespace bitlamb_b200;
  const std::string dir = argc > 1 ? argv[1] : ".";
  try {
    // ---- compressed allreduce, 4 simulated workers ----
    const int n = 4;
    const std::size_t d = 10007;
    SimCluster::Config cfg;
    cfg.n_workers = n;
    cfg.dim = d;
    SimCluster cluster(cfg);
    Rng rng{42};
    for (int call = 0; call < 3; ++call) {
      std::vector<std::vector<float>> in(n, std::vector<float>(d));
      std::vector<float> flat;
      for (auto& v : in)
        for (auto& x : v) {
          x = rng.next();
          flat.push_back(x);
        }
      const std::vector<float> out = cluster.compressed_allreduce(in);
      dump(dir + "/ar_in" + std::to_string(call) + ".bin", flat);
      dump(dir + "/ar_out" + std::to_string(call) + ".bin", out);
    }
    try {  // DimensionError mirrors comm_sim.cpp:123-126
      std::vector<std::vector<float>> bad(n - 1, std::vector<float>(d));
      cluster.compressed_allreduce(bad);
      std::printf("no error\n");
    } catch (const DimensionError&) {
      std::printf("DimensionError ok\n");
    }

    // ---- 1-bit LAMB optimizer: warmup, freeze, compression stage ----
    const std::vector<Optimizer::LayerSpec> layout = {{"w", 3000}, {"b", 2}, {"ln", 1023}, {"out", 4099}};
    std::size_t dd = 0;
    for (const auto& l : layout) dd += l.size;
    SimCluster::Config c2;
    c2.n_workers = 2;
    c2.dim = dd;
    SimCluster cl2(c2);
    HyperParams hp;
    hp.total_steps = 12;
    hp.warmup_steps = 4;
    Optimizer opt(OptimizerVariant::kOneBitLamb, layout, hp, cl2);
    std::vector<float> x0(dd);
    for (auto& x : x0) x = rng.next() * 0.02f;
    opt.set_state(BL_STATE_X, x0);
    dump(dir + "/opt_x0.bin", x0);
    for (std::size_t t = 0; t < hp.total_steps; ++t) {
      std::vector<std::vector<float>> g(2, std::vector<float>(dd));
      std::vector<float> flat;
      for (auto& v : g)
        for (auto& x : v) {
          x = rng.next() * 1e-3f;
          flat.push_back(x);
        }
      const StepTrace tr = opt.step(g, t, 1e-3, cl2);
      dump(dir + "/opt_g" + std::to_string(t) + ".bin", flat);
      std::vector<float> c(tr.c.begin(), tr.c.end());
      dump(dir + "/opt_c" + std::to_string(t) + ".bin", c);
    }
    dump(dir + "/opt_x.bin", opt.state(BL_STATE_X));
    dump(dir + "/opt_v.bin", opt.state(BL_STATE_V));
    std::printf("frozen=%d\n", opt.frozen() ? 1 : 0);
    std::printf("facade ok\n");
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
  return 0;
}

// train_dist_b200.cpp — TEST INFRASTRUCTURE.
//
// The reference's training loop (trainer.cpp:135-327: its quadratic task,
// batch sharding and schedule, linked from oracle/_ref) on the B200 backend
// in two deployments:
//   * one process, n workers simulated in one GPU (bitlamb_b200 SIM mode);
//   * n processes under torchrun (`--no-python`), one GPU each, every rank
//     computing only its own shard's gradient and stepping the optimizer
//     over NCCL mode (fused NVLink exchange).
// Both write the per-step loss and per-layer c, r, ||v|| (%.17g) to a CSV;
// tests/test_gpu_multi.py requires the two files to be byte-identical.
//
//   train_dist_b200 <out.csv> <n_workers> <id_file>
// (under torchrun n_workers is WORLD_SIZE; rank 0 writes the NCCL unique id
// to <id_file> for the others and writes the CSV.)
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "bitlamb/config.hpp"
#include "bitlamb/tasks.hpp"
#include "bitlamb/trainer.hpp"
#include "bitlamb_b200.hpp"

namespace {

namespace ref = bitlamb;
namespace b2 = bitlamb_b200;

int env_int(const char* k, int dflt) {
  const char* v = std::getenv(k);
  return v ? std::atoi(v) : dflt;
}

std::string fmt17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// NCCL unique id: rank 0 creates it and publishes it through a file.
std::array<std::uint8_t, BL_NCCL_UNIQUE_ID_BYTES> share_id(int rank, const std::string& path) {
  std::array<std::uint8_t, BL_NCCL_UNIQUE_ID_BYTES> id{};
  if (rank == 0) {
    id = b2::SimCluster::nccl_unique_id();
    const std::string tmp = path + ".tmp";
    std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<const char*>(id.data()), id.size());
    std::filesystem::rename(tmp, path);
  } else {
    for (int i = 0; i < 6000 && !std::filesystem::exists(path); ++i)
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    std::ifstream(path, std::ios::binary).read(reinterpret_cast<char*>(id.data()), id.size());
  }
  return id;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s out.csv n_workers id_file\n", argv[0]);
    return 2;
  }
  const int world = env_int("WORLD_SIZE", 1), rank = env_int("RANK", 0);
  const bool dist = world > 1;
  const int n = dist ? world : std::atoi(argv[2]);

  // The acceptance protocol (acceptance.cpp:60-83), shortened.
  ref::RunConfig cfg;
  cfg.task = "quadratic";
  cfg.n_workers = n;
  cfg.batch_per_worker = 8;
  cfg.hyper.total_steps = 600;
  cfg.hyper.warmup_steps = 150;
  cfg.schedule.kind = ref::ScheduleKind::kExpStep;
  cfg.schedule.peak = 0.02;
  cfg.schedule.initial = 0.002;
  cfg.schedule.warmup_steps = 100;
  cfg.schedule.decay_factor = 0.85;
  cfg.schedule.decay_interval = 100;
  cfg.schedule.total_steps = cfg.hyper.total_steps;
  auto task = ref::make_task(cfg.task, cfg.seed, cfg.task_options);

  std::vector<b2::Optimizer::LayerSpec> specs;
  std::vector<std::size_t> sizes;
  std::size_t d = 0;
  for (const auto& s : task->layers()) {
    specs.push_back({s.name, s.size});
    sizes.push_back(s.size);
    d += s.size;
  }
  b2::SimCluster::Config cc;
  cc.n_workers = n;
  cc.dim = d;
  cc.device = dist ? env_int("LOCAL_RANK", 0) : 0;
  b2::HyperParams hp;
  hp.total_steps = cfg.hyper.total_steps;
  hp.warmup_steps = cfg.hyper.warmup_steps;
  std::unique_ptr<b2::SimCluster> cluster =
      dist ? std::make_unique<b2::SimCluster>(cc, rank, share_id(rank, argv[3]))
           : std::make_unique<b2::SimCluster>(cc);
  b2::Optimizer opt(b2::OptimizerVariant::kOneBitLamb, specs, hp, *cluster);
  {
    std::vector<float> x0;
    for (const auto& layer : task->initial_params(cfg.seed)) x0.insert(x0.end(), layer.begin(), layer.end());
    opt.set_state(BL_STATE_X, x0);
  }

  std::ostringstream csv;
  csv << "step,loss";
  for (const auto& s : task->layers()) csv << ",c." << s.name << ",r." << s.name << ",v." << s.name;
  csv << "\n";
  std::vector<std::vector<double>> xh(sizes.size()), gl(sizes.size());
  ref::ParamsView view;
  auto read_x = [&] {
    const std::vector<float> x = opt.state(BL_STATE_X);
    view.clear();
    std::size_t o = 0;
    for (std::size_t l = 0; l < sizes.size(); ++l) {
      xh[l].assign(x.begin() + static_cast<std::ptrdiff_t>(o), x.begin() + static_cast<std::ptrdiff_t>(o + sizes[l]));
      view.push_back(std::span<const double>(xh[l]));
      o += sizes[l];
    }
  };
  read_x();
  const int first = dist ? rank : 0, count = dist ? 1 : n;  // workers this process computes
  std::vector<std::vector<float>> g(static_cast<std::size_t>(count), std::vector<float>(d));
  for (std::size_t t = 0; t < cfg.hyper.total_steps; ++t) {
    task->at_step(t);
    const auto shards = ref::shard_batch(task->dataset_size(), t, n, cfg.batch_per_worker);
    for (int i = 0; i < count; ++i) {
      ref::GradSink sink;
      for (std::size_t l = 0; l < sizes.size(); ++l) {
        gl[l].assign(sizes[l], 0.0);
        sink.push_back(std::span<double>(gl[l]));
      }
      task->gradient(view, shards[static_cast<std::size_t>(first + i)], sink);
      std::size_t o = 0;
      for (const auto& v : gl)
        for (double e : v) g[static_cast<std::size_t>(i)][o++] = static_cast<float>(e);
    }
    const b2::StepTrace tr = opt.step(g, t, cfg.schedule.at(t), *cluster);
    read_x();
    csv << t << ',' << fmt17(task->full_loss(view));
    for (std::size_t l = 0; l < sizes.size(); ++l)
      csv << ',' << fmt17(tr.c[l]) << ',' << fmt17(tr.r[l]) << ',' << fmt17(tr.v_norm[l]);
    csv << "\n";
  }
  if (rank == 0) std::ofstream(argv[1]) << csv.str();
  std::printf("rank %d done: %zu steps, n=%d, %s\n", rank, cfg.hyper.total_steps, n,
              dist ? "NCCL mode" : "SIM mode");
  return 0;
}

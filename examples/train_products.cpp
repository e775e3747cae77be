// Drop-in usage of the reference's C++ training API on B200 (mggcn/rowgcn.hpp over libmggcn.so):
// the same calls a rowgcn user makes (synth_graph, GcnConfig, train_run, TrainOptions::on_epoch).
//   g++ -std=c++17 -O2 -I include examples/train_products.cpp -L paper_2110_08688_b200 -lmggcn
//       -Wl,-rpath,$PWD/paper_2110_08688_b200 -o train_products
//   ./train_products [n] [epochs] [workers]
#include <cstdio>
#include <cstdlib>

#include "mggcn/rowgcn.hpp"

namespace R = mggcn::rowgcn;

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 20000;
  const int epochs = argc > 2 ? std::atoi(argv[2]) : 5;
  const int workers = argc > 3 ? std::atoi(argv[3]) : 1;
  try {
    const R::Dataset<float> ds = R::synth_graph<float>(n, 50.6, 0.7, 1, 100, 47);
    R::GcnConfig cfg;
    cfg.layer_dims = {100, 256, 256, 47};
    cfg.epochs = epochs;
    cfg.permute = true;
    cfg.overlap = workers > 1;
    R::TrainOptions opts;
    opts.workers = workers;
    opts.on_epoch = [](int e, double loss, double acc, double wall_us) {
      std::printf("{\"epoch\": %d, \"loss\": %.7f, \"acc\": %.5f, \"wall_us\": %.1f}\n", e, loss, acc, wall_us);
    };
    const auto art = R::train_run(ds, cfg, opts);
    std::printf("final loss %.7f over %zu epochs, %zu W matrices\n", art.final_loss(), art.epoch_loss.size(),
                art.final_w.size());
    R::audit_timeline(art.timeline);  // the CUDA-event timeline obeys the reference's audit rules
    R::export_timeline("/tmp/mggcn_products.timeline.json", art.timeline);
    std::printf("timeline: %zu events\n", art.timeline.size());
    R::write_checkpoint("/tmp/mggcn_products.ckpt", art.final_w, cfg);
    const auto back = R::read_checkpoint<float>("/tmp/mggcn_products.ckpt");
    return back.size() == art.final_w.size() ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}

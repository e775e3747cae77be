// Loads a dataset from disk through the C++ drop-in (mggcn::rowgcn::load_dataset, the reference's
// rowgcn::load_dataset, inc/dataset.hpp:264-276) and prints its shape. Host-only: no GPU needed.
//   load_dataset <graph (.mtx | edge list)> <features (MGDM | CSV)> <labels> [masks.json]
#include <cstdio>

#include "mggcn/rowgcn.hpp"

namespace R = mggcn::rowgcn;

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s graph features labels [masks]\n", argv[0]);
    return 2;
  }
  try {
    const R::Dataset<float> ds = R::load_dataset<float>(argv[1], argv[2], argv[3], argc > 4 ? argv[4] : "");
    long train = 0;
    for (auto m : ds.train_mask) train += m;
    double fsum = 0;
    for (R::index_t i = 0; i < ds.features.size(); ++i) fsum += ds.features.data()[i];
    std::printf("n=%lld nnz=%lld d0=%lld classes=%d train=%ld val=%zu test=%zu fsum=%.6f\n",
                static_cast<long long>(ds.n()), static_cast<long long>(ds.graph.nnz()),
                static_cast<long long>(ds.features.cols()), ds.num_classes(), train, ds.val_mask.size(),
                ds.test_mask.size(), fsum);
  } catch (const R::ParseError& e) {
    std::printf("ParseError: %s\n", e.what());
    return 1;
  } catch (const R::ShapeError& e) {
    std::printf("ShapeError: %s\n", e.what());
    return 1;
  }
  return 0;
}

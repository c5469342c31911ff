// kern_btile.cu -- instantiation and launch of btile_kernel (btile.cuh) with
// the default warp roles: the four same-kind pairs (mixed pairs run on the
// other staged tiles), update modes 0-3 (3: beta != 0 with B read directly,
// not through the ring), 1-16 column elements per consumer lane or the linear
// walk (0).  Tiles of 32 KB and more run with twice the warps
// (kern_btile_big.cu), selected by the launch's block size.
#include <map>
#include <mutex>
#include <utility>

#include "btile_dispatch.cuh"

namespace ttb {

unsigned int* btile_counter(cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, unsigned int*> counters;  // kept for the process
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = counters.find({dev, s});
  if (it != counters.end()) return it->second;
  void* p = nullptr;
  if (cudaMalloc(&p, 2 * sizeof(unsigned int)) != cudaSuccess ||
      cudaMemset(p, 0, 2 * sizeof(unsigned int)) != cudaSuccess) {
    cudaGetLastError();
    if (p) cudaFree(p);
    return nullptr;
  }
  counters[{dev, s}] = static_cast<unsigned int*>(p);
  return static_cast<unsigned int*>(p);
}

using BtileSmall = BtileCfg<kBtileConsumerWarps, kBtileProducerWarps, 0, 1, 2, 4, 8, 16>;

cudaError_t launch_btile(int ka, int kb, int mode, const SmemParams& p, const Launch& l,
                         cudaStream_t s) {
  if (l.block == 32 * (kBtileBigConsumerWarps + kBtileBigProducerWarps))
    return launch_btile_big(ka, kb, mode, p, l, s);
  return BtileSmall::launch(ka, kb, mode, p, l, s);
}

int occupancy_btile(int ka, int kb, int mode, int jy, int block, int smem) {
  if (block == 32 * (kBtileBigConsumerWarps + kBtileBigProducerWarps))
    return occupancy_btile_big(ka, kb, mode, jy, block, smem);
  return BtileSmall::occupancy(ka, kb, mode, jy, block, smem);
}

}  // namespace ttb

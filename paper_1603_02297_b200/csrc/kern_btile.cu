// kern_btile.cu -- instantiation and launch of btile_kernel (btile.cuh) with
// the default warp roles: the eight kind pairs, update modes 0-3 (3: beta != 0 with B read directly,
// not through the ring), 1-16 column elements per consumer lane or the linear
// walk (0).  Tiles of 32 KB and more run with twice the warps
// (kern_btile_big.cu), selected by the launch's block size.
#include <atomic>
#include <mutex>

#include "btile_dispatch.cuh"

namespace ttb {

// Tile counters [next, done] for btile launches: a ring of slots per device,
// each launch takes the next slot (a host-side atomic), so launches that run
// at the same time -- other streams, other host threads on one stream handle
// -- never share one; the kernel leaves its slot zeroed.  A graph launch
// keeps the slot it was captured with (a graph exec never runs concurrently
// with itself).  The ring is allocated by btile_counters_init() when a plan
// is prepared (not during a stream capture); a launch that finds none falls
// back to the static tile order.
constexpr int kCounterSlots = 4096;
constexpr int kMaxDevices = 64;
std::atomic<unsigned int*> g_ring[kMaxDevices];
std::atomic<uint32_t> g_next{0};

void btile_counters_init() {
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return;
  }
  if (g_ring[dev].load()) return;
  std::lock_guard<std::mutex> lk(mu);
  if (g_ring[dev].load()) return;
  void* p = nullptr;
  if (cudaMalloc(&p, 2 * sizeof(unsigned int) * kCounterSlots) != cudaSuccess ||
      cudaMemset(p, 0, 2 * sizeof(unsigned int) * kCounterSlots) != cudaSuccess) {
    cudaGetLastError();
    if (p) cudaFree(p);
    return;
  }
  g_ring[dev].store(static_cast<unsigned int*>(p));
}

unsigned int* btile_counter(cudaStream_t) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return nullptr;
  }
  unsigned int* ring = g_ring[dev].load();
  if (!ring) return nullptr;
  const uint32_t slot = g_next.fetch_add(1) % kCounterSlots;
  return ring + 2 * slot;
}

using BtileSmall = BtileCfg<kBtileConsumerWarps, kBtileProducerWarps, 0, 1, 2, 4, 8, 16>;

cudaError_t launch_btile(int ka, int kb, int mode, const SmemParams& p, const BtileTma& bt, const Launch& l,
                         cudaStream_t s) {
  if (l.block == 32 * (kBtileBigConsumerWarps + kBtileBigProducerWarps))
    return launch_btile_big(ka, kb, mode, p, bt, l, s);
  return BtileSmall::launch(ka, kb, mode, p, bt, l, s);
}

int occupancy_btile(int ka, int kb, int mode, int jy, int block, int smem) {
  if (block == 32 * (kBtileBigConsumerWarps + kBtileBigProducerWarps))
    return occupancy_btile_big(ka, kb, mode, jy, block, smem);
  return BtileSmall::occupancy(ka, kb, mode, jy, block, smem);
}

}  // namespace ttb

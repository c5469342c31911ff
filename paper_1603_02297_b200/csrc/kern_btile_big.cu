// kern_btile_big.cu -- btile_kernel for tiles of 32 KB and more (e.g. 128 x 128
// fp32, 512-byte runs on both sides): one CTA per SM, so twice the consumer
// and producer warps of the default roles.  Column walk with 2, 4 or 8
// elements per lane.
#include "btile_dispatch.cuh"

namespace ttb {

using BtileBig = BtileCfg<kBtileBigConsumerWarps, kBtileBigProducerWarps, 2, 4, 8>;

cudaError_t launch_btile_big(int ka, int kb, int mode, const SmemParams& p, const BtileTma& bt, const Launch& l,
                             cudaStream_t s) {
  return BtileBig::launch(ka, kb, mode, p, bt, l, s);
}

int occupancy_btile_big(int ka, int kb, int mode, int jy, int block, int smem) {
  return BtileBig::occupancy(ka, kb, mode, jy, block, smem);
}

}  // namespace ttb

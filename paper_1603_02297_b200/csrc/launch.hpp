// launch.hpp -- host entry points into the templated kernels (kern_*.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "params.hpp"

namespace ttb {

// dynamic shared memory above this opts in (cudaFuncAttributeMaxDynamicSharedMemorySize):
// below 48 KB, with room for the kernels' static barriers and tables
constexpr int kSmemOptIn = 40 * 1024;

// mode: 0 move (alpha == 1, beta == 0), 1 scale (beta == 0), 2 update (beta != 0)
cudaError_t launch_copy(int ka, int kb, int v, int mode, const CopyParams& p, const Launch& l,
                        cudaStream_t s);
cudaError_t launch_rt(int ka, int kb, int mx, int my, int mode, const RtParams& p,
                      const Launch& l, cudaStream_t s);
cudaError_t launch_smem(int ka, int kb, int mode, const SmemParams& p, const Launch& l,
                        cudaStream_t s);

// resident CTAs per SM for a variant (cudaOccupancyMaxActiveBlocksPerMultiprocessor)
int occupancy_copy(int ka, int kb, int v, int mode, bool long_rows, int block);
int occupancy_rt(int ka, int kb, int mx, int my, int mode, int block);
int occupancy_smem(int ka, int kb, int mode, int dense, int ept, int block, int smem);
// vtile_kernel (SmemParams::dense == 4), kern_vtile.cu
cudaError_t launch_vtile(int ka, int kb, int mode, const SmemParams& p, const Launch& l,
                         cudaStream_t s);
int occupancy_vtile(int ka, int kb, int mode, int va, int vb, int sh, int block, int smem);
int smem_carveout();
// btile_kernel (SmemParams::dense == 5, bulk-copy ring), kern_btile.cu
cudaError_t launch_btile(int ka, int kb, int mode, const SmemParams& p, const BtileTma& bt, const Launch& l,
                         cudaStream_t s);
int occupancy_btile(int ka, int kb, int mode, int jy, int block, int smem);
cudaError_t launch_btile_big(int ka, int kb, int mode, const SmemParams& p, const BtileTma& bt, const Launch& l,
                             cudaStream_t s);
int occupancy_btile_big(int ka, int kb, int mode, int jy, int block, int smem);
// btile_kernel's tile counter [next, done] for one launch: the next slot of a
// per-device ring (kern_btile.cu), or null before btile_counters_init() ran
// on this device (static tile order)
unsigned int* btile_counter(cudaStream_t s);
void btile_counters_init();

// tma_kernel (Variant kTma, tensor maps encoded per launch from A and B), kern_tma.cu
cudaError_t launch_tma(int ka, int kb, int mode, const TmaPlan& p, const void* A, void* B, const Launch& l,
                       cudaStream_t s);
int occupancy_tma(int ka, int kb, int mode, bool runs, int block, int smem);
bool tma_available();
// encode one side's tensor map over `base` (kern_tma.cu)
cudaError_t tma_encode(CUtensorMap* m, const TmaView& v, const void* base);

// rowcopy_kernel (CopyParams::bulk), kern_rows.cu
cudaError_t launch_rowcopy(int ka, int kb, int mode, const CopyParams& p, const Launch& l, cudaStream_t s);
int occupancy_rowcopy(int ka, int kb, int mode, int block, int smem);

// data utilities (util.cu)
struct BoxParams {
  int rank = 0;
  int C = 1;
  int64_t ext[16];
  int64_t st[16];    // memory strides (elements)
  int64_t gst[16];   // global logical strides
  int64_t gbase = 0; // global logical index of the box origin
  int64_t total = 1;
};
cudaError_t launch_fill_uniform(bool dbl, const BoxParams& p, uint64_t seed, void* buf,
                                cudaStream_t s);
cudaError_t launch_fill_sentinel(bool dbl, int64_t scalars, void* buf, cudaStream_t s);
cudaError_t launch_checksum(bool dbl, const BoxParams& p, const void* buf,
                            unsigned long long* dev_out, cudaStream_t s);

// number of kernels launched by this library (ttb_launch_count)
void count_launch();

}  // namespace ttb

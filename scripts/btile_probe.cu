// btile_probe.cu -- kernel-design probe for btile_kernel (not product code):
// a 2D fp32 transpose N x N through btile_kernel with experiment switches
// (EXP bit 0: no stores, bit 1: no bulk copies), stage counts and tiles.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1603_02297_b200/csrc \
//        scripts/btile_probe.cu -o scripts/_bin/btile_probe
#include <cstdio>
#include <vector>

#include "btile.cuh"

using namespace ttb;

static Space space1(uint32_t n, int64_t sa, int64_t sb) {
  Space s;
  s.nd = 1;
  s.total = n;
  s.ext[0] = Div32::make(n);
  s.sa[0] = sa;
  s.sb[0] = sb;
  return s;
}

template <int JY, int EXP, int PW = 4, int NC = 8, int MODE = 0>
float run(const float* A, float* B, uint32_t N, uint32_t tx, uint32_t ty, uint32_t ns, int ctas,
          int order = 0, uint32_t ly = 32) {
  SmemParams P{};
  P.A = A;
  P.B = B;
  P.sc = Scale{1.0, MODE >= 2 ? 0.5 : 0.0};
  P.X = space1(N, 1, N);  // A axis 0: stride 1 in A, stride N in B
  P.Y = space1(N, N, 1);
  P.O = Space{};
  P.O.nd = 0;
  P.O.total = 1;
  P.S = 1;
  P.tx = tx;
  P.ty = ty;
  P.nxc = (N + tx - 1) / tx;
  P.nyc = (N + ty - 1) / ty;
  P.dnx = Div32::make(P.nxc);
  P.dny = Div32::make(P.nyc);
  P.order = order;
  P.grp = order >= 2 ? order : 1;
  P.dplane = Div32::make(P.nxc * P.nyc);
  P.dgrp = Div32::make(P.grp * P.nxc);
  P.dG = Div32::make(P.grp);
  P.items = P.nxc * P.nyc;
  P.dense = 5;
  P.ly = ly;
  P.pa = ((tx * 4 + 12 + 15) & ~15u);
  if ((P.pa / 16) % 2 == 0) P.pa += 16;
  P.pb = ((ty * 4 + 12 + 15) & ~15u);
  P.ns = ns;
  const int smem = ns * btile_stage_bytes(tx, ty, P.pa, P.pb, MODE == 2);
  auto fn = &btile_kernel<float, float, 1, MODE, JY, PW, NC, EXP>;
  const int block = 32 * (NC + PW);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem);
  const int grid = 148 * (ctas > 0 ? ctas : occ);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    cudaEventRecord(e0);
    fn<<<grid, block, smem>>>(P);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it && ms < best) best = ms;
  }
  const double gbs = (MODE >= 2 ? 3.0 : 2.0) * 4.0 * N * N / (best * 1e6);
  printf("ly=%u mode=%d order=%d N=%u nc=%d pw=%d tile %ux%u ns=%u occ=%d grid=%d exp=%d: %.1f us %.1f GB/s  (%s)\n", ly, MODE, order, N, NC, PW, tx, ty, ns,
         occ, grid, EXP, best * 1e3, gbs, cudaGetErrorString(cudaGetLastError()));
  return best;
}

int main() {
  const uint32_t N = 14527;  // odd: every tile row / column misaligned
  float *A, *B;
  cudaMalloc(&A, sizeof(float) * N * N);
  cudaMalloc(&B, sizeof(float) * N * N);
  cudaMemset(A, 0, sizeof(float) * N * N);
  run<2, 0, 4, 4, 2>(A, B, N, 64, 64, 2, 0, 0, 32);
  run<8, 0, 4, 4, 2>(A, B, N, 64, 64, 2, 0, 0, 8);
  run<4, 0, 4, 4, 2>(A, B, N, 64, 64, 2, 0, 0, 16);
  run<2, 0, 4, 4, 0>(A, B, N, 64, 64, 2, 0, 1, 32);
  run<8, 0, 4, 4, 0>(A, B, N, 64, 64, 2, 0, 1, 8);
  run<4, 0, 4, 4, 0>(A, B, N, 64, 64, 2, 0, 1, 16);
  run<4, 0, 4, 8, 0>(A, B, N, 128, 128, 2, 0, 0, 32);
  run<16, 0, 4, 8, 0>(A, B, N, 128, 128, 2, 0, 0, 8);
  run<8, 0, 4, 8, 0>(A, B, N, 128, 128, 2, 0, 0, 16);
  return 0;
}

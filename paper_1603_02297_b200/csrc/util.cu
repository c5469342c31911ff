// util.cu -- device data utilities: seeded generator, sentinel fill, checksum.
// These define the bench's synthetic inputs and the multi-GPU verification
// checksum; they are not on the transposition hot path.
#include <atomic>

#include "launch.hpp"

namespace ttb {

namespace {

std::atomic<unsigned long long> g_launches{0};

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// logical index i of the box -> memory offset and global column-major index
__device__ __forceinline__ void box_decode(const BoxParams& p, int64_t i, int64_t& off,
                                           int64_t& g) {
  off = 0;
  g = p.gbase;
  for (int d = 0; d < p.rank; ++d) {
    const int64_t q = i / p.ext[d];
    const int64_t r = i - q * p.ext[d];
    off += r * p.st[d];
    g += r * p.gst[d];
    i = q;
  }
}

template <bool DBL>
__global__ void __launch_bounds__(256) fill_kernel(const BoxParams p, uint64_t key, void* buf) {
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < p.total;
       i += nth) {
    int64_t off, g;
    box_decode(p, i, off, g);
    for (int q = 0; q < p.C; ++q) {
      const uint64_t u = splitmix64(key + static_cast<uint64_t>(g * p.C + q));
      if constexpr (DBL)
        static_cast<double*>(buf)[off * p.C + q] =
            static_cast<double>(u >> 11) * 0x1.0p-53 * 2.0 - 1.0;
      else
        static_cast<float*>(buf)[off * p.C + q] =
            static_cast<float>(u >> 40) * 0x1.0p-24f * 2.0f - 1.0f;
    }
  }
}

template <bool DBL>
__global__ void __launch_bounds__(256) sentinel_kernel(int64_t n, void* buf) {
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += nth) {
    if constexpr (DBL)
      static_cast<unsigned long long*>(buf)[i] = 0x7FF8DEADBEEF0001ull;
    else
      static_cast<unsigned int*>(buf)[i] = 0x7FC0FFEEu;
  }
}

template <bool DBL>
__global__ void __launch_bounds__(256) checksum_kernel(const BoxParams p, const void* buf,
                                                       unsigned long long* out) {
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned long long acc = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < p.total;
       i += nth) {
    int64_t off, g;
    box_decode(p, i, off, g);
    for (int q = 0; q < p.C; ++q) {
      uint64_t bits;
      if constexpr (DBL)
        bits = static_cast<const unsigned long long*>(buf)[off * p.C + q];
      else
        bits = static_cast<const unsigned int*>(buf)[off * p.C + q];
      const uint64_t j = static_cast<uint64_t>(g * p.C + q);
      acc += splitmix64((j * 0xD1B54A32D192ED03ull) ^ bits);
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

unsigned long long launch_total() { return g_launches.load(); }

cudaError_t launch_fill_uniform(bool dbl, const BoxParams& p, uint64_t seed, void* buf,
                                cudaStream_t s) {
  const uint64_t key = seed * 0x9E3779B97F4A7C15ull;
  if (dbl)
    fill_kernel<true><<<grid_for(p.total), 256, 0, s>>>(p, key, buf);
  else
    fill_kernel<false><<<grid_for(p.total), 256, 0, s>>>(p, key, buf);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_fill_sentinel(bool dbl, int64_t scalars, void* buf, cudaStream_t s) {
  if (dbl)
    sentinel_kernel<true><<<grid_for(scalars), 256, 0, s>>>(scalars, buf);
  else
    sentinel_kernel<false><<<grid_for(scalars), 256, 0, s>>>(scalars, buf);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_checksum(bool dbl, const BoxParams& p, const void* buf,
                            unsigned long long* dev_out, cudaStream_t s) {
  if (dbl)
    checksum_kernel<true><<<grid_for(p.total), 256, 0, s>>>(p, buf, dev_out);
  else
    checksum_kernel<false><<<grid_for(p.total), 256, 0, s>>>(p, buf, dev_out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ttb

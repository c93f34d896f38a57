// Shared-memory LDS.128 conflict model on B200: SM cycles per warp-wide
// 16-byte load for controlled address patterns (one CTA of 512 threads per
// SM, 128 KiB of shared memory, addresses from a per-thread list).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds lds_conflicts.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

constexpr int NT = 512, NA = 64, ITERS = 256;

__global__ void __launch_bounds__(NT, 1) lds_kernel(const uint32_t* __restrict__ addrs, unsigned long long* cycles, uint4* sink) {
  extern __shared__ __align__(16) uint8_t smem[];
  for (int i = threadIdx.x; i < 128 * 1024 / 16; i += NT)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(i, i * 3, i * 5, i * 7);
  uint32_t a[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) a[i] = addrs[(blockIdx.x * NT + threadIdx.x) * NA + i];
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(smem);
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      uint4 v;
      const uint32_t ad = smem_base + (a[i] ^ ((it & 1) << 7));  // row flip keeps the bank group
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ad));
      acc.x ^= v.x; acc.y += v.y; acc.z ^= v.z; acc.w += v.w;
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc.x == 0x12345678u) sink[threadIdx.x] = acc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nthr = nsm * NT;
  std::vector<uint32_t> h((size_t)nthr * NA);
  uint32_t* d; unsigned long long* dc; uint4* sink;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&dc, nsm * 8); cudaMalloc(&sink, NT * 16);
  cudaFuncSetAttribute(lds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  std::mt19937 rng(1);
  auto rnd = [&](uint32_t n) { return (uint32_t)(rng() % n); };
  const char* names[] = {
    "P0 linear (lane*16)", "P1 uniform random 16B slots in 128KiB",
    "P2 4-table interleave, rotation (g+lane)%4, random entry (current row-block)",
    "P3 quarter-warp conflict-free, all quarters same bank groups",
    "P4 lanes l,l+4 same bank group (2-way in every quarter)",
    "P5 each quarter: 8 lanes one bank group (8-way), warp balanced",
    "P6 broadcast: all lanes same address",
    "P7 half-warp conflict-free (16 lanes, 8 bank groups x2 rows?)",
    "P8 lanes l,l+8 same bank group, quarter-free",
    "P9 8-table interleave (16B), lane l -> table l%8, random entry",
  };
  for (int p = 0; p < 10; ++p) {
    for (int t = 0; t < nthr; ++t) {
      int lane = t & 31;
      for (int i = 0; i < NA; ++i) {
        uint32_t a = 0;
        uint32_t row = rnd(1024);            // 128-byte row
        switch (p) {
          case 0: a = ((t & (NT - 1)) * 16 + i * 16 * 32) % (128 * 1024); break;
          case 1: a = rnd(8192) * 16; break;
          case 2: { uint32_t g = (i + lane) & 3, f = rnd(2048);
                    a = ((f >> 1) << 7) | ((f & 1) << 4) | (g << 5); } break;
          case 3: a = row * 128 + (lane & 7) * 16; break;
          case 4: a = row * 128 + (lane & 3) * 16 + 0; break;  // lanes l, l+4 same bg
          case 5: a = row * 128 + ((lane >> 3) & 7) * 16; break;
          case 6: a = (i * 16 * 33) % (128 * 1024); break;
          case 7: a = row * 128 + ((lane & 7)) * 16; break;
          case 8: a = row * 128 + ((lane & 7) ^ ((lane >> 3) & 1 ? 0 : 0)) * 16; break;
          case 9: { uint32_t g = lane & 7, f = rnd(1024); a = (f * 8 + g) * 16; } break;
        }
        h[(size_t)t * NA + i] = a;
      }
    }
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    lds_kernel<<<nsm, NT, 128 * 1024>>>(d, dc, sink);
    lds_kernel<<<nsm, NT, 128 * 1024>>>(d, dc, sink);
    std::vector<unsigned long long> c(nsm);
    cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
    double mean = 0; for (auto v : c) mean += v; mean /= nsm;
    double per = mean / ((double)ITERS * NA * (NT / 32));
    printf("%-80s  %.3f SM cycles per warp-LDS.128 (%.2fx the 4-wavefront ideal)\n", names[p], per, per / 4);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}

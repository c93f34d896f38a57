// How fast can one kernel stream a 8192 x 4096-byte matrix (cfg4's packed
// int4 weights, 33.5 MB) from HBM, as a function of the access pattern and
// the bytes in flight?  nvcc -O3 -arch=sm_100a stream_pattern.cu -o stream_pattern
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t fold(uint4 v) { return v.x ^ v.y ^ v.z ^ v.w; }

// flat: warp w of the grid reads 512 B per instruction, D instructions in flight, grid-stride
template <int D>
__global__ void flat(const uint8_t* p, size_t bytes, uint32_t* out) {
  const size_t nw = (size_t)gridDim.x * blockDim.x / 32, w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0;
  for (size_t o = w * 512 * D; o < bytes; o += nw * 512 * D) {
    uint4 v[D];
#pragma unroll
    for (int i = 0; i < D; ++i) v[i] = ldg(p + o + i * 512 + lane * 16);
#pragma unroll
    for (int i = 0; i < D; ++i) acc ^= fold(v[i]);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// rows16: a warp owns 16 rows x a k slice; lane (g, t) reads 16 B of rows g and g + 8 per chunk
// (64 B per row and chunk), D chunks in flight (rolling).  grid = (rows / 128, S), 8 warps per CTA.
template <int D, int TB>   // TB = bytes per thread and row per chunk (16 or 32)
__global__ void rows16(const uint8_t* p, int rb, int chunks_per_cta, uint32_t* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const size_t ra = (size_t)blockIdx.x * 128 + warp * 16 + g;
  const uint8_t* pa = p + ra * rb + t * TB;
  const uint8_t* pb = pa + (size_t)8 * rb;
  const int c0 = blockIdx.y * chunks_per_cta, c1 = c0 + chunks_per_cta;
  constexpr int NV = TB / 16;
  uint4 a[D][NV], b[D][NV];
#pragma unroll
  for (int u = 0; u < D; ++u)
#pragma unroll
    for (int v = 0; v < NV; ++v) { a[u][v] = ldg(pa + (size_t)(c0 + u) * 4 * TB + 16 * v); b[u][v] = ldg(pb + (size_t)(c0 + u) * 4 * TB + 16 * v); }
  uint32_t acc = 0;
  for (int c = c0; c < c1; c += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
#pragma unroll
      for (int v = 0; v < NV; ++v) acc ^= fold(a[u][v]) ^ fold(b[u][v]);
      const int cn = min(c + u + D, c1 - 1);
#pragma unroll
      for (int v = 0; v < NV; ++v) { a[u][v] = ldg(pa + (size_t)cn * 4 * TB + 16 * v); b[u][v] = ldg(pb + (size_t)cn * 4 * TB + 16 * v); }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// rowwarp: a warp owns ONE row slice at a time (512 B per instruction), D in flight; rows strided over warps
template <int D>
__global__ void rowwarp(const uint8_t* p, int rows, int rb, uint32_t* out) {
  const int nw = gridDim.x * blockDim.x / 32, w = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  uint32_t acc = 0;
  for (int r = w; r < rows; r += nw) {
    const uint8_t* q = p + (size_t)r * rb + lane * 16;
    for (int o = 0; o < rb; o += 512 * D) {
      uint4 v[D];
#pragma unroll
      for (int i = 0; i < D; ++i) v[i] = ldg(q + o + i * 512);
#pragma unroll
      for (int i = 0; i < D; ++i) acc ^= fold(v[i]);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const int rows = 8192, rb = 4096, NB = 12;
  const size_t bytes = (size_t)rows * rb;
  uint8_t* buf[NB];
  for (int i = 0; i < NB; ++i) { CK(cudaMalloc(&buf[i], bytes)); CK(cudaMemset(buf[i], i + 1, bytes)); }
  uint32_t* out; CK(cudaMalloc(&out, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    for (int i = 0; i < NB; ++i) launch(buf[i]);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) for (int i = 0; i < NB; ++i) launch(buf[i]);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / (reps * NB);
    printf("%-34s %7.2f us  %6.0f GB/s  (%s)\n", name, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("flat D=4 148x4 CTAs x256", [&](uint8_t* p) { flat<4><<<148 * 4, 256>>>(p, bytes, out); });
  timeit("flat D=8 148x4 CTAs x256", [&](uint8_t* p) { flat<8><<<148 * 4, 256>>>(p, bytes, out); });
  timeit("flat D=8 148x8 CTAs x256", [&](uint8_t* p) { flat<8><<<148 * 8, 256>>>(p, bytes, out); });
  timeit("flat D=16 148x2 CTAs x256", [&](uint8_t* p) { flat<16><<<148 * 2, 256>>>(p, bytes, out); });
  timeit("flat D=8 148x2 CTAs x512", [&](uint8_t* p) { flat<8><<<148 * 2, 512>>>(p, bytes, out); });
  timeit("flat D=4 one-shot (all in flight)", [&](uint8_t* p) { flat<4><<<(unsigned)(bytes / (256 / 32 * 512 * 4)), 256>>>(p, bytes, out); });
  timeit("flat D=8 one-shot", [&](uint8_t* p) { flat<8><<<(unsigned)(bytes / (256 / 32 * 512 * 8)), 256>>>(p, bytes, out); });
  timeit("rowwarp D=8 148x8 CTAs", [&](uint8_t* p) { rowwarp<8><<<148 * 8, 256>>>(p, rows, rb, out); });
  timeit("rowwarp D=8 1024 CTAs (1 row/warp)", [&](uint8_t* p) { rowwarp<8><<<1024, 256>>>(p, rows, rb, out); });
  timeit("rows16 16B D=4 S=4 (256 CTAs)", [&](uint8_t* p) { rows16<4, 16><<<dim3(64, 4), 256>>>(p, rb, 16, out); });
  timeit("rows16 16B D=4 S=8 (512 CTAs)", [&](uint8_t* p) { rows16<4, 16><<<dim3(64, 8), 256>>>(p, rb, 8, out); });
  timeit("rows16 16B D=8 S=4", [&](uint8_t* p) { rows16<8, 16><<<dim3(64, 4), 256>>>(p, rb, 16, out); });
  timeit("rows16 16B D=8 S=8", [&](uint8_t* p) { rows16<8, 16><<<dim3(64, 8), 256>>>(p, rb, 8, out); });
  timeit("rows16 16B D=16 S=4 (all)", [&](uint8_t* p) { rows16<16, 16><<<dim3(64, 4), 256>>>(p, rb, 16, out); });
  timeit("rows16 32B D=2 S=4", [&](uint8_t* p) { rows16<2, 32><<<dim3(64, 4), 256>>>(p, rb, 8, out); });
  timeit("rows16 32B D=4 S=4", [&](uint8_t* p) { rows16<4, 32><<<dim3(64, 4), 256>>>(p, rb, 8, out); });
  timeit("rows16 32B D=4 S=8", [&](uint8_t* p) { rows16<4, 32><<<dim3(64, 8), 256>>>(p, rb, 4, out); });
  timeit("rows16 32B D=8 S=4 (all)", [&](uint8_t* p) { rows16<8, 32><<<dim3(64, 4), 256>>>(p, rb, 8, out); });
  return 0;
}

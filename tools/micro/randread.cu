// DRAM efficiency of the search's access pattern: read ~1 GB as (a) random
// 512-B rows, (b) random 4-KB blocks of 8 consecutive rows, (c) sequentially;
// 240 CTAs x 256 threads like the search kernel, plus a full-GPU variant.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__global__ void rd(const float4* __restrict__ base, const int* __restrict__ idx, int nidx, int rows_per_unit,
                   float* sink) {
  float acc = 0.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int u = blockIdx.x * nw + warp; u < nidx; u += gridDim.x * nw) {
    const float4* row = base + (size_t)idx[u] * rows_per_unit * 32;
    float4 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = r < rows_per_unit ? __ldcg(row + r * 32 + lane) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < 8; ++r) acc += v[r].x + v[r].y + v[r].z + v[r].w;
  }
  if (acc == 12345.f) sink[0] = acc;
}
int main() {
  const size_t bytes = 4ull << 30;   // 4 GB table (like the lift array)
  float4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 0, bytes);
  float* sink; cudaMalloc(&sink, 4);
  const size_t nrows = bytes / 512;
  for (int rpu : {1, 8}) {
    const size_t units = (1ull << 30) / (512ull * rpu);   // read 1 GB
    std::vector<int> h(units);
    uint64_t s = 12345;
    for (auto& x : h) { s = s * 6364136223846793005ull + 1442695040888963407ull; x = (int)((s >> 33) % (nrows / rpu)); }
    int* d; cudaMalloc(&d, units * 4); cudaMemcpy(d, h.data(), units * 4, cudaMemcpyHostToDevice);
    for (int grid : {240, 148 * 8}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      rd<<<grid, 256>>>(buf, d, (int)units, rpu, sink);
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) rd<<<grid, 256>>>(buf, d, (int)units, rpu, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("random %4d-B units, grid %5d: %.2f TB/s\n", 512 * rpu, grid, 5.0 * (1 << 30) / (ms * 1e-3) / 1e12);
    }
    cudaFree(d);
  }
  // sequential
  {
    const size_t units = (1ull << 30) / 4096;
    std::vector<int> h(units);
    for (size_t i = 0; i < units; ++i) h[i] = (int)i;
    int* d; cudaMalloc(&d, units * 4); cudaMemcpy(d, h.data(), units * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    rd<<<148 * 8, 256>>>(buf, d, (int)units, 8, sink);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) rd<<<148 * 8, 256>>>(buf, d, (int)units, 8, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("sequential 4-KB units, full grid: %.2f TB/s\n", 5.0 * (1 << 30) / (ms * 1e-3) / 1e12);
  }
  return 0;
}

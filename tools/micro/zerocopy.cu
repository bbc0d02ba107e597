// Host-link ceilings for the KV-offload gather (BASELINE config 3): reading
// pinned, device-mapped host memory from kernels vs the copy engine.
//   (a) cudaMemcpyAsync H2D, 256 MB (the copy-engine peak the bench reports)
//   (b) kernel, 16-B loads, random 4-KB blocks (a page's K or V rows), 8 in
//       flight per thread, stores to HBM: what gather_pages does
//   (c) kernel, TMA 1-D bulk copies (cp.async.bulk) of the same 4-KB blocks
//       host -> shared memory, then bulk store shared -> HBM
// Each kernel variant on the full GPU (2 CTAs x 148 SMs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zerocopy zerocopy.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void ld16(const uint4* __restrict__ host, const int* __restrict__ blk, int nblk, uint4* dst) {
  // one 4-KB block = 256 x 16 B; items (block, chunk) strided over the grid, 8 in flight per thread
  const long long items = (long long)nblk * 256;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long x0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; x0 < items; x0 += stride * 8) {
    uint4 v[8];
    long long d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long x = x0 + u * stride;
      d[u] = -1;
      if (x < items) {
        const int b = (int)(x >> 8), c = (int)(x & 255);
        v[u] = host[(size_t)blk[b] * 256 + c];
        d[u] = x;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (d[u] >= 0) dst[d[u]] = v[u];
  }
}

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void tma_bulk(const char* host, const int* __restrict__ blk, int nblk, char* dst) {
  // each warp: 4 stages of 4 KB; lane 0 issues host -> smem bulk copies, then
  // smem -> HBM bulk stores once a stage lands
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar[8][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  char* my = sm + (size_t)warp * 4 * 4096;
  if (lane == 0)
    for (int s = 0; s < 4; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[warp][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * nw + warp, ngw = gridDim.x * nw;
  int it = 0;
  for (int b0 = gw; b0 < nblk; b0 += ngw * 4, ++it) {
    if (lane == 0) {
      for (int s = 0; s < 4; ++s) {
        const int b = b0 + s * ngw;
        if (b >= nblk) break;
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // stage free (previous store read it)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(su32(&bar[warp][s])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                         su32(my + s * 4096)),
                     "l"(host + (size_t)blk[b] * 4096), "r"(su32(&bar[warp][s]))
                     : "memory");
      }
      for (int s = 0; s < 4; ++s) {
        const int b = b0 + s * ngw;
        if (b >= nblk) break;
        asm volatile(
            "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
                su32(&bar[warp][s])),
            "r"(it & 1)
            : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(dst + (size_t)b * 4096),
                     "r"(su32(my + s * 4096))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t hbytes = 2ull << 30;   // 2 GB pinned host store
  const int nblk = (256 << 20) / 4096;   // gather 256 MB per launch
  char* h;
  cudaHostAlloc(&h, hbytes, cudaHostAllocMapped | cudaHostAllocPortable);
  for (size_t i = 0; i < hbytes; i += 4096) h[i] = (char)i;
  char* hd;
  cudaHostGetDevicePointer((void**)&hd, h, 0);
  char* d;
  cudaMalloc(&d, 256 << 20);
  std::vector<int> blk(nblk);
  uint64_t s = 7;
  for (int i = 0; i < nblk; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    blk[i] = (int)((s >> 33) % (hbytes / 4096));
  }
  int* dblk;
  cudaMalloc(&dblk, nblk * 4);
  cudaMemcpy(dblk, blk.data(), nblk * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    for (int i = 0; i < 4; ++i) cudaMemcpyAsync(d, h + (size_t)i * (256 << 20), 256 << 20, cudaMemcpyHostToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("{\"variant\": \"cudaMemcpyAsync H2D 256MB x4\", \"GBps\": %.1f}\n", 4.0 * (256 << 20) / ms / 1e6);
    cudaEventRecord(e0);
    for (int i = 0; i < 4; ++i) ld16<<<296, 256>>>((const uint4*)hd, dblk, nblk, (uint4*)d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("{\"variant\": \"kernel 16-B loads, random 4-KB blocks\", \"GBps\": %.1f}\n", 4.0 * (256 << 20) / ms / 1e6);
    cudaFuncSetAttribute(tma_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4096);
    cudaEventRecord(e0);
    for (int i = 0; i < 4; ++i) tma_bulk<<<148, 256, 8 * 4 * 4096>>>(hd, dblk, nblk, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("{\"variant\": \"TMA 1-D bulk host->smem->HBM, random 4-KB blocks\", \"GBps\": %.1f, \"err\": \"%s\"}\n",
                    4.0 * (256 << 20) / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

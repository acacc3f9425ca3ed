// pcie_probe.cu -- host->device transfer probe for the host-resident compress path.
// Measures (pinned host memory, 1 GPU):
//   1. cudaMemcpyAsync H2D (copy engine), contiguous
//   2. cudaMemcpy2DAsync H2D of every other chunk (the K halves of [L][2][H][T][D])
//   3. zero-copy kernel read of contiguous host memory (UVA), 16-B loads, grid sweep
//   4. zero-copy gather of 256-B rows at 50% / 25% density (kept V rows)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pcie_probe pcie_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n, int unroll) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

// one warp per group of rows; each row = 256 B = 16 lanes x 16 B; 2 rows per warp iteration
__global__ void zc_gather(const uint4* __restrict__ src, const int* __restrict__ idx, int nrows,
                          uint4* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r0 = warp * 8; r0 < nrows; r0 += nwarps * 8) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int r = r0 + u * 2 + (lane >> 4);
      if (r < nrows) v[u] = src[(size_t)idx[r] * 16 + (lane & 15)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int r = r0 + u * 2 + (lane >> 4);
      if (r < nrows) dst[(size_t)r * 16 + (lane & 15)] = v[u];
    }
  }
}

int main() {
  const size_t bytes = 4ull << 30;
  char* host;
  CK(cudaHostAlloc(&host, bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < bytes; i += 4096) host[i] = (char)i;
  char* dev;
  CK(cudaMalloc(&dev, bytes));
  char* hdev;
  CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;
  auto timeit = [&](auto fn, int reps) {
    fn();
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) fn();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
  };
  double t = timeit([&] { CK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s)); }, 3);
  printf("memcpy H2D contiguous: %.1f GB/s\n", bytes / t / 1e6);
  // K halves: chunks of 8.9 MB (32 heads x 1088 tok x 256 B) at stride 2x
  const size_t w = 32ull * 1088 * 256, rows = bytes / (2 * w);
  t = timeit([&] { CK(cudaMemcpy2DAsync(dev, w, host, 2 * w, w, rows, cudaMemcpyHostToDevice, s)); }, 3);
  printf("memcpy2D H2D half (w=%zu, %zu rows): %.1f GB/s\n", w, rows, rows * w / t / 1e6);
  for (int grid : {148, 296, 592, 1184, 2368}) {
    for (int blk : {256, 512}) {
      size_t n = bytes / 16;
      t = timeit([&] { zc_read<<<grid, blk, 0, s>>>((const uint4*)hdev, (uint4*)dev, n, 4); }, 3);
      printf("zero-copy read grid %d x %d: %.1f GB/s\n", grid, blk, bytes / t / 1e6);
    }
  }
  // kept-row gathers at 50% / 25% density over the whole 4 GB (16.7M rows of 256 B)
  const size_t nrows_all = bytes / 256;
  for (double dens : {0.5, 0.25}) {
    std::vector<int> idx;
    srand(1);
    for (size_t r = 0; r < nrows_all; ++r)
      if ((rand() / (double)RAND_MAX) < dens) idx.push_back((int)r);
    int* didx;
    CK(cudaMalloc(&didx, idx.size() * 4));
    CK(cudaMemcpy(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice));
    for (int grid : {296, 592, 1184, 2368}) {
      t = timeit([&] { zc_gather<<<grid, 256, 0, s>>>((const uint4*)hdev, didx, (int)idx.size(), (uint4*)dev); }, 3);
      printf("zero-copy gather dens %.2f grid %d: %.1f GB/s useful (%.2f ms for %zu rows)\n", dens, grid,
             idx.size() * 256.0 / t / 1e6, t, idx.size());
    }
    CK(cudaFree(didx));
  }
  return 0;
}

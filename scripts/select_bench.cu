// select_bench.cu -- microbenchmark of the segmented top-k (select_emit) in isolation and
// next to compactor-like memory traffic (the situation inside the warp-specialised presses).
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I<select header dir> \
//        scripts/select_bench.cu -o select_bench && ./select_bench
//
// Prints cycles per select for SnapKV-like (1100 keys, keep 25%, 32 forced keeps) and
// EA-like (7700 keys, keep 25%, 4 forced keeps) segments, with and without 8 warps of
// streaming loads/stores beside the selecting warps.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <random>
#include <vector>

__device__ long long g_marks[16];
#ifndef NO_MARKS  // phase stamps: thread 0 of CTA 0 stores clock64 (fire-and-forget, every rep)
#define FC_SEL_MARK(i) \
  do { if (threadIdx.x == 0 && blockIdx.x == 0) g_marks[i] = clock64(); } while (0)
#endif
#include "fc_select.cuh"

using namespace fc;
using Sel = NamedGroup<0, 1>;

__global__ void __launch_bounds__(512, 1)
    bench_kernel(const uint32_t* keys_in, int n, int K, int reps, bool noise, char* buf,
                 int64_t buf_bytes, long long* cycles, int32_t* out_idx, int key_off, bool global_keys,
                 int32_t* gidx, int* first_drop) {
  extern __shared__ uint32_t sm[];
  __shared__ SelectScratch ss;
  __shared__ volatile int done;
  const uint32_t* keys = global_keys ? keys_in + key_off : sm + key_off;
  int32_t* idx = global_keys ? gidx + (int64_t)blockIdx.x * K : reinterpret_cast<int32_t*>(sm + ((n + key_off + 3) & ~3));
  if (threadIdx.x == 0) done = 0;
  if (!global_keys)
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[key_off + i] = keys_in[key_off + i];
  __syncthreads();
  if (threadIdx.x < kThreads) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (Sel::tid() == 0) ss.first_drop = INT_MAX;
      Sel::sync();
      select_emit<Sel>(keys, n, K, idx, 0, 0, ss);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      cycles[blockIdx.x] = (t1 - t0) / reps;
      done = 1;
    }
    if (blockIdx.x == 0) {
      for (int j = threadIdx.x; j < K; j += kThreads) out_idx[j] = idx[j];
      if (threadIdx.x == 0) *first_drop = ss.first_drop;
    }
  } else if (noise) {
    // compactor-like traffic: 32-KB chunks of 16-B loads then stores, per CTA region
    const int t = threadIdx.x - kThreads;
    const int64_t region = (buf_bytes / gridDim.x) & ~(int64_t)65535;
    char* base = buf + region * blockIdx.x;
    int64_t off = 0;
    while (!done) {
      uint4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = ld_stream(base + ((off + (i * kThreads + t) * 16) % (region / 2)));
#pragma unroll
      for (int i = 0; i < 8; ++i) st_stream(base + region / 2 + ((off + (i * kThreads + t) * 16) % (region / 2)), v[i]);
      off += 8 * kThreads * 16;
    }
  }
}

static uint32_t fkey(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t buf_bytes = (int64_t)8 << 30;
  char* buf;
  cudaMalloc(&buf, buf_bytes);
  cudaMemset(buf, 1, buf_bytes);
  long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(long long));
  struct Case { const char* name; int n, K, forced_lo, forced_hi; float sigma; int distinct, off; bool glob; };
  const Case cases[] = {{"snapkv-like 1100/275 (+32 win)", 1100, 275, 1068, 1100, 1.0f, 0, 0, false},
                        {"ea-like 7700/1925 (+4 sinks)", 7700, 1925, 0, 4, 0.3f, 0, 0, false},
                        {"knorm-like 1088/544", 1088, 544, 0, 0, 0.25f, 0, 0, false},
                        {"ties 3000/1000 (5 values)", 3000, 1000, 0, 0, 1.f, 5, 0, false},
                        {"all equal 500/100", 500, 100, 0, 0, 1.f, 1, 0, false},
                        {"forced only 40/10 (+32)", 40, 10, 8, 40, 1.f, 0, 0, false},
                        {"unaligned 1100/275", 1100, 275, 0, 0, 1.f, 0, 1, false},
                        {"super-tile 20000/5000", 20000, 5000, 0, 4, 0.5f, 0, 0, false},
                        {"unpacked 70000/17500 (global)", 70000, 17500, 0, 4, 0.5f, 0, 0, true},
                        {"ties unpacked 70000/30000", 70000, 30000, 0, 0, 1.f, 3, 3, true}};
  std::mt19937 rng(1);
  int bad = 0;
  int32_t* gidx;
  cudaMalloc(&gidx, (int64_t)sms * 70000 * 4);
  int* dfd;
  cudaMalloc(&dfd, 4);
  for (const Case& c : cases) {
    std::lognormal_distribution<float> ln(-8.f, c.sigma);
    std::vector<uint32_t> hall(c.n + c.off);
    for (int i = 0; i < c.n; ++i) {
      float v = ln(rng);
      if (c.distinct) v = (float)(rng() % c.distinct);
      hall[c.off + i] = (i >= c.forced_lo && i < c.forced_hi) ? fkey(INFINITY) : fkey(v);
    }
    const uint32_t* h = hall.data() + c.off;
    uint32_t* d;
    int32_t* oi;
    cudaMalloc(&d, (c.n + c.off) * 4);
    cudaMalloc(&oi, c.K * 4);
    cudaMemcpy(d, hall.data(), (c.n + c.off) * 4, cudaMemcpyHostToDevice);
    const int smem = c.glob ? 0 : (((c.n + c.off + 3) & ~3) + c.K) * 4;
    cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int noise = 0; noise < 2; ++noise) {
      bench_kernel<<<sms, 512, smem>>>(d, c.n, c.K, 20, noise, buf, buf_bytes, cyc, oi, c.off, c.glob, gidx, dfd);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<long long> hc(sms);
      cudaMemcpy(hc.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
      double m = 0;
      for (long long x : hc) m += x;
      m /= sms;
      // check: kept set = top-K by (key desc, index asc), ascending; first dropped index
      std::vector<int> order(c.n);
      for (int i = 0; i < c.n; ++i) order[i] = i;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return h[a] > h[b]; });
      std::vector<int> ref(order.begin(), order.begin() + c.K);
      std::sort(ref.begin(), ref.end());
      int ref_fd = c.n;
      for (int i = 0, j = 0; i < c.n; ++i) {
        if (j < c.K && ref[j] == i) { ++j; continue; }
        ref_fd = i;
        break;
      }
      std::vector<int32_t> got(c.K);
      cudaMemcpy(got.data(), oi, c.K * 4, cudaMemcpyDeviceToHost);
      int fd = 0;
      cudaMemcpy(&fd, dfd, 4, cudaMemcpyDeviceToHost);
      const bool ok = std::vector<int>(got.begin(), got.end()) == ref && fd == ref_fd;
      bad += !ok;
      printf("%-34s noise=%d  %8.0f cycles/select (%.2f us)  %s\n", c.name, noise, m, m / 1965.0,
             ok ? "ok" : "MISMATCH");
      long long mk[16];
      cudaMemcpyFromSymbol(mk, g_marks, sizeof(mk));
      printf("   phases (cycles): range %lld", mk[1] - mk[0]);
      long long prev = mk[1];
      for (int p = 0; p < 4; ++p)
        if (mk[3 + 2 * p] > prev) {
          printf(" | pass%d hist %lld scan %lld", p, mk[2 + 2 * p] - prev, mk[3 + 2 * p] - mk[2 + 2 * p]);
          prev = mk[3 + 2 * p];
        }
      printf(" | ->emit %lld | emit %lld (classify %lld redux+sts %lld bar %lld lds %lld scans %lld) | sync %lld\n",
             mk[9] - prev, mk[10] - mk[9], mk[12] - mk[9], mk[13] - mk[12], mk[14] - mk[13], mk[15] - mk[14],
             mk[10] - mk[15], mk[11] - mk[10]);
      long long z[16] = {0};
      cudaMemcpyToSymbol(g_marks, z, sizeof(z));
    }
    cudaFree(d);
    cudaFree(oi);
  }
  printf("%s\n", bad ? "FAILED" : "ALL OK");
  return bad ? 1 : 0;
}

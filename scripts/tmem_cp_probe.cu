// tmem_cp_probe.cu -- where does tcgen05.cp.128x256b put a 128B-swizzled K-major SMEM tile?
//
// A 128-row x 64-element (16-bit) tile is written in the layout TMA's SWIZZLE_128B
// produces (row r at (r/8)*1024 + (r%8)*128, 16-B chunk c at chunk c ^ (r % 8)), with
// element (r, e) = r * 64 + e. Four tcgen05.cp.128x256b copies (descriptor start +32 B
// each, as the MMA K-steps advance) land it in 32 TMEM columns; tcgen05.ld reads them
// back. Prints whether lane r, column c holds elements (2c, 2c + 1) of row r.
//
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2503_08461_b200/csrc \
//        scripts/tmem_cp_probe.cu -o tmem_cp_probe
#include <cstdio>
#include <vector>

#include "fc_tc.cuh"

using namespace fc;

__global__ void probe(uint32_t* out) {
  __shared__ __align__(1024) uint16_t tile[128 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, e = i % 64, c = e / 8, w = e % 8;
    const int off = (r / 8) * 512 + (r % 8) * 64 + ((c ^ (r % 8)) * 8) + w;   // in 16-bit units
    tile[off] = (uint16_t)(r * 64 + e);
  }
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(&s_tmem, 32);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s_tmem;
  if (tid == 0) {
    const uint32_t a = tc::smem_u32(tile);
    for (int j = 0; j < 4; ++j) {
      const uint64_t d = tc::desc_k_sw128(a + 32 * j);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 8 * j), "l"(d) : "memory");
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  float v[32];
  tc::tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int c = 0; c < 32; ++c) out[(warp * 32 + lane) * 32 + c] = __float_as_uint(v[c]);
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 32);
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 32 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<uint32_t> h(128 * 32);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 32; ++c) {
      const uint32_t want = (uint32_t)(r * 64 + 2 * c) | ((uint32_t)(r * 64 + 2 * c + 1) << 16);
      if (h[r * 32 + c] != want && bad++ < 8)
        printf("lane %d col %d: got %u,%u want %u,%u\n", r, c, h[r * 32 + c] & 0xFFFF, h[r * 32 + c] >> 16,
               want & 0xFFFF, want >> 16);
    }
  for (int r : {0, 1, 9}) {
    printf("lane %3d:", r);
    for (int c = 0; c < 12; ++c) printf(" %u,%u", h[r * 32 + c] & 0xFFFF, h[r * 32 + c] >> 16);
    printf("\n");
  }
  printf("%s (%d mismatches)\n", bad ? "LAYOUT DIFFERS" : "row-major pairs", bad);
  return 0;
}

// lat_probe.cu -- dependent-chain latencies of the warp/SMEM primitives the select and
// consumer code is built from (B200): SHFL, REDUX, VOTE, LDS, generic LD of SMEM, ATOMS,
// RED, named barriers. One CTA of 256 threads (8 warps, as a consumer group), 1000-long
// chains, cycles per link.
#include <cstdio>

#define N 1000
__device__ long long g_out[16];
__device__ unsigned g_sink;

__global__ void probe(int seed) {
  __shared__ unsigned sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i + 1) & 1023;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned x = seed + lane;
  long long t0, t1;
  int k = 0;
#define TIME(name, body)                                  \
  __syncthreads();                                        \
  t0 = clock64();                                         \
  for (int i = 0; i < N; ++i) { body; }                   \
  t1 = clock64();                                         \
  if (threadIdx.x == 0) g_out[k] = (t1 - t0);             \
  ++k;
  TIME("shfl", x = __shfl_sync(0xffffffffu, x, (x + 1) & 31));
  TIME("redux", x = __reduce_add_sync(0xffffffffu, x) + lane);
  TIME("reduxmin", x = __reduce_min_sync(0xffffffffu, x) + lane);
  TIME("ballot", x = __ballot_sync(0xffffffffu, x & 1) + lane);
  TIME("lds", x = sm[x & 1023]);
  unsigned* gp = sm;  // generic pointer to SMEM
  asm volatile("" : "+l"(gp));
  TIME("ld generic", x = gp[x & 1023]);
  TIME("atoms", x = atomicAdd(&sm[(x + lane) & 1023], 1u) & 1023);
  TIME("bar 256", asm volatile("bar.sync 1, 256;" ::: "memory"); x += 1);
  TIME("popc", x = __popc(x) + x);
  TIME("iadd", x = x * 3 + 1);
  if (x == 0x12345678) g_sink = x;
}

int main() {
  probe<<<1, 256>>>(1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  long long h[16];
  cudaMemcpyFromSymbol(h, g_out, sizeof(h));
  const char* names[] = {"shfl", "redux.sum", "redux.min", "ballot", "lds", "ld generic(smem)",
                         "atoms (returning)", "bar.sync 256", "popc+add", "imad"};
  for (int i = 0; i < 10; ++i) printf("%-20s %6.1f cycles/link\n", names[i], (double)h[i] / N);
  return 0;
}

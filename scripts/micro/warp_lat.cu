// Micro-benchmark: dependent latency of the warp primitives the simulator's
// round is built from (one warp, clock64 around a dependent chain).
#include <cstdio>
#include <cuda_runtime.h>
#define N 4096
__global__ void lat(int mode, unsigned *out, long long *cyc) {
  __shared__ unsigned sm[1024];
  __shared__ unsigned long long sm64[64];
  int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = i & 31;
  if (lane < 32) sm64[lane] = lane;
  __syncwarp();
  unsigned x = lane + 1;
  long long t0 = clock64();
  switch (mode) {
    case 0: for (int i = 0; i < N; ++i) x = __reduce_min_sync(0xffffffffu, x) + lane; break;
    case 1: for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31); break;
    case 2: for (int i = 0; i < N; ++i) x = __ballot_sync(0xffffffffu, (x >> (lane & 7)) & 1) + lane; break;
    case 3: for (int i = 0; i < N; ++i) x = __match_any_sync(0xffffffffu, x & 7) + lane; break;
    case 4: for (int i = 0; i < N; ++i) { sm[lane] = x; __syncwarp(); x = sm[(lane + 1) & 31] + 1; __syncwarp(); } break;
    case 5: for (int i = 0; i < N; ++i) x = atomicAdd(&sm[lane], x) & 1023; break;
    case 6: for (int i = 0; i < N; ++i) x = sm[x & 1023]; break;
    case 7: for (int i = 0; i < N; ++i) { x = __any_sync(0xffffffffu, x & 1) + x; } break;
    case 8: for (int i = 0; i < N; ++i) { unsigned long long v = atomicMax(&sm64[lane], (unsigned long long)x); x = (unsigned)v + 1; } break;
    case 9: { double d = x; for (int i = 0; i < N; ++i) d = d * 1.0000001 + 0.5; x = (unsigned)d; } break;
    case 10: { double d = x; for (int i = 0; i < N; ++i) d = 1.0 / (d + 1.0); x = (unsigned)(d * 1e9); } break;
  }
  long long t1 = clock64();
  out[lane] = x;
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  unsigned *o; long long *c;
  cudaMalloc(&o, 128); cudaMalloc(&c, 8);
  const char *nm[] = {"REDUX min", "SHFL", "VOTE ballot", "MATCH any", "STS+syncwarp+LDS+syncwarp", "ATOMS add (ret)",
                      "LDS chase", "VOTE any", "ATOMS max64 (ret)", "DFMA chain (mul+add)", "fp64 div"};
  for (int m = 0; m < 11; ++m) {
    for (int r = 0; r < 2; ++r) {
      lat<<<1, 32>>>(m, o, c);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      if (r) printf("%-30s %6.1f cycles\n", nm[m], h / (double)N);
    }
  }
  return 0;
}

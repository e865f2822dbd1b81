// Micro-benchmark: dependent-load latency through shared memory with an
// explicit shared pointer (LDS) versus a generic pointer (LD) to the same data.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chase(int mode, int iters, int *out, long long *cyc, int *gbuf) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 37 + 11) & 1023;
  __syncthreads();
  int *p = buf;
  if (mode == 2) p = gbuf;
  volatile int sel = mode;
  int *gp = sel >= 1 ? p : (int *)nullptr;  // opaque: compiler cannot prove shared
  int x = threadIdx.x;
  long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < iters; ++i) x = buf[x];
  } else {
    for (int i = 0; i < iters; ++i) x = gp[x];
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  int *out, *g; long long *c;
  cudaMalloc(&out, 4096); cudaMalloc(&c, 8); cudaMalloc(&g, 4096);
  int h[1024]; for (int i = 0; i < 1024; ++i) h[i] = (i * 37 + 11) & 1023;
  cudaMemcpy(g, h, 4096, cudaMemcpyHostToDevice);
  const char *names[3] = {"LDS (shared ptr)", "LD generic -> shared", "LD generic -> global (L1 hit)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      chase<<<1, 32>>>(mode, 10000, out, c, g);
      long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%-32s %.1f cycles/load\n", names[mode], hc / 10000.0);
    }
  }
  return 0;
}

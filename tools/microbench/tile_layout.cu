// Does the DRAM layout of a marching tile matter?  Each block owns a column
// of TY x TK points and marches over planes, reading 7 and writing 4 fields
// per point (LDG/STG, no smem).  Layout A: rows of RS doubles (tile rows are
// 512-B segments at RS*8 stride).  Layout B: tile-contiguous (each tile's
// TY*TK values of a field are one contiguous chunk).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TY = 4, TK = 64, NY = 1024, NK = 512, RS = 516, NX = 256;
constexpr long PP = (long)(NY + 2) * RS;  // per field per plane (layout A)
constexpr long PS = 4 * PP;

template <bool TILED>
__global__ void march(const double* __restrict__ oth, double* __restrict__ own, int units) {
  const int lk = threadIdx.x % TK, ly = threadIdx.x / TK;
  const int nkt = NK / TK;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int kt = u % nkt, yt = u / nkt;
    long off;
    if (TILED) off = (long)(yt * nkt + kt) * (TY * TK) + ly * TK + lk;
    else off = (long)(yt * TY + ly + 1) * RS + kt * TK + lk + 2;
    for (int x = 0; x < NX; ++x) {
      const double* o = oth + x * PS + off;
      double* w = own + x * PS + off;
      double s = o[0] + o[PP] + o[2 * PP];
      double a = w[0], b = w[PP], c = w[2 * PP], d = w[3 * PP];
      w[0] = a + s; w[PP] = b + s; w[2 * PP] = c + s; w[3 * PP] = d + s;
    }
  }
}

template <bool TILED>
void run(const double* oth, double* own, int blocks, int threads) {
  const int units = (NY / TY) * (NK / TK);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  march<TILED><<<blocks, threads>>>(oth, own, units);
  cudaEventRecord(a);
  march<TILED><<<blocks, threads>>>(oth, own, units);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 8.0 * NX * NY * NK * (3 + 4 + 4);
  printf("%s blocks=%d: %.3f ms %.1f GB/s\n", TILED ? "tiled" : "rows ", blocks, ms,
         bytes / ms / 1e6);
}

int main() {
  double *oth, *own;
  const size_t bytes = sizeof(double) * NX * PS;
  if (cudaMalloc(&oth, bytes) || cudaMalloc(&own, bytes)) { printf("alloc\n"); return 1; }
  cudaMemset(oth, 0, bytes);
  cudaMemset(own, 0, bytes);
  for (int blocks : {148 * 4, 148 * 8, 2048 * 4}) {
    run<false>(oth, own, blocks, TY * TK);
    run<true>(oth, own, blocks, TY * TK);
  }
  return 0;
}

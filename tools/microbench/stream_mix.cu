// Achievable HBM bandwidth for the colour pass's stream mix: R read streams
// and W write streams of doubles, contiguous, grid-stride (no tiling).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_mix stream_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void mix(const double* __restrict__ in, double* __restrict__ out, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += in[r * n + i];
#pragma unroll
    for (int w = 0; w < W; ++w) out[w * n + i] = s + w;
  }
}

template <int R, int W>
void run(double* in, double* out, long n, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) mix<R, W><<<blocks, 256>>>(in, out, n);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) mix<R, W><<<blocks, 256>>>(in, out, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  double bytes = 8.0 * n * (R + W);
  printf("R=%d W=%d blocks=%d: %.3f ms  %.1f GB/s\n", R, W, blocks, ms, bytes / ms / 1e6);
}

int main() {
  const long n = 1L << 29;  // 4 GiB per stream
  double *in, *out;
  if (cudaMalloc(&in, 8 * n * 7) != cudaSuccess || cudaMalloc(&out, 8 * n * 4) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(in, 0, 8 * n * 7);
  for (int blocks : {148 * 8, 148 * 32}) {
    run<1, 1>(in, out, n, blocks);
    run<7, 4>(in, out, n, blocks);
    run<7, 0>(in, out, n, blocks);
    run<4, 4>(in, out, n, blocks);
    run<3, 1>(in, out, n, blocks);
  }
  return 0;
}

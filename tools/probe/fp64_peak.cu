// FP64 pipe probe for B200 (sm_100a): DFMA vs DMMA (mma.sync m8n8k4 f64) issue throughput.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int ACC>
__global__ void dmma_peak(double* out, int iters) {
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < ACC; ++i) dmma(c[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int tpb : {256, 512, 1024}) {
    for (int bps : {1, 2}) {
      int iters = 4000;
      int grid = sms * bps;
      dfma_peak<<<grid, tpb>>>(d, 10, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_peak<<<grid, tpb>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 16 * (double)iters * grid * tpb;
      printf("DFMA tpb=%d blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, bps, flops / ms / 1e9, ms);
    }
  }
  for (int tpb : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 2000;
      int grid = sms * bps;
      dmma_peak<8><<<grid, tpb>>>(d, 10);
      cudaEventRecord(e0);
      dmma_peak<8><<<grid, tpb>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * 8 * (double)iters * grid * (tpb / 32);
      printf("DMMA tpb=%d blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, bps, flops / ms / 1e9, ms);
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}

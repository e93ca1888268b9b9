// Per-warp DMMA issue rate of the leaf engine's mainloop shape, without TMA or
// barriers: a 32 x 32 warp block (4 x 4 m8n8k4 accumulators), fragments read from
// shared memory at the padded strides of the wide tiles (A 20, B 132 doubles), or
// held in registers.  Run with 1 .. 4 warps per SM sub-partition.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// mode 0: fragments from smem every k-step; 1: distinct fragments in registers (no LDS);
// 2: same two operands for all DMMAs (the fp64_peak probe pattern, 16 accumulators)
template <int MODE>
__global__ void __launch_bounds__(512, 1) mainloop(double* out, int iters) {
  __shared__ double sa[64 * 20];
  __shared__ double sb[16 * 132];
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) sa[i] = 1e-3 * i;
  for (int i = threadIdx.x; i < 16 * 132; i += blockDim.x) sb[i] = 1e-4 * i;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  const int wm = (warp >> 2) & 1, wn = warp & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double af[4], bf[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) af[i] = sa[(wm * 32 + i * 8 + lr) * 20 + lc];
#pragma unroll
  for (int j = 0; j < 4; ++j) bf[j] = sb[lc * 132 + wn * 32 + j * 8 + lr];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ks = 0; ks < 16; ks += 4) {
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = sa[(wm * 32 + i * 8 + lr) * 20 + ks + lc];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = sb[(ks + lc) * 132 + wn * 32 + j * 8 + lr];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (MODE == 2) dmma(acc[i][j], af[0], bf[0]);
          else dmma(acc[i][j], af[i], bf[j]);
        }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    for (int tpb : {128, 256, 384, 512}) {
      const int iters = 4000;
      kern<<<sms, tpb>>>(d, 10);
      cudaEventRecord(e0);
      kern<<<sms, tpb>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 512.0 * 16 * 4 * (double)iters * sms * (tpb / 32);
      printf("%-22s warps/SMSP=%d: %6.2f TFLOP/s\n", name, tpb / 128, flops / ms / 1e9);
    }
  };
  run(mainloop<0>, "smem fragments");
  run(mainloop<1>, "register fragments");
  run(mainloop<2>, "same operands");
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

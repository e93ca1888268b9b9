// Issue cost of cp.async.bulk.tensor (UTMALDG) from inside a consumer warp: clock64
// around expect_tx + two 3-D tile loads (the leaf engine's A 20 x 64 and B 132 x 16
// boxes), issued (a) by lane 0 alone inside `if (lane == 0)`, (b) by the lane picked
// with elect.sync in a converged warp, (c) like (b) with uniform coordinates.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  unsigned pred = 0;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
  return pred != 0;
}

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, long long* out,
                      int iters) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long tot = 0;
  const unsigned bytes = (64 * 20 + 16 * 132) * 8;
  for (int it = 0; it < iters; ++it) {
    const int kc = (it * 16) % 1024, row = (it % 8) * 64;
    long long t0 = clock64();
    if (warp != 0) {
    } else if (MODE == 0) {
      if (lane == 0) {
        expect_tx(&bar, bytes);
        tma3(sm, &ma, kc, row, blockIdx.x, &bar);
        tma3(sm + 64 * 20, &mb, row, kc, blockIdx.x, &bar);
      }
    } else {
      const int kcu = __shfl_sync(0xffffffffu, kc, 0), rowu = __shfl_sync(0xffffffffu, row, 0);
      if (elect_one()) {
        expect_tx(&bar, bytes);
        tma3(sm, &ma, MODE == 2 ? kcu : kc, MODE == 2 ? rowu : row, blockIdx.x, &bar);
        tma3(sm + 64 * 20, &mb, MODE == 2 ? rowu : row, MODE == 2 ? kcu : kc, blockIdx.x, &bar);
      }
    }
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
    wait(&bar, it & 1);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot / iters;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int sms = 148, cols = 2048, rows = 2048;
  double* buf;
  cudaMalloc(&buf, (size_t)sms * rows * cols * 8);
  CUtensorMap ma, mb;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)sms};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 8, (cuuint64_t)cols * rows * 8};
  cuuint32_t boxa[3] = {20, 64, 1}, boxb[3] = {132, 16, 1}, es[3] = {1, 1, 1};
  enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, dims, strides, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, dims, strides, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long* out;
  cudaMalloc(&out, sms * 8);
  long long h[148];
  const int smem = (64 * 20 + 16 * 132) * 8;
  auto run = [&](auto k, const char* name) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<sms, 256, smem>>>(ma, mb, out, 200);
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    long long s = 0;
    for (int i = 0; i < sms; ++i) s += h[i];
    printf("%-34s mean issue cycles (expect_tx + 2 tile loads): %lld  [%s]\n", name, s / sms,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(probe<0>, "lane 0 in if (lane == 0)");
  run(probe<1>, "elect.sync, per-lane coordinates");
  run(probe<2>, "elect.sync, shuffled coordinates");
  return 0;
}

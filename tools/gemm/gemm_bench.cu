// Standalone throughput probe of the leaf engine's TMA/DMMA GEMM device routine.
// Each CTA (one per SM) runs C[MxN] -= A[MxK] B[KxN] on its own slot, `reps` times.
#include "../../paper_2503_04033_b200/csrc/hps_leaf.cu"

namespace {
#ifndef GB_MINB
#define GB_MINB CTAS_PER_SM  // minimum CTAs per SM in the probe's launch bounds (1: up to 255 registers)
#endif
__global__ void __launch_bounds__(NT, GB_MINB) gemm_probe(double* base, size_t stride, int ld, int M, int N,
                                                    int K, int reps, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(1024) double smem[];
  __shared__ __align__(8) uint64_t bars[2 * STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&bars[s], 1); mbar_init(&bars[STAGES + s], NT / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
#ifdef GB_PFTMAP
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a_work)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b_work)) : "memory");
  }
#endif
  Ctx c;
  c.M = base + (size_t)blockIdx.x * stride;
  c.ld = ld; c.slot = blockIdx.x; c.smem = smem; c.maps = &maps;
  c.full = bars; c.empty = bars + STAGES; c.pipe = 0; c.prof = nullptr;
  c.sh = nullptr; c.role = 0; c.seq = 0; c.cur_op = 0; c.leaf_counter = nullptr; c.n_leaves = 0;
#ifdef GB_L2  // every CTA reads the same A and B (slot 0: L2-resident after first touch); C per CTA
  for (int r = 0; r < reps; ++r) gemm(c, true, 2, 0, 0, 1, M, 0, M + K, 0, M, N, K);
#else
  for (int r = 0; r < reps; ++r) gemm(c, true, 0, 0, 0, 0, M, 0, M + K, 0, M, N, K);
#endif
}
}  // namespace

int main(int argc, char** argv) {
  int sms = 0;
  const int cps = argc > 1 ? atoi(argv[1]) : CTAS_PER_SM;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Shape { int M, N, K; };
  Shape shapes[] = {{2560, 1376, 1376}, {1184, 1184, 2752}, {1024, 1024, 128}, {2048, 128, 128},
                    {3936, 64, 64}, {128, 1184, 128}, {3936, 32, 32}};
  cudaFuncSetAttribute(gemm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM_BYTES);
  cudaFuncSetAttribute(gemm_probe, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_probe, NT, GEMM_SMEM_BYTES);
  printf("occupancy: %d CTAs/SM at %d B dynamic smem\n", occ, GEMM_SMEM_BYTES);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto s : shapes) {
    int ld = ((s.K > s.N ? s.K : s.N) + 15) / 16 * 16;
    int NR = 2 * s.M + s.K;
    size_t stride = (size_t)NR * ld;
    double* buf;
    cudaMalloc(&buf, stride * CTAS_PER_SM * sms * 8);
    cudaMemset(buf, 0, stride * CTAS_PER_SM * sms * 8);
    TmaMaps maps;
    make_map(&maps.a_work, buf, ld, NR, CTAS_PER_SM * sms, ld, stride, A_STRIDE, TM, !A_PAD);
    make_map(&maps.b_work, buf, ld, NR, CTAS_PER_SM * sms, ld, stride, B_STRIDE, KC);
    maps.a_scratch = maps.a_work;
    maps.a_abi = maps.a_work;
    maps.b_q = maps.b_work;
    make_map(&maps.c_red, buf, ld, NR, CTAS_PER_SM * sms, ld, stride, 16, 8);
    make_map(&maps.a_work_n, buf, ld, NR, CTAS_PER_SM * sms, ld, stride, GemmNarrow::AS, GemmNarrow::TM_);
    make_map(&maps.b_work_n, buf, ld, NR, CTAS_PER_SM * sms, ld, stride, GemmNarrow::BS, GemmNarrow::KC_);
    double fl = 2.0 * s.M * s.N * s.K;
    int reps = (int)(2e10 / fl + 1);
    if (reps > 200) reps = 200;
    gemm_probe<<<cps * sms, NT, GEMM_SMEM_BYTES>>>(buf, stride, ld, s.M, s.N, s.K, 1, maps);
    cudaEventRecord(e0);
    gemm_probe<<<cps * sms, NT, GEMM_SMEM_BYTES>>>(buf, stride, ld, s.M, s.N, s.K, reps, maps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double tiles = (double)((s.M + TM - 1) / TM) * ((s.N + 127) / 128) * TM * 128 * 2.0 * s.K;
    printf("M=%5d N=%5d K=%5d: %6.2f TFLOP/s useful, %6.2f tile-TFLOP/s (%.1f GF/s/SM useful) %s\n",
           s.M, s.N, s.K, fl * reps * cps * sms / ms / 1e9, tiles * reps * cps * sms / ms / 1e9,
           cps * fl * reps / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
#ifdef HPS_TRACE
    if (s.M == 2560) {  // timeline of CTA 0's first chunks (last launch), relative to its first wait
      static long long tr[NT / 32][HPS_TRACE][3], tp[HPS_TRACE][4];
      cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
      cudaMemcpyFromSymbol(tp, g_trace_prod, sizeof(tp));
      const long long t0 = tr[0][0][0];
      for (int g = 0; g < HPS_TRACE; ++g) {
        printf("chunk %3d prod_wait %7lld..%7lld tma %7lld..%7lld |", g, tp[g][0] ? tp[g][0] - t0 : -1, tp[g][1] ? tp[g][1] - t0 : -1, tp[g][2] - t0, tp[g][3] - t0);
        for (int w = 0; w < NT / 32; ++w) printf(" w%d %7lld %7lld %7lld", w, tr[w][g][0] - t0, tr[w][g][1] - t0, tr[w][g][2] - t0);
        printf("\n");
      }
    }
#endif
    cudaFree(buf);
  }
  return 0;
}

// Calibration probe: cycles per tcgen05.mma (kind::f16, cta_group::1, M=128) for SS and TS operands
// at N = 32..256, K = 16.  One CTA per SM; one elected thread issues `iters` MMAs back to back into one
// accumulator, commits, waits.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2411_10548_b200/csrc/sm100.cuh"
using namespace esm::sm100;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sA = dyn;                 // 128 rows x 128 B
  uint8_t* sB = dyn + 128 * 128;     // 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 384 * 128; i += blockDim.x) dyn[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, false);
    const uint64_t ad = make_sdesc_sw128(smem_u32(sA), 16, 1024);
    const uint64_t bd = make_sdesc_sw128(smem_u32(sB), 16, 1024);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) mma_ts(t, t + 256, bd, idesc, 1u);
      else mma_bf16_ss(t, ad, bd, idesc, 1u);
    }
    unsigned long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(t); }
}

template <int N, bool TS>
void run(unsigned long long* d, int blocks) {
  const int iters = 4096;
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 384 * 128);
  probe<N, TS><<<blocks, 128, 384 * 128>>>(d, iters);
  probe<N, TS><<<blocks, 128, 384 * 128>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double mac = 128.0 * N * 16;
  printf("%s N=%3d blocks=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma, %.0f MAC/cyc/SM\n", TS ? "TS" : "SS", N, blocks,
         (double)h[0] / iters, (double)h[1] / iters, mac * iters / h[1]);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  for (int blocks : {1, 148}) {
    run<32, false>(d, blocks); run<64, false>(d, blocks); run<128, false>(d, blocks); run<256, false>(d, blocks);
    run<32, true>(d, blocks); run<64, true>(d, blocks); run<128, true>(d, blocks); run<256, true>(d, blocks);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

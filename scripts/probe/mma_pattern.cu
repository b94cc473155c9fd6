// Probe: cycles per tcgen05.mma (M=128, N=64, K=16) for the access patterns of the attention backward:
// varying K-step smem addresses, alternating accumulators, MN-major operands, commits every 8 MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_pattern mma_pattern.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2411_10548_b200/csrc/sm100.cuh"
using namespace esm::sm100;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// mode 0: SS K-major, same desc; 1: SS K-major, K-step addresses + 2 accumulators; 2: SS A MN-major
// (dQ pattern); 3: TS with A columns stepping; 4: mode 1 + commit every 8; 5: SS N=128 K-steps
__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sA = dyn;                 // 32 KB
  uint8_t* sB = dyn + 32768;         // 32 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) dyn[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = slot;
  if (MODE == 13 && warp == 0) {  // warp-wide issue, elect.sync inside the asm, hoisted descriptors
    constexpr uint32_t idesc = make_idesc_bf16(128, 64, false, false);
    const uint64_t ad = make_sdesc_sw128(smem_u32(sA), 16, 1024), bd = make_sdesc_sw128(smem_u32(sB), 16, 1024);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        mma_ss_elect(t + (j >> 2) * 128, ad + (j & 3) * 2, bd + (j & 3) * 2, idesc, 1u);
      commit_elect(&bar);
    }
    unsigned long long t1 = clock64();
    mbar_wait(&bar, ((iters / 8) - 1) & 1);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  } else if (MODE != 13 && threadIdx.x == 0) {
    constexpr int N = MODE == 5 ? 128 : (MODE == 9 || MODE == 12) ? 256 : 64;
    constexpr int CE = MODE == 9 ? 4 : MODE == 10 ? 16 : MODE == 11 ? 32 : MODE == 12 ? 1 << 30 : 8;
    constexpr uint32_t idesc = make_idesc_bf16(128, N, MODE == 2, MODE == 2);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    int ph = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int k = i & 3;
      if (MODE == 0) {
        mma_bf16_ss(t, make_sdesc_sw128(a0, 16, 1024), make_sdesc_sw128(b0, 16, 1024), idesc, 1u);
      } else if (MODE == 1 || MODE == 4 || MODE == 5 || MODE == 6 || MODE == 7 || MODE >= 9) {
        mma_bf16_ss(t + (i >> 2 & 1) * 128, make_sdesc_sw128(a0 + k * 32, 16, 1024),
                    make_sdesc_sw128(b0 + k * 32, 16, 1024), idesc, 1u);
        if ((MODE == 4 || MODE == 6 || MODE == 7 || MODE >= 9) && (i % CE) == CE - 1) {
          mma_commit(&bar);
          if (MODE == 4) mbar_wait(&bar, ph);
          if (MODE == 7) {  // spin on the non-blocking test_wait
            uint32_t ok = 0;
            while (!ok)
              asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                           "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(smem_u32(&bar)), "r"((uint32_t)ph) : "memory");
          }
          ph ^= 1;
        }
      } else if (MODE == 2) {  // A: M-major SW128 (16 K rows x 128 M), B: MN-major (16 K rows x 64 N)
        mma_bf16_ss(t, make_sdesc_sw128(a0 + (i & 7) * 16 * 128 * 2 % 16384, 128 * 128, 1024),
                    make_sdesc_sw128(b0 + (i & 7) * 16 * 128 % 16384, 8192, 1024), idesc, 1u);
      } else if (MODE == 8) {  // single MMA + commit + wait: round-trip latency
        mma_bf16_ss(t, make_sdesc_sw128(a0, 16, 1024), make_sdesc_sw128(b0, 16, 1024), idesc, 1u);
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      } else if (MODE == 3) {
        mma_ts(t, t + 256 + k * 8, make_sdesc_sw128(b0 + k * 16 * 128, 8192, 1024),
               make_idesc_bf16(128, 64, false, true), 1u);
      }
    }
    unsigned long long t1 = clock64();
    if (MODE == 6 || MODE >= 9) ph = (iters / CE) & 1;  // commits without waits: wait for the last phase
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(t); }
}

template <int MODE>
void run(unsigned long long* d, int blocks, const char* name) {
  const int iters = 4096;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  probe<MODE><<<blocks, 128, 65536>>>(d, iters);
  probe<MODE><<<blocks, 128, 65536>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-40s blocks=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", name, blocks, (double)h[0] / iters,
         (double)h[1] / iters);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  for (int blocks : {1, 148}) {
    run<0>(d, blocks, "SS N=64 same desc");
    run<1>(d, blocks, "SS N=64 K-steps, 2 accumulators");
    run<4>(d, blocks, "SS N=64 K-steps + commit/wait every 8");
    run<2>(d, blocks, "SS N=64 MN-major A and B (dQ pattern)");
    run<3>(d, blocks, "TS N=64 B MN-major (dV/dK pattern)");
    run<5>(d, blocks, "SS N=128 K-steps, 2 accumulators");
    run<6>(d, blocks, "SS N=64 K-steps + commit (no wait) every 8");
    run<7>(d, blocks, "SS N=64 K-steps + commit/test_wait spin /8");
    run<8>(d, blocks, "single MMA + commit + wait (latency)");
    run<12>(d, blocks, "SS N=256 no commits");
    run<9>(d, blocks, "SS N=256 commit (no wait) every 4");
    run<10>(d, blocks, "SS N=64 commit (no wait) every 16");
    run<11>(d, blocks, "SS N=64 commit (no wait) every 32");
    run<13>(d, blocks, "SS N=64 warp-wide elect.sync, commit /8");
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Linear layers of the ESM-2 encoder: C[M,N] = A[M,K] · B[N,K]^T with fused epilogues.
//
//   forward  (HF nn.Linear, HF:modeling_esm.py:300-302,365-375,406-427):  A = X  (K-major), B = W (K-major)
//   dgrad    dX = dY · W                                                  A = dY (K-major), B = W (N-major)
//   wgrad    dW += dYᵀ · X                                                A = dY (M-major), B = X (N-major)
//
// bf16 path: persistent warp-specialised tcgen05 kernel.  TMA (SWIZZLE_128B) feeds a
// STAGES-deep smem ring; one elected thread issues tcgen05.mma (M=128, N=BN, K=16)
// into a double-buffered TMEM accumulator; four epilogue warps drain TMEM with
// tcgen05.ld and apply bias / GELU / residual / GELU' (+ fused bias-grad column sums)
// or fp32 red.add (split-K weight gradients).
// fp32 path (parity mode): tiled SIMT FFMA kernel with the same epilogues.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace esm {
namespace attn {
void zero_f32(float* p, int64_t n, cudaStream_t st);  // attention.cu: PDL-launched zero fill
}

struct EpiParams {
  int M, N;
  void* C;
  int64_t ldc;
  const float* bias;
  const void* aux_in;
  int64_t ld_aux_in;
  void* aux_out;
  int64_t ld_aux_out;
  float* col_sum;
  // QKV + RoPE epilogue
  const float* rope_cos;
  const float* rope_sin;
  __nv_bfloat16* qkv_out[3];
  int seq_len, n_heads, head_dim;
  float q_scale;
  // LayerNorm-gradient statistics epilogue
  const float* row_mean;
  const float* row_rstd;
  float* col_sum2;
  // RESID: C = R + dropout(acc + bias)
  esm_dropout drop;
  // DELTA: per-head row dot products of the bf16 output with aux_in, [B, n_heads, seq_len]
  float* row_dot;
};

// ============================================================================
// tcgen05 kernel
// ============================================================================
namespace sm100 {

constexpr int BM = 128;
constexpr int BK = 64;
// Bottleneck experiments (scripts/gemm_exp.sh builds them into a separate library; never defined in the product
// build): 1 = no TMA operand loads (MMAs read stale shared memory), 2 = no MMAs (the epilogue drains stale TMEM).
#ifndef ESM_GEMM_EXP
#define ESM_GEMM_EXP 0
#endif
// warp0 TMA, warp1 MMA (+TMEM alloc), warps 2.. epilogue: EW warps per TMEM lane quarter take interleaved
// 32-column chunks (EpiCfg::EW).

// Epilogue staging per warp: a 32x32 output chunk in swizzled smem, written to HBM by TMA.
template <int EPI>
struct EpiCfg {
  static constexpr bool QKV = EPI >= 16;  // ESM_EPI_QKV_ROPE specialised per head dim: EPI = 16 + dh
  static constexpr bool F32 = EPI == ESM_EPI_F32_ACC;
#ifndef ESM_GEMM_EW
#define ESM_GEMM_EW 2
#endif
  static constexpr int EW = ESM_GEMM_EW;  // epilogue warps per TMEM lane quarter (3 measured slower: smem for staging
                                // costs mainloop stages)
  static constexpr int WARPS = 4 * EW;
  static constexpr int THREADS = 64 + 32 * WARPS;
  static constexpr int CHUNK = F32 ? 32 * 32 * 4 : 32 * 32 * 2;  // bytes per 32x32 chunk
  static constexpr bool GELU2 = EPI == ESM_EPI_GELU || EPI == ESM_EPI_GELU_GRADAUX;  // C + aux output
  static constexpr int NOUT = GELU2 ? 2 : 1;  // outputs per chunk (GELU: C and Z; GELU_GRADAUX: C and GELU'(Z))
  static constexpr bool AUX = EPI == ESM_EPI_RESID || EPI == ESM_EPI_DGELU || EPI == ESM_EPI_STORE_LN ||
                              EPI == ESM_EPI_MUL_AUX || EPI == ESM_EPI_DELTA;
#ifndef ESM_GEMM_OBUF
#define ESM_GEMM_OBUF 1
#endif
  // output staging buffers per epilogue warp: 1 leaves room for one more operand stage (650M step 85.4 -> 84.6 ms
  // with 2 -> 1; the epilogue waits for its previous TMA store to finish reading, off the critical path)
  static constexpr int OBUF = ESM_GEMM_OBUF;
  static constexpr int WARP_BYTES = QKV ? 0 : OBUF * NOUT * CHUNK + (AUX ? 2 * CHUNK : 0);
  static constexpr int BYTES = WARPS * WARP_BYTES;
};

template <int BN, int EPI, int CG = 1>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;  // a CTA pair splits B's columns
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BUDGET = 224 * 1024 - EpiCfg<EPI>::BYTES - 1024 - 512;
  static constexpr int STAGES = BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES;
  // BN = 512: two N = 256 MMAs per k-step into one accumulator that fills TMEM (no double buffering; a quarter
  // less operand traffic per FLOP than BN = 256)
  static constexpr int NSUB = BN > 256 ? 2 : 1;   // MMAs per K = 16 step
  static constexpr int MMA_N = BN / NSUB;
  static constexpr int BSUB = BN / CG / NSUB;     // B columns per CTA per MMA
  static constexpr int NACC = BN > 256 ? 1 : 2;   // TMEM accumulator buffers
  static constexpr uint32_t TMEM_COLS = (NACC * BN <= 32) ? 32 : (NACC * BN <= 64) ? 64 : (NACC * BN <= 128) ? 128
                                                          : (NACC * BN <= 256) ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EpiCfg<EPI>::BYTES + 1024 /*align*/ + 512 /*barriers*/;
  static_assert(STAGES >= 2, "not enough shared memory for the pipeline");
};

struct TileInfo {
  int num_m, num_n, splits, kb_total, kb_per_split;
  int num_ng;  // column-tile groups: ceil(num_n / MC), MC pairs of a cluster take adjacent column tiles
};

// unit tile t -> (row block, column tile of pair `pi` of the cluster, k range); n fastest: concurrent units
// share the A row-block in L2
template <int MC>
__device__ __forceinline__ void decode_tile(const TileInfo& ti, int t, int pi, int& mb, int& nb, int& kb0, int& kb1) {
  const int per_split = ti.num_m * ti.num_ng;
  const int split = t / per_split;
  const int rem = t - split * per_split;
  mb = rem / ti.num_ng;
  nb = (rem - mb * ti.num_ng) * MC + pi;
  kb0 = split * ti.kb_per_split;
  kb1 = min(ti.kb_total, kb0 + ti.kb_per_split);
}

// ---- TMA store / reduce of a staged chunk, and bulk-group bookkeeping
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Swizzled 16-byte chunk offset inside a staged chunk: bf16 32x32 (64 B rows, SWIZZLE_64B) or
// fp32 32x32 (128 B rows, SWIZZLE_128B) -- the layouts TMA uses for the matching tensor maps.
template <bool F32>
__device__ __forceinline__ uint32_t stage_off(int row, int chunk16) {
  if constexpr (F32) return row * 128 + ((chunk16 ^ (row & 7)) << 4);
  else return row * 64 + ((chunk16 ^ ((row >> 1) & 3)) << 4);
}

struct EpiMaps {
  CUtensorMap c, z, r;
};

// CG = 2: a CTA pair computes a 256 x BN tile with tcgen05.mma.cta_group::2 -- each CTA loads its 128 rows of
// A and half of B's columns, so per-SM operand traffic drops by a third.
// MC = 2 (CG = 2 only): a cluster of two pairs computes two adjacent column tiles of the same row block; the
// shared A rows are loaded once by pair 0 and multicast into both pairs (TMA .multicast::cluster), a quarter
// less L2 -> SM operand traffic (the GEMMs are bound by it: scripts/gemm_exp.sh); every stage is released by
// both pairs' MMA commits before it is refilled.
template <int BN, bool A_MN, bool B_MN, int EPI, int CG, int MC = 1>
__global__ void __launch_bounds__(EpiCfg<EPI>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ EpiMaps maps, TileInfo ti, EpiParams ep) {
  using C = Cfg<BN, EPI, CG>;
  using E = EpiCfg<EPI>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps shared provenance
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sEpi = smem + STAGES * C::STAGE_BYTES;  // 1 KB aligned (stage sizes are multiples of 1 KB)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sEpi + E::BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar = tempty_bar + 2;  // [E::WARPS][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + 2 * E::WARPS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  static_assert(MC == 1 || CG == 2, "multicast clusters are built from CTA pairs");
  constexpr int CL = CG * MC;  // cluster size
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int rank = crank & (CG - 1);  // rank within the pair
  const int pi = crank / CG;          // pair index within the cluster
  const int unit = (int)blockIdx.x / CL;  // tile-processing unit (CTA, pair or cluster of pairs)
  const int nunits = (int)gridDim.x / CL;
  constexpr uint16_t kAllMask = (uint16_t)((1u << CL) - 1u);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], MC);  // released by every pair of the cluster
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], E::WARPS * CG);
    }
    for (int i = 0; i < 2 * E::WARPS; ++i) mbar_init(&aux_bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
    else tmem_alloc<C::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();     // predecessor's outputs (our operands) complete and visible
  pdl_trigger();  // the successor may start its prologue on SMs this grid frees

  const int num_tiles = ti.num_m * ti.num_ng * ti.splits;

  if (warp == 0) {
    // ===================== TMA producer =====================
    int stage = 0;
    uint32_t phase = 0;
    auto load = [&](void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
      if constexpr (CG == 2) tma_load_2d_pair(dst, map, bar, c0, c1);
      else tma_load_2d(dst, map, bar, c0, c1);
    };
    for (int t = unit; t < num_tiles; t += nunits) {
      int mb, nb, kb0, kb1;
      decode_tile<MC>(ti, t, pi, mb, nb, kb0, kb1);
      const int m0 = mb * BM * CG + rank * BM;   // this CTA's A rows
      const int n0 = nb * BN + rank * C::BSUB;   // this CTA's B columns (per MMA sub-tile j: + j * MMA_N)
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (ESM_GEMM_EXP == 1) {
          if (lane == 0 && rank == 0) mbar_arrive(&full_bar[stage]);
        } else if (lane == 0) {
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          if (rank == 0) mbar_expect_tx(&full_bar[stage], C::STAGE_BYTES * CG);  // both CTAs' bytes
          if constexpr (MC == 2) {  // A: pair 0 loads it into its own and pair 1's CTA of the same rank
            if (pi == 0) {
              const uint16_t mask = (uint16_t)((1u << rank) | (1u << (rank + CG)));
              if constexpr (!A_MN) {
                tma_load_2d_pair_mc(a_dst, &tmA, &full_bar[stage], kb * BK, m0, mask);
              } else {
#pragma unroll
                for (int i = 0; i < BM / 64; ++i)
                  tma_load_2d_pair_mc(a_dst + i * 64 * BK * 2, &tmA, &full_bar[stage], m0 + i * 64, kb * BK, mask);
              }
            }
          } else if constexpr (!A_MN) {
            load(a_dst, &tmA, &full_bar[stage], kb * BK, m0);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              load(a_dst + i * 64 * BK * 2, &tmA, &full_bar[stage], m0 + i * 64, kb * BK);
          }
#pragma unroll
          for (int j = 0; j < C::NSUB; ++j) {
            uint8_t* bj = b_dst + j * C::BSUB * BK * 2;
            if constexpr (!B_MN) {
              load(bj, &tmB, &full_bar[stage], kb * BK, n0 + j * C::MMA_N);
            } else {
#pragma unroll
              for (int i = 0; i < C::BSUB / 64; ++i)
                load(bj + i * 64 * BK * 2, &tmB, &full_bar[stage], n0 + j * C::MMA_N + i * 64, kb * BK);
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ===================== MMA issuer (leader CTA of a pair) =====================
    constexpr uint32_t idesc = make_idesc_bf16(BM * CG, C::MMA_N, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = unit; t < num_tiles; t += nunits, ++it) {
      int mb, nb, kb0, kb1;
      decode_tile<MC>(ti, t, pi, mb, nb, kb0, kb1);
      const int buf = C::NACC == 2 ? (it & 1) : 0;
      const uint32_t aphase = C::NACC == 2 ? ((it >> 1) & 1) : (it & 1);
      mbar_wait(&tempty_bar[buf], aphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * BN;
      const int nsub = (C::NSUB == 2 && nb * BN + C::MMA_N >= ep.N) ? 1 : C::NSUB;  // skip an all-padding sub-tile
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_base = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sdesc_sw128(a_base + k * 16 * 128, BK * 128, 1024)
                                     : make_sdesc_sw128(a_base + k * 32, 16, 1024);
            if (ESM_GEMM_EXP == 2) break;
#pragma unroll
            for (int j = 0; j < C::NSUB; ++j) {
              if (j >= nsub) break;
              const uint32_t bj = b_base + j * C::BSUB * BK * 2;
              const uint64_t bd = B_MN ? make_sdesc_sw128(bj + k * 16 * 128, BK * 128, 1024)
                                       : make_sdesc_sw128(bj + k * 32, 16, 1024);
              const uint32_t dj = d_tmem + j * C::MMA_N;
              if constexpr (CG == 2) mma_bf16_ss_pair(dj, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
              else mma_bf16_ss(dj, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          if constexpr (CG == 2) {
            mma_commit_pair(&empty_bar[stage], kAllMask);  // every CTA of the cluster: its stage may be refilled
            if (kb == kb1 - 1) mma_commit_pair(&tfull_bar[buf], (uint16_t)(3u << (pi * CG)));
          } else {
            mma_commit(&empty_bar[stage]);
            if (kb == kb1 - 1) mma_commit(&tfull_bar[buf]);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 2) {
    // ===================== epilogue warps =====================
    const int ew = warp - 2;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = ew >> 2;
    uint8_t* my = sEpi + ew * E::WARP_BYTES;
    uint8_t* obuf = my;                              // [2][NOUT][CHUNK]
    uint8_t* abuf = my + E::OBUF * E::NOUT * E::CHUNK;  // [2][CHUNK]  (AUX only)
    uint64_t* abar = aux_bar + 2 * ew;
    uint32_t aux_phase = 0;  // bit b = expected parity of aux buffer b
    int ob = 0, ab = 0;
    int it = 0;
    for (int t = unit; t < num_tiles; t += nunits, ++it) {
      int mb, nb, kb0, kb1;
      decode_tile<MC>(ti, t, pi, mb, nb, kb0, kb1);
      const int buf = C::NACC == 2 ? (it & 1) : 0;
      const uint32_t aphase = C::NACC == 2 ? ((it >> 1) & 1) : (it & 1);
      const int row0 = mb * BM * CG + rank * BM + q * 32;
      const int ncols = min(BN, ep.N - nb * BN);
      if constexpr (E::AUX) {  // prefetch the residual / pre-activation chunk of the first column block
        if (lane == 0 && half * 32 < ncols) {
          mbar_expect_tx(&abar[ab], E::CHUNK);
          tma_load_2d(abuf + ab * E::CHUNK, &maps.r, &abar[ab], nb * BN + half * 32, row0);
        }
      }
      mbar_wait(&tfull_bar[buf], aphase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * BN;
      if constexpr (E::QKV) {
        // thread = token row; one head (DH columns) at a time: bias, q-scale, RoPE, scatter
        constexpr int DH = EPI - 16, HALF = DH / 2;
        const int t = row0 + lane;
        const int Hd = ep.n_heads * DH;
        const int sq = t % ep.seq_len, bb = t / ep.seq_len;
        for (int hh = half; hh * DH < ncols; hh += E::EW) {
          uint32_t u[DH];
#pragma unroll
          for (int j = 0; j < DH; j += 8)
            tmem_ld8(taddr + hh * DH + j, u[j], u[j + 1], u[j + 2], u[j + 3], u[j + 4], u[j + 5], u[j + 6], u[j + 7]);
          tmem_ld_wait();
          float x[DH];
#pragma unroll
          for (int j = 0; j < DH; ++j) x[j] = __uint_as_float(u[j]);
          const int gcol = nb * BN + hh * DH;
          const int part = gcol / Hd, head = (gcol - part * Hd) / DH;
          const float4* b4 = reinterpret_cast<const float4*>(ep.bias + gcol);
#pragma unroll
          for (int j = 0; j < DH / 4; ++j) {
            const float4 bb4 = __ldg(b4 + j);
            x[4 * j] += bb4.x;
            x[4 * j + 1] += bb4.y;
            x[4 * j + 2] += bb4.z;
            x[4 * j + 3] += bb4.w;
          }
          if (part < 2) {
            const float sc = part == 0 ? ep.q_scale : 1.0f;
            const float4* c4 = reinterpret_cast<const float4*>(ep.rope_cos + (int64_t)sq * HALF);
            const float4* s4 = reinterpret_cast<const float4*>(ep.rope_sin + (int64_t)sq * HALF);
#pragma unroll
            for (int j = 0; j < HALF / 4; ++j) {
              const float4 cc = __ldg(c4 + j), ss = __ldg(s4 + j);
              const float cv[4] = {cc.x, cc.y, cc.z, cc.w}, sv[4] = {ss.x, ss.y, ss.z, ss.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int jj = 4 * j + u;
                const float a = x[jj] * sc, b2 = x[jj + HALF] * sc;
                x[jj] = a * cv[u] - b2 * sv[u];
                x[jj + HALF] = b2 * cv[u] + a * sv[u];
              }
            }
          }
          if (t < ep.M) {
            __nv_bfloat16* base = part == 0 ? ep.qkv_out[0] : (part == 1 ? ep.qkv_out[1] : ep.qkv_out[2]);
            __nv_bfloat16* dst = base + (((int64_t)bb * ep.n_heads + head) * ep.seq_len + sq) * DH;
#pragma unroll
            for (int j = 0; j < DH; j += 8) store_vec(dst + j, x + j);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_leader(&tempty_bar[buf]);
          else mbar_arrive(&tempty_bar[buf]);
        }
        continue;
      }
#pragma unroll 1
      for (int c = half * 32; c < ncols; c += 32 * E::EW) {
        const int col0 = nb * BN + c;
        uint32_t r[32];
        tmem_ld32(taddr + c, r);
        if constexpr (E::AUX) {
          if (lane == 0 && c + 32 * E::EW < ncols) {  // prefetch the next chunk into the other buffer
            fence_async_smem();
            mbar_expect_tx(&abar[ab ^ 1], E::CHUNK);
            tma_load_2d(abuf + (ab ^ 1) * E::CHUNK, &maps.r, &abar[ab ^ 1], col0 + 32 * E::EW, row0);
          }
        }
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if constexpr (EPI != ESM_EPI_F32_ACC && EPI != ESM_EPI_DGELU && EPI != ESM_EPI_STORE_LN &&
                      EPI != ESM_EPI_MUL_AUX && EPI != ESM_EPI_DELTA) {
          if (ep.bias != nullptr) {
            if (col0 + 32 <= ep.N) {
              const float4* b4 = reinterpret_cast<const float4*>(ep.bias + col0);  // 1 KB aligned groups
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 bb = __ldg(b4 + j);  // packed adds: same rounding as scalar FADD
                f2_unpack(f2_add(f2_pack(v[4 * j], v[4 * j + 1]), f2_pack(bb.x, bb.y)), v[4 * j], v[4 * j + 1]);
                f2_unpack(f2_add(f2_pack(v[4 * j + 2], v[4 * j + 3]), f2_pack(bb.z, bb.w)), v[4 * j + 2], v[4 * j + 3]);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += (col0 + j < ep.N) ? __ldg(ep.bias + col0 + j) : 0.f;
            }
          }
        }
        if constexpr (EPI == ESM_EPI_RESID) {
          if (ep.drop.threshold != 0u) {  // hidden dropout of the branch, before the residual add
            const DropKeys dk = drop_keys(ep.drop);
            const uint32_t rh = drop_row(dk, (uint32_t)(row0 + lane));
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const uint32_t kb = drop_pair(dk, rh, (uint32_t)(col0 + j) >> 1);
              v[j] = (kb & 1u) ? v[j] * dk.scale : 0.f;
              v[j + 1] = (kb & 2u) ? v[j + 1] * dk.scale : 0.f;
            }
          }
        }
        if constexpr (E::AUX) {
          mbar_wait(&abar[ab], (aux_phase >> ab) & 1u);
          aux_phase ^= 1u << ab;
          const uint8_t* a = abuf + ab * E::CHUNK;
          if constexpr (EPI == ESM_EPI_STORE_LN) {
            // dbeta += colsum(dy), dgamma += colsum(dy * xhat); rows >= M carry dy == 0
            const int row = row0 + lane;
            const float mu = row < ep.M ? __ldg(ep.row_mean + row) : 0.f;
            const float rs = row < ep.M ? __ldg(ep.row_rstd + row) : 0.f;
            float w[32];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float xv[8];
              load_vec(reinterpret_cast<const __nv_bfloat16*>(a + stage_off<false>(lane, k)), xv);
#pragma unroll
              for (int e = 0; e < 8; ++e) w[8 * k + e] = v[8 * k + e] * (xv[e] - mu) * rs;
            }
            __syncwarp();
            const float s2 = warp_transpose_sum32(w, lane);
            if (col0 + lane < ep.N) red_add_f32(ep.col_sum2 + col0 + lane, s2);
#pragma unroll
            for (int j = 0; j < 32; ++j) w[j] = v[j];
            const float s1 = warp_transpose_sum32(w, lane);
            if (col0 + lane < ep.N) red_add_f32(ep.col_sum + col0 + lane, s1);
          } else if constexpr (EPI == ESM_EPI_DELTA) {
            // Delta[b, h, s] += sum over this chunk's columns of head h of bf16(dO) * O; a chunk of 32 columns
            // may span several heads (dh = 24) and a head several chunks (dh = 64): partial sums are reduced
            // with fp32 red.add into the caller-zeroed row_dot (head boundaries are warp-uniform)
            const int row = row0 + lane;
            const int dh = ep.head_dim;
            const int64_t bb = row / ep.seq_len, ss = row - bb * ep.seq_len;
            float* rd = ep.row_dot + bb * ep.n_heads * (int64_t)ep.seq_len + ss;
            int h = col0 / dh, hend = (h + 1) * dh;
            float part = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float ov[8];
              load_vec(reinterpret_cast<const __nv_bfloat16*>(a + stage_off<false>(lane, k)), ov);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int c = col0 + 8 * k + e;
                if (c == hend) {
                  if (row < ep.M) red_add_f32(rd + (int64_t)h * ep.seq_len, part);
                  part = 0.f;
                  ++h;
                  hend += dh;
                }
                if (c < ep.N) part = fmaf(__bfloat162float(__float2bfloat16_rn(v[8 * k + e])), ov[e], part);
              }
            }
            if (row < ep.M && h * dh < ep.N) red_add_f32(rd + (int64_t)h * ep.seq_len, part);
            __syncwarp();
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float rv[8];
              load_vec(reinterpret_cast<const __nv_bfloat16*>(a + stage_off<false>(lane, k)), rv);
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                float& a0 = v[8 * k + e];
                float& a1 = v[8 * k + e + 1];
                if constexpr (EPI == ESM_EPI_RESID) {
                  f2_unpack(f2_add(f2_pack(a0, a1), f2_pack(rv[e], rv[e + 1])), a0, a1);
                } else if constexpr (EPI == ESM_EPI_MUL_AUX) {
                  f2_unpack(f2_mul(f2_pack(a0, a1), f2_pack(rv[e], rv[e + 1])), a0, a1);
                } else {
                  float g0, g1;
                  gelu_grad_fast2(rv[e], rv[e + 1], g0, g1);
                  f2_unpack(f2_mul(f2_pack(a0, a1), f2_pack(g0, g1)), a0, a1);
                }
              }
            }
            __syncwarp();
          }
          ab ^= 1;
        }
        // stage the outputs (wait until the TMA store that last read this buffer is done)
        if (lane == 0) bulk_wait_read<E::OBUF - 1>();
        __syncwarp();
        uint8_t* o = obuf + ob * E::NOUT * E::CHUNK;
        if constexpr (EPI == ESM_EPI_F32_ACC) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<float4*>(o + stage_off<true>(lane, k)) =
                make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        } else {
          if constexpr (EPI == ESM_EPI_GELU) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              store_vec(reinterpret_cast<__nv_bfloat16*>(o + E::CHUNK + stage_off<false>(lane, k)), v + 8 * k);
#pragma unroll
            for (int j = 0; j < 32; j += 2) gelu_fast2(v[j], v[j + 1]);
          } else if constexpr (EPI == ESM_EPI_GELU_GRADAUX) {
            float gd[32];
#pragma unroll
            for (int j = 0; j < 32; j += 2) gelu_and_grad_fast2(v[j], v[j + 1], gd[j], gd[j + 1]);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              store_vec(reinterpret_cast<__nv_bfloat16*>(o + E::CHUNK + stage_off<false>(lane, k)), gd + 8 * k);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
            store_vec(reinterpret_cast<__nv_bfloat16*>(o + stage_off<false>(lane, k)), v + 8 * k);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if constexpr (EPI == ESM_EPI_F32_ACC) {
            tma_reduce_add_2d(&maps.c, o, col0, row0);
          } else {
            tma_store_2d(&maps.c, o, col0, row0);
            if constexpr (E::GELU2) tma_store_2d(&maps.z, o + E::CHUNK, col0, row0);
          }
          bulk_commit();
        }
        if constexpr (E::OBUF == 2) ob ^= 1;
        if constexpr (EPI == ESM_EPI_DGELU || EPI == ESM_EPI_MUL_AUX) {
          if (ep.col_sum != nullptr) {  // rows >= M are exactly 0 (TMA zero-filled A)
            const float s = warp_transpose_sum32(v, lane);
            if (col0 + lane < ep.N) red_add_f32(ep.col_sum + col0 + lane, s);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_leader(&tempty_bar[buf]);
        else mbar_arrive(&tempty_bar[buf]);
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // every CTA done with TMEM and remote barriers
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
    else tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// 2D tensor map over a row-major [outer, inner] matrix with row stride ld (elements).
static int make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, int64_t ld, uint32_t box_inner,
                    uint32_t box_outer, bool f32 = false, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return ESM_EDRIVER;
  }
  const int es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * es};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%lld box=%u,%u", (int)r,
                   (unsigned long long)inner, (unsigned long long)outer, (long long)ld, box_inner, box_outer);
    return ESM_EDRIVER;
  }
  return 0;
}

static int num_sms() { return device_sm_count(); }

template <int BN, bool A_MN, bool B_MN, int EPI, int CG, int MC = 1>
static int launch_cg(const esm_gemm_args& a, cudaStream_t st) {
  using C = Cfg<BN, EPI, CG>;
  CUtensorMap tA, tB;
  EpiMaps maps;
  memset(&maps, 0, sizeof(maps));
  int rc;
  if (!A_MN)
    rc = make_map(&tA, a.A, a.K, a.M, a.lda, BK, BM);
  else
    rc = make_map(&tA, a.A, a.M, a.K, a.lda, 64, BK);
  if (rc) return rc;
  if (!B_MN)
    rc = make_map(&tB, a.B, a.K, a.N, a.ldb, BK, C::BSUB);
  else
    rc = make_map(&tB, a.B, a.N, a.K, a.ldb, 64, BK);
  if (rc) return rc;
  // epilogue maps: 32x32 chunks; bf16 -> SWIZZLE_64B (64 B rows), fp32 -> SWIZZLE_128B (128 B rows)
  if (EPI >= 16) {
    // QKV epilogue stores directly (no TMA maps)
  } else if (EPI == ESM_EPI_F32_ACC) {
    rc = make_map(&maps.c, a.C, a.N, a.M, a.ldc, 32, 32, true, CU_TENSOR_MAP_SWIZZLE_128B);
  } else {
    rc = make_map(&maps.c, a.C, a.N, a.M, a.ldc, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
    if (!rc && (EPI == ESM_EPI_GELU || EPI == ESM_EPI_GELU_GRADAUX))
      rc = make_map(&maps.z, a.aux_out, a.N, a.M, a.ld_aux_out, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
    if (!rc && (EPI == ESM_EPI_RESID || EPI == ESM_EPI_DGELU || EPI == ESM_EPI_STORE_LN || EPI == ESM_EPI_MUL_AUX ||
                EPI == ESM_EPI_DELTA))
      rc = make_map(&maps.r, a.aux_in, a.N, a.M, a.ld_aux_in, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
  }
  if (rc) return rc;

  TileInfo ti;
  ti.num_m = (a.M + BM * CG - 1) / (BM * CG);
  ti.num_n = (a.N + BN - 1) / BN;
  ti.kb_total = (a.K + BK - 1) / BK;
  ti.num_ng = (ti.num_n + MC - 1) / MC;
  int splits = 1;
  const int tiles = ti.num_m * ti.num_ng;
  const int sms = num_sms() / (CG * MC);  // tile-processing units (CTAs, CTA pairs or clusters of pairs)
  if (EPI == ESM_EPI_F32_ACC) {
    if (a.split_k > 0) {
      splits = a.split_k;
    } else {
      // minimise (waves of work units) / splits, i.e. the per-SM k-block count, with >= 8 k-blocks per unit
      const int max_splits = ti.kb_total / 8 > 0 ? ti.kb_total / 8 : 1;
      double best = 1e30;
      for (int sp = 1; sp <= max_splits && sp <= 64; ++sp) {
        const int units = tiles * sp;
        const double waves = (double)((units + sms - 1) / sms);
        const double cost = waves / sp * (1.0 + 0.01 * sp);  // small penalty for extra reduce traffic
        if (cost < best - 1e-12) {
          best = cost;
          splits = sp;
        }
      }
    }
  }
  ti.kb_per_split = (ti.kb_total + splits - 1) / splits;
  splits = (ti.kb_total + ti.kb_per_split - 1) / ti.kb_per_split;
  ti.splits = splits;

  EpiParams ep{a.M, a.N, a.C, a.ldc, a.bias, a.aux_in, a.ld_aux_in, a.aux_out, a.ld_aux_out, a.col_sum,
               a.rope_cos, a.rope_sin,
               {(__nv_bfloat16*)a.q_out, (__nv_bfloat16*)a.k_out, (__nv_bfloat16*)a.v_out},
               a.seq_len, a.n_heads, a.head_dim, a.q_scale, a.row_mean, a.row_rstd, a.col_sum2, a.drop, a.row_dot};
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, EPI, CG, MC>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);  // per device: every launch
  const int total = tiles * splits;
  int units = total < sms ? total : sms;
  if constexpr (CG * MC > 1) {
    // persistent clusters must all be co-resident: a cluster that waits for a free GPC slot runs as a second
    // wave.  Size the grid by the occupancy API (per device and configuration, cached).
    static int cached[16] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& maxc = cached[dev & 15];
    if (maxc == 0) {
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3(CG * MC * sms);
      qc.blockDim = dim3(EpiCfg<EPI>::THREADS);
      qc.dynamicSmemBytes = C::SMEM;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = CG * MC;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      qc.attrs = qa;
      qc.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &qc) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = sms;
      }
      maxc = n;
      if (getenv("ESM_GEMM_VERBOSE"))
        fprintf(stderr, "esm gemm: BN %d CG %d MC %d EPI %d: %d co-resident clusters (%d wanted)\n", BN, CG, MC, EPI,
                n, sms);
    }
    if (units > maxc) units = maxc;
  }
  launch_pdl(kern, dim3(units * CG * MC), dim3(EpiCfg<EPI>::THREADS), C::SMEM, st, CG * MC, tA, tB, maps, ti, ep);
  ESM_LAUNCH_RET();
}

static int g_pair_mode = -1;  // ESM_GEMM_PAIR=0 disables the CTA-pair kernels
static bool pair_enabled() {
  if (g_pair_mode < 0) {
    const char* e = getenv("ESM_GEMM_PAIR");
    g_pair_mode = (e && e[0] == '0') ? 0 : 1;
  }
  return g_pair_mode == 1;
}
// ESM_GEMM_MC=1 enables the multicast clusters of two pairs.  Off by default: per SM they are ~8 % faster (a
// quarter less L2 -> SM operand traffic), but only 33 clusters of 4 CTAs are co-resident on a B200 (132 of 148
// SMs: GPC placement), so every 650M GEMM measured 2-12 % slower than pairs on all 148 SMs (fc1 fwd 0.193 vs
// 0.186 ms, qkv dgrad 0.135 vs 0.122).
static bool mc_enabled() {
  static const bool on = [] {
    const char* e = getenv("ESM_GEMM_MC");
    return e && e[0] == '1';
  }();
  return on;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static int launch(const esm_gemm_args& a, cudaStream_t st) {
  // CTA pairs (M = 256 tiles) when M fills them; B columns are split across the pair, so for an
  // N-major B each half must be a whole number of 64-column TMA boxes.
  constexpr bool pair_ok = (BN % 32 == 0) && (!B_MN || (BN / 2) % 64 == 0) && BN <= 512;
  if constexpr (pair_ok) {
    if (pair_enabled() && a.M >= 2 * BM * 8) {
      if (mc_enabled() && a.N > BN) return launch_cg<BN, A_MN, B_MN, EPI, 2, 2>(a, st);
      return launch_cg<BN, A_MN, B_MN, EPI, 2>(a, st);
    }
  }
  return launch_cg<BN, A_MN, B_MN, EPI, 1>(a, st);
}

// ESM_GEMM_BN overrides the tile width (A/B measurements).  A wave-quantisation-aware choice (BN 160 / 128 for
// N = 1280, which fills the last wave) measured 16-55 % SLOWER than BN = 256 on the 650M shapes (fc2 fwd 0.202 vs
// 0.168 ms, fc1 dgrad 0.253 vs 0.163, qkv dgrad 0.192 vs 0.122): per-MMA operand reads, not the idle tail of the
// last wave, set the time, so the widest tile wins.
static int env_bn() {
  static const int v = [] {
    const char* e = getenv("ESM_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  return v;
}

static int pick_bn_kmajor(int N) {
  if (env_bn() > 0) return env_bn();
  // largest tile with <= ~6% column waste; all multiples of 32
  static const int cands[] = {256, 224, 192, 160, 128, 96, 64};
  int best = 64;
  double best_cost = 1e30;
  for (int bn : cands) {
    const int tiles = (N + bn - 1) / bn;
    const double waste = double(tiles * bn - N) / N;
    const double cost = tiles * (1.0 + 0.15 * (256.0 / bn)) * (1.0 + waste);  // favour wide tiles
    if (cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

// BN = 512 (256 x 512 pair tiles, two N = 256 MMAs per k-step, a single TMEM accumulator): a quarter less L2 -> SM
// operand traffic per FLOP, measured 1551 vs 1351 TF/s at 8192^3 and 1502 vs 1415 at 16384 x 8192 x 4096.  With
// no second accumulator the epilogue cannot overlap the next tile's mainloop, and all CTAs reach it together, so
// its output burst is HBM-write bound: every ESM-2 shape measured slower (650M fc1 fwd 0.205 vs 0.185 ms, K = 1280;
// 3B fc2 fwd 0.326 vs 0.319 ms, K = 10240 but 3 rounds of 160 tiles on 74 pairs vs 5 of 320).  Chosen only for long
// K (>= 4096, epilogue amortised) when the wide tiles quantise onto the CTA pairs no worse than BN = 256 does.
static bool prefer_bn512(const esm_gemm_args& a) {
  if (env_bn() > 0 || !pair_enabled() || a.M < 2 * BM * 8 || a.K < 4096 || a.N % 512 != 0) return false;
  const int pairs = num_sms() / 2;
  const int64_t mt = (a.M + 2 * BM - 1) / (2 * BM);
  const int64_t r512 = (mt * (a.N / 512) + pairs - 1) / pairs, r256 = (mt * (a.N / 256) + pairs - 1) / pairs;
  return 2 * r512 <= r256;
}

template <bool A_MN, bool B_MN, int EPI>
static int dispatch_bn(const esm_gemm_args& a, int bn, cudaStream_t st) {
  switch (bn) {
    case 512: return launch<512, A_MN, B_MN, EPI>(a, st);
    case 256: return launch<256, A_MN, B_MN, EPI>(a, st);
    case 128: return launch<128, A_MN, B_MN, EPI>(a, st);
    case 64: return launch<64, A_MN, B_MN, EPI>(a, st);
    default: break;
  }
  if constexpr (!B_MN) {
    switch (bn) {
      case 224: return launch<224, A_MN, B_MN, EPI>(a, st);
      case 192: return launch<192, A_MN, B_MN, EPI>(a, st);
      case 160: return launch<160, A_MN, B_MN, EPI>(a, st);
      case 96: return launch<96, A_MN, B_MN, EPI>(a, st);
      default: break;
    }
  }
  set_last_error("unsupported BN %d", bn);
  return ESM_ENOTSUP;
}

int gemm_bf16(const esm_gemm_args& a, cudaStream_t st) {
  const bool amn = a.a_mn_major != 0, bmn = a.b_mn_major != 0;
  // TMA constraints: 16-byte aligned bases and row strides
  ESM_CHECK_ARG(((uintptr_t)a.A & 15) == 0 && ((uintptr_t)a.B & 15) == 0, "gemm: A/B must be 16B aligned");
  ESM_CHECK_ARG((a.lda * 2) % 16 == 0 && (a.ldb * 2) % 16 == 0, "gemm: lda/ldb must be multiples of 8");
  if (a.epilogue == ESM_EPI_F32_ACC) {
    ESM_CHECK_ARG(amn && bmn, "gemm: F32_ACC (wgrad) expects A and B MN-major");
    ESM_CHECK_ARG(a.ldc % 4 == 0 && ((uintptr_t)a.C & 15) == 0, "gemm: fp32 C must be 16B aligned");
    const int bn = env_bn() == 512 ? 512 : (a.N > 128 ? 256 : 128);
    return dispatch_bn<true, true, ESM_EPI_F32_ACC>(a, bn, st);
  }
  ESM_CHECK_ARG(!amn, "gemm: activation-output GEMMs expect K-major A");
  ESM_CHECK_ARG(!a.aux_in || (((uintptr_t)a.aux_in & 15) == 0 && a.ld_aux_in % 8 == 0), "gemm: aux_in alignment");
  ESM_CHECK_ARG(!a.aux_out || (((uintptr_t)a.aux_out & 15) == 0 && a.ld_aux_out % 8 == 0), "gemm: aux_out alignment");
  ESM_CHECK_ARG(a.epilogue == ESM_EPI_QKV_ROPE || (a.ldc % 8 == 0 && ((uintptr_t)a.C & 15) == 0),
                "gemm: C must be 16B aligned, ldc %% 8 == 0");
  if (a.epilogue == ESM_EPI_QKV_ROPE) {
    ESM_CHECK_ARG(!bmn && a.bias && a.rope_cos && a.rope_sin && a.q_out && a.k_out && a.v_out,
                  "gemm: QKV_ROPE needs bias, rope tables and q/k/v outputs");
    ESM_CHECK_ARG(a.N == 3 * a.n_heads * a.head_dim && a.M % a.seq_len == 0, "gemm: QKV_ROPE shape");
    switch (a.head_dim) {
      case 16: return launch<256, false, false, 16 + 16>(a, st);
      case 24: return launch<240, false, false, 16 + 24>(a, st);
      case 32: return launch<256, false, false, 16 + 32>(a, st);
      case 64: return launch<256, false, false, 16 + 64>(a, st);
      default: set_last_error("gemm: QKV_ROPE head_dim %d unsupported", a.head_dim); return ESM_ENOTSUP;
    }
  }
  if (!bmn) {
    const int bn = prefer_bn512(a) ? 512 : pick_bn_kmajor(a.N);
    switch (a.epilogue) {
      case ESM_EPI_STORE: return dispatch_bn<false, false, ESM_EPI_STORE>(a, bn, st);
      case ESM_EPI_GELU: return dispatch_bn<false, false, ESM_EPI_GELU>(a, bn, st);
      case ESM_EPI_GELU_GRADAUX: return dispatch_bn<false, false, ESM_EPI_GELU_GRADAUX>(a, bn, st);
      case ESM_EPI_RESID: return dispatch_bn<false, false, ESM_EPI_RESID>(a, bn, st);
      default: break;
    }
  } else {
    const int bn = env_bn() == 128 || env_bn() == 256 || env_bn() == 512 ? env_bn()
                   : prefer_bn512(a)                                     ? 512
                   : (a.N > 128 ? 256 : 128);
    switch (a.epilogue) {
      case ESM_EPI_STORE: return dispatch_bn<false, true, ESM_EPI_STORE>(a, bn, st);
      case ESM_EPI_DGELU: return dispatch_bn<false, true, ESM_EPI_DGELU>(a, bn, st);
      case ESM_EPI_MUL_AUX: return dispatch_bn<false, true, ESM_EPI_MUL_AUX>(a, bn, st);
      case ESM_EPI_STORE_LN:
        ESM_CHECK_ARG(a.aux_in && a.row_mean && a.row_rstd && a.col_sum && a.col_sum2, "gemm: STORE_LN args");
        return dispatch_bn<false, true, ESM_EPI_STORE_LN>(a, bn, st);
      case ESM_EPI_DELTA:
        ESM_CHECK_ARG(a.aux_in && a.row_dot && a.seq_len > 0 && a.n_heads > 0 && a.head_dim > 0 &&
                          a.N == a.n_heads * a.head_dim && a.M % a.seq_len == 0,
                      "gemm: DELTA needs aux_in (O), row_dot and N = n_heads * head_dim, M = B * seq_len");
        attn::zero_f32(a.row_dot, (int64_t)a.M * a.n_heads, st);  // partial sums red.add into it
        return dispatch_bn<false, true, ESM_EPI_DELTA>(a, bn, st);
      default: break;
    }
  }
  set_last_error("gemm: unsupported epilogue %d for this operand layout", a.epilogue);
  return ESM_ENOTSUP;
}

}  // namespace sm100

// ============================================================================
// fp32 SIMT path (parity mode)
// ============================================================================
namespace simt {
constexpr int TM = 64, TN = 64, TK = 16;

template <int EPI>
__device__ __forceinline__ void apply_epi(const EpiParams& p, int row, int col, float v) {
  if (row >= p.M || col >= p.N) return;
  if constexpr (EPI == ESM_EPI_F32_ACC) {
    atomicAdd(reinterpret_cast<float*>(p.C) + (int64_t)row * p.ldc + col, v);
    return;
  } else {
    if (p.bias && EPI != ESM_EPI_DGELU) v += p.bias[col];
    if constexpr (EPI == ESM_EPI_RESID) {
      if (p.drop.threshold != 0u) {
        const DropKeys dk = drop_keys(p.drop);
        const uint32_t kb = drop_pair(dk, drop_row(dk, (uint32_t)row), (uint32_t)col >> 1);
        v = ((kb >> (col & 1)) & 1u) ? v * dk.scale : 0.f;
      }
      v += reinterpret_cast<const float*>(p.aux_in)[(int64_t)row * p.ld_aux_in + col];
    }
    if constexpr (EPI == ESM_EPI_DGELU) {
      v *= gelu_grad_f(reinterpret_cast<const float*>(p.aux_in)[(int64_t)row * p.ld_aux_in + col]);
      if (p.col_sum) atomicAdd(p.col_sum + col, v);
    }
    if constexpr (EPI == ESM_EPI_GELU) {
      reinterpret_cast<float*>(p.aux_out)[(int64_t)row * p.ld_aux_out + col] = v;
      v = gelu_f(v);
    }
    reinterpret_cast<float*>(p.C)[(int64_t)row * p.ldc + col] = v;
  }
}

template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int64_t lda, int amn,
                                                       const float* __restrict__ B, int64_t ldb, int bmn, int K,
                                                       int kchunk, EpiParams ep) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int k_begin = blockIdx.z * kchunk;
  const int k_end = min(K, k_begin + kchunk);
  float acc[4][4] = {};
  for (int k0 = k_begin; k0 < k_end; k0 += TK) {
    for (int i = threadIdx.x; i < TK * TM; i += 256) {
      int kk, mm;
      if (amn) { kk = i / TM; mm = i % TM; } else { mm = i / TK; kk = i % TK; }
      const int gm = m0 + mm, gk = k0 + kk;
      float a = 0.f;
      if (gm < ep.M && gk < k_end) a = amn ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk];
      As[kk][mm] = a;
    }
    for (int i = threadIdx.x; i < TK * TN; i += 256) {
      int kk, nn;
      if (bmn) { kk = i / TN; nn = i % TN; } else { nn = i / TK; kk = i % TK; }
      const int gn = n0 + nn, gk = k0 + kk;
      float b = 0.f;
      if (gn < ep.N && gk < k_end) b = bmn ? B[(int64_t)gk * ldb + gn] : B[(int64_t)gn * ldb + gk];
      Bs[kk][nn] = b;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) apply_epi<EPI>(ep, m0 + ty * 4 + i, n0 + tx * 4 + j, acc[i][j]);
}

int gemm_f32(const esm_gemm_args& a, cudaStream_t st) {
  EpiParams ep{a.M, a.N, a.C, a.ldc, a.bias, a.aux_in, a.ld_aux_in, a.aux_out, a.ld_aux_out, a.col_sum};
  ep.drop = a.drop;
  int splits = 1;
  if (a.epilogue == ESM_EPI_F32_ACC) splits = a.split_k > 0 ? a.split_k : (a.K >= 4096 ? 8 : 1);
  int kchunk = (a.K + splits - 1) / splits;
  kchunk = (kchunk + TK - 1) / TK * TK;
  splits = (a.K + kchunk - 1) / kchunk;
  if (splits < 1) splits = 1;
  dim3 grid((a.N + TN - 1) / TN, (a.M + TM - 1) / TM, splits);
  const float* A = reinterpret_cast<const float*>(a.A);
  const float* B = reinterpret_cast<const float*>(a.B);
  switch (a.epilogue) {
    case ESM_EPI_STORE: gemm_f32_kernel<ESM_EPI_STORE><<<grid, 256, 0, st>>>(A, a.lda, a.a_mn_major, B, a.ldb, a.b_mn_major, a.K, kchunk, ep); break;
    case ESM_EPI_GELU: gemm_f32_kernel<ESM_EPI_GELU><<<grid, 256, 0, st>>>(A, a.lda, a.a_mn_major, B, a.ldb, a.b_mn_major, a.K, kchunk, ep); break;
    case ESM_EPI_RESID: gemm_f32_kernel<ESM_EPI_RESID><<<grid, 256, 0, st>>>(A, a.lda, a.a_mn_major, B, a.ldb, a.b_mn_major, a.K, kchunk, ep); break;
    case ESM_EPI_DGELU: gemm_f32_kernel<ESM_EPI_DGELU><<<grid, 256, 0, st>>>(A, a.lda, a.a_mn_major, B, a.ldb, a.b_mn_major, a.K, kchunk, ep); break;
    case ESM_EPI_F32_ACC: gemm_f32_kernel<ESM_EPI_F32_ACC><<<grid, 256, 0, st>>>(A, a.lda, a.a_mn_major, B, a.ldb, a.b_mn_major, a.K, kchunk, ep); break;
    default: set_last_error("gemm_f32: bad epilogue %d", a.epilogue); return ESM_EINVAL;
  }
  ESM_LAUNCH_RET();
}
}  // namespace simt

}  // namespace esm

extern "C" int esm_gemm(const esm_gemm_args* args, esm_stream_t stream) {
  ESM_CHECK_ARG(args != nullptr, "esm_gemm: null args");
  const esm_gemm_args& a = *args;
  ESM_CHECK_ARG(a.M > 0 && a.N > 0 && a.K > 0, "esm_gemm: bad shape %d %d %d", a.M, a.N, a.K);
  ESM_CHECK_ARG(a.epilogue >= 0 && a.epilogue <= ESM_EPI_DELTA, "esm_gemm: bad epilogue");
  ESM_CHECK_ARG(a.epilogue < ESM_EPI_GELU_GRADAUX || a.dtype == ESM_BF16,
                "esm_gemm: GELU_GRADAUX / MUL_AUX / DELTA are bf16-only");
  ESM_CHECK_ARG(a.epilogue != ESM_EPI_GELU_GRADAUX || a.aux_out, "esm_gemm: GELU_GRADAUX needs aux_out");
  ESM_CHECK_ARG(a.epilogue != ESM_EPI_MUL_AUX || a.aux_in, "esm_gemm: MUL_AUX needs aux_in");
  ESM_CHECK_ARG(a.epilogue != ESM_EPI_STORE_LN || a.dtype == ESM_BF16, "esm_gemm: STORE_LN is bf16-only");
  ESM_CHECK_ARG(a.epilogue != ESM_EPI_QKV_ROPE || a.dtype == ESM_BF16, "esm_gemm: QKV_ROPE is bf16-only");
  ESM_CHECK_ARG(a.epilogue != ESM_EPI_RESID || a.aux_in, "esm_gemm: RESID needs aux_in");
  ESM_CHECK_ARG(a.epilogue != ESM_EPI_DGELU || a.aux_in, "esm_gemm: DGELU needs aux_in");
  ESM_CHECK_ARG(a.epilogue != ESM_EPI_GELU || a.aux_out, "esm_gemm: GELU needs aux_out");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.dtype == ESM_BF16) return esm::sm100::gemm_bf16(a, st);
  if (a.dtype == ESM_F32) return esm::simt::gemm_f32(a, st);
  esm::set_last_error("esm_gemm: bad dtype %d", a.dtype);
  return ESM_EINVAL;
}

// Flash attention forward on Blackwell tensor cores (tcgen05 + TMEM + TMA), ESM-2 semantics:
// non-causal, q pre-scaled (scaling = 1), key-padding mask (HF:modeling_esm.py:257-282).
//
// One CTA = 128 queries of one (batch, head).  Warp roles:
//   warp 0      TMA producer: Q once, then K/V tiles of 128 keys into a 2-stage smem ring
//   warp 1      MMA issuer (one elected lane): S_j = Q K_jᵀ into TMEM (double buffered),
//               O += P_{j-1} V_{j-1} with P read straight from TMEM (A-from-TMEM "TS" MMA)
//   warps 2..5  softmax: thread = one query row (its TMEM lane); exp2 online softmax with
//               lazy O rescaling (only when the running max grows by > 2^8), P written back
//               to TMEM as packed bf16 over its own S buffer; final O / l and LSE to HBM.
// Head dims 16/24/32/64 are zero-padded by TMA (OOB fill) to DP = 16/32/32/64 and use the
// matching 32/64/64/128-byte swizzle.  Right-padded (prefix) key masks skip whole key tiles;
// arbitrary masks fall back to per-key mask loads.
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace esm {
namespace fa {
using namespace sm100;

constexpr int BM = 128;
constexpr int kThreads = 192;
// Bottleneck experiments for the backward (scripts/attn_bwd_exp.sh builds them into a separate library; the
// product library is compiled without ESM_ATTN_EXP): 1 = softmax math skipped, 2 = no dQ MMAs, 3 = no dV / dK
// MMAs, 4 = no S^T / dP^T MMAs, 5 = no dQ reduce-add into global memory.  Results are wrong by construction;
// only the timing is of interest.
#ifndef ESM_ATTN_EXP
#define ESM_ATTN_EXP 0
#endif
#ifndef ESM_ATTN_FENCE_EVERY_BLOCK
#define ESM_ATTN_FENCE_EVERY_BLOCK 0
#endif
#ifndef ESM_ATTN_QST64
#define ESM_ATTN_QST64 4  // backward Q / dO stages at dh 64 (3: the previous layout with two dQ staging boxes)
#endif
constexpr float L2E = 1.4426950408889634f;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units

template <int DH, int BN_, int NSB_ = 2>
struct Shape {
  static constexpr int BN = BN_;                                    // keys per tile
  static constexpr int NSB = NSB_;                                  // S (and P) TMEM buffers
  static constexpr int DP = DH <= 16 ? 16 : (DH <= 32 ? 32 : 64);  // padded head dim (MMA K / N)
  static constexpr int ROWB = DP * 2;                               // smem row bytes = swizzle span
  static constexpr uint32_t LAYOUT = ROWB == 128 ? 2u : (ROWB == 64 ? 4u : 6u);  // SW128 / SW64 / SW32
  static constexpr int Q_BYTES = BM * ROWB;
  static constexpr int KV_BYTES = BN * ROWB;
  static constexpr int STAGES = BN >= 128 ? 2 : 3;  // K/V ring (shared memory: 2 CTAs per SM)
  // TMEM: S0 [0,BN) (S1 [BN,2BN)) O0 / O1 [NSB*BN, NSB*BN + 2*DP) (O double-buffered across items)
  static constexpr uint32_t TMEM_COLS = (NSB * BN + 2 * DP) <= 128 ? 128 : (NSB * BN + 2 * DP) <= 256 ? 256 : 512;
};

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// D[tmem] (+)= A[tmem] * B[smem]^T
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// N consecutive 32-bit TMEM columns of this warp's lane quarter (N = 16 or 32)
template <int N>
__device__ __forceinline__ void tmem_ldq(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 32) tmem_ld32(taddr, r);
  else tmem_ld16(taddr, r);
}
template <int N>
__device__ __forceinline__ void tmem_stq(uint32_t taddr, const uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_st16(taddr, r);
  else tmem_st8(taddr, r);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (offloads part of the softmax exponentials from MUFU, 16/clk/SM): round-to-nearest
// split x = j + f, f in [-0.5, 0.5], degree-3 minimax for 2^f (max rel. error 7.5e-5, far below the bf16
// rounding of P), exponent added in the integer domain.  Inputs below -126 flush to ~2^-126.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: the low mantissa bits of t hold round(x)
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517166853f, f, 0.24261115491f), f, 0.69326096773f), f, 0.99992805719f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// exp2_poly on two values with the float arithmetic in f32x2 (FADD2/FFMA2); exponent insertion is one LEA each
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& y0, float& y1) {
  const uint64_t x = f2_pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t t = f2_add(x, f2_splat(12582912.f));
  const uint64_t f = f2_fma(f2_add(t, f2_splat(-12582912.f)), f2_splat(-1.f), x);
  uint64_t p = f2_fma(f2_splat(0.05517166853f), f, f2_splat(0.24261115491f));
  p = f2_fma(p, f, f2_splat(0.69326096773f));
  p = f2_fma(p, f, f2_splat(0.99992805719f));
  float p0, p1, t0, t1;
  f2_unpack(p, p0, p1);
  f2_unpack(t, t0, t1);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}


// Scheduling workspace (caller-owned int32, ESM_ATTN_SCHED_WORDS(B) words; no global mutable state):
//   [0] forward item counter   [1] forward CTAs finished   [2] backward tile counter   [3] backward CTAs finished
//   [16 + 2b, 17 + 2b] batch row b: number of valid keys, 1 if they do not form a prefix
// esm_attn_prepare (mask_info_kernel) fills it once per batch; each persistent kernel's last CTA to finish
// resets its two counters to zero, so a prepared buffer serves every layer of the step.
constexpr int kSchedHdr = 16;

__global__ void mask_info_kernel(const int32_t* __restrict__ km, int S, int* __restrict__ sched) {
  __shared__ int s_len, s_np;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    s_len = 0;
    s_np = 0;
  }
  __syncthreads();
  int cnt = 0;
  for (int s = threadIdx.x; s < S; s += blockDim.x) cnt += km ? (km[(int64_t)b * S + s] != 0) : 1;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_len, cnt);
  __syncthreads();
  const int len = s_len;
  int bad = 0;
  if (km)
    for (int s = threadIdx.x; s < S; s += blockDim.x) bad |= ((km[(int64_t)b * S + s] != 0) != (s < len));
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(&s_np, 1);
  __syncthreads();
  if (threadIdx.x == 0) reinterpret_cast<int2*>(sched + kSchedHdr)[b] = make_int2(len, s_np);
  if (b == 0 && threadIdx.x < 4) sched[threadIdx.x] = 0;
}

__device__ __forceinline__ int2 mask_info(const int* sched, int b) {
  return reinterpret_cast<const int2*>(sched + kSchedHdr)[b];
}

// called by one thread per CTA after the CTA's last work claim: the last CTA of the grid zeroes the
// claim counter (at sched[c]) and the finished-CTA count (sched[c + 1]) for the next launch
__device__ __forceinline__ void sched_finish(int* sched, int c) {
  __threadfence();
  if (atomicAdd(&sched[c + 1], 1) == (int)gridDim.x - 1) {
    atomicExch(&sched[c], 0);
    atomicExch(&sched[c + 1], 0);
  }
}

// backward tile (head, 128-key block) whose keys are all right-padding (prefix mask): skipped by every role
__device__ __forceinline__ bool tile_skipped(const int* sched, int tile, int nkb, int nh) {
  const int b = (tile / nkb) / nh, k0 = (tile % nkb) * 128;
  const int2 mi = mask_info(sched, b);
  return mi.y == 0 && k0 >= mi.x;
}

// Persistent forward: CTA c processes items (query tile, head) c, c + gridDim.x, ... (query tile fastest).
// Q and the O accumulator are double-buffered across items (q_empty / o_free handshakes), the K/V ring and
// the S / P barriers follow a global tile counter, so the next item's loads and first MMAs overlap this
// item's softmax tail and epilogue.
template <int DH, int BN, int NSB>
constexpr int fwd_ctas_per_sm() {  // resident CTAs per SM: TMEM allocations (NSB * BN + 2 * DP columns, power of two)
  return 512 / Shape<DH, BN, NSB>::TMEM_COLS > 4 ? 4 : 512 / Shape<DH, BN, NSB>::TMEM_COLS;
}

template <int DH, int BN, int NSB, int FP>
__global__ void __launch_bounds__(kThreads, fwd_ctas_per_sm<DH, BN, NSB>())
    fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const int32_t* __restrict__ key_mask,
               int* __restrict__ sched, __nv_bfloat16* __restrict__ O, float* __restrict__ LSE, int S, int nh,
               int nbh, const esm_dropout drop) {
  using SH = Shape<DH, BN, NSB>;
  constexpr int DP = SH::DP, ROWB = SH::ROWB, ST = SH::STAGES;
  constexpr int QB = SH::Q_BYTES, TB = SH::KV_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps shared provenance
  uint8_t* sQ = smem;                      // [2][QB]
  uint8_t* sK = sQ + 2 * QB;
  uint8_t* sV = sK + ST * TB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + ST * TB);
  uint64_t* q_full = bars;                 // 2
  uint64_t* q_empty = q_full + 2;          // 2
  uint64_t* kv_full = q_empty + 2;         // ST
  uint64_t* kv_empty = kv_full + ST;       // ST
  uint64_t* s_full = kv_empty + ST;        // 2
  uint64_t* p_full = s_full + 2;           // 2
  uint64_t* o_done = p_full + 2;           // 1
  uint64_t* o_free = o_done + 1;           // 2
  uint64_t* o_full = o_free + 2;           // 2: all PV MMAs of the item using O buffer qs are complete
  uint64_t* item_full = o_full + 2;        // [4] item-id ring (TMA warp -> MMA / softmax warps)
  uint64_t* item_empty = item_full + 4;    // [4]
  int* item_ring = reinterpret_cast<int*>(item_empty + 4);  // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(item_ring + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = nh * DH;
  const int nqb = (S + BM - 1) / BM;
  const int nitem = nqb * nbh;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&o_free[i], 4);
      mbar_init(&o_full[i], 1);
    }
    for (int i = 0; i < ST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
    }
    mbar_init(o_done, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&item_full[i], 1);
      mbar_init(&item_empty[i], 1 + 4);  // MMA warp + 4 softmax warps
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<SH::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  pdl_wait();  // programmatic dependent launch: predecessor complete (common.cuh)
  pdl_trigger();

  int G0 = 0;  // KV tiles processed by this CTA before the current item (same in every role)
  // dynamic item scheduler: the TMA warp claims items (first = blockIdx.x) and publishes them through the
  // ring; -1 terminates.  Items of short (padded) rows cost less, so claiming balances the CTAs.
  int next_item = blockIdx.x;
  for (int it = 0;; ++it) {
    const int slot = it & 3;
    int item;
    if (warp == 0) {
      mbar_wait(&item_empty[slot], ((it >> 2) & 1) ^ 1);
      item = next_item < nitem ? next_item : -1;
      if (lane == 0) {
        item_ring[slot] = item;
        mbar_arrive(&item_full[slot]);
      }
      __syncwarp();
    } else {
      mbar_wait(&item_full[slot], (it >> 2) & 1);
      item = item_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&item_empty[slot]);
    }
    if (item < 0) break;
    const int bh = item / nqb, q0 = (item % nqb) * BM, b = bh / nh, h = bh % nh;
    const int2 mi = mask_info(sched, b);
    const int kv_len = mi.x;
    const bool nonprefix = mi.y != 0;
    const int ntiles = nonprefix ? (S + BN - 1) / BN : (kv_len + BN - 1) / BN;
    const int row0 = bh * S;  // first row of this head in the [B*nh*S, DH] views
    const int qs = it & 1;
    const uint32_t t_o = tbase + NSB * BN + qs * DP;  // O accumulator of this item (double-buffered)
    if (warp == 0) {
      // ======================= TMA producer =======================
      if (lane == 0 && it == 0) {
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
      }
      mbar_wait(&q_empty[qs], ((it >> 1) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&q_full[qs], QB);
        tma_load_2d(sQ + qs * QB, &tmQ, &q_full[qs], 0, row0 + q0);
      }
      for (int j = 0; j < ntiles; ++j) {
        const int gj = G0 + j, st = gj % ST;
        mbar_wait(&kv_empty[st], ((gj / ST) & 1) ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&kv_full[st], 2 * TB);
          tma_load_2d(sK + st * TB, &tmK, &kv_full[st], 0, row0 + j * BN);
          tma_load_2d(sV + st * TB, &tmV, &kv_full[st], 0, row0 + j * BN);
        }
        __syncwarp();
      }
      int t = 0;
      if (lane == 0) t = atomicAdd(&sched[0], 1) + gridDim.x;
      next_item = __shfl_sync(0xffffffffu, t, 0);
    } else if (warp == 1) {
      // ======================= MMA issuer =======================
      constexpr uint32_t idesc_s = make_idesc_bf16(BM, BN, false, false);  // S = Q Kᵀ, both K-major
      constexpr uint32_t idesc_o = make_idesc_bf16(BM, DP, false, true);   // O += P V, V N-major
      // descriptors hoisted; stage offsets are added to the start-address field (bytes >> 4)
      const uint64_t qd = make_sdesc(smem_u32(sQ + qs * QB), 16, 8 * ROWB, SH::LAYOUT);
      const uint64_t kd = make_sdesc(smem_u32(sK), 16, 8 * ROWB, SH::LAYOUT);
      const uint64_t vd = make_sdesc(smem_u32(sV), BN * ROWB, 8 * ROWB, SH::LAYOUT);
      mbar_wait(&q_full[qs], (it >> 1) & 1);
      auto issue_s = [&](int j) {  // S_j = Q K_j^T into buffer gj % NSB
        const int gj = G0 + j, st = gj % ST;
        mbar_wait(&kv_full[st], (gj / ST) & 1);
        tc_fence_after();
        const uint64_t so = (uint64_t)((st * TB) >> 4);
        const uint32_t d = tbase + (gj % NSB) * BN;
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) mma_ss_w(d, qd + 2 * k, kd + so + 2 * k, idesc_s, k > 0 ? 1u : 0u);
        mma_commit_w(&s_full[gj % NSB]);
        if (j == ntiles - 1) mma_commit_w(&q_empty[qs]);  // last use of this Q buffer
      };
      auto issue_pv = [&](int i) {  // O += P_i V_i
        const int gi = G0 + i, st = gi % ST;
        if (i == 0 && it >= 2) mbar_wait(&o_free[qs], ((it >> 1) - 1) & 1);  // item it-2 read this O buffer
        mbar_wait(&p_full[gi % NSB], (gi / NSB) & 1);
        tc_fence_after();
        const uint64_t so = (uint64_t)((st * TB) >> 4);
        const uint32_t p_tmem = tbase + (gi % NSB) * BN;
#pragma unroll
        for (int k = 0; k < BN / 16; ++k)  // V tile: BN key rows (K) x DP (N, contiguous); 16 keys per MMA
          mma_ts_w(t_o, p_tmem + k * 8, vd + so + k * ROWB, idesc_o, (i > 0 || k > 0) ? 1u : 0u);
        mma_commit_w(&kv_empty[st]);
        mma_commit_w(o_done);
        if (i == ntiles - 1) mma_commit_w(&o_full[qs]);
      };
      for (int j = 0; j <= ntiles; ++j) {
        if (NSB == 1) {  // one S buffer: P_{j-1} (packed over S) must be consumed before S_j overwrites it
          if (j >= 1) issue_pv(j - 1);
          if (j < ntiles) issue_s(j);
        } else {
          if (j < ntiles) issue_s(j);
          if (j >= 1) issue_pv(j - 1);
        }
      }
      if (ntiles == 0) {
        mma_commit_w(&q_empty[qs]);
        mma_commit_w(&o_full[qs]);  // keeps the per-buffer phase count of o_full in step with the items
      }
    } else {
      // ======================= softmax warps =======================
      const int qq = warp & 3;
      const int r = qq * 32 + lane;  // query row within tile == TMEM lane
      const uint32_t lane_off = (uint32_t)(qq * 32) << 16;
      float m_used = -INFINITY, l = 0.f;
      // attention-probability dropout (HF: dropout(softmax(S)) @ V): the row sum l keeps every probability, the
      // P fed to P.V is masked and scaled; keep(q, k) = esm_dropout bit of row bh*S + q, column k
      const DropKeys dk = drop_keys(drop);
      const uint32_t drh = dk.on ? drop_row(dk, (uint32_t)(row0 + q0 + r)) : 0u;
      for (int j = 0; j < ntiles; ++j) {
        const int gj = G0 + j;
        mbar_wait(&s_full[gj % NSB], (gj / NSB) & 1);
        tc_fence_after();
        const uint32_t sbase = tbase + lane_off + (gj % NSB) * BN;
        float ls = 0.f;
        auto rescale = [&](float mx) {
          const float mnew = mx * L2E;
          const bool grow = mnew > m_used + RESCALE_THRESHOLD;
          if (__any_sync(0xffffffffu, grow)) {  // warp-uniform: tcgen05.ld/st are warp-collective
            // raise the reference max; rescale running sum and (if any PV issued) O in TMEM
            const float f = grow ? ex2(m_used - mnew) : 1.0f;  // 0 on the first tile
            l *= f;
            if (j > 0) {
              mbar_wait(o_done, (gj - 1) & 1);
              tc_fence_after();
#pragma unroll
              for (int c = 0; c < DP; c += 16) {
                uint32_t u[16];
                tmem_ld16(t_o + lane_off + c, u);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 16; ++e) u[e] = __float_as_uint(__uint_as_float(u[e]) * f);
                tmem_st16(t_o + lane_off + c, u);
              }
            }
            if (grow) m_used = mnew;
          }
        };
        if constexpr (BN <= 64) {
          static_assert(BN == 64 || BN == 32, "the softmax holds one 32- or 64-key tile as 32-column TMEM loads");
          uint32_t ua[32], ub[BN == 64 ? 32 : 1];  // S row, used in place (no register copies)
          tmem_ld32(sbase, ua);
          if constexpr (BN == 64) tmem_ld32(sbase + 32, ub);
          else ub[0] = 0u;  // never read (BN = 32)
          tmem_ld_wait();
          auto sv = [&](int c) -> float { return __uint_as_float(c < 32 ? ua[c] : ub[c - 32]); };
          auto kill = [&](int c) {
            if (c < 32) ua[c] = __float_as_uint(-INFINITY);
            else ub[c - 32] = __float_as_uint(-INFINITY);
          };
          const int kbase = j * BN;
          bool full = !nonprefix;
          if (!nonprefix) {
            const int valid = kv_len - kbase;  // keys [0, valid) of this tile are real
            if (valid < BN) {
              full = false;
#pragma unroll
              for (int c = 0; c < BN; ++c)
                if (c >= valid) kill(c);
            }
          } else {
#pragma unroll
            for (int c = 0; c < BN; ++c) {
              const int kk = kbase + c;
              if (!(kk < S && key_mask[(int64_t)b * S + kk] != 0)) kill(c);
            }
          }
          // row max as a 4-way tree (FMNMX3 chains of 8 instead of one of 32)
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < BN; c += 8)
#pragma unroll
            for (int q = 0; q < 4; ++q) m4[q] = fmaxf(m4[q], fmaxf(sv(c + 2 * q), sv(c + 2 * q + 1)));
          const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
          rescale(mx);
          const float moff = m_used == -INFINITY ? 0.f : m_used;
          // exponentials: x = s log2e - m in FFMA2, row sums in two FADD2 chains; on full tiles FP of every four
          // pairs go to the FMA pipe (exp2_poly2) to relieve MUFU (masked tiles stay on MUFU: exact zeros)
          const uint64_t l2e = f2_splat(L2E), nm = f2_splat(-moff);
          uint64_t ls0 = f2_splat(0.f), ls1 = ls0;
          uint32_t pk[BN / 2];
          auto exps = [&](auto fp_tag, auto drop_tag) {
            constexpr int F = decltype(fp_tag)::value;
#pragma unroll
            for (int e = 0; e < BN / 2; e += 4) {  // 8 keys: 4 pairs
              float x[8], pr[8];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                f2_unpack(f2_fma(f2_pack(sv(2 * e + 2 * q), sv(2 * e + 2 * q + 1)), l2e, nm), x[2 * q], x[2 * q + 1]);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (q >= 4 - F) {
                  exp2_poly2(x[2 * q], x[2 * q + 1], pr[2 * q], pr[2 * q + 1]);
                } else {
                  pr[2 * q] = ex2(x[2 * q]);
                  pr[2 * q + 1] = ex2(x[2 * q + 1]);
                }
              }
              ls0 = f2_add(ls0, f2_pack(pr[0], pr[1]));
              ls1 = f2_add(ls1, f2_pack(pr[2], pr[3]));
              ls0 = f2_add(ls0, f2_pack(pr[4], pr[5]));
              ls1 = f2_add(ls1, f2_pack(pr[6], pr[7]));
              if constexpr (decltype(drop_tag)::value) {  // keys kbase + 2(e + q) + {0, 1}
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t kb = drop_pair(dk, drh, (uint32_t)(kbase / 2 + e + q));
                  pr[2 * q] = (kb & 1u) ? pr[2 * q] * dk.scale : 0.f;
                  pr[2 * q + 1] = (kb & 2u) ? pr[2 * q + 1] * dk.scale : 0.f;
                }
              }
#pragma unroll
              for (int q = 0; q < 4; ++q) pk[e + q] = pack2(pr[2 * q], pr[2 * q + 1]);
            }
          };
          if (dk.on) exps(std::integral_constant<int, 0>{}, std::true_type{});
          else if (FP > 0 && full) exps(std::integral_constant<int, FP>{}, std::false_type{});
          else exps(std::integral_constant<int, 0>{}, std::false_type{});
          if constexpr (BN == 64) tmem_st32(sbase, pk);  // P (bf16x2) over the first BN/2 columns of this S buffer
          else tmem_st16(sbase, pk);
          float l0, l1, l2, l3;
          f2_unpack(ls0, l0, l1);
          f2_unpack(ls1, l2, l3);
          ls = (l0 + l1) + (l2 + l3);
        } else {
          // 128-key tiles (NSB = 1): two passes over the S row in TMEM, 32 columns at a time (the row does not fit
          // in registers): the max, then exp2 / row sum / P packing, P (bf16x2) written over the columns already
          // read (chunk c -> columns [16c, 16c + 16))
          static_assert(BN == 128, "tile width");
          const int kbase = j * BN;
          const int valid = nonprefix ? BN : kv_len - kbase;
          bool full = !nonprefix && valid >= BN;
          auto chunk = [&](int c, uint32_t (&u)[32]) {
            tmem_ld32(sbase + 32 * c, u);
            tmem_ld_wait();
            if (!full) {
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const int kk = kbase + 32 * c + e;
                const bool ok = nonprefix ? (kk < S && key_mask[(int64_t)b * S + kk] != 0) : (32 * c + e < valid);
                if (!ok) u[e] = __float_as_uint(-INFINITY);
              }
            }
          };
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t u[32];
            chunk(c, u);
#pragma unroll
            for (int e = 0; e < 32; e += 8)
#pragma unroll
              for (int q = 0; q < 4; ++q)
                m4[q] = fmaxf(m4[q], fmaxf(__uint_as_float(u[e + 2 * q]), __uint_as_float(u[e + 2 * q + 1])));
          }
          rescale(fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
          const float moff = m_used == -INFINITY ? 0.f : m_used;
          const uint64_t l2e = f2_splat(L2E), nm = f2_splat(-moff);
          uint64_t ls0 = f2_splat(0.f), ls1 = ls0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t u[32], pk[16];
            chunk(c, u);
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              float x[8], pr[8];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                f2_unpack(f2_fma(f2_pack(__uint_as_float(u[e + 2 * q]), __uint_as_float(u[e + 2 * q + 1])), l2e, nm),
                          x[2 * q], x[2 * q + 1]);
#pragma unroll
              for (int q = 0; q < 8; ++q) pr[q] = ex2(x[q]);
              ls0 = f2_add(ls0, f2_pack(pr[0], pr[1]));
              ls1 = f2_add(ls1, f2_pack(pr[2], pr[3]));
              ls0 = f2_add(ls0, f2_pack(pr[4], pr[5]));
              ls1 = f2_add(ls1, f2_pack(pr[6], pr[7]));
#pragma unroll
              for (int q = 0; q < 4; ++q) pk[e / 2 + q] = pack2(pr[2 * q], pr[2 * q + 1]);
            }
            tmem_st16(sbase + 16 * c, pk);
          }
          float l0, l1, l2, l3;
          f2_unpack(ls0, l0, l1);
          f2_unpack(ls1, l2, l3);
          ls = (l0 + l1) + (l2 + l3);
        }
        l += ls;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[gj % NSB]);
      }
      // ---- epilogue: wait for the last PV, O / l, LSE; release the O buffer.  (Not o_done: another softmax
      // warp may still be two tiles behind, so o_done's phase count can trail by two and a parity wait on it
      // would pass early; o_full[qs] completes exactly once per item on this buffer.)
      const int qrow = q0 + r;
      float inv = l > 0.f ? 1.f / l : 0.f;
      mbar_wait(&o_full[qs], (it >> 1) & 1);
      tc_fence_after();
      float o[DP];
#pragma unroll
      for (int c = 0; c < DP; c += 16) {
        uint32_t u[16];
        tmem_ld16(t_o + lane_off + c, u);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) o[c + e] = ntiles > 0 ? __uint_as_float(u[e]) * inv : 0.f;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[qs]);
      if (qrow < S) {
        __nv_bfloat16* dst = O + ((int64_t)b * S + qrow) * H + h * DH;
#pragma unroll
        for (int c = 0; c < DH; c += 8) {
          uint4 w;
          w.x = pack2(o[c], o[c + 1]);
          w.y = pack2(o[c + 2], o[c + 3]);
          w.z = pack2(o[c + 4], o[c + 5]);
          w.w = pack2(o[c + 6], o[c + 7]);
          *reinterpret_cast<uint4*>(dst + c) = w;
        }
        LSE[(int64_t)bh * S + qrow] = l > 0.f ? -(m_used + log2f(l)) : INFINITY;  // -LSE log2 e (ABI form)
      }
    }
    G0 += ntiles;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sched_finish(sched, 0);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<SH::TMEM_COLS>(tbase);
  }
}

// ============================================================================ backward
// CTA = 128 keys of one (batch, head); loop over 64-query blocks (processed in pairs).
//   warp 0     TMA: K, V once; Q_i, dO_i tiles + LSE_i / Delta_i (bulk copies) per block (QST stages)
//   warp 1     MMA: S^T = K Q_i^T, dP^T = V dO_i^T into TMEM; after softmax-bwd:
//              dV += P^T dO_i, dK += dS^T Q_i (A = P^T / dS^T read from TMEM); once per block pair
//              dQ_pair = dS K (M = 128 queries; A = dS^T of both blocks staged in smem, M-major)
//   warps 2..  softmax-bwd: SW warps per TMEM lane quarter, 64 / SW queries each, thread = key row:
//              P^T = exp2(S^T - LSE), dS^T = P^T (dP^T - Delta); P^T / dS^T written back to TMEM (bf16,
//              over S^T / dP^T), dS^T also to smem (the A operand of dQ)
//   last 4     dQ drain (one per lane quarter, thread = query row): TMEM -> swizzled smem boxes ->
//              TMA reduce-add into the fp32 dQ accumulator, overlapped with the softmax warps
// SW = 2 (448 threads) is the default; SW = 4 (16 softmax warps, 704 threads, 80 registers) doubles the softmax
// warps in flight and measured slower (see bwd_softmax_warps).
// TMEM (512 columns, one CTA per SM): NBUF x {S^T, dP^T} (64 columns each), dV, dK, 2 x dQ (DP each);
// NBUF = 3 for dh <= 32, 2 for dh = 64.
// Prefix (right-padded) masks: key blocks past the valid length write zero dK/dV and exit.
template <int SW>
struct BwdWarps {
  static constexpr int QW = 64 / SW;                 // queries per softmax warp
  static constexpr int SOFT = 4 * SW;                // softmax warps
  static constexpr int DRAIN0 = 2 + SOFT;            // first dQ-drain warp
  static constexpr int THREADS = 32 * (2 + SOFT + 4);
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Optional fused output of the backward (esm_attn_bwd_qkv): dK (RoPE^T applied) and dV written straight
// into the token-major dqkv [T, 3H] buffer the QKV dgrad/wgrad GEMMs consume, with their bias-gradient
// column sums; dQ accumulated token-major [T, H] (finalised by dq_finalize_kernel).
struct FusedOut {
  __nv_bfloat16* dqkv;  // nullptr -> classic [B, nh, S, dh] outputs
  float* col_sum;       // [3H]
  const float* cos_t;   // [S, dh/2]
  const float* sin_t;
  int H;
  esm_dropout drop;     // attention-probability dropout (threshold 0: off); keep(q, k) at (row bh*S + q, column k)
};

__device__ __forceinline__ void tma_reduce_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int DH>
struct BwdShape {
  static constexpr int DP = Shape<DH, 64>::DP, ROWB = Shape<DH, 64>::ROWB;
  static constexpr uint32_t LAYOUT = Shape<DH, 64>::LAYOUT;
  static constexpr int QB = 64 * ROWB, KB = 128 * ROWB;
  static constexpr int NBUF = DP <= 32 ? 3 : 2;  // {S^T, dP^T} TMEM buffers (128 columns each)
  // Q / dO / LSE / Delta stages (>= NBUF + 1): a stage freed by block i's dV / dK MMAs is refilled for block
  // i + QST, which the MMA warp needs right after block i + QST - NBUF's dV / dK: QST - NBUF block periods of
  // TMA latency budget
  static constexpr int QST = DH == 64 ? ESM_ATTN_QST64 : 6;
  // FOLD: the TMA warp folds block j's Delta into dO after loading block j + LAG; that load waits for block
  // j + LAG - QST's dV / dK MMAs, which the MMA warp issues before it needs block j (at j - NBUF):
  // LAG <= QST - NBUF keeps the cycle open
  static constexpr int LAG = QST - NBUF < 2 ? QST - NBUF : 2;
  static_assert(LAG >= 1, "prep lag");
  // dh padded with >= 3 zero columns (dh = 24): Delta rides in dO's padding columns and V's hold -1, so the
  // dP^T MMA directly yields dP^T - Delta (Delta split into three bf16 parts: ~24-bit exact)
  static constexpr bool FOLD = DP - DH >= 3;
  static constexpr int DS_BUF = 2 * 128 * 128;  // one pair: [2 query chunks of 64][128 key rows][128 B]
  // dQ drain: fp32 boxes of BOXC columns x 32 rows, swizzled (128B or 64B rows), staged per drain warp for
  // TMA reduce-add.  DH = 24 drains its zero-padded 32-column tile: the 8 extra columns either fall outside
  // the tensor map (clipped) or add exact zeros to the neighbouring head's accumulator.
  static constexpr int BOXC = DP < 32 ? DP : 32;
  static constexpr int NBOX = DP / BOXC;
  static constexpr int BOX_BYTES = 32 * BOXC * 4;
  // dQ staging boxes per drain warp: all NBOX, or one reused box (dh 64 with 4 Q/dO stages: shared memory)
  static constexpr int SBOX = (DH == 64 && QST > 3) ? 1 : NBOX;
  static constexpr int DQ_STAGE = 4 * SBOX * BOX_BYTES;
  static constexpr int SMEM = 2 * DS_BUF + 4 * KB + 2 * QST * QB + 2 * QST * 64 * 4 + DQ_STAGE + 1024 + 512;
};

// TMEM: {S^T, dP^T} x NBUF buffers (64 columns each) at [0, 128*NBUF); dV, dK, 2 x dQ (DP columns each).
// Persistent: CTA c processes key-block tiles c, c + gridDim.x, ... (tile = (b, h, 128-key block), key block
// fastest).  All barrier phases follow global block / pair counters (every tile has nqe blocks); K / V are
// double-buffered so the next tile's loads and first S^T / dP^T MMAs overlap this tile's tail, and the
// dK / dV epilogue runs on the dQ-drain warps, which release the accumulators (dkv_free) for the next tile.
template <int DH, int SW>
__global__ void __launch_bounds__(BwdWarps<SW>::THREADS, 1)
    bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
               const __grid_constant__ CUtensorMap tmdQ, const int32_t* __restrict__ key_mask,
               int* __restrict__ sched, const float* __restrict__ LSE, const float* __restrict__ Delta,
               float* __restrict__ dQ, __nv_bfloat16* __restrict__ dK, __nv_bfloat16* __restrict__ dV, int S,
               int nh, int nbh, const FusedOut fo) {
  using BS = BwdShape<DH>;
  using BW = BwdWarps<SW>;
  constexpr int DP = BS::DP, ROWB = BS::ROWB, QB = BS::QB, KB = BS::KB, QST = BS::QST, NBUF = BS::NBUF;
  constexpr int QW = BW::QW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps shared provenance
  uint8_t* sdS = smem;               // [2][DS_BUF]
  uint8_t* sK = sdS + 2 * BS::DS_BUF;  // [2][KB]
  uint8_t* sV = sK + 2 * KB;           // [2][KB]
  uint8_t* sQ = sV + 2 * KB;         // [QST][QB]
  uint8_t* sdO = sQ + QST * QB;      // [QST][QB]
  uint8_t* sDQ = sdO + QST * QB;     // [4 warps][NBOX][32 rows][BOXC fp32] (1024-aligned: swizzled)
  float* sL = reinterpret_cast<float*>(sDQ + BS::DQ_STAGE);  // [QST][64]
  float* sD = sL + QST * 64;                                 // [QST][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + QST * 64);
  uint64_t* kv_full = bars;                // [2]
  uint64_t* kv_empty = kv_full + 2;        // [2]
  uint64_t* qdo_full = kv_empty + 2;       // [QST]
  uint64_t* qdo_empty = qdo_full + QST;    // [QST]
  uint64_t* qdo_ready = qdo_empty + QST;   // [QST] (FOLD: dO padding columns written)
  uint64_t* s_full = qdo_ready + QST;      // [NBUF]
  uint64_t* ds_full = s_full + NBUF;       // [NBUF]
  uint64_t* dq_full = ds_full + NBUF;      // [2]
  uint64_t* dq_empty = dq_full + 2;        // [2]
  uint64_t* dsm_empty = dq_empty + 2;      // [2]
  uint64_t* dkv_done = dsm_empty + 2;
  uint64_t* dkv_free = dkv_done + 1;
  uint64_t* tile_full = dkv_free + 1;     // [4] tile-id ring (TMA warp -> MMA / softmax / drain warps)
  uint64_t* tile_empty = tile_full + 4;   // [4]
  int* tile_ring = reinterpret_cast<int*>(tile_empty + 4);  // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = (S + 127) / 128;
  const int ntile = nkb * nbh;
  const int nq = (S + 63) / 64;
  const int nqe = nq + (nq & 1);  // whole pairs (a trailing virtual block holds no queries)
  const int npairs = nqe / 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < QST; ++i) {
      mbar_init(&qdo_full[i], 1);
      mbar_init(&qdo_empty[i], 1);
      mbar_init(&qdo_ready[i], 1);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&ds_full[i], BW::SOFT);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dsm_empty[i], 1);
      mbar_init(&dq_full[i], 1);
      mbar_init(&dq_empty[i], 4);
    }
    mbar_init(dkv_done, 1);
    mbar_init(dkv_free, 4);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tile_full[i], 1);
      mbar_init(&tile_empty[i], 1 + BW::SOFT + 4);  // MMA warp, softmax warps, 4 drain warps
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  pdl_wait();  // programmatic dependent launch: predecessor complete (common.cuh)
  pdl_trigger();
  const uint32_t tdV = tbase + 128 * NBUF, tdK = tdV + DP, tdQ0 = tdK + DP;  // dQ double buffered

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmdO);
    }
    // dynamic tile scheduler: claim tiles from the global counter (first tile = blockIdx.x), zero-fill the
    // dK / dV rows of fully padded key blocks here, publish real tiles through the ring, -1 terminates
    auto claim = [&]() {
      int t = 0;
      if (lane == 0) t = atomicAdd(&sched[2], 1) + gridDim.x;
      return __shfl_sync(0xffffffffu, t, 0);
    };
    int tile = blockIdx.x;
    for (int it = 0;; ++it) {
      while (tile < ntile && tile_skipped(sched, tile, nkb, nh)) {
        const int bh = tile / nkb, k0 = (tile % nkb) * 128, b = bh / nh, h = bh % nh;
        for (int i = lane; i < 128; i += 32) {
          const int key = k0 + i;
          if (key >= S) break;
          for (int hf = 0; hf < 2; ++hf) {
            __nv_bfloat16* dst = fo.dqkv ? fo.dqkv + ((int64_t)b * S + key) * 3 * fo.H + (1 + hf) * fo.H + h * DH
                                         : (hf == 0 ? dK : dV) + ((int64_t)bh * S + key) * DH;
            for (int cc = 0; cc < DH; cc += 8) *reinterpret_cast<uint4*>(dst + cc) = make_uint4(0u, 0u, 0u, 0u);
          }
        }
        tile = claim();
      }
      const int slot = it & 3;
      mbar_wait(&tile_empty[slot], ((it >> 2) & 1) ^ 1);
      if (lane == 0) {
        tile_ring[slot] = tile < ntile ? tile : -1;
        mbar_arrive(&tile_full[slot]);
      }
      __syncwarp();
      if (tile >= ntile) break;
      const int bh = tile / nkb, k0 = (tile % nkb) * 128, b = bh / nh, h = bh % nh;
      const int row0 = bh * S;
      const int kvs = it & 1;
      mbar_wait(&kv_empty[kvs], ((it >> 1) & 1) ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&kv_full[kvs], 2 * KB);
        tma_load_2d(sK + kvs * KB, &tmK, &kv_full[kvs], 0, row0 + k0);
        tma_load_2d(sV + kvs * KB, &tmV, &kv_full[kvs], 0, row0 + k0);
      }
      // FOLD: once block i's tiles have landed, write its Delta (three bf16 parts) into dO's padding columns
      // 24..26 (SW64: logical 16-byte chunk 3 of a row sits at chunk 3 ^ ((row >> 1) & 3)), then release it
      auto fold = [&](int i) {
        const int g = it * nqe + i, st = g % QST;
        mbar_wait(&qdo_full[st], (g / QST) & 1);
        for (int rr = lane; rr < 64; rr += 32) {
          const float d = sD[st * 64 + rr];  // rows past S hold stale values: their P is masked to 0
          const __nv_bfloat16 h0 = __float2bfloat16_rn(d);
          const float r1 = d - __bfloat162float(h0);
          const __nv_bfloat16 h1 = __float2bfloat16_rn(r1);
          const __nv_bfloat16 h2 = __float2bfloat16_rn(r1 - __bfloat162float(h1));
          __nv_bfloat16* dst =
              reinterpret_cast<__nv_bfloat16*>(sdO + st * QB + rr * ROWB + ((3 ^ ((rr >> 1) & 3)) << 4));
          dst[0] = h0;
          dst[1] = h1;
          dst[2] = h2;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&qdo_ready[st]);
      };
      for (int i = 0; i < nqe; ++i) {
        const int g = it * nqe + i;
        const int st = g % QST, use = g / QST;
        mbar_wait(&qdo_empty[st], (use & 1) ^ 1);
        if (lane == 0) {
          const int q0 = i * 64;
          const int nvalid = max(0, min(64, S - q0));
          const uint32_t vb = (uint32_t)nvalid * 4;
          mbar_expect_tx(&qdo_full[st], 2 * QB + 2 * vb);
          tma_load_2d(sQ + st * QB, &tmQ, &qdo_full[st], 0, row0 + q0);
          tma_load_2d(sdO + st * QB, &tmdO, &qdo_full[st], h * DH, b * S + q0);
          if (vb) {
            bulk_load(sL + st * 64, LSE + (int64_t)bh * S + q0, vb, &qdo_full[st]);
            bulk_load(sD + st * 64, Delta + (int64_t)bh * S + q0, vb, &qdo_full[st]);
          }
        }
        __syncwarp();
        if constexpr (BS::FOLD) {
          if (i >= BS::LAG) fold(i - BS::LAG);
        }
      }
      if constexpr (BS::FOLD) {
        for (int i = max(0, nqe - BS::LAG); i < nqe; ++i) fold(i);
      }
      tile = claim();
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);  // S^T, dP^T: 128 keys x 64 queries
    constexpr uint32_t idesc_kv = make_idesc_bf16(128, DP, false, true);  // dV, dK (A from TMEM)
    constexpr uint32_t idesc_q = make_idesc_bf16(128, DP, true, true);    // dQ (A = dS^T smem, M-major)
    // descriptors hoisted: per-use offsets are added to the 14-bit start-address field (bytes >> 4)
    const uint64_t kd_s = make_sdesc(smem_u32(sK), 16, 8 * ROWB, BS::LAYOUT);     // K  (A of S^T)
    const uint64_t vd_s = make_sdesc(smem_u32(sV), 16, 8 * ROWB, BS::LAYOUT);     // V  (A of dP^T)
    const uint64_t qd_s = make_sdesc(smem_u32(sQ), 16, 8 * ROWB, BS::LAYOUT);     // Q  (B of S^T)
    const uint64_t od_s = make_sdesc(smem_u32(sdO), 16, 8 * ROWB, BS::LAYOUT);    // dO (B of dP^T)
    const uint64_t od_kv = make_sdesc(smem_u32(sdO), QB, 8 * ROWB, BS::LAYOUT);   // dO (B of dV, MN-major)
    const uint64_t qd_kv = make_sdesc(smem_u32(sQ), QB, 8 * ROWB, BS::LAYOUT);    // Q  (B of dK, MN-major)
    const uint64_t kd_q = make_sdesc(smem_u32(sK), KB, 8 * ROWB, BS::LAYOUT);     // K  (B of dQ, MN-major)
    const uint64_t dsd = make_sdesc(smem_u32(sdS), 128 * 128, 1024, 2u);          // dS^T (A of dQ, M-major)
    for (int it = 0;; ++it) {
      const int slot = it & 3;
      mbar_wait(&tile_full[slot], (it >> 2) & 1);
      const int tile = tile_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_empty[slot]);
      if (tile < 0) break;
      const int kvs = it & 1;
      const uint64_t ko = (uint64_t)((kvs * KB) >> 4);
      auto issue_s = [&](int j) {  // S^T(j), dP^T(j) into buffer g % NBUF
        const int g = it * nqe + j;
        const int st = g % QST;
        if constexpr (BS::FOLD) mbar_wait(&qdo_ready[st], (g / QST) & 1);
        else mbar_wait(&qdo_full[st], (g / QST) & 1);
        tc_fence_after();
        const uint64_t so = (uint64_t)((st * QB) >> 4);
        const uint32_t tS = tbase + (g % NBUF) * 128, tDP = tS + 64;
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) {
          if (ESM_ATTN_EXP == 4) break;
          mma_ss_w(tS, kd_s + ko + 2 * k, qd_s + so + 2 * k, idesc_s, k > 0 ? 1u : 0u);
          mma_ss_w(tDP, vd_s + ko + 2 * k, od_s + so + 2 * k, idesc_s, k > 0 ? 1u : 0u);
        }
        mma_commit_w(&s_full[g % NBUF]);
      };
      mbar_wait(&kv_full[kvs], (it >> 1) & 1);
      if constexpr (BS::FOLD) {  // V's padding columns 24..26 = -1 (the dP^T MMA subtracts Delta)
        for (int rr = lane; rr < 128; rr += 32) {
          __nv_bfloat16* dst =
              reinterpret_cast<__nv_bfloat16*>(sV + kvs * KB + rr * ROWB + ((3 ^ ((rr >> 1) & 3)) << 4));
          dst[0] = dst[1] = dst[2] = __float2bfloat16_rn(-1.f);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      for (int j = 0; j < NBUF && j < nqe; ++j) issue_s(j);
      for (int i = 0; i < nqe; ++i) {
        const int g = it * nqe + i, p = i >> 1, gp = it * npairs + p;
        const int st = g % QST;
        mbar_wait(&ds_full[g % NBUF], (g / NBUF) & 1);
        if (i == 0 && it > 0) mbar_wait(dkv_free, (it - 1) & 1);  // previous tile's dV / dK have been read
        tc_fence_after();
        const uint64_t so = (uint64_t)((st * QB) >> 4);
        const uint32_t tS = tbase + (g % NBUF) * 128, tDP = tS + 64;
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 16 queries per step
          const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
          // packed P^T / dS^T of queries [16k, 16k+16): the softmax warp owning them wrote them at the start of
          // its own QW fp32 columns
          const uint32_t pc = (uint32_t)((16 * k / QW) * QW + ((16 * k) % QW) / 2);
          if (ESM_ATTN_EXP == 3) break;
          mma_ts_w(tdV, tS + pc, od_kv + so + k * ROWB, idesc_kv, acc);
          mma_ts_w(tdK, tDP + pc, qd_kv + so + k * ROWB, idesc_kv, acc);
        }
        if (i & 1) {
          if (gp >= 2) {  // the drain warps have read this dQ accumulator's previous pair
            mbar_wait(&dq_empty[gp & 1], ((gp >> 1) - 1) & 1);
            tc_fence_after();
          }
          const uint64_t dso = (uint64_t)(((gp & 1) * BS::DS_BUF) >> 4);
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // 16 keys per step
            if (ESM_ATTN_EXP == 2) break;
            mma_ss_w(tdQ0 + (gp & 1) * DP, dsd + dso + k * 128, kd_q + ko + k * ROWB, idesc_q, k > 0 ? 1u : 0u);
          }
          mma_commit_w(&dq_full[gp & 1]);
          mma_commit_w(&dsm_empty[gp & 1]);
        }
        mma_commit_w(&qdo_empty[st]);
        if (i == nqe - 1) {
          mma_commit_w(dkv_done);
          mma_commit_w(&kv_empty[kvs]);
        }
        // (measured: issuing S^T / dP^T(i + NBUF) ahead of the pair's dQ MMAs is 11 % slower at dh 64 -- the
        // MMA thread then blocks on block i + NBUF's Q / dO loads before it can issue dQ)
        if (i + NBUF < nqe) issue_s(i + NBUF);  // buffer g % NBUF is free once dV/dK(g) are issued (in-order)
      }
    }
  } else if (warp >= BW::DRAIN0) {
    // ============ dQ drain + dK / dV epilogue: 4 warps, one per TMEM lane quarter ============
    // dQ (thread = query row of the pair): TMEM -> registers -> swizzled smem boxes -> asynchronous TMA
    // reduce-add into the fp32 dQ accumulator (no per-element LSU traffic to contend with the softmax).
    const int qq = warp & 3;
    const uint32_t lane_off = (uint32_t)(qq * 32) << 16;
    constexpr int BOXC = BS::BOXC, RB = BOXC * 4;           // fp32 columns / bytes per staged row
    constexpr uint32_t SWM = RB == 128 ? 7u : 3u;            // 128B / 64B swizzle: chunk ^= (addr >> 7) & SWM
    uint8_t* stage = sDQ + qq * (BS::SBOX * BS::BOX_BYTES);
    for (int it = 0;; ++it) {
      const int slot = it & 3;
      mbar_wait(&tile_full[slot], (it >> 2) & 1);
      const int tile = tile_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_empty[slot]);
      if (tile < 0) break;
      const int bh = tile / nkb, k0 = (tile % nkb) * 128, b = bh / nh, h = bh % nh;
      for (int p = 0; p < npairs; ++p) {
        const int gp = it * npairs + p;
        mbar_wait(&dq_full[gp & 1], (gp >> 1) & 1);
        tc_fence_after();
        const uint32_t tq = tdQ0 + (gp & 1) * DP + lane_off;
#pragma unroll
        for (int x = 0; x < BS::NBOX; ++x) {
          uint32_t u[BOXC];
#pragma unroll
          for (int c = 0; c < BOXC; c += 8)
            tmem_ld8(tq + x * BOXC + c, u[c], u[c + 1], u[c + 2], u[c + 3], u[c + 4], u[c + 5], u[c + 6], u[c + 7]);
          tmem_ld_wait();
          if (x == BS::NBOX - 1) {  // whole tile read: release the TMEM buffer to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&dq_empty[gp & 1]);
          }
          const int sb = BS::SBOX == 1 ? 0 : x;
          if (BS::SBOX == 1 || x == 0) {  // the previous reduce has finished reading the staging box(es)
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < BOXC / 4; ++j) {
            const uint32_t off = (uint32_t)(lane * RB + j * 16);
            *reinterpret_cast<float4*>(stage + sb * BS::BOX_BYTES + (off ^ (((off >> 7) & SWM) << 4))) =
                make_float4(__uint_as_float(u[4 * j]), __uint_as_float(u[4 * j + 1]), __uint_as_float(u[4 * j + 2]),
                            __uint_as_float(u[4 * j + 3]));
          }
          // rows past this sequence carry exact zeros (dS = 0 there), so spilling into the next rows is harmless
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            const int row = (fo.dqkv ? b * S : bh * S) + p * 128 + qq * 32;
            const int col = fo.dqkv ? h * DH : 0;
            if (ESM_ATTN_EXP != 5) tma_reduce_2d(&tmdQ, stage + sb * BS::BOX_BYTES, col + x * BOXC, row);
            bulk_commit_group();
          }
        }
      }
      // ---- final key rows of this tile: dK, dV (thread = key row kr of lane quarter qq).  Both accumulators
      // are read out of TMEM and packed to bf16 (the output precision) first, and released to the MMA warp
      // (dkv_free: the next tile's first dV / dK MMAs wait on it) before any RoPE / store / bias-sum work.
      mbar_wait(dkv_done, it & 1);
      tc_fence_after();
      const int key = k0 + qq * 32 + lane;
      const bool live = key < S;
      uint32_t kp[DP / 2], vp[DP / 2];  // bf16x2 pairs of dK, dV
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const uint32_t src = (hf == 0 ? tdK : tdV) + lane_off;
#pragma unroll
        for (int cc = 0; cc < DP; cc += 8) {
          uint32_t u[8];
          tmem_ld8(src + cc, u[0], u[1], u[2], u[3], u[4], u[5], u[6], u[7]);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const uint32_t pk = live ? pack2(__uint_as_float(u[j]), __uint_as_float(u[j + 1])) : 0u;
            if (hf == 0) kp[(cc + j) / 2] = pk;
            else vp[(cc + j) / 2] = pk;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dkv_free);
      auto lo = [](uint32_t w) { return __uint_as_float(w << 16); };
      auto hi = [](uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); };
      if (fo.dqkv) {
        // fused: RoPE^T on dK (pairs (j, j + DH/2) are packed words m and m + DH/4), token-major stores into
        // dqkv, q/k/v bias-gradient column sums (from the bf16 values, as the classic qkv_rope_bwd path)
        constexpr int HALF = DH / 2, HW = HALF / 2;
        if (live) {
          const float* cs = fo.cos_t + (int64_t)key * HALF;
          const float* sn = fo.sin_t + (int64_t)key * HALF;
#pragma unroll
          for (int m = 0; m < HW; ++m) {
            const float2 c2 = __ldg(reinterpret_cast<const float2*>(cs + 2 * m));
            const float2 s2 = __ldg(reinterpret_cast<const float2*>(sn + 2 * m));
            const float a0 = lo(kp[m]), a1 = hi(kp[m]), b0 = lo(kp[m + HW]), b1 = hi(kp[m + HW]);
            kp[m] = pack2(a0 * c2.x + b0 * s2.x, a1 * c2.y + b1 * s2.y);
            kp[m + HW] = pack2(b0 * c2.x - a0 * s2.x, b1 * c2.y - a1 * s2.y);
          }
          __nv_bfloat16* row = fo.dqkv + ((int64_t)b * S + key) * 3 * fo.H + fo.H + h * DH;
#pragma unroll
          for (int cc = 0; cc < DH; cc += 8) {
            *reinterpret_cast<uint4*>(row + cc) = make_uint4(kp[cc / 2], kp[cc / 2 + 1], kp[cc / 2 + 2], kp[cc / 2 + 3]);
            *reinterpret_cast<uint4*>(row + fo.H + cc) =
                make_uint4(vp[cc / 2], vp[cc / 2 + 1], vp[cc / 2 + 2], vp[cc / 2 + 3]);
          }
        }
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int c0 = 0; c0 < DH; c0 += 32) {
            float t32[32];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const uint32_t w = (c0 + j < DH) ? (hf == 0 ? kp[(c0 + j) / 2] : vp[(c0 + j) / 2]) : 0u;
              t32[j] = lo(w);
              t32[j + 1] = hi(w);
            }
            const float csum = warp_transpose_sum32(t32, lane);
            if (c0 + lane < DH) red_add_f32(fo.col_sum + (1 + hf) * fo.H + h * DH + c0 + lane, csum);
          }
        }
      } else if (live) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          __nv_bfloat16* dst = (hf == 0 ? dK : dV) + ((int64_t)bh * S + key) * DH;
          const uint32_t* w = hf == 0 ? kp : vp;
#pragma unroll
          for (int cc = 0; cc < DH; cc += 8)
            *reinterpret_cast<uint4*>(dst + cc) = make_uint4(w[cc / 2], w[cc / 2 + 1], w[cc / 2 + 2], w[cc / 2 + 3]);
        }
      }
    }
    if (lane == 0) bulk_wait_all0();
  } else {
    // ============ softmax-bwd (thread = key row; SW warps per lane quarter, QW queries each) ============
    const int qq = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int kr = qq * 32 + lane;
    const DropKeys dk = drop_keys(fo.drop);
    const uint32_t lane_off = (uint32_t)(qq * 32) << 16;
    const int c = hf * QW;
    for (int it = 0;; ++it) {
      const int slot = it & 3;
      mbar_wait(&tile_full[slot], (it >> 2) & 1);
      const int tile = tile_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_empty[slot]);
      if (tile < 0) break;
      const int bh = tile / nkb, k0 = (tile % nkb) * 128, b = bh / nh;
      const int key = k0 + kr;
      const bool kvalid = key < S && key_mask[(int64_t)b * S + key] != 0;
      for (int i = 0; i < nqe; ++i) {
        const int g = it * nqe + i, p = i >> 1, ch = i & 1, gp = it * npairs + p;
        const int st = g % QST;
        const float* lse = sL + st * 64 + c;
        const float* dl = sD + st * 64 + c;
        const uint32_t tS = tbase + (g % NBUF) * 128, tDP = tS + 64;
        mbar_wait(&s_full[g % NBUF], (g / NBUF) & 1);
        tc_fence_after();
        uint32_t us[QW], ud[QW];
        tmem_ldq<QW>(tS + lane_off + c, us);
        tmem_ldq<QW>(tDP + lane_off + c, ud);
        if (ch == 0 && gp >= 2) mbar_wait(&dsm_empty[gp & 1], ((gp >> 1) - 1) & 1);
        tmem_ld_wait();
        uint32_t pp[QW / 2], dd[QW / 2];
        const int qmax = S - i * 64 - c;
        bool dropped = false;
        {
          if (dk.on) {
            // attention-probability dropout: dV uses Z o P^T, dS^T = P^T o (Z o dP^T - Delta), Z = keep / (1 - p).
            // FOLD (dh 24): the MMA left dP^T - Delta, so Z o dP^T - Delta = Z o (dP^T - Delta) + (Z - 1) Delta
            const uint32_t kpair = (uint32_t)key >> 1;
            const int kodd = key & 1;
            // row hashes of this warp's QW queries: lane e computes query e's, the others read it by shuffle
            const uint32_t rh_lane = drop_row(dk, (uint32_t)(bh * S + i * 64 + c) + (uint32_t)(lane % QW));
#pragma unroll
            for (int e = 0; e < QW; e += 4) {
              const float4 l4 = *reinterpret_cast<const float4*>(lse + e);
              const float4 d4 = *reinterpret_cast<const float4*>(dl + e);
              const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv4[4] = {d4.x, d4.y, d4.z, d4.w};
              // one hash covers both keys of a pair (lanes 2j, 2j + 1): each lane hashes two of the four queries
              // and swaps with its partner lane
              uint32_t hv[4];
#pragma unroll
              for (int t = 0; t < 2; ++t) {
                const uint32_t mine =
                    lowbias32(__shfl_sync(0xffffffffu, rh_lane, e + 2 * t + kodd) ^ (kpair + dk.k1));
                const uint32_t other = __shfl_xor_sync(0xffffffffu, mine, 1);
                hv[2 * t] = kodd ? other : mine;
                hv[2 * t + 1] = kodd ? mine : other;
              }
              // packed f32x2 arithmetic as the no-dropout path; 1 in 4 exponentials on the FMA pipe
              const uint64_t l2e = f2_splat(L2E);
              float x[4], pr[4], z[4];
              f2_unpack(f2_fma(f2_pack(__uint_as_float(us[e]), __uint_as_float(us[e + 1])), l2e, f2_pack(lv[0], lv[1])),
                        x[0], x[1]);
              f2_unpack(f2_fma(f2_pack(__uint_as_float(us[e + 2]), __uint_as_float(us[e + 3])), l2e,
                               f2_pack(lv[2], lv[3])),
                        x[2], x[3]);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float pe = u == 3 ? exp2_poly(x[u]) : ex2(x[u]);
                pr[u] = (kvalid && e + u < qmax) ? pe : 0.f;
                const uint32_t bits = kodd ? (hv[u] >> 16) : (hv[u] & 0xFFFFu);
                z[u] = bits >= dk.thr ? dk.scale : 0.f;
              }
              float pz[4], ds[4];
#pragma unroll
              for (int u = 0; u < 4; u += 2) {
                const uint64_t p2 = f2_pack(pr[u], pr[u + 1]), z2 = f2_pack(z[u], z[u + 1]);
                f2_unpack(f2_mul(p2, z2), pz[u], pz[u + 1]);
                const uint64_t add = BS::FOLD ? f2_pack((z[u] - 1.f) * dv4[u], (z[u + 1] - 1.f) * dv4[u + 1])
                                              : f2_pack(-dv4[u], -dv4[u + 1]);
                const uint64_t g2 =
                    f2_fma(f2_pack(__uint_as_float(ud[e + u]), __uint_as_float(ud[e + u + 1])), z2, add);
                f2_unpack(f2_mul(p2, g2), ds[u], ds[u + 1]);
              }
              pp[e >> 1] = pack2(pz[0], pz[1]);
              pp[(e >> 1) + 1] = pack2(pz[2], pz[3]);
              dd[e >> 1] = pack2(ds[0], ds[1]);
              dd[(e >> 1) + 1] = pack2(ds[2], ds[3]);
            }
            dropped = true;
          }
        }
        if (dropped) {
        } else if (ESM_ATTN_EXP == 1) {
#pragma unroll
          for (int e = 0; e < QW / 2; ++e) pp[e] = dd[e] = us[e] ^ ud[e];
        } else if (__all_sync(0xffffffffu, kvalid) && qmax >= QW) {  // full tile: no masking
          // packed f32x2 arithmetic; 1 in 4 exponentials (a pair per 8) on the FMA pipe
#pragma unroll
          for (int e = 0; e < QW; e += 8) {
            const float4 la = *reinterpret_cast<const float4*>(lse + e), lb = *reinterpret_cast<const float4*>(lse + e + 4);
            const uint64_t l2e = f2_splat(L2E);
            float x[8], pr[8];
            f2_unpack(f2_fma(f2_pack(__uint_as_float(us[e]), __uint_as_float(us[e + 1])), l2e, f2_pack(la.x, la.y)),
                      x[0], x[1]);
            f2_unpack(f2_fma(f2_pack(__uint_as_float(us[e + 2]), __uint_as_float(us[e + 3])), l2e, f2_pack(la.z, la.w)),
                      x[2], x[3]);
            f2_unpack(f2_fma(f2_pack(__uint_as_float(us[e + 4]), __uint_as_float(us[e + 5])), l2e, f2_pack(lb.x, lb.y)),
                      x[4], x[5]);
            f2_unpack(f2_fma(f2_pack(__uint_as_float(us[e + 6]), __uint_as_float(us[e + 7])), l2e, f2_pack(lb.z, lb.w)),
                      x[6], x[7]);
            pr[0] = ex2(x[0]);
            pr[1] = ex2(x[1]);
            pr[2] = ex2(x[2]);
            pr[4] = ex2(x[4]);
            pr[5] = ex2(x[5]);
            pr[6] = ex2(x[6]);
            exp2_poly2(x[3], x[7], pr[3], pr[7]);
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
              pp[(e + u) >> 1] = pack2(pr[u], pr[u + 1]);
              uint64_t dv = f2_pack(__uint_as_float(ud[e + u]), __uint_as_float(ud[e + u + 1]));
              if constexpr (!BS::FOLD) {  // ud holds dP^T; subtract Delta (FOLD: the MMA already did)
                const float2 d2 = *reinterpret_cast<const float2*>(dl + e + u);
                dv = f2_sub(dv, f2_pack(d2.x, d2.y));
              }
              float d0, d1;
              f2_unpack(f2_mul(f2_pack(pr[u], pr[u + 1]), dv), d0, d1);
              dd[(e + u) >> 1] = pack2(d0, d1);
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < QW; e += 4) {
            const float4 l4 = *reinterpret_cast<const float4*>(lse + e);
            const float4 d4 = BS::FOLD ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(dl + e);
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv4[4] = {d4.x, d4.y, d4.z, d4.w};
            float pr[4], ds[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float xe = fmaf(__uint_as_float(us[e + u]), L2E, lv[u]);  // lv = -LSE (log2 domain)
              const float pe = u == 3 ? exp2_poly(xe) : ex2(xe);
              pr[u] = (kvalid && e + u < qmax) ? pe : 0.f;
              ds[u] = pr[u] * (__uint_as_float(ud[e + u]) - dv4[u]);
            }
            pp[e >> 1] = pack2(pr[0], pr[1]);
            pp[(e >> 1) + 1] = pack2(pr[2], pr[3]);
            dd[e >> 1] = pack2(ds[0], ds[1]);
            dd[(e >> 1) + 1] = pack2(ds[2], ds[3]);
          }
        }
        // packed P^T / dS^T go into the first QW/2 of this warp's own QW columns of the S^T / dP^T buffers
        // (which it has finished reading), so the warps of a lane quarter need no barrier
        tmem_stq<QW / 2>(tS + lane_off + c, pp);
        tmem_stq<QW / 2>(tDP + lane_off + c, dd);
        uint8_t* rowp = sdS + (gp & 1) * BS::DS_BUF + ch * (128 * 128) + kr * 128;
#pragma unroll
        for (int gg = 0; gg < QW / 8; ++gg) {
          const int c16 = c / 8 + gg;
          *reinterpret_cast<uint4*>(rowp + ((c16 ^ (kr & 7)) << 4)) =
              make_uint4(dd[4 * gg], dd[4 * gg + 1], dd[4 * gg + 2], dd[4 * gg + 3]);
        }
        tmem_st_wait();
        // dS^T in shared memory is read (async proxy) only by the pair's dQ MMA, issued after the pair's second
        // block: one proxy fence per pair covers both blocks' stores of this thread
        if (ch == 1 || ESM_ATTN_FENCE_EVERY_BLOCK) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_full[g % NBUF]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sched_finish(sched, 2);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ---------------------------------------------------------------------------- host
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled encoder() {
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

template <int DH, int ROWS>
static int head_map(CUtensorMap* m, const void* base, int64_t rows) {
  using SH = Shape<DH, 64>;
  PFN_encodeTiled enc = encoder();
  if (!enc) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return ESM_EDRIVER;
  }
  cuuint64_t dims[2] = {(cuuint64_t)DH, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)DH * 2};
  cuuint32_t box[2] = {(cuuint32_t)SH::DP, (cuuint32_t)ROWS};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = SH::ROWB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : SH::ROWB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                 : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("attention tensor map encode failed (%d)", (int)r);
    return ESM_EDRIVER;
  }
  return 0;
}

// exponential pairs (of every four) evaluated on the FMA pipe in the forward softmax: ESM_ATTN_FWD_POLY=0/1/2.
// Measured (B200, 35M / 650M layer shapes): 0 -> 0.238 / 0.133 ms, 1 -> 0.237 / 0.136, 2 -> 0.245 / 0.137: the
// forward is not MUFU-throughput-bound once the S registers are used in place, so the default is 0.
static int fwd_poly_pairs() {
  static const int fp = [] {
    const char* e = getenv("ESM_ATTN_FWD_POLY");
    return e ? atoi(e) : 0;
  }();
  return fp;
}

// Key-tile width of the forward (ESM_ATTN_FWD_BN): 64 (two S buffers, 2 CTAs/SM, default); 32 for dh <= 32 (4
// CTAs / 16 softmax warps per SM; measured slower: 35M layer 0.249 vs 0.238 ms, 80 registers spill); 128 (one
// S buffer -- the next tile's S waits for this tile's P.V -- two-pass softmax over TMEM, 2 CTAs/SM).
static int fwd_bn() {
  static const int v = [] {
    const char* e = getenv("ESM_ATTN_FWD_BN");
    const int x = e ? atoi(e) : 64;
    return (x == 32 || x == 128) ? x : 64;
  }();
  return v;
}
static bool fwd_small_tiles() { return fwd_bn() == 32; }

template <int DH, int BN, int NSB>
int launch_fwd(const void* q, const void* k, const void* v, const int32_t* km, int* sched, void* o, float* lse, int B,
               int nh, int S, cudaStream_t st, const esm_dropout& drop) {
  using SH = Shape<DH, BN, NSB>;
  CUtensorMap tq, tk, tv;
  const int64_t rows = (int64_t)B * nh * S;
  int rc;
  if ((rc = head_map<DH, BM>(&tq, q, rows)) || (rc = head_map<DH, BN>(&tk, k, rows)) ||
      (rc = head_map<DH, BN>(&tv, v, rows)))
    return rc;
  const int smem = 2 * SH::Q_BYTES + 2 * SH::STAGES * SH::KV_BYTES + 1024 + 256;
  const int nitem = ((S + BM - 1) / BM) * B * nh;
  const int per_sm = fwd_ctas_per_sm<DH, BN, NSB>();  // CTAs resident per SM
  const int grid = min(nitem, per_sm * device_sm_count());
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    launch_pdl(kern, dim3(grid), dim3(kThreads), smem, st, 1, tq, tk, tv, km, sched, (__nv_bfloat16*)o, lse, S, nh,
               B * nh, drop);
  };
  switch (fwd_poly_pairs()) {
    case 0: go(fwd_kernel<DH, BN, NSB, 0>); break;
    case 2: go(fwd_kernel<DH, BN, NSB, 2>); break;
    default: go(fwd_kernel<DH, BN, NSB, 1>); break;
  }
  ESM_LAUNCH_RET();
}


// softmax warps per TMEM lane quarter of the backward: 2 (448 threads, default) or 4 (704 threads,
// ESM_ATTN_BWD_SW=4).  Measured on B200: SW = 4 is 5-6 % slower at dh 24 and 64 (0.499 vs 0.471 ms, 0.361 vs
// 0.342 ms per launch incl. Delta) -- the stage is bound by the MMA <-> softmax hand-offs, not by warps in flight.
static int bwd_softmax_warps() {
  static const int sw = [] {
    const char* e = getenv("ESM_ATTN_BWD_SW");
    return (e && atoi(e) == 4) ? 4 : 2;
  }();
  return sw;
}

template <int DH>
int launch_bwd(const void* q, const void* k, const void* v, const void* dout, const float* lse, const float* delta,
               const int32_t* km, int* sched, float* dq, void* dk, void* dv, int B, int nh, int S, cudaStream_t st,
               FusedOut fo) {
  using SH = Shape<DH, 64>;
  using BS = BwdShape<DH>;
  CUtensorMap tq, tk, tv, tdo, tdq;
  const int64_t rows = (int64_t)B * nh * S;
  int rc;
  if ((rc = head_map<DH, 64>(&tq, q, rows)) || (rc = head_map<DH, 128>(&tk, k, rows)) ||
      (rc = head_map<DH, 128>(&tv, v, rows)))
    return rc;
  PFN_encodeTiled enc = encoder();
  {  // dO is token-major [B*S, nh*DH]; box = DP columns of one head x 64 tokens
    cuuint64_t dims[2] = {(cuuint64_t)nh * DH, (cuuint64_t)B * S};
    cuuint64_t strides[1] = {(cuuint64_t)nh * DH * 2};
    cuuint32_t box[2] = {(cuuint32_t)SH::DP, 64};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = SH::ROWB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : SH::ROWB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                   : CU_TENSOR_MAP_SWIZZLE_32B;
    if (!enc || enc(&tdo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dout), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_last_error("attention bwd: dO tensor map encode failed");
      return ESM_EDRIVER;
    }
  }
  {  // fp32 dQ accumulator (fused: token-major [B*S, nh*DH]; classic: [B*nh*S, DH]); box BOXC cols x 32 rows
    const bool fused = fo.dqkv != nullptr;
    cuuint64_t dims[2] = {(cuuint64_t)(fused ? nh * DH : DH), (cuuint64_t)(fused ? (int64_t)B * S : rows)};
    cuuint64_t strides[1] = {(cuuint64_t)(fused ? nh * DH : DH) * 4};
    cuuint32_t box[2] = {(cuuint32_t)BS::BOXC, 32};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&tdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            BS::BOXC == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_last_error("attention bwd: dQ tensor map encode failed");
      return ESM_EDRIVER;
    }
  }
  const int ntile = ((S + 127) / 128) * B * nh;
  // persistent: one CTA per SM loops over key-block tiles
  const int grid = min(device_sm_count(), ntile);
  if (bwd_softmax_warps() == 2) {
    cudaFuncSetAttribute(bwd_kernel<DH, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, BS::SMEM);
    launch_pdl(bwd_kernel<DH, 2>, dim3(grid), dim3(BwdWarps<2>::THREADS), BS::SMEM, st, 1, tq, tk, tv, tdo, tdq, km,
               sched, lse, delta, dq, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, S, nh, B * nh, fo);
  } else {
    cudaFuncSetAttribute(bwd_kernel<DH, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, BS::SMEM);
    launch_pdl(bwd_kernel<DH, 4>, dim3(grid), dim3(BwdWarps<4>::THREADS), BS::SMEM, st, 1, tq, tk, tv, tdo, tdq, km,
               sched, lse, delta, dq, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, S, nh, B * nh, fo);
  }
  ESM_LAUNCH_RET();
}

}  // namespace fa

int attn_prepare_tc(const int32_t* km, int* sched, int B, int S, cudaStream_t st) {
  fa::mask_info_kernel<<<B, 256, 0, st>>>(km, S, sched);
  ESM_LAUNCH_RET();
}

int attn_bwd_tc(const void* q, const void* k, const void* v, const void* dout, const float* lse, const float* delta,
                const int32_t* km, int* sched, float* dq, void* dk, void* dv, int B, int nh, int S, int dh,
                cudaStream_t st, void* dqkv, float* col_sum, const float* cos_t, const float* sin_t,
                const esm_dropout* drop) {
  ESM_CHECK_ARG(S % 4 == 0, "attention bwd (tcgen05): S %% 4 == 0 required");
  const esm_dropout dr = (drop && drop->threshold != 0u) ? *drop : esm_dropout{nullptr, 0u, 0u, 1.f};
  ESM_CHECK_ARG(dr.threshold == 0u || dr.seed != nullptr, "attention dropout: needs a seed");
  fa::FusedOut fo{(__nv_bfloat16*)dqkv, col_sum, cos_t, sin_t, nh * dh, dr};
  switch (dh) {
    case 16: return fa::launch_bwd<16>(q, k, v, dout, lse, delta, km, sched, dq, dk, dv, B, nh, S, st, fo);
    case 24: return fa::launch_bwd<24>(q, k, v, dout, lse, delta, km, sched, dq, dk, dv, B, nh, S, st, fo);
    case 32: return fa::launch_bwd<32>(q, k, v, dout, lse, delta, km, sched, dq, dk, dv, B, nh, S, st, fo);
    case 64: return fa::launch_bwd<64>(q, k, v, dout, lse, delta, km, sched, dq, dk, dv, B, nh, S, st, fo);
    default: set_last_error("attention: head dim %d unsupported", dh); return ESM_ENOTSUP;
  }
}

int attn_fwd_tc(const void* q, const void* k, const void* v, const int32_t* km, int* sched, void* o, float* lse,
                int B, int nh, int S, int dh, cudaStream_t st, const esm_dropout* drop) {
  ESM_CHECK_ARG(((uintptr_t)q & 15) == 0 && ((uintptr_t)k & 15) == 0 && ((uintptr_t)v & 15) == 0,
                "attention: q/k/v must be 16B aligned");
  const esm_dropout dr = (drop && drop->threshold != 0u) ? *drop : esm_dropout{nullptr, 0u, 0u, 1.f};
  ESM_CHECK_ARG(dr.threshold == 0u || (dr.seed != nullptr && fa::fwd_bn() != 128),
                "attention dropout: needs a seed and the 64-key forward tiles");
  // two S buffers per CTA, 2 CTAs/SM (a single-buffer 3-CTA/SM variant measured equal at dh 24, slower at 64)
  switch (dh) {
    case 16:
      return fa::fwd_small_tiles() ? fa::launch_fwd<16, 32, 2>(q, k, v, km, sched, o, lse, B, nh, S, st, dr)
                                   : fa::launch_fwd<16, 64, 2>(q, k, v, km, sched, o, lse, B, nh, S, st, dr);
    case 24:
      if (fa::fwd_bn() == 128) return fa::launch_fwd<24, 128, 1>(q, k, v, km, sched, o, lse, B, nh, S, st, dr);
      return fa::fwd_small_tiles() ? fa::launch_fwd<24, 32, 2>(q, k, v, km, sched, o, lse, B, nh, S, st, dr)
                                   : fa::launch_fwd<24, 64, 2>(q, k, v, km, sched, o, lse, B, nh, S, st, dr);
    case 32:
      return fa::fwd_small_tiles() ? fa::launch_fwd<32, 32, 2>(q, k, v, km, sched, o, lse, B, nh, S, st, dr)
                                   : fa::launch_fwd<32, 64, 2>(q, k, v, km, sched, o, lse, B, nh, S, st, dr);
    case 64:
      return fa::fwd_bn() == 128 ? fa::launch_fwd<64, 128, 1>(q, k, v, km, sched, o, lse, B, nh, S, st, dr)
                                 : fa::launch_fwd<64, 64, 2>(q, k, v, km, sched, o, lse, B, nh, S, st, dr);
    default: set_last_error("attention: head dim %d unsupported", dh); return ESM_ENOTSUP;
  }
}

}  // namespace esm

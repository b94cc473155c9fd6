// Attention C-ABI entry points (esm_attn_fwd / esm_attn_bwd / esm_attn_bwd_qkv) for ESM-2 (non-causal,
// key-padding mask, scaling = 1 because q is pre-scaled before RoPE: HF:modeling_esm.py:257-282, 313, 341-344).
//
// bf16 production path: the persistent tcgen05/TMEM kernels in attention_tc.cu; this file holds the
//       helpers around them (Delta / log2-LSE, dQ finalisation with RoPE^T) and the legacy FA2-style
//       mma.sync.m16n8k16 kernels kept as the baseline (ESM_ATTN_LEGACY=1): cp.async double buffering,
//       ldmatrix(.trans) fragments, exp2 online softmax, dQ via fp32 vector reductions.
// fp32: SIMT reference-precision kernels (parity mode).
#include <cstdlib>

#include "common.cuh"

namespace esm {
namespace attn {

constexpr float L2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x2(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// smem pitch (elements) such that 8 consecutive rows of 16 B hit distinct bank groups
__host__ __device__ constexpr int pitch_for(int cols) {
  return ((cols / 8) % 2 == 1) ? cols : cols + 8;
}

// Copy a [64 x DH] bf16 tile (rows at stride `ld` elements) into smem with pitch P.
template <int DH, int P>
__device__ __forceinline__ void load_tile(__nv_bfloat16* s, const __nv_bfloat16* g, int64_t ld, int row0,
                                          int nrows_valid) {
  constexpr int CH = DH / 8;
  for (int i = threadIdx.x; i < 64 * CH; i += blockDim.x) {
    const int r = i / CH, c = (i % CH) * 8;
    const bool ok = (row0 + r) < nrows_valid;
    const __nv_bfloat16* src = g + (int64_t)(ok ? row0 + r : 0) * ld + c;
    cp_async16(s + r * P + c, src, ok);
  }
}
template <int DH, int KD, int P>
__device__ __forceinline__ void zero_pad(__nv_bfloat16* s) {
  if constexpr (KD > DH) {
    for (int i = threadIdx.x; i < 64 * (KD - DH); i += blockDim.x) {
      const int r = i / (KD - DH), c = DH + i % (KD - DH);
      s[r * P + c] = __float2bfloat16_rn(0.f);
    }
  }
}

// ---------------------------------------------------------------------------- forward
template <int DH>
__global__ void __launch_bounds__(128) fwd_bf16_kernel(const __nv_bfloat16* __restrict__ Q,
                                                       const __nv_bfloat16* __restrict__ K,
                                                       const __nv_bfloat16* __restrict__ V,
                                                       const int32_t* __restrict__ key_mask,
                                                       __nv_bfloat16* __restrict__ O, float* __restrict__ LSE, int S,
                                                       int nh) {
  constexpr int KD = (DH + 15) / 16 * 16;
  constexpr int KP = pitch_for(KD);
  constexpr int VP = pitch_for(DH);
  constexpr int KS = KD / 16;  // k16 steps for QK^T
  constexpr int ND = DH / 8;   // n8 blocks over d for PV
  __shared__ __align__(16) __nv_bfloat16 sQ[64 * KP];
  __shared__ __align__(16) __nv_bfloat16 sK[2][64 * KP];
  __shared__ __align__(16) __nv_bfloat16 sV[2][64 * VP];
  __shared__ float sMask[2][64];

  const int bh = blockIdx.y, b = bh / nh, h = bh % nh;
  const int q0 = blockIdx.x * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)bh * S * DH;
  const int H = nh * DH;

  zero_pad<DH, KD, KP>(sQ);
  zero_pad<DH, KD, KP>(sK[0]);
  zero_pad<DH, KD, KP>(sK[1]);
  load_tile<DH, KP>(sQ, Q + base, DH, q0, S);
  const int ntiles = (S + 63) / 64;
  auto issue = [&](int j, int buf) {
    load_tile<DH, KP>(sK[buf], K + base, DH, j * 64, S);
    load_tile<DH, VP>(sV[buf], V + base, DH, j * 64, S);
    if (threadIdx.x < 64) {
      const int kk = j * 64 + threadIdx.x;
      sMask[buf][threadIdx.x] = (kk < S && (key_mask == nullptr || key_mask[(int64_t)b * S + kk] != 0)) ? 0.f : -INFINITY;
    }
  };
  issue(0, 0);
  cp_commit();

  uint32_t qa[KS][4];
  float o[ND][4];
#pragma unroll
  for (int i = 0; i < ND; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

  for (int j = 0; j < ntiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < ntiles) {
      issue(j + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = ks * 16 + (lane >> 4) * 8;
        ldsm_x4(qa[ks], sQ + r * KP + c);
      }
    }
    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) s[nb][0] = s[nb][1] = s[nb][2] = s[nb][3] = 0.f;
#pragma unroll
    for (int nb = 0; nb < 8; nb += 2) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        uint32_t kb[4];
        const int r = nb * 8 + (lane & 7) + (lane >> 4) * 8;
        const int c = ks * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(kb, sK[buf] + r * KP + c);
        mma16816(s[nb], qa[ks], kb[0], kb[1]);
        mma16816(s[nb + 1], qa[ks], kb[2], kb[3]);
      }
    }
    // mask + online softmax (rows lane/4 and lane/4+8)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const int c = nb * 8 + 2 * (lane & 3);
      const float m0 = sMask[buf][c], m1 = sMask[buf][c + 1];
      s[nb][0] = s[nb][0] * L2E + m0;
      s[nb][1] = s[nb][1] * L2E + m1;
      s[nb][2] = s[nb][2] * L2E + m0;
      s[nb][3] = s[nb][3] * L2E + m1;
      mx[0] = fmaxf(mx[0], fmaxf(s[nb][0], s[nb][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nb][2], s[nb][3]));
    }
    float scale[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mnew = fmaxf(m_r[r], mx[r]);
      const float msafe = mnew == -INFINITY ? 0.f : mnew;
      scale[r] = exp2f(m_r[r] - msafe);
      m_r[r] = mnew;
      mx[r] = msafe;
    }
    float rs[2] = {0.f, 0.f};
    uint32_t pa[4][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const float p0 = exp2f(s[nb][0] - mx[0]), p1 = exp2f(s[nb][1] - mx[0]);
      const float p2 = exp2f(s[nb][2] - mx[1]), p3 = exp2f(s[nb][3] - mx[1]);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pa[nb >> 1][(nb & 1) * 2 + 0] = pack_bf16(p0, p1);
      pa[nb >> 1][(nb & 1) * 2 + 1] = pack_bf16(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      l_r[r] = l_r[r] * scale[r] + rs[r];
    }
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      o[i][0] *= scale[0];
      o[i][1] *= scale[0];
      o[i][2] *= scale[1];
      o[i][3] *= scale[1];
    }
    // O += P V  (k = 64 keys in 4 k16 steps; n = d)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // A fragment order {a0,a1,a2,a3} = {rows0-7 k0-7, rows8-15 k0-7, rows0-7 k8-15, rows8-15 k8-15}
      const uint32_t a[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
#pragma unroll
      for (int nd = 0; nd < ND; nd += 2) {
        if (nd + 1 < ND) {
          uint32_t vb[4];
          const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int c = nd * 8 + (lane >> 4) * 8;
          ldsm_x4_t(vb, sV[buf] + r * VP + c);
          mma16816(o[nd], a, vb[0], vb[1]);
          mma16816(o[nd + 1], a, vb[2], vb[3]);
        } else {
          uint32_t b0, b1;
          const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          ldsm_x2_t(b0, b1, sV[buf] + r * VP + nd * 8);
          mma16816(o[nd], a, b0, b1);
        }
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qrow = q0 + warp * 16 + (lane >> 2) + r * 8;
    if (qrow < S) {
      const float inv = l_r[r] > 0.f ? 1.f / l_r[r] : 0.f;
      __nv_bfloat16* dst = O + ((int64_t)b * S + qrow) * H + h * DH;
#pragma unroll
      for (int nd = 0; nd < ND; ++nd) {
        const int c = nd * 8 + 2 * (lane & 3);
        *reinterpret_cast<uint32_t*>(dst + c) = pack_bf16(o[nd][2 * r] * inv, o[nd][2 * r + 1] * inv);
      }
      if ((lane & 3) == 0) {
        const float m = m_r[r] == -INFINITY ? 0.f : m_r[r];
        LSE[(int64_t)bh * S + qrow] = (m + log2f(l_r[r])) / L2E;
      }
    }
  }
}

// ---------------------------------------------------------------------------- backward
// delta[q] = sum_d dO[q,d] * O[q,d]; one thread per (token, head): consecutive threads read consecutive
// heads of a token, i.e. contiguous 16-byte vectors of the token-major [T, H] rows.
template <typename T>
__global__ void delta_kernel(const T* __restrict__ O, const T* __restrict__ dO, float* __restrict__ delta,
                             const float* __restrict__ lse, float* __restrict__ lse2, int64_t T_, int S, int nh,
                             int dh) {
  constexpr int VEC = vec16<T>::N;
  const int H = nh * dh;
  const int64_t total = T_ * nh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / nh;
    const int h = (int)(i - t * nh);
    const T* o = O + t * H + h * dh;
    const T* g = dO + t * H + h * dh;
    float acc = 0.f;
    for (int d = 0; d < dh; d += VEC) {
      float a[VEC], c[VEC];
      load_vec(o + d, a);
      load_vec(g + d, c);
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc += a[e] * c[e];
    }
    const int64_t b = t / S, s = t % S;
    const int64_t idx = (b * nh + h) * S + s;
    delta[idx] = acc;
    if (lse2) lse2[idx] = -lse[idx] * L2E;  // negated log2-domain LSE (an FFMA2 addend in the tcgen05 backward)
  }
}

template <int DH>
__global__ void __launch_bounds__(128) bwd_bf16_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
    const __nv_bfloat16* __restrict__ dO, const float* __restrict__ LSE, const float* __restrict__ Delta,
    const int32_t* __restrict__ key_mask, float* __restrict__ dQ, __nv_bfloat16* __restrict__ dK,
    __nv_bfloat16* __restrict__ dV, int S, int nh) {
  constexpr int KD = (DH + 15) / 16 * 16;
  constexpr int KP = pitch_for(KD);
  constexpr int KS = KD / 16;
  constexpr int ND = DH / 8;
  constexpr int SP = 72;  // dS^T pitch (64 + 8)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sV = sK + 64 * KP;
  __nv_bfloat16* sQ = sV + 64 * KP;       // [2][64*KP]
  __nv_bfloat16* sdO = sQ + 2 * 64 * KP;  // [2][64*KP]
  __nv_bfloat16* sdS = sdO + 2 * 64 * KP; // [64 keys][SP]
  float* sL = reinterpret_cast<float*>(sdS + 64 * SP);  // [2][64]
  float* sD = sL + 128;                                 // [2][64]

  const int bh = blockIdx.y, b = bh / nh, h = bh % nh;
  const int k0 = blockIdx.x * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)bh * S * DH;
  const int H = nh * DH;

  zero_pad<DH, KD, KP>(sK);
  zero_pad<DH, KD, KP>(sV);
  zero_pad<DH, KD, KP>(sQ);
  zero_pad<DH, KD, KP>(sQ + 64 * KP);
  zero_pad<DH, KD, KP>(sdO);
  zero_pad<DH, KD, KP>(sdO + 64 * KP);
  load_tile<DH, KP>(sK, K + base, DH, k0, S);
  load_tile<DH, KP>(sV, V + base, DH, k0, S);
  const int nq = (S + 63) / 64;
  const __nv_bfloat16* dOb = dO + (int64_t)b * S * H + h * DH;
  auto issue = [&](int i, int buf) {
    load_tile<DH, KP>(sQ + buf * 64 * KP, Q + base, DH, i * 64, S);
    load_tile<DH, KP>(sdO + buf * 64 * KP, dOb, H, i * 64, S);
    if (threadIdx.x < 64) {
      const int qq = i * 64 + threadIdx.x;
      sL[buf * 64 + threadIdx.x] = qq < S ? LSE[(int64_t)bh * S + qq] * L2E : INFINITY;
      sD[buf * 64 + threadIdx.x] = qq < S ? Delta[(int64_t)bh * S + qq] : 0.f;
    }
  };
  issue(0, 0);
  cp_commit();

  // my 16 keys: validity of rows lane/4 and lane/4+8
  bool kval[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int kk = k0 + warp * 16 + (lane >> 2) + r * 8;
    kval[r] = kk < S && (key_mask == nullptr || key_mask[(int64_t)b * S + kk] != 0);
  }
  uint32_t ka[KS][4], va[KS][4];
  float dk[ND][4], dv[ND][4];
#pragma unroll
  for (int i = 0; i < ND; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

  for (int i = 0; i < nq; ++i) {
    const int buf = i & 1;
    if (i + 1 < nq) {
      issue(i + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __nv_bfloat16* q_s = sQ + buf * 64 * KP;
    const __nv_bfloat16* do_s = sdO + buf * 64 * KP;
    const float* l_s = sL + buf * 64;
    const float* d_s = sD + buf * 64;
    if (i == 0) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = ks * 16 + (lane >> 4) * 8;
        ldsm_x4(ka[ks], sK + r * KP + c);
        ldsm_x4(va[ks], sV + r * KP + c);
      }
    }
    // S^T = K Q^T and dP^T = V dO^T : 16 keys x 64 queries
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[nb][e] = dpt[nb][e] = 0.f;
#pragma unroll
    for (int nb = 0; nb < 8; nb += 2) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int r = nb * 8 + (lane & 7) + (lane >> 4) * 8;
        const int c = ks * 16 + ((lane >> 3) & 1) * 8;
        uint32_t qb[4], ob[4];
        ldsm_x4(qb, q_s + r * KP + c);
        ldsm_x4(ob, do_s + r * KP + c);
        mma16816(st[nb], ka[ks], qb[0], qb[1]);
        mma16816(st[nb + 1], ka[ks], qb[2], qb[3]);
        mma16816(dpt[nb], va[ks], ob[0], ob[1]);
        mma16816(dpt[nb + 1], va[ks], ob[2], ob[3]);
      }
    }
    // P^T, dS^T
    uint32_t pa[4][4], da[4][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const int c = nb * 8 + 2 * (lane & 3);
      const float l0 = l_s[c], l1 = l_s[c + 1];
      const float d0 = d_s[c], d1 = d_s[c + 1];
      float p[4];
      p[0] = kval[0] ? exp2f(st[nb][0] * L2E - l0) : 0.f;
      p[1] = kval[0] ? exp2f(st[nb][1] * L2E - l1) : 0.f;
      p[2] = kval[1] ? exp2f(st[nb][2] * L2E - l0) : 0.f;
      p[3] = kval[1] ? exp2f(st[nb][3] * L2E - l1) : 0.f;
      const float ds0 = p[0] * (dpt[nb][0] - d0), ds1 = p[1] * (dpt[nb][1] - d1);
      const float ds2 = p[2] * (dpt[nb][2] - d0), ds3 = p[3] * (dpt[nb][3] - d1);
      pa[nb >> 1][(nb & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
      pa[nb >> 1][(nb & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
      da[nb >> 1][(nb & 1) * 2 + 0] = pack_bf16(ds0, ds1);
      da[nb >> 1][(nb & 1) * 2 + 1] = pack_bf16(ds2, ds3);
      // stash dS^T (keys x queries) for the dQ product
      const int kr = warp * 16 + (lane >> 2);
      *reinterpret_cast<uint32_t*>(sdS + kr * SP + c) = da[nb >> 1][(nb & 1) * 2 + 0];
      *reinterpret_cast<uint32_t*>(sdS + (kr + 8) * SP + c) = da[nb >> 1][(nb & 1) * 2 + 1];
    }
    // dV += P^T dO ; dK += dS^T Q   (k = 64 queries, n = d)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t ap[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
      const uint32_t ad[4] = {da[kk][0], da[kk][1], da[kk][2], da[kk][3]};
      const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int nd = 0; nd < ND; nd += 2) {
        if (nd + 1 < ND) {
          const int c = nd * 8 + (lane >> 4) * 8;
          uint32_t ob[4], qb[4];
          ldsm_x4_t(ob, do_s + r * KP + c);
          ldsm_x4_t(qb, q_s + r * KP + c);
          mma16816(dv[nd], ap, ob[0], ob[1]);
          mma16816(dv[nd + 1], ap, ob[2], ob[3]);
          mma16816(dk[nd], ad, qb[0], qb[1]);
          mma16816(dk[nd + 1], ad, qb[2], qb[3]);
        } else {
          uint32_t o0, o1, q0_, q1_;
          ldsm_x2_t(o0, o1, do_s + r * KP + nd * 8);
          ldsm_x2_t(q0_, q1_, q_s + r * KP + nd * 8);
          mma16816(dv[nd], ap, o0, o1);
          mma16816(dk[nd], ad, q0_, q1_);
        }
      }
    }
    __syncthreads();  // sdS complete
    // dQ[16 queries of this warp] = dS K : A = dS (from dS^T via ldmatrix.trans), B = K (trans)
    {
      float dq[ND][4];
#pragma unroll
      for (int nd = 0; nd < ND; ++nd) dq[nd][0] = dq[nd][1] = dq[nd][2] = dq[nd][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t a[4];
        {
          // matrices: (q0-7,k0-7) (q8-15,k0-7) (q0-7,k8-15) (q8-15,k8-15); rows of sdS are keys
          const int key = kk * 16 + (lane & 7) + (lane >> 4) * 8;
          const int qc = warp * 16 + ((lane >> 3) & 1) * 8;
          ldsm_x4_t(a, sdS + key * SP + qc);
        }
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int nd = 0; nd < ND; nd += 2) {
          if (nd + 1 < ND) {
            uint32_t kb[4];
            ldsm_x4_t(kb, sK + r * KP + nd * 8 + (lane >> 4) * 8);
            mma16816(dq[nd], a, kb[0], kb[1]);
            mma16816(dq[nd + 1], a, kb[2], kb[3]);
          } else {
            uint32_t b0, b1;
            ldsm_x2_t(b0, b1, sK + r * KP + nd * 8);
            mma16816(dq[nd], a, b0, b1);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int qq = i * 64 + warp * 16 + (lane >> 2) + r * 8;
        if (qq < S) {
          float* dst = dQ + base + (int64_t)qq * DH;
#pragma unroll
          for (int nd = 0; nd < ND; ++nd) {
            const int c = nd * 8 + 2 * (lane & 3);
            asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dst + c), "f"(dq[nd][2 * r]),
                         "f"(dq[nd][2 * r + 1])
                         : "memory");
          }
        }
      }
    }
    __syncthreads();  // before the next prefetch overwrites buffers / sdS
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int kk = k0 + warp * 16 + (lane >> 2) + r * 8;
    if (kk < S) {
#pragma unroll
      for (int nd = 0; nd < ND; ++nd) {
        const int c = nd * 8 + 2 * (lane & 3);
        *reinterpret_cast<uint32_t*>(dK + base + (int64_t)kk * DH + c) = pack_bf16(dk[nd][2 * r], dk[nd][2 * r + 1]);
        *reinterpret_cast<uint32_t*>(dV + base + (int64_t)kk * DH + c) = pack_bf16(dv[nd][2 * r], dv[nd][2 * r + 1]);
      }
    }
  }
}

template <int DH>
constexpr int bwd_smem_bytes() {
  constexpr int KD = (DH + 15) / 16 * 16;
  constexpr int KP = pitch_for(KD);
  return (6 * 64 * KP + 64 * 72) * 2 + 4 * 64 * 4;
}

// ---------------------------------------------------------------------------- fp32 SIMT
constexpr int MAXD = 64;

__global__ void __launch_bounds__(64) fwd_f32_kernel(const float* __restrict__ Q, const float* __restrict__ K,
                                                     const float* __restrict__ V, const int32_t* __restrict__ km,
                                                     float* __restrict__ O, float* __restrict__ LSE, int S, int nh,
                                                     int dh) {
  __shared__ float sK[64][MAXD + 1], sV[64][MAXD + 1];
  __shared__ bool sM[64];
  const int bh = blockIdx.y, b = bh / nh, h = bh % nh;
  const int qi = blockIdx.x * 64 + threadIdx.x;
  const int64_t base = (int64_t)bh * S * dh;
  float q[MAXD], o[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    q[d] = (qi < S && d < dh) ? Q[base + (int64_t)qi * dh + d] : 0.f;
    o[d] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int k0 = 0; k0 < S; k0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * dh; i += 64) {
      const int r = i / dh, d = i % dh;
      const bool ok = k0 + r < S;
      sK[r][d] = ok ? K[base + (int64_t)(k0 + r) * dh + d] : 0.f;
      sV[r][d] = ok ? V[base + (int64_t)(k0 + r) * dh + d] : 0.f;
    }
    {
      const int kk = k0 + threadIdx.x;
      sM[threadIdx.x] = kk < S && (km == nullptr || km[(int64_t)b * S + kk] != 0);
    }
    __syncthreads();
    for (int j = 0; j < 64; ++j) {
      if (!sM[j]) continue;
      float s = 0.f;
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) s += q[d] * sK[j][d];
      const float mn = fmaxf(m, s);
      const float sc = expf(m - mn), p = expf(s - mn);
      l = l * sc + p;
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) o[d] = o[d] * sc + p * sV[j][d];
      m = mn;
    }
  }
  if (qi < S) {
    const int H = nh * dh;
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < dh) O[((int64_t)b * S + qi) * H + h * dh + d] = o[d] * inv;
    LSE[(int64_t)bh * S + qi] = m + logf(l);
  }
}

// dQ (per query thread) and dK/dV (per key thread), recomputing P from LSE
__global__ void __launch_bounds__(64) bwd_dq_f32_kernel(const float* __restrict__ Q, const float* __restrict__ K,
                                                        const float* __restrict__ V, const float* __restrict__ dO,
                                                        const float* __restrict__ LSE,
                                                        const float* __restrict__ Delta,
                                                        const int32_t* __restrict__ km, float* __restrict__ dQ, int S,
                                                        int nh, int dh) {
  __shared__ float sK[64][MAXD + 1], sV[64][MAXD + 1];
  __shared__ bool sM[64];
  const int bh = blockIdx.y, b = bh / nh, h = bh % nh;
  const int qi = blockIdx.x * 64 + threadIdx.x;
  const int64_t base = (int64_t)bh * S * dh;
  const int H = nh * dh;
  float q[MAXD], go[MAXD], dq[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    const bool ok = qi < S && d < dh;
    q[d] = ok ? Q[base + (int64_t)qi * dh + d] : 0.f;
    go[d] = ok ? dO[((int64_t)b * S + qi) * H + h * dh + d] : 0.f;
    dq[d] = 0.f;
  }
  const float lse = qi < S ? LSE[(int64_t)bh * S + qi] : 0.f;
  const float delta = qi < S ? Delta[(int64_t)bh * S + qi] : 0.f;
  for (int k0 = 0; k0 < S; k0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * dh; i += 64) {
      const int r = i / dh, d = i % dh;
      const bool ok = k0 + r < S;
      sK[r][d] = ok ? K[base + (int64_t)(k0 + r) * dh + d] : 0.f;
      sV[r][d] = ok ? V[base + (int64_t)(k0 + r) * dh + d] : 0.f;
    }
    {
      const int kk = k0 + threadIdx.x;
      sM[threadIdx.x] = kk < S && (km == nullptr || km[(int64_t)b * S + kk] != 0);
    }
    __syncthreads();
    for (int j = 0; j < 64; ++j) {
      if (!sM[j]) continue;
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) {
          s += q[d] * sK[j][d];
          dp += go[d] * sV[j][d];
        }
      const float p = expf(s - lse);
      const float ds = p * (dp - delta);
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) dq[d] += ds * sK[j][d];
    }
  }
  if (qi < S)
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < dh) dQ[base + (int64_t)qi * dh + d] = dq[d];
}

__global__ void __launch_bounds__(64) bwd_dkv_f32_kernel(const float* __restrict__ Q, const float* __restrict__ K,
                                                         const float* __restrict__ V, const float* __restrict__ dO,
                                                         const float* __restrict__ LSE,
                                                         const float* __restrict__ Delta,
                                                         const int32_t* __restrict__ km, float* __restrict__ dK,
                                                         float* __restrict__ dV, int S, int nh, int dh) {
  __shared__ float sQ[64][MAXD + 1], sO[64][MAXD + 1];
  __shared__ float sL[64], sD[64];
  const int bh = blockIdx.y, b = bh / nh, h = bh % nh;
  const int ki = blockIdx.x * 64 + threadIdx.x;
  const int64_t base = (int64_t)bh * S * dh;
  const int H = nh * dh;
  const bool kval = ki < S && (km == nullptr || km[(int64_t)b * S + ki] != 0);
  float k[MAXD], v[MAXD], dk[MAXD], dv[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    const bool ok = ki < S && d < dh;
    k[d] = ok ? K[base + (int64_t)ki * dh + d] : 0.f;
    v[d] = ok ? V[base + (int64_t)ki * dh + d] : 0.f;
    dk[d] = dv[d] = 0.f;
  }
  for (int q0 = 0; q0 < S; q0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * dh; i += 64) {
      const int r = i / dh, d = i % dh;
      const bool ok = q0 + r < S;
      sQ[r][d] = ok ? Q[base + (int64_t)(q0 + r) * dh + d] : 0.f;
      sO[r][d] = ok ? dO[((int64_t)b * S + q0 + r) * H + h * dh + d] : 0.f;
    }
    {
      const int qq = q0 + threadIdx.x;
      sL[threadIdx.x] = qq < S ? LSE[(int64_t)bh * S + qq] : INFINITY;
      sD[threadIdx.x] = qq < S ? Delta[(int64_t)bh * S + qq] : 0.f;
    }
    __syncthreads();
    if (!kval) continue;
    for (int j = 0; j < 64; ++j) {
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) {
          s += sQ[j][d] * k[d];
          dp += sO[j][d] * v[d];
        }
      const float p = expf(s - sL[j]);
      const float ds = p * (dp - sD[j]);
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) {
          dv[d] += p * sO[j][d];
          dk[d] += ds * sQ[j][d];
        }
    }
  }
  if (ki < S)
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < dh) {
        dK[base + (int64_t)ki * dh + d] = dk[d];
        dV[base + (int64_t)ki * dh + d] = dv[d];
      }
}

// dq (fp32, token-major [T, H]) -> dqkv[:, 0:H] with RoPE^T and q_scale; col_sum[0:H] += column sums.
// RoPE^T + q-scale of the token-major fp32 dQ accumulator -> the q part of dqkv (bf16) + q bias-grad column
// sums.  Thread = two adjacent rotation pairs (vector accesses), RU tokens in flight per iteration.
__global__ void __launch_bounds__(64) dq_finalize_kernel(const float* __restrict__ dq, __nv_bfloat16* __restrict__ dqkv,
                                                         float* __restrict__ csum, const float* __restrict__ cs,
                                                         const float* __restrict__ sn, int64_t T_, int S, int nh,
                                                         int dh, float qs, int rows_per_block) {
  constexpr int RU = 4;
  const int half = dh >> 1;
  const int H = nh * dh;
  const int unit = blockIdx.x * blockDim.x + threadIdx.x;
  if (unit >= nh * (half >> 1)) return;
  const int h = unit / (half >> 1), j = (unit % (half >> 1)) * 2;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(T_, r0 + rows_per_block);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  for (int64_t t0 = r0; t0 < r1; t0 += RU) {
    float2 g0[RU], g1[RU], c[RU], sv[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int64_t t = min(t0 + u, r1 - 1);
      const int s = (int)(t % S);
      c[u] = __ldg(reinterpret_cast<const float2*>(cs + (int64_t)s * half + j));
      sv[u] = __ldg(reinterpret_cast<const float2*>(sn + (int64_t)s * half + j));
      g0[u] = *reinterpret_cast<const float2*>(dq + t * H + h * dh + j);
      g1[u] = *reinterpret_cast<const float2*>(dq + t * H + h * dh + j + half);
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      if (t0 + u >= r1) break;
      const float qa0 = (g0[u].x * c[u].x + g1[u].x * sv[u].x) * qs, qb0 = (g0[u].y * c[u].y + g1[u].y * sv[u].y) * qs;
      const float qa1 = (g1[u].x * c[u].x - g0[u].x * sv[u].x) * qs, qb1 = (g1[u].y * c[u].y - g0[u].y * sv[u].y) * qs;
      __nv_bfloat16* row = dqkv + (t0 + u) * 3 * H + h * dh;
      *reinterpret_cast<__nv_bfloat162*>(row + j) = __floats2bfloat162_rn(qa0, qb0);
      *reinterpret_cast<__nv_bfloat162*>(row + j + half) = __floats2bfloat162_rn(qa1, qb1);
      a0 += qa0; a1 += qb0; a2 += qa1; a3 += qb1;
    }
  }
  if (csum) {
    atomicAdd(csum + h * dh + j, a0);
    atomicAdd(csum + h * dh + j + 1, a1);
    atomicAdd(csum + h * dh + j + half, a2);
    atomicAdd(csum + h * dh + j + half + 1, a3);
  }
}

}  // namespace attn
}  // namespace esm

namespace esm {
int attn_fwd_tc(const void* q, const void* k, const void* v, const int32_t* km, void* o, float* lse, int B, int nh,
                int S, int dh, cudaStream_t st);
int attn_bwd_tc(const void* q, const void* k, const void* v, const void* dout, const float* lse2, const float* delta,
                const int32_t* km, float* dq, void* dk, void* dv, int B, int nh, int S, int dh, cudaStream_t st,
                void* dqkv, float* col_sum, const float* cos_t, const float* sin_t);
static int legacy_attention() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ESM_ATTN_LEGACY");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}
}  // namespace esm

using namespace esm;

extern "C" int esm_attn_fwd(int dtype, const void* q, const void* k, const void* v, const int32_t* key_mask, void* o,
                            float* lse, int B, int nh, int S, int dh, esm_stream_t stream) {
  ESM_CHECK_ARG(q && k && v && o && lse && B > 0 && nh > 0 && S > 0, "esm_attn_fwd: bad args");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid((S + 63) / 64, B * nh);
  if (dtype == ESM_BF16 && !legacy_attention()) {
    return attn_fwd_tc(q, k, v, key_mask, o, lse, B, nh, S, dh, st);
  }
  if (dtype == ESM_BF16) {
    auto* Q = (const __nv_bfloat16*)q;
    auto* K = (const __nv_bfloat16*)k;
    auto* V = (const __nv_bfloat16*)v;
    auto* O = (__nv_bfloat16*)o;
    switch (dh) {
      case 16: attn::fwd_bf16_kernel<16><<<grid, 128, 0, st>>>(Q, K, V, key_mask, O, lse, S, nh); break;
      case 24: attn::fwd_bf16_kernel<24><<<grid, 128, 0, st>>>(Q, K, V, key_mask, O, lse, S, nh); break;
      case 32: attn::fwd_bf16_kernel<32><<<grid, 128, 0, st>>>(Q, K, V, key_mask, O, lse, S, nh); break;
      case 64: attn::fwd_bf16_kernel<64><<<grid, 128, 0, st>>>(Q, K, V, key_mask, O, lse, S, nh); break;
      default: esm::set_last_error("esm_attn_fwd: head dim %d unsupported (16/24/32/64)", dh); return ESM_ENOTSUP;
    }
  } else {
    ESM_CHECK_ARG(dh <= attn::MAXD, "esm_attn_fwd: dh <= 64");
    attn::fwd_f32_kernel<<<grid, 64, 0, st>>>((const float*)q, (const float*)k, (const float*)v, key_mask, (float*)o,
                                              lse, S, nh, dh);
  }
  ESM_LAUNCH_RET();
}

extern "C" int esm_attn_bwd(int dtype, const void* q, const void* k, const void* v, const void* o, const void* dout,
                            const float* lse, const int32_t* key_mask, float* delta, float* dq, void* dk, void* dv,
                            int B, int nh, int S, int dh, esm_stream_t stream) {
  ESM_CHECK_ARG(q && k && v && o && dout && lse && delta && dq && dk && dv, "esm_attn_bwd: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t T_ = (int64_t)B * S;
  dim3 grid((S + 63) / 64, B * nh);
  int dgrid = (int)((T_ * nh + 255) / 256);
  if (dgrid > 148 * 32) dgrid = 148 * 32;
  if (dtype == ESM_BF16) {
    const bool tc = !legacy_attention() && S % 4 == 0;
    float* lse2 = delta + T_ * nh;  // workspace [2, B, nh, S]: Delta then log2-domain LSE
    attn::delta_kernel<__nv_bfloat16><<<dgrid, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout,
                                                             delta, lse, tc ? lse2 : nullptr, T_, S, nh, dh);
    cudaMemsetAsync(dq, 0, sizeof(float) * T_ * nh * dh, st);
    if (tc) {
      const int rc = attn_bwd_tc(q, k, v, dout, lse2, delta, key_mask, dq, dk, dv, B, nh, S, dh, st, nullptr, nullptr,
                                 nullptr, nullptr);
      if (rc) return rc;
      ESM_LAUNCH_RET();
    }
    auto* Q = (const __nv_bfloat16*)q;
    auto* K = (const __nv_bfloat16*)k;
    auto* V = (const __nv_bfloat16*)v;
    auto* dO = (const __nv_bfloat16*)dout;
    auto* dK = (__nv_bfloat16*)dk;
    auto* dV = (__nv_bfloat16*)dv;
#define BWD(D)                                                                                      \
  {                                                                                                 \
    constexpr int smem = attn::bwd_smem_bytes<D>();                                                 \
    cudaFuncSetAttribute(attn::bwd_bf16_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    attn::bwd_bf16_kernel<D><<<grid, 128, smem, st>>>(Q, K, V, dO, lse, delta, key_mask, dq, dK, dV, S, nh); \
  }
    switch (dh) {
      case 16: BWD(16); break;
      case 24: BWD(24); break;
      case 32: BWD(32); break;
      case 64: BWD(64); break;
      default: esm::set_last_error("esm_attn_bwd: head dim %d unsupported", dh); return ESM_ENOTSUP;
    }
#undef BWD
  } else {
    ESM_CHECK_ARG(dh <= attn::MAXD, "esm_attn_bwd: dh <= 64");
    attn::delta_kernel<float><<<dgrid, 256, 0, st>>>((const float*)o, (const float*)dout, delta, lse, nullptr, T_, S, nh,
                                                     dh);
    attn::bwd_dq_f32_kernel<<<grid, 64, 0, st>>>((const float*)q, (const float*)k, (const float*)v,
                                                 (const float*)dout, lse, delta, key_mask, dq, S, nh, dh);
    attn::bwd_dkv_f32_kernel<<<grid, 64, 0, st>>>((const float*)q, (const float*)k, (const float*)v,
                                                  (const float*)dout, lse, delta, key_mask, (float*)dk, (float*)dv, S,
                                                  nh, dh);
  }
  ESM_LAUNCH_RET();
}

extern "C" int esm_attn_bwd_qkv(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                const float* lse, const int32_t* key_mask, float* delta, float* dq_ws, void* dqkv,
                                float* col_sum, const float* cos_t, const float* sin_t, float q_scale, int B, int nh,
                                int S, int dh, esm_stream_t stream) {
  ESM_CHECK_ARG(q && k && v && o && dout && lse && delta && dq_ws && dqkv && col_sum && cos_t && sin_t,
                "esm_attn_bwd_qkv: null pointer");
  ESM_CHECK_ARG(S % 4 == 0 && dh % 8 == 0, "esm_attn_bwd_qkv: needs S %% 4 == 0 and dh %% 8 == 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t T_ = (int64_t)B * S;
  int dgrid = (int)((T_ * nh + 255) / 256);
  if (dgrid > 148 * 32) dgrid = 148 * 32;
  float* lse2 = delta + T_ * nh;
  attn::delta_kernel<__nv_bfloat16><<<dgrid, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout,
                                                           delta, lse, lse2, T_, S, nh, dh);
  cudaMemsetAsync(dq_ws, 0, sizeof(float) * T_ * nh * dh, st);
  const int rc = attn_bwd_tc(q, k, v, dout, lse2, delta, key_mask, dq_ws, nullptr, nullptr, B, nh, S, dh, st, dqkv,
                             col_sum, cos_t, sin_t);
  if (rc) return rc;
  const int pairs = nh * dh / 2;
  const int rpb = 32;
  const int units = pairs / 2;  // two rotation pairs per thread
  dim3 grid((units + 63) / 64, (unsigned)((T_ + rpb - 1) / rpb));
  attn::dq_finalize_kernel<<<grid, 64, 0, st>>>(dq_ws, (__nv_bfloat16*)dqkv, col_sum, cos_t, sin_t, T_, S, nh, dh,
                                                 q_scale, rpb);
  ESM_LAUNCH_RET();
}

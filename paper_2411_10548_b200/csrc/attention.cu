// Attention C-ABI entry points (esm_attn_fwd / esm_attn_bwd / esm_attn_bwd_qkv) for ESM-2 (non-causal,
// key-padding mask, scaling = 1 because q is pre-scaled before RoPE: HF:modeling_esm.py:257-282, 313, 341-344).
//
// bf16 production path: the persistent tcgen05/TMEM kernels in attention_tc.cu; this file holds the
//       helpers around them (Delta / log2-LSE, dQ finalisation with RoPE^T) and the C entry points.
// fp32: SIMT reference-precision kernels (parity mode).
#include <cstdlib>

#include "common.cuh"

namespace esm {
namespace attn {

constexpr float L2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
// The attention row normaliser crosses the C ABI in the form the tcgen05 backward consumes:
// lse2 = -log2(sum_k exp(s_k)) = -LSE * log2(e) (an FFMA2 addend there); the fp32 kernels convert at the edges.

// ---------------------------------------------------------------------------- backward
// delta[b,h,s] = sum_d dO[t,h,d] * O[t,h,d] (t = b*S + s) (the model computes it in the dO GEMM's epilogue,
// ESM_EPI_DELTA; this pass serves esm_attn_bwd callers that pass O, and the fp32 parity path).  Block = a tile of 64
// tokens x all heads, transposed through shared memory: the dot products run with consecutive threads on
// consecutive heads of a token (contiguous 16-byte reads of the token-major [T, H] rows of O and dO), the
// per-(b, h, s) results leave with consecutive threads on consecutive tokens of a head (contiguous writes, and
// contiguous lse reads).  All of a thread's vector loads are unrolled at compile time.
template <typename T, int DH>
__global__ void __launch_bounds__(256) delta_kernel(const T* __restrict__ O, const T* __restrict__ dO,
                                                    float* __restrict__ delta, int64_t T_, int S, int nh) {
  constexpr int VEC = vec16<T>::N;
  constexpr int NV = DH / VEC;
  constexpr int TT = 64;
  extern __shared__ float tile[];  // [nh][TT]
  const int H = nh * DH;
  const int64_t t0 = (int64_t)blockIdx.x * TT;
  const int pairs = TT * nh;
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    const int tl = i / nh, h = i - tl * nh;
    const int64_t t = t0 + tl;
    float acc = 0.f;
    if (t < T_) {
      const T* o = O + t * H + h * DH;
      const T* g = dO + t * H + h * DH;
      uint4 ov[NV], gv[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        ov[k] = *reinterpret_cast<const uint4*>(o + k * VEC);
        gv[k] = *reinterpret_cast<const uint4*>(g + k * VEC);
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        float a[VEC], c[VEC];
        load_vec(reinterpret_cast<const T*>(&ov[k]), a);
        load_vec(reinterpret_cast<const T*>(&gv[k]), c);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc = fmaf(a[e], c[e], acc);
      }
    }
    tile[h * TT + tl] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    const int h = i / TT, tl = i - h * TT;
    const int64_t t = t0 + tl;
    if (t >= T_) continue;
    const int64_t b = t / S, s = t - b * S;
    const int64_t idx = (b * nh + h) * S + s;
    delta[idx] = tile[h * TT + tl];
  }
}

// generic head dim (fp32 parity mode): one thread per (token, head)
template <typename T>
__global__ void delta_generic_kernel(const T* __restrict__ O, const T* __restrict__ dO, float* __restrict__ delta,
                                     int64_t T_, int S, int nh, int dh) {
  const int H = nh * dh;
  const int64_t total = T_ * nh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = i / T_, t = i - h * T_;
    float acc = 0.f;
    for (int d = 0; d < dh; ++d) acc += io<T>::ld(O + t * H + h * dh + d) * io<T>::ld(dO + t * H + h * dh + d);
    const int64_t b = t / S, s = t - b * S;
    const int64_t idx = (b * nh + h) * S + s;
    delta[idx] = acc;
  }
}

template <typename T>
int launch_delta(const void* o, const void* dout, float* delta, int64_t T_, int S, int nh, int dh, cudaStream_t st) {
  const int64_t work = T_ * nh;
  int grid = (int)((work + 255) / 256);
  if (grid > device_sm_count() * 16) grid = device_sm_count() * 16;
  const T* O = (const T*)o;
  const T* dO = (const T*)dout;
  const int tiles = (int)((T_ + 63) / 64);
  const size_t sm = (size_t)64 * nh * sizeof(float);
  if (sm > 48 * 1024 || dh % vec16<T>::N != 0) {
    delta_generic_kernel<T><<<grid, 256, 0, st>>>(O, dO, delta, T_, S, nh, dh);
    return 0;
  }
  switch (dh) {
    case 16: delta_kernel<T, 16><<<tiles, 256, sm, st>>>(O, dO, delta, T_, S, nh); break;
    case 24: delta_kernel<T, 24><<<tiles, 256, sm, st>>>(O, dO, delta, T_, S, nh); break;
    case 32: delta_kernel<T, 32><<<tiles, 256, sm, st>>>(O, dO, delta, T_, S, nh); break;
    case 64: delta_kernel<T, 64><<<tiles, 256, sm, st>>>(O, dO, delta, T_, S, nh); break;
    default: delta_generic_kernel<T><<<grid, 256, 0, st>>>(O, dO, delta, T_, S, nh, dh); break;
  }
  return 0;
}

// ---------------------------------------------------------------------------- fp32 SIMT
constexpr int MAXD = 64;

// attention-probability dropout multiplier of (query q, key k) of head bh: keep / (1 - p) (1 when off); the
// esm_dropout bit of row bh*S + q, column k, as the tcgen05 kernels (attention_tc.cu) and the oracle
__device__ __forceinline__ float attn_drop_z(const DropKeys& dk, int bh, int S, int q, int k) {
  if (!dk.on) return 1.f;
  const uint32_t kb = drop_pair(dk, drop_row(dk, (uint32_t)((int64_t)bh * S + q)), (uint32_t)k >> 1);
  return ((kb >> (k & 1)) & 1u) ? dk.scale : 0.f;
}

__global__ void __launch_bounds__(64) fwd_f32_kernel(const float* __restrict__ Q, const float* __restrict__ K,
                                                     const float* __restrict__ V, const int32_t* __restrict__ km,
                                                     float* __restrict__ O, float* __restrict__ LSE, int S, int nh,
                                                     int dh, const esm_dropout drop) {
  const DropKeys dkeys = drop_keys(drop);
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
      l = l * sc + p;  // the normaliser keeps every probability
      const float pz = p * attn_drop_z(dkeys, bh, S, qi, k0 + j);
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) o[d] = o[d] * sc + pz * sV[j][d];
      m = mn;
    }
  }
  if (qi < S) {
    const int H = nh * dh;
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < dh) O[((int64_t)b * S + qi) * H + h * dh + d] = o[d] * inv;
    LSE[(int64_t)bh * S + qi] = -(m + logf(l)) * L2E;
  }
}

// dQ (per query thread) and dK/dV (per key thread), recomputing P from LSE
__global__ void __launch_bounds__(64) bwd_dq_f32_kernel(const float* __restrict__ Q, const float* __restrict__ K,
                                                        const float* __restrict__ V, const float* __restrict__ dO,
                                                        const float* __restrict__ LSE,
                                                        const float* __restrict__ Delta,
                                                        const int32_t* __restrict__ km, float* __restrict__ dQ, int S,
                                                        int nh, int dh, const esm_dropout drop) {
  const DropKeys dkeys = drop_keys(drop);
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
  const float lse = qi < S ? -LSE[(int64_t)bh * S + qi] * LN2 : 0.f;
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
      const float ds = p * (dp * attn_drop_z(dkeys, bh, S, qi, k0 + j) - delta);
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
                                                         float* __restrict__ dV, int S, int nh, int dh,
                                                         const esm_dropout drop) {
  const DropKeys dkeys = drop_keys(drop);
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
      sL[threadIdx.x] = qq < S ? -LSE[(int64_t)bh * S + qq] * LN2 : INFINITY;
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
      const float z = attn_drop_z(dkeys, bh, S, q0 + j, ki);
      const float ds = p * (dp * z - sD[j]);
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dh) {
          dv[d] += p * z * sO[j][d];
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

// zero fill of the fp32 dQ accumulator as a kernel (a memset node would break the programmatic-dependent-launch
// chain of the backward)
__global__ void __launch_bounds__(256) zero_f32_kernel(float4* __restrict__ p, int64_t n4) {
  pdl_wait();
  pdl_trigger();
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z;
}

void zero_f32(float* p, int64_t n, cudaStream_t st) {
  if (n % 4 == 0 && ((uintptr_t)p & 15) == 0) {
    const int64_t n4 = n / 4;
    int64_t g = (n4 + 255) / 256;
    if (g > device_sm_count() * 8) g = device_sm_count() * 8;
    launch_pdl(zero_f32_kernel, dim3((unsigned)g), dim3(256), 0, st, 1, reinterpret_cast<float4*>(p), n4);
  } else {
    cudaMemsetAsync(p, 0, sizeof(float) * n, st);
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

// Vector variant: thread = (token, head, 4-column chunk of the first rotation half + its partner chunk); the
// lanes of a token cover the whole fp32 dQ row (16-byte loads, whole sectors) and its bf16 q-slice of the dqkv
// row (8-byte stores); tokens strided over the grid; bias partial sums leave with vector reductions.
__global__ void __launch_bounds__(256) dq_finalize_vec_kernel(const float* __restrict__ dq,
                                                              __nv_bfloat16* __restrict__ dqkv,
                                                              float* __restrict__ csum, const float* __restrict__ cs,
                                                              const float* __restrict__ sn, int64_t T_, int S, int nh,
                                                              int dh, float qs) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  const int half = dh >> 1, cpr = half >> 2;
  const int lanes = nh * cpr;
  const int slots = blockDim.x / lanes;
  const int slot = threadIdx.x / lanes, li = threadIdx.x - slot * lanes;
  if (slot >= slots) return;
  const int h = li / cpr, j = (li - h * cpr) * 4;
  const int H = nh * dh;
  float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
  const int64_t stride = (int64_t)gridDim.x * slots;
  for (int64_t t = (int64_t)blockIdx.x * slots + slot; t < T_; t += stride) {
    const int s = (int)(t % S);
    const float4 g0 = *reinterpret_cast<const float4*>(dq + t * H + h * dh + j);
    const float4 g1 = *reinterpret_cast<const float4*>(dq + t * H + h * dh + j + half);
    const float4 c = __ldg(reinterpret_cast<const float4*>(cs + (int64_t)s * half + j));
    const float4 sv = __ldg(reinterpret_cast<const float4*>(sn + (int64_t)s * half + j));
    const float4 q0 = make_float4((g0.x * c.x + g1.x * sv.x) * qs, (g0.y * c.y + g1.y * sv.y) * qs,
                                  (g0.z * c.z + g1.z * sv.z) * qs, (g0.w * c.w + g1.w * sv.w) * qs);
    const float4 q1 = make_float4((g1.x * c.x - g0.x * sv.x) * qs, (g1.y * c.y - g0.y * sv.y) * qs,
                                  (g1.z * c.z - g0.z * sv.z) * qs, (g1.w * c.w - g0.w * sv.w) * qs);
    __nv_bfloat16* row = dqkv + t * 3 * H + h * dh + j;
    __nv_bfloat162 p0 = __floats2bfloat162_rn(q0.x, q0.y), p1 = __floats2bfloat162_rn(q0.z, q0.w);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(q1.x, q1.y), p3 = __floats2bfloat162_rn(q1.z, q1.w);
    *reinterpret_cast<uint2*>(row) = make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
    *reinterpret_cast<uint2*>(row + half) =
        make_uint2(*reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
    a0.x += q0.x; a0.y += q0.y; a0.z += q0.z; a0.w += q0.w;
    a1.x += q1.x; a1.y += q1.y; a1.z += q1.z; a1.w += q1.w;
  }
  if (csum) {
    red_add_v4_f32(csum + h * dh + j, a0.x, a0.y, a0.z, a0.w);
    red_add_v4_f32(csum + h * dh + j + half, a1.x, a1.y, a1.z, a1.w);
  }
}

}  // namespace attn
}  // namespace esm

namespace esm {
int attn_prepare_tc(const int32_t* km, int* sched, int B, int S, cudaStream_t st);
int attn_fwd_tc(const void* q, const void* k, const void* v, const int32_t* km, int* sched, void* o, float* lse,
                int B, int nh, int S, int dh, cudaStream_t st, const esm_dropout* drop);
int attn_bwd_tc(const void* q, const void* k, const void* v, const void* dout, const float* lse, const float* delta,
                const int32_t* km, int* sched, float* dq, void* dk, void* dv, int B, int nh, int S, int dh,
                cudaStream_t st, void* dqkv, float* col_sum, const float* cos_t, const float* sin_t,
                const esm_dropout* drop);
static bool drop_on(const esm_dropout* d) { return d != nullptr && d->threshold != 0u; }
}  // namespace esm

using namespace esm;

extern "C" int esm_attn_prepare(const int32_t* key_mask, int32_t* sched, int B, int S, esm_stream_t stream) {
  ESM_CHECK_ARG(sched && B > 0 && S > 0, "esm_attn_prepare: bad args");
  return attn_prepare_tc(key_mask, sched, B, S, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int esm_attn_fwd_dropout(int dtype, const void* q, const void* k, const void* v, const int32_t* key_mask,
                                    int32_t* sched, void* o, float* lse, int B, int nh, int S, int dh,
                                    const esm_dropout* drop, esm_stream_t stream) {
  ESM_CHECK_ARG(q && k && v && o && lse && B > 0 && nh > 0 && S > 0, "esm_attn_fwd: bad args");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == ESM_BF16) {
    ESM_CHECK_ARG(sched != nullptr, "esm_attn_fwd: bf16 needs the scheduling workspace (esm_attn_prepare)");
    ESM_CHECK_ARG(S % 4 == 0, "esm_attn_fwd: bf16 needs S %% 4 == 0 (pad the batch)");
    return attn_fwd_tc(q, k, v, key_mask, sched, o, lse, B, nh, S, dh, st, drop);
  }
  ESM_CHECK_ARG(dh <= attn::MAXD, "esm_attn_fwd: dh <= 64");
  dim3 grid((S + 63) / 64, B * nh);
  attn::fwd_f32_kernel<<<grid, 64, 0, st>>>((const float*)q, (const float*)k, (const float*)v, key_mask, (float*)o,
                                            lse, S, nh, dh, drop_on(drop) ? *drop : esm_dropout{nullptr, 0u, 0u, 1.f});
  ESM_LAUNCH_RET();
}

extern "C" int esm_attn_fwd(int dtype, const void* q, const void* k, const void* v, const int32_t* key_mask,
                            int32_t* sched, void* o, float* lse, int B, int nh, int S, int dh, esm_stream_t stream) {
  return esm_attn_fwd_dropout(dtype, q, k, v, key_mask, sched, o, lse, B, nh, S, dh, nullptr, stream);
}

extern "C" int esm_attn_bwd_dropout(int dtype, const void* q, const void* k, const void* v, const void* o,
                                    const void* dout, const float* lse, const int32_t* key_mask, int32_t* sched,
                                    float* delta, float* dq, void* dk, void* dv, int B, int nh, int S, int dh,
                                    const esm_dropout* drop, esm_stream_t stream) {
  ESM_CHECK_ARG(q && k && v && dout && lse && delta && dq && dk && dv, "esm_attn_bwd: null pointer");
  ESM_CHECK_ARG(o || dtype == ESM_BF16, "esm_attn_bwd: fp32 needs o");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t T_ = (int64_t)B * S;
  if (dtype == ESM_BF16) {
    ESM_CHECK_ARG(sched != nullptr, "esm_attn_bwd: bf16 needs the scheduling workspace (esm_attn_prepare)");
    ESM_CHECK_ARG(S % 4 == 0, "esm_attn_bwd: bf16 needs S %% 4 == 0 (pad the batch)");
    // o == NULL: Delta was accumulated by the dO-producing GEMM (ESM_EPI_DELTA)
    if (o) attn::launch_delta<__nv_bfloat16>(o, dout, delta, T_, S, nh, dh, st);
    attn::zero_f32(dq, T_ * nh * dh, st);
    const int rc = attn_bwd_tc(q, k, v, dout, lse, delta, key_mask, sched, dq, dk, dv, B, nh, S, dh, st, nullptr,
                               nullptr, nullptr, nullptr, drop);
    if (rc) return rc;
    ESM_LAUNCH_RET();
  }
  ESM_CHECK_ARG(dh <= attn::MAXD, "esm_attn_bwd: dh <= 64");
  dim3 grid((S + 63) / 64, B * nh);
  attn::launch_delta<float>(o, dout, delta, T_, S, nh, dh, st);
  const esm_dropout dr = drop_on(drop) ? *drop : esm_dropout{nullptr, 0u, 0u, 1.f};
  attn::bwd_dq_f32_kernel<<<grid, 64, 0, st>>>((const float*)q, (const float*)k, (const float*)v, (const float*)dout,
                                               lse, delta, key_mask, dq, S, nh, dh, dr);
  attn::bwd_dkv_f32_kernel<<<grid, 64, 0, st>>>((const float*)q, (const float*)k, (const float*)v,
                                                (const float*)dout, lse, delta, key_mask, (float*)dk, (float*)dv, S,
                                                nh, dh, dr);
  ESM_LAUNCH_RET();
}

extern "C" int esm_attn_bwd(int dtype, const void* q, const void* k, const void* v, const void* o, const void* dout,
                            const float* lse, const int32_t* key_mask, int32_t* sched, float* delta, float* dq,
                            void* dk, void* dv, int B, int nh, int S, int dh, esm_stream_t stream) {
  return esm_attn_bwd_dropout(dtype, q, k, v, o, dout, lse, key_mask, sched, delta, dq, dk, dv, B, nh, S, dh, nullptr,
                              stream);
}

extern "C" int esm_attn_bwd_qkv_dropout(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                        const float* lse, const int32_t* key_mask, int32_t* sched, float* delta,
                                        float* dq_ws, void* dqkv, float* col_sum, const float* cos_t,
                                        const float* sin_t, float q_scale, int B, int nh, int S, int dh,
                                        const esm_dropout* drop, esm_stream_t stream) {
  ESM_CHECK_ARG(q && k && v && dout && lse && sched && delta && dq_ws && dqkv && col_sum && cos_t && sin_t,
                "esm_attn_bwd_qkv: null pointer");
  ESM_CHECK_ARG(S % 4 == 0 && dh % 8 == 0, "esm_attn_bwd_qkv: needs S %% 4 == 0 and dh %% 8 == 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t T_ = (int64_t)B * S;
  if (o) attn::launch_delta<__nv_bfloat16>(o, dout, delta, T_, S, nh, dh, st);
  attn::zero_f32(dq_ws, T_ * nh * dh, st);
  const int rc = attn_bwd_tc(q, k, v, dout, lse, delta, key_mask, sched, dq_ws, nullptr, nullptr, B, nh, S, dh, st,
                             dqkv, col_sum, cos_t, sin_t, drop);
  if (rc) return rc;
  const int lanes = nh * (dh / 8);  // vector path: threads per token
  if (dh % 8 == 0 && lanes <= 256 && ((uintptr_t)col_sum & 15) == 0) {
    const int slots = 256 / lanes;
    const int64_t want = (T_ + (int64_t)slots * 16 - 1) / ((int64_t)slots * 16);  // ~16 tokens per thread
    const int grid = (int)(want < device_sm_count() * 8 ? (want < 1 ? 1 : want) : device_sm_count() * 8);
    launch_pdl(attn::dq_finalize_vec_kernel, dim3(grid), dim3(slots * lanes), 0, st, 1, (const float*)dq_ws,
               (__nv_bfloat16*)dqkv, col_sum, cos_t, sin_t, T_, S, nh, dh, q_scale);
    ESM_LAUNCH_RET();
  }
  const int pairs = nh * dh / 2;
  const int rpb = 32;
  const int units = pairs / 2;  // two rotation pairs per thread
  dim3 grid((units + 63) / 64, (unsigned)((T_ + rpb - 1) / rpb));
  attn::dq_finalize_kernel<<<grid, 64, 0, st>>>(dq_ws, (__nv_bfloat16*)dqkv, col_sum, cos_t, sin_t, T_, S, nh, dh,
                                                 q_scale, rpb);
  ESM_LAUNCH_RET();
}

extern "C" int esm_attn_bwd_qkv(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                const float* lse, const int32_t* key_mask, int32_t* sched, float* delta, float* dq_ws,
                                void* dqkv, float* col_sum, const float* cos_t, const float* sin_t, float q_scale,
                                int B, int nh, int S, int dh, esm_stream_t stream) {
  return esm_attn_bwd_qkv_dropout(q, k, v, o, dout, lse, key_mask, sched, delta, dq_ws, dqkv, col_sum, cos_t, sin_t,
                                  q_scale, B, nh, S, dh, nullptr, stream);
}

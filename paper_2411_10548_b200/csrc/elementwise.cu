// Memory-bound kernels of the ESM-2 MLM step: masking, embeddings (+token dropout),
// LayerNorm fwd/bwd (+ fused bias-grad column sums, fused GELU'), rotary/head
// re-layout, LM-head decoder + masked cross-entropy, fused AdamW.
// All are coalesced, 16-byte vectorised, warp-shuffle reductions; one warp per row
// for the row-wise ops.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include <algorithm>

#include "common.cuh"

namespace esm {

static thread_local char g_err[512] = "";
void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static inline cudaStream_t S(esm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ============================================================================
// MLM masking (bit-exact with oracle/esm2_oracle.py:mlm_mask)
// ============================================================================
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__global__ void mlm_mask_kernel(const int32_t* __restrict__ ids, int32_t* __restrict__ inp, int32_t* __restrict__ lab,
                                int32_t* __restrict__ n_labels, int64_t n, uint64_t key, int elig_lo, int elig_hi,
                                int mask_id, int rand_lo, uint32_t rand_n) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = ids[i];
    const uint64_t base = key + (uint64_t)i * kGolden;
    const uint64_t r0 = mix64(base), r1 = mix64(base + 1), r2 = mix64(base + 2);
    const bool eligible = id >= elig_lo && id <= elig_hi;
    const bool sel = eligible && (int64_t)(r0 >> 40) < 2516582;
    const int64_t a = (int64_t)(r1 >> 40);
    int32_t out = id;
    if (sel && a < 13421773) out = mask_id;
    else if (sel && a < 15099494) out = rand_lo + (int32_t)(r2 % (uint64_t)rand_n);
    inp[i] = out;
    lab[i] = sel ? id : -100;
    local += sel ? 1 : 0;
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(&cnt, local);
  __syncthreads();
  if (threadIdx.x == 0 && n_labels && cnt) atomicAdd(n_labels, cnt);
}

__global__ void inv_count_kernel(const int32_t* n, float* inv) {
  const int c = *n;
  *inv = 1.0f / (float)(c > 1 ? c : 1);
}

// ============================================================================
// embeddings (HF:modeling_esm.py:203-234)
// ============================================================================
__global__ void row_scale_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ am, float* row_scale,
                                 int S, int token_dropout, int mask_id) {
  const int b = blockIdx.x;
  int nm = 0, len = 0;
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    nm += ids[(int64_t)b * S + s] == mask_id;
    len += am ? (am[(int64_t)b * S + s] != 0) : 1;
  }
  __shared__ int sm[2][32];
  nm = __reduce_add_sync(0xffffffffu, nm);
  len = __reduce_add_sync(0xffffffffu, len);
  if ((threadIdx.x & 31) == 0) {
    sm[0][threadIdx.x >> 5] = nm;
    sm[1][threadIdx.x >> 5] = len;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, l = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += sm[0][w];
      l += sm[1][w];
    }
    float scale = 1.0f;
    if (token_dropout) {
      const float observed = (float)a / (float)(l > 0 ? l : 1);
      scale = (1.0f - 0.15f * 0.8f) / (1.0f - observed);
    }
    row_scale[b] = scale;
  }
}

template <typename T>
__global__ void embed_fwd_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ am,
                                 const T* __restrict__ E, const float* __restrict__ row_scale, T* __restrict__ x,
                                 int64_t T_, int S, int H, int token_dropout, int mask_id) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  constexpr int VEC = vec16<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < T_; t += nwarps) {
    const int id = ids[t];
    float sc = row_scale[t / S] * (am ? (float)(am[t] != 0) : 1.0f);
    if (token_dropout && id == mask_id) sc = 0.f;
    for (int h = lane * VEC; h < H; h += 32 * VEC) {
      float v[VEC];
      load_vec(E + (int64_t)id * H + h, v);
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] *= sc;
      store_vec(x + t * H + h, v);
    }
  }
}

// dE[v, :] += sum over rows with ids == v (small V: the ESM alphabet).  Thread = one 16-byte column vector
// (VEC columns), block = up to 1280 columns x a contiguous block of rows; per-(id, column) partial sums live in
// shared memory ([V][VEC * blockDim] fp32), RU rows' vectors are loaded before they are accumulated, and each
// block adds its partials to dE with vector reductions (red.global.add.v4.f32).
template <typename T>
__global__ void __launch_bounds__(256) embed_bwd_smem_kernel(const int32_t* __restrict__ ids,
                                                             const int32_t* __restrict__ am,
                                                             const float* __restrict__ row_scale,
                                                             const T* __restrict__ dx, float* __restrict__ dE,
                                                             int64_t T_, int S, int H, int V, int rows_per_block,
                                                             int mask_id, int pad_id) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  constexpr int VEC = vec16<T>::N;
  constexpr int RU = 4;
  extern __shared__ float acc[];  // [V][BC]
  const int BC = VEC * blockDim.x;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * VEC;  // first column of this thread
  const int lc = threadIdx.x * VEC;
  for (int i = threadIdx.x; i < V * BC; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(T_, r0 + rows_per_block);
  if (c < H) {
    for (int64_t t0 = r0; t0 < r1; t0 += RU) {
      uint4 raw[RU];
      int id[RU];
      float sc[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int64_t t = t0 + u < r1 ? t0 + u : r1 - 1;
        id[u] = t0 + u < r1 ? ids[t] : pad_id;
        sc[u] = row_scale[t / S] * (am ? (float)(am[t] != 0) : 1.0f);
        raw[u] = *reinterpret_cast<const uint4*>(dx + t * H + c);
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (id[u] == pad_id || id[u] == mask_id || sc[u] == 0.f) continue;  // no grad for padding / masked rows
        float v[VEC];
        load_vec(reinterpret_cast<const T*>(&raw[u]), v);
        float* a = acc + id[u] * BC + lc;
#pragma unroll
        for (int e = 0; e < VEC; e += 4) {
          float4 q = *reinterpret_cast<float4*>(a + e);
          q.x += v[e] * sc[u];
          q.y += v[e + 1] * sc[u];
          q.z += v[e + 2] * sc[u];
          q.w += v[e + 3] * sc[u];
          *reinterpret_cast<float4*>(a + e) = q;
        }
      }
    }
  }
  __syncthreads();
  if (c < H)
    for (int v = 0; v < V; ++v) {
      const float* a = acc + v * BC + lc;
#pragma unroll
      for (int e = 0; e < VEC; e += 4) {
        const float4 q = *reinterpret_cast<const float4*>(a + e);
        if (q.x != 0.f || q.y != 0.f || q.z != 0.f || q.w != 0.f)
          red_add_v4_f32(dE + (int64_t)v * H + c + e, q.x, q.y, q.z, q.w);
      }
    }
}

// large vocabularies (Geneformer V ~ 25k): one warp per token row, vector fp32 reductions into dE[id]
template <typename T>
__global__ void embed_bwd_atomic_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ am,
                                        const float* __restrict__ row_scale, const T* __restrict__ dx,
                                        float* __restrict__ dE, int64_t T_, int S, int H, int mask_id, int pad_id) {
  constexpr int VEC = vec16<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < T_; t += warps) {
    const int id = ids[t];
    if (id == pad_id || id == mask_id) continue;
    const float sc = row_scale[t / S] * (am ? (float)(am[t] != 0) : 1.0f);
    if (sc == 0.f) continue;
    for (int c = lane * VEC; c < H; c += 32 * VEC) {
      float v[VEC];
      load_vec(dx + t * H + c, v);
#pragma unroll
      for (int e = 0; e < VEC; e += 4)
        atomicAdd(reinterpret_cast<float4*>(dE + (int64_t)id * H + c + e),
                  make_float4(v[e] * sc, v[e + 1] * sc, v[e + 2] * sc, v[e + 3] * sc));
    }
  }
}

// ============================================================================
// LayerNorm: a row is owned by a group of WPR warps (WPR*32 lanes); each lane owns MAXV fixed
// 16-byte column vectors, so gamma/beta and the backward's dgamma/dbeta/column-sum
// accumulators live in registers across all rows the group processes.
// ============================================================================
template <int WPR>
__device__ __forceinline__ float2 group_sum2(float2 v, float2* red, int wig, int lane, int bar_id, int& parity) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  if constexpr (WPR == 1) {
    return v;
  } else {
    float2* buf = red + parity * WPR;
    if (lane == 0) buf[wig] = v;
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(WPR * 32) : "memory");
    float2 r = make_float2(0.f, 0.f);
#pragma unroll
    for (int w = 0; w < WPR; ++w) {
      r.x += buf[w].x;
      r.y += buf[w].y;
    }
    parity ^= 1;
    return r;
  }
}

template <typename T>
__device__ __forceinline__ void unpack_vec(const uint4& u, float* out) {  // 16 raw bytes -> VEC floats
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      out[2 * i] = f.x;
      out[2 * i + 1] = f.y;
    }
  } else {
    out[0] = __uint_as_float(u.x); out[1] = __uint_as_float(u.y);
    out[2] = __uint_as_float(u.z); out[3] = __uint_as_float(u.w);
  }
}

__device__ __forceinline__ void load_f32x(const float* p, float* o, int n) {
  // n = 8 (bf16 VEC) or 4 (fp32 VEC); p 16B aligned
  const float4 a = *reinterpret_cast<const float4*>(p);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  if (n == 8) {
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
  }
}

// Bulk prefetch of a contiguous byte range into L2 (one thread issues it; no registers held).  Used by
// the RoPE-backward scatter (+7 % at 650M); measured neutral in the LayerNorm kernels.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// SG: gamma/beta read from shared memory ([2][H] floats, dynamic) instead of being held in registers, so
// the bf16 kernel fits 64 (MAXV <= 2) / 80 (MAXV = 3) registers and 4 / 3 CTAs per SM keep more row bytes
// in flight than the register-resident variant's 2.
template <typename T, int MAXV, int WPR, bool SG = false>
__global__ void __launch_bounds__(256, SG ? (MAXV <= 2 ? 4 : 3) : 1) ln_fwd_kernel(const T* __restrict__ x, const float* __restrict__ g,
                                                     const float* __restrict__ b, T* __restrict__ y,
                                                     float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                     int64_t rows, int H, float eps) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  constexpr int VEC = vec16<T>::N;
  constexpr int GPB = 8 / WPR;  // groups per block
  __shared__ float2 red[GPB][2 * WPR];
  extern __shared__ float sgb[];  // SG: gamma [H], beta [H]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp / WPR, wig = warp % WPR;
  const int glane = wig * 32 + lane;
  int parity = 0;
  float gv[SG ? 1 : MAXV][VEC], bv[SG ? 1 : MAXV][VEC];
  if constexpr (SG) {
    for (int i = threadIdx.x; i < H; i += blockDim.x) {
      sgb[i] = g[i];
      sgb[H + i] = b[i];
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        load_f32x(g + h, gv[i], VEC);
        load_f32x(b + h, bv[i], VEC);
      }
    }
  }
  const float invH = 1.0f / H;
  // two rows per group iteration: both rows' loads are in flight together and their statistics are
  // reduced as one float2 (half the cross-lane reductions per row).  Rows stay packed (raw 16-byte
  // vectors, unpacked on the fly) so a lane can hold 2 rows x 3 vectors without spilling occupancy.
  const int64_t rstep = (int64_t)gridDim.x * GPB * 2;
  for (int64_t r0 = ((int64_t)blockIdx.x * GPB + grp) * 2; r0 < rows; r0 += rstep) {
    const bool has1 = r0 + 1 < rows;
    uint4 raw[2][MAXV];
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        raw[0][i] = *reinterpret_cast<const uint4*>(x + r0 * H + h);
        raw[1][i] = has1 ? *reinterpret_cast<const uint4*>(x + (r0 + 1) * H + h) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        float v0[VEC], v1[VEC];
        unpack_vec<T>(raw[0][i], v0);
        unpack_vec<T>(raw[1][i], v1);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          s0 += v0[j];
          s1 += v1[j];
        }
      }
    }
    const float2 mu = group_sum2<WPR>(make_float2(s0, s1), red[grp], wig, lane, grp + 1, parity);
    const float mu0 = mu.x * invH, mu1 = mu.y * invH;
    float ss0 = 0.f, ss1 = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        float v0[VEC], v1[VEC];
        unpack_vec<T>(raw[0][i], v0);
        unpack_vec<T>(raw[1][i], v1);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const float d0 = v0[j] - mu0, d1 = v1[j] - mu1;
          ss0 += d0 * d0;
          ss1 += d1 * d1;
        }
      }
    }
    const float2 var = group_sum2<WPR>(make_float2(ss0, ss1), red[grp], wig, lane, grp + 1, parity);
    const float rs0 = rsqrtf(var.x * invH + eps), rs1 = rsqrtf(var.y * invH + eps);
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        float v[VEC], o[VEC], gs[VEC], bs[VEC];
        const float* gi = gs;
        const float* bi = bs;
        if constexpr (SG) {
          load_f32x(sgb + h, gs, VEC);
          load_f32x(sgb + H + h, bs, VEC);
        } else {
          gi = gv[i];
          bi = bv[i];
        }
        unpack_vec<T>(raw[0][i], v);
#pragma unroll
        for (int j = 0; j < VEC; ++j) o[j] = (v[j] - mu0) * rs0 * gi[j] + bi[j];
        store_vec(y + r0 * H + h, o);
        if (has1) {
          unpack_vec<T>(raw[1][i], v);
#pragma unroll
          for (int j = 0; j < VEC; ++j) o[j] = (v[j] - mu1) * rs1 * gi[j] + bi[j];
          store_vec(y + (r0 + 1) * H + h, o);
        }
      }
    }
    if (glane == 0) {
      mean_out[r0] = mu0;
      rstd_out[r0] = rs0;
      if (has1) {
        mean_out[r0 + 1] = mu1;
        rstd_out[r0 + 1] = rs1;
      }
    }
  }
}

// Backward.  STATS: also accumulate dgamma / dbeta here (otherwise the dgrad GEMM that produced dy
// computes them in its epilogue, ESM_EPI_STORE_LN).  Rows are held as raw 16-byte vectors (bf16 packed)
// and all of a row's loads are issued before the reduction.
// SG (bf16, no dgamma/dbeta, <= 2 vectors per lane): gamma from shared memory, 3 CTAs per SM.
template <typename T, int MAXV, int WPR, bool STATS, bool SG = false, bool DROP = false>
__global__ void __launch_bounds__(256, SG ? 3 : (sizeof(T) == 2 && (MAXV <= 2 || !STATS)) ? 2 : 1)
    ln_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ g,
                  const float* __restrict__ mean, const float* __restrict__ rstd, const T* __restrict__ dres,
                  const T* __restrict__ gelu_z, T* __restrict__ dx, float* __restrict__ dg, float* __restrict__ db,
                  float* __restrict__ csum, int64_t rows, int H, const esm_dropout drop, T* __restrict__ dxd) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  constexpr int VEC = vec16<T>::N;
  constexpr int GPB = 8 / WPR;
  DropKeys dk{0u, 0u, 0u, 1.f, false};
  if constexpr (DROP) dk = drop_keys(drop);
  __shared__ float2 red[GPB][2 * WPR];
  extern __shared__ float sacc[];  // [3][H] block-level partial sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp / WPR, wig = warp % WPR;
  const int glane = wig * 32 + lane;
  int parity = 0;
  for (int i = threadIdx.x; i < 3 * H; i += blockDim.x) sacc[i] = 0.f;
  const float* sg = sacc + 3 * H;  // SG: gamma [H] after the partial sums
  if constexpr (SG) {
    for (int i = threadIdx.x; i < H; i += blockDim.x) sacc[3 * H + i] = g[i];
    __syncthreads();
  }
  float gv[SG ? 1 : MAXV][VEC], ac[MAXV][VEC];
  float ag[STATS ? MAXV : 1][VEC], ab[STATS ? MAXV : 1][VEC];
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int h = (i * WPR * 32 + glane) * VEC;
    if constexpr (!SG) {
      if (h < H) load_f32x(g + h, gv[i], VEC);
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) ac[i][j] = 0.f;
    if constexpr (STATS) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) ag[i][j] = ab[i][j] = 0.f;
    }
  }
  const float invH = 1.0f / H;
  const int64_t rstep = (int64_t)gridDim.x * GPB;
  for (int64_t r = (int64_t)blockIdx.x * GPB + grp; r < rows; r += rstep) {
    const float mu = mean[r], rs = rstd[r];
    uint4 xr[MAXV], dr[MAXV], rr[MAXV], zr[MAXV];
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        xr[i] = *reinterpret_cast<const uint4*>(x + r * H + h);
        dr[i] = *reinterpret_cast<const uint4*>(dy + r * H + h);
        if (dres) rr[i] = *reinterpret_cast<const uint4*>(dres + r * H + h);
        if (gelu_z) zr[i] = *reinterpret_cast<const uint4*>(gelu_z + r * H + h);
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        float xv[VEC], dv[VEC], gs[VEC];
        const float* gi = gs;
        if constexpr (SG) load_f32x(sg + h, gs, VEC); else gi = gv[i];
        load_vec(reinterpret_cast<const T*>(&xr[i]), xv);
        load_vec(reinterpret_cast<const T*>(&dr[i]), dv);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const float xh = (xv[j] - mu) * rs;
          const float gy = dv[j] * gi[j];
          s1 += gy;
          s2 += gy * xh;
          if constexpr (STATS) {
            ag[i][j] += dv[j] * xh;
            ab[i][j] += dv[j];
          }
        }
      }
    }
    const float2 red2 = group_sum2<WPR>(make_float2(s1, s2), red[grp], wig, lane, grp + 1, parity);
    s1 = red2.x * invH;
    s2 = red2.y * invH;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * WPR * 32 + glane) * VEC;
      if (h < H) {
        float xv[VEC], dv[VEC], o[VEC], gs[VEC];
        const float* gi = gs;
        if constexpr (SG) load_f32x(sg + h, gs, VEC); else gi = gv[i];
        load_vec(reinterpret_cast<const T*>(&xr[i]), xv);
        load_vec(reinterpret_cast<const T*>(&dr[i]), dv);
#pragma unroll
        for (int j = 0; j < VEC; ++j) o[j] = rs * (dv[j] * gi[j] - s1 - (xv[j] - mu) * rs * s2);
        if (dres) {
          float rv[VEC];
          load_vec(reinterpret_cast<const T*>(&rr[i]), rv);
#pragma unroll
          for (int j = 0; j < VEC; ++j) o[j] += rv[j];
        }
        if (gelu_z) {
          float zv[VEC];
          load_vec(reinterpret_cast<const T*>(&zr[i]), zv);
#pragma unroll
          for (int j = 0; j < VEC; ++j) o[j] *= gelu_grad_f(zv[j]);
        }
        if constexpr (DROP) {  // gradient of the dropped-out branch (its bias gradient goes to csum)
          const uint32_t rh = drop_row(dk, (uint32_t)r);
          float od[VEC];
#pragma unroll
          for (int j = 0; j < VEC; j += 2) {
            const uint32_t kb = drop_pair(dk, rh, (uint32_t)(h + j) >> 1);
            od[j] = (kb & 1u) ? o[j] * dk.scale : 0.f;
            od[j + 1] = (kb & 2u) ? o[j + 1] * dk.scale : 0.f;
          }
#pragma unroll
          for (int j = 0; j < VEC; ++j) ac[i][j] += od[j];
          store_vec(dxd + r * H + h, od);
        } else {
#pragma unroll
          for (int j = 0; j < VEC; ++j) ac[i][j] += o[j];
        }
        store_vec(dx + r * H + h, o);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int h = (i * WPR * 32 + glane) * VEC;
    if (h < H) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        atomicAdd(&sacc[2 * H + h + j], ac[i][j]);
        if constexpr (STATS) {
          atomicAdd(&sacc[h + j], ag[i][j]);
          atomicAdd(&sacc[H + h + j], ab[i][j]);
        }
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    if (STATS && dg) atomicAdd(dg + c, sacc[c]);
    if (STATS && db) atomicAdd(db + c, sacc[H + c]);
    if (csum) atomicAdd(csum + c, sacc[2 * H + c]);
  }
}

// ============================================================================
// rotary embedding + [T,3H] <-> [B,nh,S,dh] re-layout (HF:modeling_esm.py:318-344, 45-54)
// ============================================================================
template <typename T>
__global__ void qkv_rope_fwd_kernel(const T* __restrict__ qkv, T* __restrict__ q, T* __restrict__ k,
                                    T* __restrict__ v, const float* __restrict__ cs, const float* __restrict__ sn,
                                    int64_t T_, int S, int nh, int dh, float qs) {
  const int half = dh >> 1;
  const int H = nh * dh;
  const int64_t total = T_ * nh * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % half);
    const int64_t th = i / half;
    const int h = (int)(th % nh);
    const int64_t t = th / nh;
    const int s = (int)(t % S);
    const int64_t b = t / S;
    const float c = cs[(int64_t)s * half + j], sv = sn[(int64_t)s * half + j];
    const T* row = qkv + t * 3 * H + h * dh;
    const int64_t o = ((b * nh + h) * S + s) * dh;
    float q0 = io<T>::ld(row + j) * qs, q1 = io<T>::ld(row + j + half) * qs;
    io<T>::st(q + o + j, q0 * c - q1 * sv);
    io<T>::st(q + o + j + half, q1 * c + q0 * sv);
    float k0 = io<T>::ld(row + H + j), k1 = io<T>::ld(row + H + j + half);
    io<T>::st(k + o + j, k0 * c - k1 * sv);
    io<T>::st(k + o + j + half, k1 * c + k0 * sv);
    v[o + j] = row[2 * H + j];
    v[o + j + half] = row[2 * H + j + half];
  }
}

// each thread owns one (head, j) column pair of q, k and v; loops rows; column sums -> bias grads
template <typename T>
struct pair2;  // two adjacent elements
template <> struct pair2<float> {
  static __device__ __forceinline__ float2 ld(const float* p) { return *reinterpret_cast<const float2*>(p); }
  static __device__ __forceinline__ void st(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }
};
template <> struct pair2<__nv_bfloat16> {
  static __device__ __forceinline__ float2 ld(const __nv_bfloat16* p) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float a, float b) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
  }
};

// RoPE^T + q-scale + [B, nh, S, dh] -> token-major dqkv [T, 3H] relayout + q/k/v bias-gradient column sums.
// Thread = two adjacent rotation pairs (j, j+1) of one head (float2 / bf16x2 accesses), a block-row of
// tokens processed RU at a time so each thread keeps RU tokens' loads in flight.
template <typename T>
__global__ void __launch_bounds__(256) qkv_rope_bwd_kernel(const float* __restrict__ dq, const T* __restrict__ dk,
                                                           const T* __restrict__ dv, T* __restrict__ dqkv,
                                                           float* __restrict__ csum, const float* __restrict__ cs,
                                                           const float* __restrict__ sn, int64_t T_, int S, int nh,
                                                           int dh, float qs, int rows_per_block) {
  constexpr int RU = 4;
  const int half = dh >> 1;
  const int H = nh * dh;
  const int unit = blockIdx.x * blockDim.x + threadIdx.x;  // 0 .. nh*half/2
  if (unit >= nh * (half >> 1)) return;
  const int h = unit / (half >> 1), j = (unit % (half >> 1)) * 2;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(T_, r0 + rows_per_block);
  if (j == 0 && (r0 % S) + (r1 - r0) <= S) {  // this head's rows are contiguous (head-major): pull them into L2
    const int64_t o = ((r0 / S * nh + h) * S + r0 % S) * dh;
    const uint32_t n = (uint32_t)((r1 - r0) * dh);
    if ((o * sizeof(T)) % 16 == 0 && (n * sizeof(T)) % 16 == 0) {
      prefetch_l2(dq + o, n * 4);
      prefetch_l2(dk + o, n * (uint32_t)sizeof(T));
      prefetch_l2(dv + o, n * (uint32_t)sizeof(T));
    }
  }
  float a[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) a[i] = 0.f;
  for (int64_t t0 = r0; t0 < r1; t0 += RU) {
    float2 g0[RU], g1[RU], e0[RU], e1[RU], v0[RU], v1[RU], c[RU], sv[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int64_t t = min(t0 + u, r1 - 1);  // tail rows re-read the last row; only valid rows are stored
      const int s = (int)(t % S);
      const int64_t o = ((t / S * nh + h) * S + s) * dh;
      g0[u] = *reinterpret_cast<const float2*>(dq + o + j);
      g1[u] = *reinterpret_cast<const float2*>(dq + o + j + half);
      e0[u] = pair2<T>::ld(dk + o + j);
      e1[u] = pair2<T>::ld(dk + o + j + half);
      v0[u] = pair2<T>::ld(dv + o + j);
      v1[u] = pair2<T>::ld(dv + o + j + half);
      c[u] = *reinterpret_cast<const float2*>(cs + (int64_t)s * half + j);
      sv[u] = *reinterpret_cast<const float2*>(sn + (int64_t)s * half + j);
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      if (t0 + u >= r1) break;
      // RoPE^T: dx_j = dy_j c + dy_{j+h} s ; dx_{j+h} = dy_{j+h} c - dy_j s
      const float qa0 = (g0[u].x * c[u].x + g1[u].x * sv[u].x) * qs, qb0 = (g0[u].y * c[u].y + g1[u].y * sv[u].y) * qs;
      const float qa1 = (g1[u].x * c[u].x - g0[u].x * sv[u].x) * qs, qb1 = (g1[u].y * c[u].y - g0[u].y * sv[u].y) * qs;
      const float ka0 = e0[u].x * c[u].x + e1[u].x * sv[u].x, kb0 = e0[u].y * c[u].y + e1[u].y * sv[u].y;
      const float ka1 = e1[u].x * c[u].x - e0[u].x * sv[u].x, kb1 = e1[u].y * c[u].y - e0[u].y * sv[u].y;
      T* row = dqkv + (t0 + u) * 3 * H + h * dh;
      pair2<T>::st(row + j, qa0, qb0);
      pair2<T>::st(row + j + half, qa1, qb1);
      pair2<T>::st(row + H + j, ka0, kb0);
      pair2<T>::st(row + H + j + half, ka1, kb1);
      pair2<T>::st(row + 2 * H + j, v0[u].x, v0[u].y);
      pair2<T>::st(row + 2 * H + j + half, v1[u].x, v1[u].y);
      a[0] += qa0; a[1] += qb0; a[2] += qa1; a[3] += qb1;
      a[4] += ka0; a[5] += kb0; a[6] += ka1; a[7] += kb1;
      a[8] += v0[u].x; a[9] += v0[u].y; a[10] += v1[u].x; a[11] += v1[u].y;
    }
  }
  if (csum) {
    const int c0 = h * dh + j;
    atomicAdd(csum + c0, a[0]);
    atomicAdd(csum + c0 + 1, a[1]);
    atomicAdd(csum + c0 + half, a[2]);
    atomicAdd(csum + c0 + half + 1, a[3]);
    atomicAdd(csum + H + c0, a[4]);
    atomicAdd(csum + H + c0 + 1, a[5]);
    atomicAdd(csum + H + c0 + half, a[6]);
    atomicAdd(csum + H + c0 + half + 1, a[7]);
    atomicAdd(csum + 2 * H + c0, a[8]);
    atomicAdd(csum + 2 * H + c0 + 1, a[9]);
    atomicAdd(csum + 2 * H + c0 + half, a[10]);
    atomicAdd(csum + 2 * H + c0 + half + 1, a[11]);
  }
}

// bf16 fast path (head_dim % 16 == 0): block = one head x a tile of TT consecutive tokens; thread = (token,
// 8-column chunk of the first rotation half + its partner chunk of the second half).  The block streams each
// head-major input as one contiguous region (TT x dh elements) and writes the token-major dqkv rows in whole
// 128-byte lines (dh = 64); q/k/v bias partial sums are reduced across the block's tokens with warp shuffles and
// shared memory before one atomic add per column.
template <int CPR>  // 8-column chunks per rotation half (dh / 16)
__global__ void __launch_bounds__(256) qkv_rope_bwd_tile_kernel(const float* __restrict__ dq,
                                                                const __nv_bfloat16* __restrict__ dk,
                                                                const __nv_bfloat16* __restrict__ dv,
                                                                __nv_bfloat16* __restrict__ dqkv,
                                                                float* __restrict__ csum, const float* __restrict__ cs,
                                                                const float* __restrict__ sn, int T_, int S, int nh,
                                                                float qs, int TT) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  constexpr int DH = CPR * 16, HALF = DH / 2, TPB = 256 / CPR;
  __shared__ float red[8][CPR][48];
  const int h = blockIdx.y;
  const int chunk = threadIdx.x % CPR, sub = threadIdx.x / CPR, j = chunk * 8;
  const int H = nh * DH;
  float acc[48];
#pragma unroll
  for (int i = 0; i < 48; ++i) acc[i] = 0.f;
  const int t_begin = blockIdx.x * TT, t_end = min(T_, t_begin + TT);
  for (int t = t_begin + sub; t < t_end; t += TPB) {
    const int b = t / S, s = t - b * S;
    const int64_t o = (((int64_t)b * nh + h) * S + s) * DH + j;
    float g0[8], g1[8], e0[8], e1[8], v0[8], v1[8], c[8], sv[8];
    load_f32x(dq + o, g0, 8);
    load_f32x(dq + o + HALF, g1, 8);
    load_vec(dk + o, e0);
    load_vec(dk + o + HALF, e1);
    load_vec(dv + o, v0);
    load_vec(dv + o + HALF, v1);
    load_f32x(cs + s * HALF + j, c, 8);
    load_f32x(sn + s * HALF + j, sv, 8);
    float q0[8], q1[8], k0[8], k1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {  // RoPE^T: dx_j = dy_j c + dy_{j+h} s ; dx_{j+h} = dy_{j+h} c - dy_j s
      q0[e] = (g0[e] * c[e] + g1[e] * sv[e]) * qs;
      q1[e] = (g1[e] * c[e] - g0[e] * sv[e]) * qs;
      k0[e] = e0[e] * c[e] + e1[e] * sv[e];
      k1[e] = e1[e] * c[e] - e0[e] * sv[e];
      acc[e] += q0[e];
      acc[8 + e] += q1[e];
      acc[16 + e] += k0[e];
      acc[24 + e] += k1[e];
      acc[32 + e] += v0[e];
      acc[40 + e] += v1[e];
    }
    __nv_bfloat16* row = dqkv + (int64_t)t * 3 * H + h * DH + j;
    store_vec(row, q0);
    store_vec(row + HALF, q1);
    store_vec(row + H, k0);
    store_vec(row + H + HALF, k1);
    store_vec(row + 2 * H, v0);
    store_vec(row + 2 * H + HALF, v1);
  }
  if (csum == nullptr) return;
  // lanes with the same chunk (lane % CPR) hold partial sums of different tokens
#pragma unroll
  for (int off = CPR; off < 32; off <<= 1)
#pragma unroll
    for (int i = 0; i < 48; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane < CPR)
#pragma unroll
    for (int i = 0; i < 48; ++i) red[w][lane][i] = acc[i];
  __syncthreads();
  for (int i = threadIdx.x; i < CPR * 48; i += blockDim.x) {
    const int ch = i / 48, k = i - ch * 48;
    float v = 0.f;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += red[ww][ch][k];
    const int part = k >> 3, e = k & 7;  // part: q lo, q hi, k lo, k hi, v lo, v hi
    const int col = (part >> 1) * H + h * DH + ch * 8 + (part & 1) * HALF + e;
    atomicAdd(csum + col, v);
  }
}

// ============================================================================
// LM head decoder (tied E) + masked cross entropy (HF:modeling_esm.py:777-784, 808-815)
// ============================================================================
template <typename T, int MAXV, int V_MAX>
__global__ void __launch_bounds__(256) xent_kernel(const T* __restrict__ n, const T* __restrict__ E,
                                                   const float* __restrict__ bias, const int32_t* __restrict__ labels,
                                                   const float* __restrict__ inv_denom, float* __restrict__ loss_sum,
                                                   float* __restrict__ dlogits, T* __restrict__ dn,
                                                   float* __restrict__ dbias, int64_t rows, int H, int V) {
  constexpr int VEC = vec16<T>::N;
  __shared__ float s_dbias[V_MAX];
  __shared__ float s_loss;
  for (int i = threadIdx.x; i < V_MAX; i += blockDim.x) s_dbias[i] = 0.f;
  if (threadIdx.x == 0) s_loss = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float inv = *inv_denom;
  float my_loss = 0.f;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const int lab = labels[r];
    if (lab < 0) {
      float z[VEC] = {};
      for (int h = lane * VEC; h < H; h += 32 * VEC) store_vec(dn + r * H + h, z);
      continue;
    }
    float x[MAXV][VEC];
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * 32 + lane) * VEC;
      if (h < H) load_vec(n + r * H + h, x[i]);
    }
    float logit[V_MAX];
#pragma unroll 8  // full unrolling hoists all V_MAX x MAXV E-row loads into registers (255 regs, 1 block/SM)
    for (int v = 0; v < V_MAX; ++v) {
      float p = 0.f;
      if (v < V) {
#pragma unroll
        for (int i = 0; i < MAXV; ++i) {
          const int h = (i * 32 + lane) * VEC;
          if (h < H) {
            float e[VEC];
            load_vec(E + (int64_t)v * H + h, e);
#pragma unroll
            for (int j = 0; j < VEC; ++j) p += x[i][j] * e[j];
          }
        }
      }
      logit[v] = v < V ? warp_sum(p) + bias[v] : -INFINITY;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int v = 0; v < V_MAX; ++v) mx = fmaxf(mx, logit[v]);
    float se = 0.f;
#pragma unroll
    for (int v = 0; v < V_MAX; ++v) se += (v < V) ? __expf(logit[v] - mx) : 0.f;
    const float lse = mx + __logf(se);
    float tgt = 0.f;
#pragma unroll
    for (int v = 0; v < V_MAX; ++v) tgt = (v == lab) ? logit[v] : tgt;
    if (lane == 0) my_loss += (lse - tgt) * inv;
    // dlogits
#pragma unroll
    for (int v = 0; v < V_MAX; ++v) {
      const float d = (v < V) ? (__expf(logit[v] - lse) - (v == lab ? 1.f : 0.f)) * inv : 0.f;
      logit[v] = d;
    }
    if (lane < V_MAX && lane < V) {
      float d = 0.f;
#pragma unroll
      for (int v = 0; v < V_MAX; ++v) d = (v == lane) ? logit[v] : d;
      dlogits[r * V + lane] = d;
      atomicAdd(&s_dbias[lane], d);
    }
    if (V > 32 && lane + 32 < V) {
      float d = 0.f;
#pragma unroll
      for (int v = 32; v < V_MAX; ++v) d = (v == lane + 32) ? logit[v] : d;
      dlogits[r * V + lane + 32] = d;
      atomicAdd(&s_dbias[lane + 32], d);
    }
    // dn = dlogits · E
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int h = (i * 32 + lane) * VEC;
      if (h < H) {
        float o[VEC] = {};
#pragma unroll 8
        for (int v = 0; v < V_MAX; ++v) {
          if (v < V) {
            float e[VEC];
            load_vec(E + (int64_t)v * H + h, e);
#pragma unroll
            for (int j = 0; j < VEC; ++j) o[j] += logit[v] * e[j];
          }
        }
        store_vec(dn + r * H + h, o);
      }
    }
  }
  my_loss = warp_sum(my_loss);
  if (lane == 0 && my_loss != 0.f) atomicAdd(&s_loss, my_loss);
  __syncthreads();
  if (threadIdx.x == 0 && s_loss != 0.f) atomicAdd(loss_sum, s_loss);
  for (int i = threadIdx.x; i < V && i < V_MAX; i += blockDim.x)
    if (s_dbias[i] != 0.f) atomicAdd(dbias + i, s_dbias[i]);
}

// Small-vocabulary decoder + masked CE (ESM V = 33), one warp per labelled row.  The tied decoder E is
// staged in shared memory with an odd 32-bit row pitch (conflict-free column access) and the row n[r] in a
// per-warp buffer: lane v computes logit v over H (lanes 32..V-1 cooperatively), the softmax runs across
// lanes, and dn = dlogits . E is computed with lanes over H.  Unlabelled rows only get dn = 0.
template <typename T>
__global__ void __launch_bounds__(256) xent_small_kernel(const T* __restrict__ n, const T* __restrict__ E,
                                                         const float* __restrict__ bias,
                                                         const int32_t* __restrict__ labels,
                                                         const float* __restrict__ inv_denom,
                                                         float* __restrict__ loss_sum, float* __restrict__ dlogits,
                                                         T* __restrict__ dn, float* __restrict__ dbias, int64_t rows,
                                                         int H, int V) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  constexpr int VEC = vec16<T>::N;
  constexpr int PAD = sizeof(T) == 2 ? 2 : 1;  // odd number of 32-bit words per staged row
  const int HP = H + PAD;
  extern __shared__ __align__(16) uint8_t xsm[];
  T* Es = reinterpret_cast<T*>(xsm);                                        // [V][HP]
  float* dlw = reinterpret_cast<float*>(xsm + (((size_t)V * HP * sizeof(T) + 15) & ~(size_t)15));  // [8][64]
  T* nrow = reinterpret_cast<T*>(dlw + 8 * 64);                             // [8][H]
  __shared__ float s_dbias[64];
  __shared__ float s_loss;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_dbias[i] = 0.f;
  if (threadIdx.x == 0) s_loss = 0.f;
  for (int i = threadIdx.x; i < V * H; i += blockDim.x) Es[(i / H) * HP + (i % H)] = E[i];
  __syncthreads();
  float* dl = dlw + w * 64;
  T* nr = nrow + (size_t)w * H;
  const float inv = *inv_denom;
  float my_loss = 0.f;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + w; r < rows; r += nwarps) {
    const int lab = labels[r];
    if (lab < 0) {
      float z[VEC] = {};
      for (int h = lane * VEC; h < H; h += 32 * VEC) store_vec(dn + r * H + h, z);
      continue;
    }
    for (int h = lane * VEC; h < H; h += 32 * VEC)
      *reinterpret_cast<uint4*>(nr + h) = *reinterpret_cast<const uint4*>(n + r * H + h);
    __syncwarp();
    // logits: lane v < min(V, 32) over all of H
    float lg = -INFINITY;
    if (lane < V) {
      float a0 = 0.f, a1 = 0.f;
      const T* er = Es + lane * HP;
#pragma unroll 8
      for (int h = 0; h < H; h += 2) {
        a0 = fmaf(io<T>::ld(nr + h), io<T>::ld(er + h), a0);
        a1 = fmaf(io<T>::ld(nr + h + 1), io<T>::ld(er + h + 1), a1);
      }
      lg = a0 + a1 + bias[lane];
    }
    // v in [32, V): cooperative dot products (all lanes get the value)
    const int nx = V > 32 ? V - 32 : 0;
#pragma unroll 1
    for (int x = 0; x < nx; ++x) {
      const T* er = Es + (32 + x) * HP;
      float a = 0.f;
      for (int h = lane; h < H; h += 32) a = fmaf(io<T>::ld(nr + h), io<T>::ld(er + h), a);
      dl[32 + x] = warp_sum(a) + bias[32 + x];  // stash the logit
    }
    __syncwarp();
    float mx = warp_max(lg);
    for (int x = 0; x < nx; ++x) mx = fmaxf(mx, dl[32 + x]);
    float se = warp_sum(lane < V ? __expf(lg - mx) : 0.f);
    for (int x = 0; x < nx; ++x) se += __expf(dl[32 + x] - mx);
    const float lse = mx + __logf(se);
    const float tgt = lab < 32 ? __shfl_sync(0xffffffffu, lg, lab) : dl[lab];
    if (lane == 0) my_loss += (lse - tgt) * inv;
    // dlogits
    if (lane < V) {
      const float d = (__expf(lg - lse) - (lane == lab ? 1.f : 0.f)) * inv;
      dl[lane] = d;
      dlogits[r * V + lane] = d;
      atomicAdd(&s_dbias[lane], d);
    }
    __syncwarp();
    for (int x = lane; x < nx; x += 32) {
      const int v = 32 + x;
      const float d = (__expf(dl[v] - lse) - (v == lab ? 1.f : 0.f)) * inv;
      dl[v] = d;
      dlogits[r * V + v] = d;
      atomicAdd(&s_dbias[v], d);
    }
    __syncwarp();
    // dn = dlogits . E, lanes over H (pairs of columns)
    for (int h = 2 * lane; h < H; h += 64) {
      float o0 = 0.f, o1 = 0.f;
#pragma unroll 4
      for (int v = 0; v < V; ++v) {
        const float d = dl[v];
        o0 = fmaf(d, io<T>::ld(Es + v * HP + h), o0);
        o1 = fmaf(d, io<T>::ld(Es + v * HP + h + 1), o1);
      }
      io<T>::st(dn + r * H + h, o0);
      io<T>::st(dn + r * H + h + 1, o1);
    }
    __syncwarp();
  }
  my_loss = warp_sum(my_loss);
  if (lane == 0 && my_loss != 0.f) atomicAdd(&s_loss, my_loss);
  __syncthreads();
  if (threadIdx.x == 0 && s_loss != 0.f) atomicAdd(loss_sum, s_loss);
  for (int i = threadIdx.x; i < V; i += blockDim.x)
    if (s_dbias[i] != 0.f) atomicAdd(dbias + i, s_dbias[i]);
}

// dE[v, h] += sum_{labelled rows r} dlogits[r, v] * n[r, h]; lane = column, warps = rows
template <typename T, int V_MAX>
__global__ void __launch_bounds__(256) xent_dE_kernel(const T* __restrict__ n, const int32_t* __restrict__ labels,
                                                      const float* __restrict__ dlogits, float* __restrict__ dE,
                                                      int64_t rows, int H, int V, int rows_per_block) {
  pdl_wait();  // programmatic dependent launch (common.cuh)
  pdl_trigger();
  __shared__ float red[8][V_MAX][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  float acc[V_MAX];
#pragma unroll
  for (int v = 0; v < V_MAX; ++v) acc[v] = 0.f;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  for (int64_t r = r0 + w; r < r1; r += 8) {
    if (labels[r] < 0) continue;
    const float x = col < H ? io<T>::ld(n + r * H + col) : 0.f;
#pragma unroll
    for (int v = 0; v < V_MAX; ++v)
      if (v < V) acc[v] += dlogits[r * V + v] * x;
  }
#pragma unroll
  for (int v = 0; v < V_MAX; ++v) red[w][v][lane] = acc[v];
  __syncthreads();
  for (int i = threadIdx.x; i < V * 32; i += blockDim.x) {
    const int v = i / 32, l = i % 32;
    float s = 0.f;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) s += red[ww][v][l];
    const int c = blockIdx.x * 32 + l;
    if (c < H && s != 0.f) atomicAdd(dE + (int64_t)v * H + c, s);
  }
}

// ============================================================================
// fused AdamW over the flat fp32 parameter buffer (+ bf16 shadow refresh)
// ============================================================================
// grads as fp32 (local / fp32 buckets) or bf16 (bf16-reduced data-parallel buckets)
__device__ __forceinline__ float4 load_grad4(const float* g, int64_t i) { return reinterpret_cast<const float4*>(g)[i]; }
__device__ __forceinline__ float4 load_grad4(const __nv_bfloat16* g, int64_t i) {
  const uint2 u = reinterpret_cast<const uint2*>(g)[i];
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

template <typename GT>
__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ p, const GT* __restrict__ g,
                                                    float* __restrict__ m, float* __restrict__ v,
                                                    __nv_bfloat16* __restrict__ p16,
                                                    const uint8_t* __restrict__ decay, int64_t n,
                                                    const float* __restrict__ hyper) {
  const float lr = hyper[0], b1 = hyper[1], b2 = hyper[2], eps = hyper[3], wd = hyper[4], step = hyper[5],
              gs = hyper[6];
  const float bc1 = 1.0f - powf(b1, step), bc2 = 1.0f - powf(b2, step);
  const float step_size = lr / bc1, inv_sqrt_bc2 = rsqrtf(bc2);
  const int64_t n4 = n >> 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i << 2;
    const float dec = decay[e >> 8] ? (1.0f - lr * wd) : 1.0f;
    float4 pp = reinterpret_cast<float4*>(p)[i];
    const float4 gg = load_grad4(g, i);
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float* P = &pp.x;
    const float* G = &gg.x;
    float* M = &mm.x;
    float* VV = &vv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gj = G[j] * gs;
      P[j] *= dec;
      M[j] = b1 * M[j] + (1.0f - b1) * gj;
      VV[j] = b2 * VV[j] + (1.0f - b2) * gj * gj;
      const float denom = sqrtf(VV[j]) * inv_sqrt_bc2 + eps;
      P[j] -= step_size * M[j] / denom;
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (p16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pp.x, pp.y), hi = __floats2bfloat162_rn(pp.z, pp.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(p16)[i] = u;
    }
  }
}

__global__ void cast_kernel(const float* __restrict__ s, __nv_bfloat16* __restrict__ d, int64_t n) {
  const int64_t n4 = n >> 2;  // 16-byte loads, 8-byte stores; n % 4 tail below
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 f = reinterpret_cast<const float4*>(s)[i];
    __nv_bfloat162 lo = __floats2bfloat162_rn(f.x, f.y), hi = __floats2bfloat162_rn(f.z, f.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(d)[i] = u;
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

__global__ void dropout_mask_kernel(const esm_dropout d, int64_t rows, int cols, uint8_t* __restrict__ out) {
  const DropKeys dk = drop_keys(d);
  const int64_t pairs = (int64_t)rows * ((cols + 1) / 2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pairs; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ((cols + 1) / 2);
    const int p = (int)(i - r * ((cols + 1) / 2));
    const uint32_t kb = dk.on ? drop_pair(dk, drop_row(dk, (uint32_t)r), (uint32_t)p) : 3u;
    out[r * cols + 2 * p] = kb & 1u;
    if (2 * p + 1 < cols) out[r * cols + 2 * p + 1] = (kb >> 1) & 1u;
  }
}

__global__ void cast_bf16_f32_kernel(const __nv_bfloat16* __restrict__ s, float* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = __bfloat162float(s[i]);
}

static int grid_for(int64_t work, int block, int cap = device_sm_count() * 16) {
  int64_t g = (work + block - 1) / block;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace esm

using namespace esm;

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int esm_version(void) { return 10000; }
const char* esm_last_error(void) { return esm::g_err; }
int esm_device_sm_count(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

int esm_tokenize(const char* seq, int len, int32_t* out, int max_out) {
  static int table[256];
  static bool init = false;
  if (!init) {
    for (int i = 0; i < 256; ++i) table[i] = 3;  // <unk>
    const char* aa = "LAGVSERTIDPKQNFYMHWC";
    for (int i = 0; i < 20; ++i) table[(unsigned char)aa[i]] = 4 + i;
    const char* ex = "XBUZO.-";
    for (int i = 0; i < 7; ++i) table[(unsigned char)ex[i]] = 24 + i;
    init = true;
  }
  const int need = len + 2;
  if (!out || max_out < need) return -need;
  out[0] = 0;
  for (int i = 0; i < len; ++i) out[i + 1] = table[(unsigned char)seq[i]];
  out[len + 1] = 2;
  return need;
}

int esm_mlm_mask_ex(const int32_t* ids, int32_t* input_ids, int32_t* labels, int32_t* n_labels, int64_t n,
                    uint64_t seed, uint64_t stream_id, int elig_lo, int elig_hi, int mask_id, int rand_lo, int rand_n,
                    esm_stream_t stream) {
  ESM_CHECK_ARG(ids && input_ids && labels && n >= 0 && rand_n > 0 && elig_lo <= elig_hi, "esm_mlm_mask: bad args");
  const uint64_t k0 = mix64(seed + kGolden);
  const uint64_t key = mix64(k0 ^ stream_id);
  if (n == 0) return 0;
  mlm_mask_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(ids, input_ids, labels, n_labels, n, key, elig_lo, elig_hi,
                                                           mask_id, rand_lo, (uint32_t)rand_n);
  ESM_LAUNCH_RET();
}

int esm_mlm_mask(const int32_t* ids, int32_t* input_ids, int32_t* labels, int32_t* n_labels, int64_t n, uint64_t seed,
                 uint64_t stream_id, esm_stream_t stream) {
  // ESM-2 alphabet: amino acids 4..30 eligible, <mask>=32, random replacement from the 20 standard residues
  return esm_mlm_mask_ex(ids, input_ids, labels, n_labels, n, seed, stream_id, 4, 30, 32, 4, 20, stream);
}

int esm_inv_count(const int32_t* n_labels, float* inv_denom, esm_stream_t stream) {
  inv_count_kernel<<<1, 1, 0, S(stream)>>>(n_labels, inv_denom);
  ESM_LAUNCH_RET();
}

int esm_embed_fwd(int dtype, const int32_t* ids, const int32_t* am, const void* E, void* x, float* row_scale, int B,
                  int Sq, int H, int token_dropout, int mask_id, esm_stream_t stream) {
  ESM_CHECK_ARG(ids && E && x && row_scale && B > 0 && Sq > 0 && H > 0, "esm_embed_fwd: bad args");
  ESM_CHECK_ARG(H % 8 == 0, "esm_embed_fwd: H %% 8");
  row_scale_kernel<<<B, 256, 0, S(stream)>>>(ids, am, row_scale, Sq, token_dropout, mask_id);
  const int64_t T_ = (int64_t)B * Sq;
  const int grid = grid_for(T_ * 32, 256);
  if (dtype == ESM_BF16)
    launch_pdl(embed_fwd_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, S(stream), 1, ids, am,
               (const __nv_bfloat16*)E, row_scale, (__nv_bfloat16*)x, T_, Sq, H, token_dropout, mask_id);
  else
    embed_fwd_kernel<float><<<grid, 256, 0, S(stream)>>>(ids, am, (const float*)E, row_scale, (float*)x, T_, Sq, H,
                                                         token_dropout, mask_id);
  ESM_LAUNCH_RET();
}

int esm_embed_bwd(int dtype, const int32_t* ids, const int32_t* am, const float* row_scale, const void* dx, float* dE,
                  int B, int Sq, int H, int V, int mask_id, int pad_id, esm_stream_t stream) {
  ESM_CHECK_ARG(ids && row_scale && dx && dE && V > 0 && H % 8 == 0, "esm_embed_bwd: bad args");
  const int64_t T_ = (int64_t)B * Sq;
  if (V > 40) {
    const int grid = grid_for(T_ * 32, 256);
    if (dtype == ESM_BF16)
      embed_bwd_atomic_kernel<__nv_bfloat16><<<grid, 256, 0, S(stream)>>>(ids, am, row_scale,
                                                                          (const __nv_bfloat16*)dx, dE, T_, Sq, H,
                                                                          mask_id, pad_id);
    else
      embed_bwd_atomic_kernel<float><<<grid, 256, 0, S(stream)>>>(ids, am, row_scale, (const float*)dx, dE, T_, Sq,
                                                                  H, mask_id, pad_id);
    ESM_LAUNCH_RET();
  }
  const int vec = dtype == ESM_BF16 ? 8 : 4;
  const int cols = std::min(H, std::min(1280, 256 * vec));    // columns per block (<= 165 KB of partials at V 33)
  const int bx = ((cols / vec) + 31) / 32 * 32;
  const int gx = (H + bx * vec - 1) / (bx * vec);
  const int gy = (int)std::max<int64_t>(1, std::min<int64_t>((T_ + 63) / 64, device_sm_count() / gx));
  const int rpb = (int)((T_ + gy - 1) / gy);
  dim3 grid(gx, gy);
  const size_t sm = (size_t)V * bx * vec * sizeof(float);
  if (dtype == ESM_BF16) {
    cudaFuncSetAttribute(embed_bwd_smem_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_pdl(embed_bwd_smem_kernel<__nv_bfloat16>, dim3(grid), dim3(bx), sm, S(stream), 1, ids, am, row_scale,
               (const __nv_bfloat16*)dx, dE, T_, Sq, H, V, rpb, mask_id, pad_id);
  } else {
    cudaFuncSetAttribute(embed_bwd_smem_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    embed_bwd_smem_kernel<float><<<grid, bx, sm, S(stream)>>>(ids, am, row_scale, (const float*)dx, dE, T_, Sq, H, V,
                                                              rpb, mask_id, pad_id);
  }
  ESM_LAUNCH_RET();
}

// choose (MAXV, WPR): WPR = smallest power of two with <= 3 vectors per lane
static inline void ln_shape(int H, int vec, int& maxv, int& wpr, int max_per_lane = 3) {
  const int vectors = H / vec;
  wpr = 1;
  while (wpr < 8 && vectors > wpr * 32 * max_per_lane) wpr <<= 1;
  maxv = (vectors + wpr * 32 - 1) / (wpr * 32);
}

#define LN_SWITCH(T, KERNEL, LAUNCH)                                                     \
  do {                                                                                   \
    if (mv == 1 && wpr == 1) LAUNCH(KERNEL<T, 1, 1>);                                    \
    else if (mv == 2 && wpr == 1) LAUNCH(KERNEL<T, 2, 1>);                               \
    else if (mv == 3 && wpr == 1) LAUNCH(KERNEL<T, 3, 1>);                               \
    else if (mv == 2 && wpr == 2) LAUNCH(KERNEL<T, 2, 2>);                               \
    else if (mv == 3 && wpr == 2) LAUNCH(KERNEL<T, 3, 2>);                               \
    else if (mv == 2 && wpr == 4) LAUNCH(KERNEL<T, 2, 4>);                               \
    else if (mv == 3 && wpr == 4) LAUNCH(KERNEL<T, 3, 4>);                               \
    else if (mv == 2 && wpr == 8) LAUNCH(KERNEL<T, 2, 8>);                               \
    else if (mv == 3 && wpr == 8) LAUNCH(KERNEL<T, 3, 8>);                               \
    else { esm::set_last_error("layernorm: H=%d unsupported", H); return ESM_ENOTSUP; }  \
  } while (0)

#define LN_SWITCH_SG(T, LAUNCH)                                                          \
  do {                                                                                   \
    if (mv == 1 && wpr == 1) LAUNCH(ln_fwd_kernel<T, 1, 1, true>);                       \
    else if (mv == 2 && wpr == 1) LAUNCH(ln_fwd_kernel<T, 2, 1, true>);                  \
    else if (mv == 3 && wpr == 1) LAUNCH(ln_fwd_kernel<T, 3, 1, true>);                  \
    else if (mv == 2 && wpr == 2) LAUNCH(ln_fwd_kernel<T, 2, 2, true>);                  \
    else if (mv == 3 && wpr == 2) LAUNCH(ln_fwd_kernel<T, 3, 2, true>);                  \
    else if (mv == 2 && wpr == 4) LAUNCH(ln_fwd_kernel<T, 2, 4, true>);                  \
    else if (mv == 3 && wpr == 4) LAUNCH(ln_fwd_kernel<T, 3, 4, true>);                  \
    else if (mv == 2 && wpr == 8) LAUNCH(ln_fwd_kernel<T, 2, 8, true>);                  \
    else if (mv == 3 && wpr == 8) LAUNCH(ln_fwd_kernel<T, 3, 8, true>);                  \
    else { esm::set_last_error("layernorm: H=%d unsupported", H); return ESM_ENOTSUP; }  \
  } while (0)

#define LN_SWITCH2(KS)                                                                   \
  do {                                                                                   \
    if (mv == 1 && wpr == 1) L_B(KS(1, 1));                                              \
    else if (mv == 2 && wpr == 1) L_B(KS(2, 1));                                         \
    else if (mv == 3 && wpr == 1) L_B(KS(3, 1));                                         \
    else if (mv == 2 && wpr == 2) L_B(KS(2, 2));                                         \
    else if (mv == 3 && wpr == 2) L_B(KS(3, 2));                                         \
    else if (mv == 2 && wpr == 4) L_B(KS(2, 4));                                         \
    else if (mv == 3 && wpr == 4) L_B(KS(3, 4));                                         \
    else if (mv == 2 && wpr == 8) L_B(KS(2, 8));                                         \
    else if (mv == 3 && wpr == 8) L_B(KS(3, 8));                                         \
    else { esm::set_last_error("layernorm: H=%d unsupported", H); return ESM_ENOTSUP; }  \
  } while (0)

int esm_layernorm_fwd(int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean, float* rstd,
                      int rows, int H, float eps, esm_stream_t stream) {
  ESM_CHECK_ARG(x && gamma && beta && y && mean && rstd && rows > 0 && H > 0, "esm_layernorm_fwd: bad args");
  const int vec = dtype == ESM_BF16 ? 8 : 4;
  ESM_CHECK_ARG(H % vec == 0, "layernorm: H %% %d", vec);
  int mv, wpr;
  ln_shape(H, vec, mv, wpr);
  const int gpb = 8 / wpr;
  int grid = (int)((rows + 2 * gpb - 1) / (2 * gpb));  // 2 rows per group iteration
  if (grid > device_sm_count() * 8) grid = device_sm_count() * 8;
#define L_SG(...)                                                                                     \
  do {                                                                                                \
    cudaFuncSetAttribute(__VA_ARGS__, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    launch_pdl(__VA_ARGS__, dim3(grid), dim3(256), smem, S(stream), 1, (const TT*)x, gamma, beta, (TT*)y, mean, \
               rstd, (int64_t)rows, H, eps);                                                          \
  } while (0)
#define L_F(...) launch_pdl(__VA_ARGS__, dim3(grid), dim3(256), 0, S(stream), 1, (const TT*)x, gamma, beta, (TT*)y, \
                            mean, rstd, (int64_t)rows, H, eps)
  static const bool sg_ok = !(getenv("ESM_LN_FWD_SG") && atoi(getenv("ESM_LN_FWD_SG")) == 0);
  if (dtype == ESM_BF16 && sg_ok) {
    using TT = __nv_bfloat16;
    const int per_sm = mv <= 2 ? 4 : 3;  // resident CTAs per SM (launch bounds): one persistent wave
    if (grid > device_sm_count() * per_sm) grid = device_sm_count() * per_sm;
    const size_t smem = (size_t)2 * H * sizeof(float);
#define L_S(...) L_SG(__VA_ARGS__)
    LN_SWITCH_SG(TT, L_S);
#undef L_S
  } else if (dtype == ESM_BF16) {
    using TT = __nv_bfloat16;
    LN_SWITCH(TT, ln_fwd_kernel, L_F);
  } else {
    using TT = float;
    LN_SWITCH(TT, ln_fwd_kernel, L_F);
  }
#undef L_F
#undef L_SG
  ESM_LAUNCH_RET();
}

int esm_layernorm_bwd(int dtype, const void* dy, const void* x, const float* gamma, const float* mean,
                      const float* rstd, const void* dres, const void* gelu_z, void* dx, float* dgamma, float* dbeta,
                      float* col_sum, int rows, int H, const esm_dropout* drop, void* dx_drop, esm_stream_t stream) {
  ESM_CHECK_ARG(dy && x && gamma && mean && rstd && dx && rows > 0, "esm_layernorm_bwd: bad args");
  const bool dropping = drop != nullptr && drop->threshold != 0u;
  ESM_CHECK_ARG(!dropping || (dx_drop != nullptr && drop->seed != nullptr), "esm_layernorm_bwd: dropout needs dx_drop");
  const esm_dropout dr = dropping ? *drop : esm_dropout{nullptr, 0u, 0u, 1.f};
  void* dxd = dropping ? dx_drop : nullptr;
  const int vec = dtype == ESM_BF16 ? 8 : 4;
  ESM_CHECK_ARG(H % vec == 0, "layernorm: H %% %d", vec);
  int mv, wpr;
  ln_shape(H, vec, mv, wpr);
  const size_t sm = (size_t)4 * H * sizeof(float);  // [3][H] partial sums + gamma (SG variant)
  ESM_CHECK_ARG(sm <= 200 * 1024, "layernorm_bwd: H too large");
  const bool stats = dgamma != nullptr || dbeta != nullptr;
  static const bool sg_ok = !(getenv("ESM_LN_BWD_SG") && atoi(getenv("ESM_LN_BWD_SG")) == 0);
  const bool sg = sg_ok && dtype == ESM_BF16 && !stats && mv <= 2;
  int grid = device_sm_count() * (sg ? 3 : 2);
  const int gpb = 8 / wpr;
  if ((int64_t)grid * gpb > rows) grid = (int)((rows + gpb - 1) / gpb);
#define L_B(...)                                                                                     \
  do {                                                                                               \
    cudaFuncSetAttribute(__VA_ARGS__, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);         \
    launch_pdl(__VA_ARGS__, dim3(grid), dim3(256), sm, S(stream), 1, (const TT*)dy, (const TT*)x, gamma, mean, \
               rstd, (const TT*)dres, (const TT*)gelu_z, (TT*)dx, dgamma, dbeta, col_sum, (int64_t)rows, H, dr,   \
               (TT*)dxd);                                                                             \
  } while (0)
  if (dxd != nullptr) {  // hidden dropout: the branch-gradient variant (no fused dgamma/dbeta in bf16)
    if (dtype == ESM_BF16) {
      using TT = __nv_bfloat16;
      if (stats) {
#define KS(A, B) ln_bwd_kernel<TT, A, B, true, false, true>
        LN_SWITCH2(KS);
#undef KS
      } else {
#define KS(A, B) ln_bwd_kernel<TT, A, B, false, false, true>
        LN_SWITCH2(KS);
#undef KS
      }
    } else {
      using TT = float;
      if (stats) {
#define KS(A, B) ln_bwd_kernel<TT, A, B, true, false, true>
        LN_SWITCH2(KS);
#undef KS
      } else {
#define KS(A, B) ln_bwd_kernel<TT, A, B, false, false, true>
        LN_SWITCH2(KS);
#undef KS
      }
    }
  } else if (dtype == ESM_BF16) {
    using TT = __nv_bfloat16;
    if (stats) {
#define KS(A, B) ln_bwd_kernel<TT, A, B, true>
      LN_SWITCH2(KS);
#undef KS
    } else if (sg) {
#define KS(A, B) ln_bwd_kernel<TT, A, B, false, ((A) <= 2)>
      LN_SWITCH2(KS);
#undef KS
    } else {
#define KS(A, B) ln_bwd_kernel<TT, A, B, false>
      LN_SWITCH2(KS);
#undef KS
    }
  } else {
    using TT = float;
    if (stats) {
#define KS(A, B) ln_bwd_kernel<TT, A, B, true>
      LN_SWITCH2(KS);
#undef KS
    } else {
#define KS(A, B) ln_bwd_kernel<TT, A, B, false>
      LN_SWITCH2(KS);
#undef KS
    }
  }
#undef L_B
  ESM_LAUNCH_RET();
}

int esm_qkv_rope_fwd(int dtype, const void* qkv, void* q, void* k, void* v, const float* cos_t, const float* sin_t,
                     int B, int Sq, int nh, int dh, float q_scale, esm_stream_t stream) {
  ESM_CHECK_ARG(qkv && q && k && v && cos_t && sin_t && dh % 2 == 0, "esm_qkv_rope_fwd: bad args");
  const int64_t T_ = (int64_t)B * Sq;
  const int grid = grid_for(T_ * nh * (dh / 2), 256);
  if (dtype == ESM_BF16)
    qkv_rope_fwd_kernel<__nv_bfloat16><<<grid, 256, 0, S(stream)>>>(
        (const __nv_bfloat16*)qkv, (__nv_bfloat16*)q, (__nv_bfloat16*)k, (__nv_bfloat16*)v, cos_t, sin_t, T_, Sq, nh,
        dh, q_scale);
  else
    qkv_rope_fwd_kernel<float><<<grid, 256, 0, S(stream)>>>((const float*)qkv, (float*)q, (float*)k, (float*)v, cos_t,
                                                            sin_t, T_, Sq, nh, dh, q_scale);
  ESM_LAUNCH_RET();
}

int esm_qkv_rope_bwd(int dtype, const float* dq, const void* dk, const void* dv, void* dqkv, float* col_sum,
                     const float* cos_t, const float* sin_t, int B, int Sq, int nh, int dh, float q_scale,
                     esm_stream_t stream) {
  ESM_CHECK_ARG(dq && dk && dv && dqkv && cos_t && sin_t && dh % 4 == 0, "esm_qkv_rope_bwd: bad args (dh %% 4)");
  const int64_t T_ = (int64_t)B * Sq;
  if (dtype == ESM_BF16 && (dh == 16 || dh == 32 || dh == 64) && T_ < (1ll << 31)) {
    const int TT = 512;  // tokens per block (one head)
    dim3 grid((unsigned)((T_ + TT - 1) / TT), (unsigned)nh);
#define QRB(CPR)                                                                                                  \
  launch_pdl(qkv_rope_bwd_tile_kernel<CPR>, dim3(grid), dim3(256), 0, S(stream), 1, dq, (const __nv_bfloat16*)dk, \
             (const __nv_bfloat16*)dv, (__nv_bfloat16*)dqkv, col_sum, cos_t, sin_t, (int)T_, Sq, nh, q_scale, TT)
    if (dh == 16) QRB(1);
    else if (dh == 32) QRB(2);
    else QRB(4);
#undef QRB
    ESM_LAUNCH_RET();
  }
  const int units = nh * dh / 4;  // two rotation pairs per thread
  const int bx = units >= 64 ? 64 : (units + 31) / 32 * 32;  // small blocks: many in flight per SM
  const int rpb = 32;
  dim3 grid((units + bx - 1) / bx, (unsigned)((T_ + rpb - 1) / rpb));
  if (dtype == ESM_BF16)
    qkv_rope_bwd_kernel<__nv_bfloat16><<<grid, bx, 0, S(stream)>>>(
        dq, (const __nv_bfloat16*)dk, (const __nv_bfloat16*)dv, (__nv_bfloat16*)dqkv, col_sum, cos_t, sin_t, T_, Sq,
        nh, dh, q_scale, rpb);
  else
    qkv_rope_bwd_kernel<float><<<grid, bx, 0, S(stream)>>>(dq, (const float*)dk, (const float*)dv, (float*)dqkv,
                                                           col_sum, cos_t, sin_t, T_, Sq, nh, dh, q_scale, rpb);
  ESM_LAUNCH_RET();
}

int esm_lmhead_xent(int dtype, const void* n, const void* E, const float* bias, const int32_t* labels,
                    const float* inv_denom, float* loss_sum, float* dlogits_ws, void* dn, float* dE, float* dbias,
                    int T_, int H, int V, esm_stream_t stream) {
  ESM_CHECK_ARG(n && E && bias && labels && inv_denom && loss_sum && dlogits_ws && dn && dE && dbias,
                "esm_lmhead_xent: null pointer");
  ESM_CHECK_ARG(V > 0 && V <= 64, "esm_lmhead_xent: V must be <= 64 (ESM alphabet is 33)");
  const int grid = grid_for((int64_t)T_ * 32, 256, device_sm_count() * 8);
  const int rpb = 512;
  dim3 g2((H + 31) / 32, (T_ + rpb - 1) / rpb);
  {  // preferred: E staged in shared memory (lanes over the vocabulary)
    const size_t esz = dtype == ESM_BF16 ? 2 : 4;
    const size_t pad = dtype == ESM_BF16 ? 2 : 1;
    const size_t smem = (((size_t)V * (H + pad) * esz + 15) & ~(size_t)15) + 8 * 64 * 4 + 8 * (size_t)H * esz;
    if (smem <= 200 * 1024 && H % 8 == 0) {
      // one resident wave (2 CTAs / SM): every CTA stages E once, so more CTAs only re-copy it
      const int g = grid_for((int64_t)T_ * 32, 256, device_sm_count() * 2);
      if (dtype == ESM_BF16) {
        cudaFuncSetAttribute(xent_small_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(xent_small_kernel<__nv_bfloat16>, dim3(g), dim3(256), smem, S(stream), 1, (const __nv_bfloat16*)n,
                   (const __nv_bfloat16*)E, bias, labels, inv_denom, loss_sum, dlogits_ws, (__nv_bfloat16*)dn, dbias,
                   T_, H, V);
        launch_pdl(xent_dE_kernel<__nv_bfloat16, 40>, dim3(g2), dim3(256), 0, S(stream), 1, (const __nv_bfloat16*)n,
                   labels, (const float*)dlogits_ws, dE, T_, H, V, rpb);
      } else {
        cudaFuncSetAttribute(xent_small_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        xent_small_kernel<float><<<g, 256, smem, S(stream)>>>((const float*)n, (const float*)E, bias, labels, inv_denom,
                                                             loss_sum, dlogits_ws, (float*)dn, dbias, T_, H, V);
        xent_dE_kernel<float, 40><<<g2, 256, 0, S(stream)>>>((const float*)n, labels, dlogits_ws, dE, T_, H, V, rpb);
      }
      ESM_LAUNCH_RET();
    }
  }
  if (V > 40) { esm::set_last_error("xent: V > 40 unsupported for this H"); return ESM_ENOTSUP; }
  if (dtype == ESM_BF16) {
    ESM_CHECK_ARG(H % 8 == 0, "xent: H %% 8");
    const int mv = (H + 255) / 256;
    auto* nn = (const __nv_bfloat16*)n;
    auto* ee = (const __nv_bfloat16*)E;
    auto* dd = (__nv_bfloat16*)dn;
#define XL(MV) xent_kernel<__nv_bfloat16, MV, 40><<<grid, 256, 0, S(stream)>>>(nn, ee, bias, labels, inv_denom, loss_sum, dlogits_ws, dd, dbias, T_, H, V)
    if (V > 40) { esm::set_last_error("xent: V > 40 unsupported in bf16 path"); return ESM_ENOTSUP; }
    if (mv <= 1) XL(1); else if (mv <= 2) XL(2); else if (mv <= 4) XL(4); else if (mv <= 6) XL(6); else if (mv <= 10) XL(10);
    else { esm::set_last_error("xent: H too large"); return ESM_ENOTSUP; }
#undef XL
    xent_dE_kernel<__nv_bfloat16, 40><<<g2, 256, 0, S(stream)>>>(nn, labels, dlogits_ws, dE, T_, H, V, rpb);
  } else {
    ESM_CHECK_ARG(H % 4 == 0, "xent: H %% 4");
    const int mv = (H + 127) / 128;
    auto* nn = (const float*)n;
    auto* ee = (const float*)E;
    auto* dd = (float*)dn;
#define XL(MV) xent_kernel<float, MV, 40><<<grid, 256, 0, S(stream)>>>(nn, ee, bias, labels, inv_denom, loss_sum, dlogits_ws, dd, dbias, T_, H, V)
    if (V > 40) { esm::set_last_error("xent: V > 40 unsupported"); return ESM_ENOTSUP; }
    if (mv <= 1) XL(1); else if (mv <= 2) XL(2); else if (mv <= 4) XL(4); else if (mv <= 6) XL(6); else if (mv <= 10) XL(10);
    else { esm::set_last_error("xent: H too large"); return ESM_ENOTSUP; }
#undef XL
    xent_dE_kernel<float, 40><<<g2, 256, 0, S(stream)>>>(nn, labels, dlogits_ws, dE, T_, H, V, rpb);
  }
  ESM_LAUNCH_RET();
}

int esm_adamw(float* p, const float* g, float* m, float* v, void* p16, const uint8_t* decay_chunk, int64_t n,
              const float* hyper, esm_stream_t stream) {
  ESM_CHECK_ARG(p && g && m && v && decay_chunk && hyper && n % 256 == 0, "esm_adamw: bad args (n %% 256 == 0)");
  adamw_kernel<float><<<grid_for(n / 4, 256, device_sm_count() * 8), 256, 0, S(stream)>>>(
      p, g, m, v, (__nv_bfloat16*)p16, decay_chunk, n, hyper);
  ESM_LAUNCH_RET();
}

int esm_adamw_bf16g(float* p, const void* g, float* m, float* v, void* p16, const uint8_t* decay_chunk, int64_t n,
                    const float* hyper, esm_stream_t stream) {
  ESM_CHECK_ARG(p && g && m && v && decay_chunk && hyper && n % 256 == 0, "esm_adamw_bf16g: bad args (n %% 256 == 0)");
  adamw_kernel<__nv_bfloat16><<<grid_for(n / 4, 256, device_sm_count() * 8), 256, 0, S(stream)>>>(
      p, (const __nv_bfloat16*)g, m, v, (__nv_bfloat16*)p16, decay_chunk, n, hyper);
  ESM_LAUNCH_RET();
}

int esm_cast_f32_bf16(const float* src, void* dst, int64_t n, esm_stream_t stream) {
  ESM_CHECK_ARG(src && dst && n >= 0 && ((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 7) == 0,
                "esm_cast_f32_bf16: bad args (src 16 B, dst 8 B aligned)");
  if (n == 0) return 0;
  cast_kernel<<<grid_for(n / 4 + 1, 256, device_sm_count() * 8), 256, 0, S(stream)>>>(src, (__nv_bfloat16*)dst, n);
  ESM_LAUNCH_RET();
}

int esm_dropout_mask(const esm_dropout* drop, int64_t rows, int cols, uint8_t* out, esm_stream_t stream) {
  ESM_CHECK_ARG(drop && out && rows >= 0 && cols > 0, "esm_dropout_mask: bad args");
  if (rows == 0) return 0;
  dropout_mask_kernel<<<grid_for(rows * ((cols + 1) / 2), 256), 256, 0, S(stream)>>>(*drop, rows, cols, out);
  ESM_LAUNCH_RET();
}

int esm_cast_bf16_f32(const void* src, float* dst, int64_t n, esm_stream_t stream) {
  ESM_CHECK_ARG(src && dst && n >= 0, "esm_cast_bf16_f32: bad args");
  if (n == 0) return 0;
  cast_bf16_f32_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>((const __nv_bfloat16*)src, dst, n);
  ESM_LAUNCH_RET();
}

}  // extern "C"

// Bulk-copy-staged LayerNorm forward / backward for bf16 activations (nn.LayerNorm, HF:modeling_esm.py:384,
// 394, 479, 511; the backward of the same).
//
// A row block of R consecutive token rows is one contiguous range of the token-major [T, H] tensors, so a
// single producer lane moves it into shared memory with one `cp.async.bulk` per tensor (completion counted on
// an mbarrier) into a 4-stage ring, while 8 consumer warps normalise the rows of the previous stages.  HBM
// reads are therefore always in flight independently of the consumers' reduction latency (the limit of the
// register-staged kernels in elementwise.cu), and the consumers read their rows from shared memory with
// conflict-free 16-byte vectors.  Persistent grid: one CTA per SM, row blocks strided over the grid.
//
//   forward   y = (x - mean) * rstd * gamma + beta;  mean, rstd per row (fp32)
//   backward  dx = rstd * (g - mean_H(g) - xhat * mean_H(g * xhat)) [+ dres],  g = dy * gamma, xhat = (x-mean)*rstd
//             col_sum += colsum(dx)  (or colsum(dx_drop) with hidden dropout: dx_drop = dx * keep * scale)
#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

namespace esm {
namespace lnb {
using namespace sm100;

constexpr int NWARP = 8;        // consumer warps
constexpr int MAX_STAGES = 4;
constexpr int SMEM_BUDGET = 192 * 1024;  // staged rows (all tensors, all stages)

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void unpack8(const uint4& u, float* o) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return u;
}

// ---------------------------------------------------------------------------------------------------- forward
// NV = 16-byte vectors per lane per row (ceil(H / 256)); gamma / beta stay in shared memory (fp32).
template <int NV>
__global__ void __launch_bounds__(32 * (NWARP + 1), 1)
    ln_fwd_bulk_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ gamma,
                       const float* __restrict__ beta, __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                       float* __restrict__ rstd_out, int64_t rows, int H, float eps, int R, int ns) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = R * H * 2;
  uint8_t* sx = smem;                                                    // [ns][R * H] bf16
  float* sg = reinterpret_cast<float*>(smem + ns * stage_bytes);    // gamma [H], beta [H]
  uint64_t* full = reinterpret_cast<uint64_t*>(sg + 2 * H);
  uint64_t* empty = full + ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    sg[i] = gamma[i];
    sg[H + i] = beta[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nblk = (rows + R - 1) / R;
  if (warp == NWARP) {  // producer
    if (lane == 0) {
      int it = 0;
      for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
        const int s = it % ns;
        mbar_wait(&empty[s], ((it / ns) & 1) ^ 1);
        const int64_t r0 = blk * R;
        const int nr = (int)(rows - r0 < R ? rows - r0 : R);
        const uint32_t bytes = (uint32_t)nr * H * 2;
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(sx + s * stage_bytes, x + r0 * H, bytes, &full[s]);
      }
    }
    return;
  }
  const float invH = 1.0f / H;
  int it = 0;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
    const int s = it % ns;
    mbar_wait(&full[s], (it / ns) & 1);
    const int64_t r0 = blk * R;
    const int nr = (int)(rows - r0 < R ? rows - r0 : R);
    const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(sx + s * stage_bytes);
    for (int rr = warp; rr < nr; rr += NWARP) {
      uint4 raw[NV];
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int h = (i * 32 + lane) * 8;
        if (h < H) {
          raw[i] = *reinterpret_cast<const uint4*>(rb + rr * H + h);
          float v[8];
          unpack8(raw[i], v);
#pragma unroll
          for (int e = 0; e < 8; ++e) sum += v[e];
        }
      }
      const float mu = warp_sum(sum) * invH;
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int h = (i * 32 + lane) * 8;
        if (h < H) {
          float v[8];
          unpack8(raw[i], v);
#pragma unroll
          for (int e = 0; e < 8; ++e) ss += (v[e] - mu) * (v[e] - mu);
        }
      }
      const float rs = rsqrtf(warp_sum(ss) * invH + eps);
      const int64_t r = r0 + rr;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int h = (i * 32 + lane) * 8;
        if (h < H) {
          float v[8], o[8];
          unpack8(raw[i], v);
          const float4 g0 = *reinterpret_cast<const float4*>(sg + h), g1 = *reinterpret_cast<const float4*>(sg + h + 4);
          const float4 b0 = *reinterpret_cast<const float4*>(sg + H + h);
          const float4 b1 = *reinterpret_cast<const float4*>(sg + H + h + 4);
          const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = (v[e] - mu) * rs * gg[e] + bb[e];
          *reinterpret_cast<uint4*>(y + r * H + h) = pack8(o);
        }
      }
      if (lane == 0) {
        mean_out[r] = mu;
        rstd_out[r] = rs;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// ---------------------------------------------------------------------------------------------------- backward
// Without dgamma / dbeta (the bf16 path fuses those into the producing dgrad GEMM's epilogue).  DROP: hidden
// dropout branch gradient dx_drop (and col_sum over it).
template <int NV, bool DROP>
__global__ void __launch_bounds__(32 * (NWARP + 1), 1)
    ln_bwd_bulk_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                       const float* __restrict__ gamma, const float* __restrict__ mean,
                       const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ dres,
                       __nv_bfloat16* __restrict__ dx, float* __restrict__ csum, int64_t rows, int H, int R,
                       int ns, const esm_dropout drop, __nv_bfloat16* __restrict__ dxd) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tb = R * H * 2;                     // one tensor's share of a stage
  const int nt = dres != nullptr ? 3 : 2;       // staged tensors: dy, x (, dres)
  const int stage_bytes = nt * tb;
  float* sg = reinterpret_cast<float*>(smem + ns * stage_bytes);   // gamma [H], col partials [H]
  float* scol = sg + H;
  uint64_t* full = reinterpret_cast<uint64_t*>(scol + H);
  uint64_t* empty = full + ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    sg[i] = gamma[i];
    scol[i] = 0.f;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nblk = (rows + R - 1) / R;
  if (warp == NWARP) {  // producer
    if (lane == 0) {
      int it = 0;
      for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
        const int s = it % ns;
        mbar_wait(&empty[s], ((it / ns) & 1) ^ 1);
        const int64_t r0 = blk * R;
        const int nr = (int)(rows - r0 < R ? rows - r0 : R);
        const uint32_t bytes = (uint32_t)nr * H * 2;
        uint8_t* st = smem + s * stage_bytes;
        mbar_expect_tx(&full[s], bytes * nt);
        bulk_g2s(st, dy + r0 * H, bytes, &full[s]);
        bulk_g2s(st + tb, x + r0 * H, bytes, &full[s]);
        if (dres != nullptr) bulk_g2s(st + 2 * tb, dres + r0 * H, bytes, &full[s]);
      }
    }
    __syncwarp();
  } else {
    DropKeys dk{0u, 0u, 0u, 1.f, false};
    if constexpr (DROP) dk = drop_keys(drop);
    const float invH = 1.0f / H;
    float acc[NV][8];
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[i][e] = 0.f;
    int it = 0;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
      const int s = it % ns;
      mbar_wait(&full[s], (it / ns) & 1);
      const int64_t r0 = blk * R;
      const int nr = (int)(rows - r0 < R ? rows - r0 : R);
      const uint8_t* st = smem + s * stage_bytes;
      const __nv_bfloat16* sdy = reinterpret_cast<const __nv_bfloat16*>(st);
      const __nv_bfloat16* sx = reinterpret_cast<const __nv_bfloat16*>(st + tb);
      const __nv_bfloat16* sr = reinterpret_cast<const __nv_bfloat16*>(st + 2 * tb);
      for (int rr = warp; rr < nr; rr += NWARP) {
        const int64_t r = r0 + rr;
        const float mu = mean[r], rs = rstd[r];
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int h = (i * 32 + lane) * 8;
          if (h < H) {
            float dv[8], xv[8];
            unpack8(*reinterpret_cast<const uint4*>(sdy + rr * H + h), dv);
            unpack8(*reinterpret_cast<const uint4*>(sx + rr * H + h), xv);
            const float4 g0 = *reinterpret_cast<const float4*>(sg + h);
            const float4 g1 = *reinterpret_cast<const float4*>(sg + h + 4);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float gy = dv[e] * gg[e];
              s1 += gy;
              s2 += gy * (xv[e] - mu) * rs;
            }
          }
        }
        s1 = warp_sum(s1) * invH;
        s2 = warp_sum(s2) * invH;
        const uint32_t rh = DROP ? drop_row(dk, (uint32_t)r) : 0u;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int h = (i * 32 + lane) * 8;
          if (h < H) {
            float dv[8], xv[8], o[8];
            unpack8(*reinterpret_cast<const uint4*>(sdy + rr * H + h), dv);
            unpack8(*reinterpret_cast<const uint4*>(sx + rr * H + h), xv);
            const float4 g0 = *reinterpret_cast<const float4*>(sg + h);
            const float4 g1 = *reinterpret_cast<const float4*>(sg + h + 4);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = rs * (dv[e] * gg[e] - s1 - (xv[e] - mu) * rs * s2);
            if (dres != nullptr) {
              float rv[8];
              unpack8(*reinterpret_cast<const uint4*>(sr + rr * H + h), rv);
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] += rv[e];
            }
            *reinterpret_cast<uint4*>(dx + r * H + h) = pack8(o);
            if constexpr (DROP) {
              float od[8];
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                const uint32_t kb = drop_pair(dk, rh, (uint32_t)(h + e) >> 1);
                od[e] = (kb & 1u) ? o[e] * dk.scale : 0.f;
                od[e + 1] = (kb & 2u) ? o[e + 1] * dk.scale : 0.f;
              }
              *reinterpret_cast<uint4*>(dxd + r * H + h) = pack8(od);
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[i][e] += od[e];
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[i][e] += o[e];
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (csum != nullptr) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int h = (i * 32 + lane) * 8;
        if (h < H)
#pragma unroll
          for (int e = 0; e < 8; ++e) atomicAdd(&scol[h + e], acc[i][e]);
      }
    }
  }
  __syncthreads();
  if (csum != nullptr)
    for (int c = threadIdx.x; c < H; c += blockDim.x) atomicAdd(csum + c, scol[c]);
}

// rows per stage for `tensors` staged tensors and `ns` stages within the shared-memory budget (0: does not fit)
inline int rows_per_stage(int H, int tensors, int ns) {
  int R = SMEM_BUDGET / ns / tensors / (H * 2);
  return R > 32 ? 32 : R;
}

}  // namespace lnb

#define LNB_NV_SWITCH(NV_, CALL)                     \
  switch (NV_) {                                     \
    case 1: CALL(1); break;                          \
    case 2: CALL(2); break;                          \
    case 3: CALL(3); break;                          \
    case 4: CALL(4); break;                          \
    case 5: CALL(5); break;                          \
    case 6: CALL(6); break;                          \
    case 8: CALL(8); break;                          \
    case 10: CALL(10); break;                        \
    case 12: CALL(12); break;                        \
    case 16: CALL(16); break;                        \
    default: return -1;                              \
  }

static int lnb_nv(int H) {
  const int nv = (H + 255) / 256;
  static const int ok[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16};
  for (int v : ok)
    if (nv <= v) return v;
  return -1;
}

// returns 0 (launched), -1 (shape not handled: caller uses the register-staged kernel), or a cudaError_t
int ln_fwd_bulk(const void* x, const float* gamma, const float* beta, void* y, float* mean, float* rstd, int64_t rows,
                int H, float eps, cudaStream_t st) {
  const int nv = lnb_nv(H);
  if (nv < 0 || H % 8 != 0 || rows <= 0) return -1;
  const int ns = lnb::MAX_STAGES;
  const int R = lnb::rows_per_stage(H, 1, ns);
  if (R < 1) return -1;
  const size_t smem = (size_t)ns * R * H * 2 + 2 * (size_t)H * 4 + 2 * ns * 8;
  const int64_t nblk = (rows + R - 1) / R;
  const int grid = (int)std::min<int64_t>(nblk, device_sm_count());
#define LNF(NV)                                                                                                   \
  {                                                                                                               \
    cudaFuncSetAttribute(lnb::ln_fwd_bulk_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    lnb::ln_fwd_bulk_kernel<NV><<<grid, 32 * (lnb::NWARP + 1), smem, st>>>(                                      \
        (const __nv_bfloat16*)x, gamma, beta, (__nv_bfloat16*)y, mean, rstd, rows, H, eps, R, ns);                   \
  }
  LNB_NV_SWITCH(nv, LNF)
#undef LNF
  return (int)cudaGetLastError();
}

int ln_bwd_bulk(const void* dy, const void* x, const float* gamma, const float* mean, const float* rstd,
                const void* dres, void* dx, float* csum, int64_t rows, int H, const esm_dropout* drop, void* dxd,
                cudaStream_t st) {
  const int nv = lnb_nv(H);
  if (nv < 0 || H % 8 != 0 || rows <= 0) return -1;
  const int nt = dres != nullptr ? 3 : 2;
  const int ns = 3;
  const int R = lnb::rows_per_stage(H, nt, ns);
  if (R < 1) return -1;
  const size_t smem = (size_t)ns * nt * R * H * 2 + 2 * (size_t)H * 4 + 2 * ns * 8;
  const int64_t nblk = (rows + R - 1) / R;
  const int grid = (int)std::min<int64_t>(nblk, device_sm_count());
  const bool dropping = drop != nullptr && drop->threshold != 0u && dxd != nullptr;
  const esm_dropout dr = dropping ? *drop : esm_dropout{nullptr, 0u, 0u, 1.f};
#define LNB(NV)                                                                                                   \
  {                                                                                                               \
    auto k = dropping ? lnb::ln_bwd_bulk_kernel<NV, true> : lnb::ln_bwd_bulk_kernel<NV, false>;                   \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                              \
    k<<<grid, 32 * (lnb::NWARP + 1), smem, st>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, gamma, mean,  \
                                                 rstd, (const __nv_bfloat16*)dres, (__nv_bfloat16*)dx, csum, rows, \
                                                 H, R, ns, dr, (__nv_bfloat16*)dxd);                               \
  }
  LNB_NV_SWITCH(nv, LNB)
#undef LNB
  return (int)cudaGetLastError();
}

}  // namespace esm

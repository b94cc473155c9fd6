// Common device helpers for the ESM-2 B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdlib>

#include "../../include/esm2_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "esm2_b200 kernels target sm_100a only"
#endif

namespace esm {

// ----------------------------------------------------------------------------
// error plumbing: every C-ABI entry returns 0 or a cudaError_t / ESM_E* code
// ----------------------------------------------------------------------------
void set_last_error(const char* fmt, ...);

#define ESM_CHECK_ARG(cond, ...)                         \
  do {                                                   \
    if (!(cond)) {                                       \
      ::esm::set_last_error(__VA_ARGS__);                \
      return ESM_EINVAL;                                 \
    }                                                    \
  } while (0)

#define ESM_LAUNCH_RET()                                                    \
  do {                                                                      \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess) {                                                \
      ::esm::set_last_error("%s:%d: %s", __FILE__, __LINE__,                \
                            cudaGetErrorString(_e));                        \
      return (int)_e;                                                       \
    }                                                                       \
    return 0;                                                               \
  } while (0)

// Counter-based dropout keep mask (include/esm2_b200.h esm_dropout; oracle/esm2_oracle.py:dropout_keep).
__host__ __device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
struct DropKeys {
  uint32_t k0, k1, thr;
  float scale;
  bool on;
};
__device__ __forceinline__ DropKeys drop_keys(const esm_dropout& d) {
  DropKeys k{0u, 0u, d.threshold, d.scale, d.seed != nullptr && d.threshold != 0};
  if (k.on) {
    const uint64_t s = *d.seed;
    k.k0 = (uint32_t)s ^ lowbias32(2u * d.site + 1u);
    k.k1 = (uint32_t)(s >> 32) ^ lowbias32(2u * d.site + 2u);
  }
  return k;
}
__device__ __forceinline__ uint32_t drop_row(const DropKeys& k, uint32_t row) {
  return lowbias32(row * 0x9E3779B1u ^ k.k0);
}
// keep bits of columns (2*pair, 2*pair + 1) of a row (rh = drop_row): bit 0 / bit 1
__device__ __forceinline__ uint32_t drop_pair(const DropKeys& k, uint32_t rh, uint32_t pair) {
  const uint32_t u = lowbias32(rh ^ (pair + k.k1));
  return ((u & 0xFFFFu) >= k.thr ? 1u : 0u) | ((u >> 16) >= k.thr ? 2u : 0u);
}

// ----------------------------------------------------------------------------
// Programmatic dependent launch (PDL): the step's kernels are launched with programmatic stream serialisation,
// so a kernel's CTAs are scheduled while its predecessor's last CTAs are still running (as SMs free up) and run
// their prologue (mbarrier init, TMEM allocation, tensor-map prefetch) early; `pdl_wait()` -- before the first
// global-memory access of every such kernel -- blocks until the predecessor grid has completed and its writes
// are visible.  `pdl_trigger()` lets the successor's launch begin.  Both are no-ops for normal launches.
// ESM_PDL=0 launches everything with full stream serialisation.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("ESM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// kernel launch with the PDL attribute (and an optional cluster size)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// SM count of the *current* device (cached per device id; launches size persistent grids with it).
// Function attributes (max dynamic shared memory) are likewise per device, so launchers set them on
// every launch rather than once per process (cheap, and legal during CUDA-graph capture).
inline int device_sm_count() {
  static int cache[64] = {0};
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v;
  }
  if (cache[d] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    cache[d] = v > 0 ? v : 148;
  }
  return cache[d];
}

// ----------------------------------------------------------------------------
// element I/O for the two activation dtypes (fp32 parity mode, bf16 production)
// ----------------------------------------------------------------------------
template <typename T> struct io;
template <> struct io<float> {
  static __device__ __forceinline__ float ld(const float* p) { return *p; }
  static __device__ __forceinline__ void st(float* p, float v) { *p = v; }
};
template <> struct io<__nv_bfloat16> {
  static __device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

// 16-byte vector of T (8 bf16 or 4 fp32)
template <typename T> struct vec16 { static constexpr int N = 16 / sizeof(T); };

template <typename T>
__device__ __forceinline__ void load_vec(const T* p, float* out) {
  if constexpr (sizeof(T) == 2) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      out[2 * i] = f.x;
      out[2 * i + 1] = f.y;
    }
  } else {
    float4 u = *reinterpret_cast<const float4*>(p);
    out[0] = u.x; out[1] = u.y; out[2] = u.z; out[3] = u.w;
  }
}

template <typename T>
__device__ __forceinline__ void store_vec(T* p, const float* v) {
  if constexpr (sizeof(T) == 2) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  } else {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// exact erf GELU (HF:modeling_esm.py:57-61) and its derivative
__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
  float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  float pdf = 0.39894228040143268f * __expf(-0.5f * x * x);
  return cdf + x * pdf;
}

// erf-GELU for the bf16 tcgen05 epilogues: one MUFU op per element.  erfc(x) = exp(-x^2) R(x) for x >= 0
// with R a degree-8 minimax fit on [0, 4] (relative error 2.8e-4: GELU / GELU' absolute error <= 4e-5 / 1.1e-4,
// ~2e-4 relative where GELU is not negligible, below the bf16 rounding of the stored result); R's argument
// is clamped at 4 (erfc(4) = 1.5e-8).  GELU(z) = max(z, 0) - |z|/2 * erfc(|z|/sqrt2).  The fp32 parity path uses erff.
__device__ __forceinline__ float erfc_core(float x, float& ex) {  // x >= 0; ex = exp(-x^2)
  const float xr = fminf(x, 4.0f);  // R fitted on [0, 4]; exp(-x^2) itself is not clamped
  float r = 1.1063529e-04f;
  r = fmaf(r, xr, -2.1946724e-03f);
  r = fmaf(r, xr, 1.8796470e-02f);
  r = fmaf(r, xr, -9.1806091e-02f);
  r = fmaf(r, xr, 2.8634080e-01f);
  r = fmaf(r, xr, -6.1150831e-01f);
  r = fmaf(r, xr, 9.4866168e-01f);
  r = fmaf(r, xr, -1.1205097e+00f);
  r = fmaf(r, xr, 9.9977970e-01f);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-1.4426950408889634f * x * x));
  ex = e;
  return e * r;
}
__device__ __forceinline__ float gelu_fast(float z) {
  const float x = fabsf(z) * 0.70710678118654752f;
  float ex;
  const float ec = erfc_core(x, ex);
  return fmaxf(z, 0.f) - 0.5f * fabsf(z) * ec;
}
// GELU(z) and GELU'(z) from one exp / erfc evaluation
__device__ __forceinline__ float gelu_and_grad_fast(float z, float& grad) {
  const float x = fabsf(z) * 0.70710678118654752f;
  float ex;
  const float ec = erfc_core(x, ex);
  const float cdf = z >= 0.f ? 1.f - 0.5f * ec : 0.5f * ec;
  grad = fmaf(z * 0.3989422804014327f, ex, cdf);
  return z * cdf;
}
// ---- packed fp32x2 arithmetic (sm_100 FFMA2/FMUL2/FADD2: two lanes' worth of fp32 per issue slot)
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_splat(float a) { return f2_pack(a, a); }

// Phi(z) and exp(-z^2/2) of two values at once: same erfc_core polynomial (coefficients pre-halved, exact),
// the arithmetic in f32x2, and Phi(z) = 0.5 + copysign(0.5 - h, z) with h = erfc(|z|/sqrt2)/2 instead of
// a compare-and-select.
__device__ __forceinline__ void phi_core2(uint64_t z, float z0, float z1, uint64_t& cdf, uint64_t& e) {
  const uint64_t x = f2_mul(z, f2_splat(0.70710678118654752f));
  float x0, x1;
  f2_unpack(x, x0, x1);
  const uint64_t xr = f2_pack(fminf(fabsf(x0), 4.0f), fminf(fabsf(x1), 4.0f));
  uint64_t r = f2_splat(0.5f * 1.1063529e-04f);
  r = f2_fma(r, xr, f2_splat(0.5f * -2.1946724e-03f));
  r = f2_fma(r, xr, f2_splat(0.5f * 1.8796470e-02f));
  r = f2_fma(r, xr, f2_splat(0.5f * -9.1806091e-02f));
  r = f2_fma(r, xr, f2_splat(0.5f * 2.8634080e-01f));
  r = f2_fma(r, xr, f2_splat(0.5f * -6.1150831e-01f));
  r = f2_fma(r, xr, f2_splat(0.5f * 9.4866168e-01f));
  r = f2_fma(r, xr, f2_splat(0.5f * -1.1205097e+00f));
  r = f2_fma(r, xr, f2_splat(0.5f * 9.9977970e-01f));
  const uint64_t t = f2_mul(f2_mul(x, x), f2_splat(-1.4426950408889634f));
  float t0, t1, e0, e1;
  f2_unpack(t, t0, t1);
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(t0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(t1));
  e = f2_pack(e0, e1);
  const uint64_t s = f2_fma(e, r, f2_splat(-0.5f));  // h - 0.5 <= 0
  float s0, s1;
  f2_unpack(s, s0, s1);
  // s ^ (~z & 0x80000000) as one LOP3 (immLut 0xD2 = a ^ (~b & c))
  asm("lop3.b32 %0, %0, %1, 0x80000000, 0xD2;" : "+f"(s0) : "f"(z0));
  asm("lop3.b32 %0, %0, %1, 0x80000000, 0xD2;" : "+f"(s1) : "f"(z1));
  cdf = f2_add(f2_pack(s0, s1), f2_splat(0.5f));
}
// GELU(z) = z Phi(z) and GELU'(z) = Phi(z) + z phi(z), two values at a time
__device__ __forceinline__ void gelu_and_grad_fast2(float& z0, float& z1, float& g0, float& g1) {
  const uint64_t z = f2_pack(z0, z1);
  uint64_t cdf, e;
  phi_core2(z, z0, z1, cdf, e);
  const uint64_t gd = f2_fma(f2_mul(z, f2_splat(0.3989422804014327f)), e, cdf);
  f2_unpack(f2_mul(z, cdf), z0, z1);
  f2_unpack(gd, g0, g1);
}
__device__ __forceinline__ void gelu_fast2(float& z0, float& z1) {
  const uint64_t z = f2_pack(z0, z1);
  uint64_t cdf, e;
  phi_core2(z, z0, z1, cdf, e);
  f2_unpack(f2_mul(z, cdf), z0, z1);
}
__device__ __forceinline__ void gelu_grad_fast2(float z0, float z1, float& g0, float& g1) {
  const uint64_t z = f2_pack(z0, z1);
  uint64_t cdf, e;
  phi_core2(z, z0, z1, cdf, e);
  f2_unpack(f2_fma(f2_mul(z, f2_splat(0.3989422804014327f)), e, cdf), g0, g1);
}
__device__ __forceinline__ float gelu_grad_fast(float z) {
  const float x = fabsf(z) * 0.70710678118654752f;
  float ex;
  const float ec = erfc_core(x, ex);
  const float cdf = z >= 0.f ? 1.f - 0.5f * ec : 0.5f * ec;
  return fmaf(z * 0.3989422804014327f, ex, cdf);  // Phi(z) + z * phi(z), phi = exp(-z^2/2) / sqrt(2 pi)
}

__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add_v4_f32(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// Sum 32 per-lane values v[0..31] across the warp so that lane j ends with
// sum_lanes v[j] (butterfly reduce-scatter, 31 shuffles).  Used for the fused
// bias-gradient column sums in GEMM epilogues.
__device__ __forceinline__ float warp_transpose_sum32(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      // keep half i (lower) or i+s (upper); send the other
      float send = upper ? v[i] : v[i + s];
      float keep = upper ? v[i + s] : v[i];
      float recv = __shfl_xor_sync(0xffffffffu, send, s);
      v[i] = keep + recv;
    }
  }
  return v[0];
}

}  // namespace esm

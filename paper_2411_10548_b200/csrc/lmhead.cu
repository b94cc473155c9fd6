// Large-vocabulary LM head (Geneformer, V ~ 25k; BASELINE configs[4]).
//
// For V <= 40 (ESM-2) the decoder + CE run fused per row in esm_lmhead_xent.  For large V the head is
// restricted to the labelled (masked) rows -- the only rows that carry loss (HF:modeling_esm.py:777-784):
//   esm_label_compact   deterministic stream compaction of labelled rows -> row index list (capacity-bounded)
//   esm_gather_rows     n_lab[i] = n[idx[i]]                               (rows past the count are zero)
//   esm_gemm            logits = n_lab · Eᵀ + bias  (tcgen05, tied decoder)
//   esm_xent_rows       per-row log-softmax CE over V, dlogits written in place (scaled by 1/N_labels)
//   esm_gemm            dn_lab = dlogits · E ;  dE += dlogitsᵀ · n_lab   (tcgen05 dgrad / wgrad)
//   esm_colsum_rows     dbias += Σ_rows dlogits
//   esm_scatter_rows    dn[idx[i]] = dn_lab[i], other rows 0
#include "common.cuh"

namespace esm {

static inline cudaStream_t S_(esm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// one block: contiguous chunks per thread, block-wide exclusive scan -> deterministic row order
__global__ void __launch_bounds__(1024) label_compact_kernel(const int32_t* __restrict__ labels, int64_t T,
                                                             int32_t* __restrict__ idx, int32_t* __restrict__ lab,
                                                             int32_t* __restrict__ count, int cap) {
  __shared__ int warp_tot[32];
  __shared__ int total;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t per = (T + blockDim.x - 1) / blockDim.x;
  const int64_t r0 = tid * per, r1 = min(T, r0 + per);
  int c = 0;
  for (int64_t r = r0; r < r1; ++r) c += labels[r] >= 0;
  // block exclusive scan of c
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive prefix over warps
    if (lane == 31) total = t;
  }
  __syncthreads();
  int pos = x - c + (w > 0 ? warp_tot[w - 1] : 0);
  for (int64_t r = r0; r < r1; ++r) {
    const int l = labels[r];
    if (l >= 0) {
      if (pos < cap) {
        idx[pos] = (int32_t)r;
        lab[pos] = l;
      }
      ++pos;
    }
  }
  __syncthreads();
  for (int i = total + tid; i < cap; i += blockDim.x) {
    idx[i] = -1;
    lab[i] = -100;
  }
  if (tid == 0) *count = total;
}

template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ src, const int32_t* __restrict__ idx, T* __restrict__ dst,
                                   int cap, int H) {
  constexpr int VEC = vec16<T>::N;
  const int64_t nv = (int64_t)cap * (H / VEC);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / (H / VEC);
    const int col = (int)(i % (H / VEC)) * VEC;
    const int r = idx[row];
    float v[VEC];
    if (r >= 0) {
      load_vec(src + (int64_t)r * H + col, v);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) v[e] = 0.f;
    }
    store_vec(dst + row * H + col, v);
  }
}

template <typename T>
__global__ void scatter_rows_kernel(const T* __restrict__ src, const int32_t* __restrict__ idx, T* __restrict__ dst,
                                    int cap, int H) {
  constexpr int VEC = vec16<T>::N;
  const int64_t nv = (int64_t)cap * (H / VEC);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / (H / VEC);
    const int col = (int)(i % (H / VEC)) * VEC;
    const int r = idx[row];
    if (r >= 0) *reinterpret_cast<uint4*>(dst + (int64_t)r * H + col) = *reinterpret_cast<const uint4*>(src + row * H + col);
  }
}

// one block per labelled row: max / sum-exp over V, loss, dlogits = (softmax - onehot) * inv (in place)
template <typename T>
__global__ void __launch_bounds__(256) xent_rows_kernel(T* __restrict__ logits, const int32_t* __restrict__ lab,
                                                        int V, int64_t ld, const float* __restrict__ inv_denom,
                                                        float* __restrict__ loss_sum) {
  __shared__ float red[8];
  __shared__ float bc;
  const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  T* x = logits + (int64_t)row * ld;
  const int l = lab[row];
  if (l < 0) {  // padding row: zero gradient
    for (int c = tid; c < ld; c += blockDim.x) io<T>::st(x + c, 0.f);
    return;
  }
  float mx = -INFINITY;
  for (int c = tid; c < V; c += blockDim.x) mx = fmaxf(mx, io<T>::ld(x + c));
  mx = warp_max(mx);
  if (lane == 0) red[w] = mx;
  __syncthreads();
  if (tid == 0) {
    float m = red[0];
    for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i]);
    bc = m;
  }
  __syncthreads();
  mx = bc;
  float se = 0.f;
  for (int c = tid; c < V; c += blockDim.x) se += __expf(io<T>::ld(x + c) - mx);
  se = warp_sum(se);
  __syncthreads();
  if (lane == 0) red[w] = se;
  __syncthreads();
  if (tid == 0) {
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += red[i];
    const float lse = mx + __logf(s);
    const float inv = *inv_denom;
    atomicAdd(loss_sum, (lse - io<T>::ld(x + l)) * inv);
    bc = lse;
  }
  __syncthreads();
  const float lse = bc, inv = *inv_denom;
  for (int c = tid; c < ld; c += blockDim.x) {
    float d = 0.f;
    if (c < V) d = (__expf(io<T>::ld(x + c) - lse) - (c == l ? 1.f : 0.f)) * inv;
    io<T>::st(x + c, d);
  }
}

// out[c] += sum_rows x[r, c] for c < V (one thread per column, coalesced rows)
template <typename T>
__global__ void colsum_rows_kernel(const T* __restrict__ x, int rows, int V, int64_t ld, float* __restrict__ out,
                                   int rows_per_block) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= V) return;
  const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  float s = 0.f;
  for (int r = r0; r < r1; ++r) s += io<T>::ld(x + (int64_t)r * ld + c);
  if (s != 0.f) atomicAdd(out + c, s);
}

}  // namespace esm

using namespace esm;

extern "C" {

int esm_label_compact(const int32_t* labels, int64_t T, int32_t* idx, int32_t* lab, int32_t* count, int cap,
                      esm_stream_t stream) {
  ESM_CHECK_ARG(labels && idx && lab && count && T > 0 && cap > 0, "esm_label_compact: bad args");
  label_compact_kernel<<<1, 1024, 0, S_(stream)>>>(labels, T, idx, lab, count, cap);
  ESM_LAUNCH_RET();
}

int esm_gather_rows(int dtype, const void* src, const int32_t* idx, void* dst, int cap, int H, esm_stream_t stream) {
  ESM_CHECK_ARG(src && idx && dst && cap > 0 && H % 8 == 0, "esm_gather_rows: bad args");
  int64_t g = ((int64_t)cap * H / 4 + 255) / 256;
  if (g > device_sm_count() * 16) g = device_sm_count() * 16;
  if (dtype == ESM_BF16)
    gather_rows_kernel<__nv_bfloat16><<<(int)g, 256, 0, S_(stream)>>>((const __nv_bfloat16*)src, idx,
                                                                      (__nv_bfloat16*)dst, cap, H);
  else
    gather_rows_kernel<float><<<(int)g, 256, 0, S_(stream)>>>((const float*)src, idx, (float*)dst, cap, H);
  ESM_LAUNCH_RET();
}

int esm_scatter_rows(int dtype, const void* src, const int32_t* idx, void* dst, int cap, int H, int64_t T,
                     esm_stream_t stream) {
  ESM_CHECK_ARG(src && idx && dst && cap > 0 && H % 8 == 0, "esm_scatter_rows: bad args");
  cudaMemsetAsync(dst, 0, (size_t)T * H * (dtype == ESM_BF16 ? 2 : 4), S_(stream));
  int64_t g = ((int64_t)cap * H / 4 + 255) / 256;
  if (g > device_sm_count() * 16) g = device_sm_count() * 16;
  if (dtype == ESM_BF16)
    scatter_rows_kernel<__nv_bfloat16><<<(int)g, 256, 0, S_(stream)>>>((const __nv_bfloat16*)src, idx,
                                                                       (__nv_bfloat16*)dst, cap, H);
  else
    scatter_rows_kernel<float><<<(int)g, 256, 0, S_(stream)>>>((const float*)src, idx, (float*)dst, cap, H);
  ESM_LAUNCH_RET();
}

int esm_xent_rows(int dtype, void* logits, const int32_t* lab, int rows, int V, int64_t ld, const float* inv_denom,
                  float* loss_sum, esm_stream_t stream) {
  ESM_CHECK_ARG(logits && lab && inv_denom && loss_sum && rows > 0 && V > 0 && ld >= V, "esm_xent_rows: bad args");
  if (dtype == ESM_BF16)
    xent_rows_kernel<__nv_bfloat16><<<rows, 256, 0, S_(stream)>>>((__nv_bfloat16*)logits, lab, V, ld, inv_denom,
                                                                   loss_sum);
  else
    xent_rows_kernel<float><<<rows, 256, 0, S_(stream)>>>((float*)logits, lab, V, ld, inv_denom, loss_sum);
  ESM_LAUNCH_RET();
}

int esm_colsum_rows(int dtype, const void* x, int rows, int V, int64_t ld, float* out, esm_stream_t stream) {
  ESM_CHECK_ARG(x && out && rows > 0 && V > 0, "esm_colsum_rows: bad args");
  const int rpb = 256;
  dim3 grid((V + 255) / 256, (rows + rpb - 1) / rpb);
  if (dtype == ESM_BF16)
    colsum_rows_kernel<__nv_bfloat16><<<grid, 256, 0, S_(stream)>>>((const __nv_bfloat16*)x, rows, V, ld, out, rpb);
  else
    colsum_rows_kernel<float><<<grid, 256, 0, S_(stream)>>>((const float*)x, rows, V, ld, out, rpb);
  ESM_LAUNCH_RET();
}

}  // extern "C"

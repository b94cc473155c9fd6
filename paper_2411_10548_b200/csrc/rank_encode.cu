// Geneformer rank-value tokenisation on the GPU (reference pkg/src/densefeed/tokenizer.py:68-83).
//
// rank_encode(row) = cols sorted by score = val / median[col] (fp64) descending, ties by ascending gene
// index, truncated to max_len, id = gene + 2.  One CTA per output row: the row's (key, col) pairs are
// staged in shared memory and bitonic-sorted; key = order-preserving uint64 image of -score, so the
// ascending (key, col) order is exactly numpy's stable argsort(cols) then stable argsort(-score):
//   * equal scores -> ascending col (the reference's tie rule), -0.0 == +0.0,
//   * NaN scores last (numpy's argsort puts NaN at the end), ascending col among them.
// The CTA then writes the padded batch row ([S] ids, PAD=0 past the length) and its attention mask, so a
// batch of CSR rows goes from the mmap'd store straight to the train step's input tensors.
#include "common.cuh"

namespace esm {

static inline cudaStream_t S_rank(esm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ uint64_t desc_key(double score) {
  if (score != score) return ~0ull;  // NaN: last
  if (score == 0.0) score = 0.0;     // fold -0.0
  const uint64_t b = (uint64_t)__double_as_longlong(score);
  const uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending image of score
  return ~asc;  // descending; ~0 only for NaN (asc == 0 is a NaN bit pattern)
}

__device__ __forceinline__ bool pair_less(uint64_t ka, uint32_t ca, uint64_t kb, uint32_t cb) {
  return ka < kb || (ka == kb && ca < cb);
}

__global__ void __launch_bounds__(1024) rank_encode_kernel(const int64_t* __restrict__ indptr,
                                                           const int64_t* __restrict__ cols,
                                                           const float* __restrict__ vals,
                                                           const float* __restrict__ medians, int64_t n_genes,
                                                           const int64_t* __restrict__ rows, int max_len, int S,
                                                           int pad_id, int offset, int32_t* __restrict__ ids,
                                                           int32_t* __restrict__ am, int32_t* __restrict__ lengths,
                                                           int32_t* __restrict__ status, int cap) {
  extern __shared__ uint64_t sm_keys[];  // [cap] keys, then [cap] uint32 cols (cap = staging capacity, pow2)
  const int b = blockIdx.x, tid = threadIdx.x;
  const int64_t r = rows ? rows[b] : b;
  const int64_t beg = indptr[r], n64 = indptr[r + 1] - beg;
  int32_t* out = ids + (int64_t)b * S;
  int32_t* mk = am + (int64_t)b * S;
  int64_t keep64 = n64 < max_len ? n64 : max_len;
  if (keep64 > S) keep64 = S;
  const int K = (int)keep64;  // tokens written
  if (n64 < 0 || (n64 > cap && K > cap / 2)) {  // a long row whose kept prefix does not fit the streaming top-K
    if (tid == 0) atomicExch(status, 2);
    for (int i = tid; i < S; i += blockDim.x) { out[i] = pad_id; mk[i] = 0; }
    if (tid == 0 && lengths) lengths[b] = 0;
    return;
  }
  // rows up to the staging capacity: one sort of the next power of two >= n.  Longer rows: streaming top-K --
  // slots [0, K) hold the best K so far, each chunk of cap - K entries is loaded behind them and the whole
  // buffer re-sorted, so [0, K) ends as the K smallest (key, col) of the row, i.e. exactly the prefix a full
  // sort would give.
  int P = 1;
  while (P < n64 && P < cap) P <<= 1;
  uint64_t* key = sm_keys;
  uint32_t* col = reinterpret_cast<uint32_t*>(sm_keys + P);
  const bool stream = n64 > P;
  const int head = stream ? K : 0;
  const int64_t chunk = P - head;
  for (int i = tid; i < head; i += blockDim.x) {
    key[i] = ~0ull;
    col[i] = 0xFFFFFFFFu;
  }
  for (int64_t c0 = 0; c0 < n64 || c0 == 0; c0 += chunk) {
    for (int i = head + tid; i < P; i += blockDim.x) {
      const int64_t e = c0 + (i - head);
      if (e < n64) {
        const int64_t c = cols[beg + e];
        if (c < 0 || c >= n_genes) {
          atomicExch(status, 1);
          key[i] = ~0ull;
          col[i] = 0xFFFFFFFFu;
        } else {
          key[i] = desc_key((double)vals[beg + e] / (double)medians[c]);
          col[i] = (uint32_t)c;
        }
      } else {  // padding sorts after every real element
        key[i] = ~0ull;
        col[i] = 0xFFFFFFFFu;
      }
    }
    __syncthreads();
    // bitonic sort, ascending by (key, col)
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < P; i += blockDim.x) {
          const int l = i ^ j;
          if (l > i) {
            const bool up = (i & k) == 0;
            const uint64_t ki = key[i], kl = key[l];
            const uint32_t ci = col[i], cl = col[l];
            if (pair_less(kl, cl, ki, ci) == up) {
              key[i] = kl; key[l] = ki;
              col[i] = cl; col[l] = ci;
            }
          }
        }
        __syncthreads();
      }
    }
    if (!stream) break;
  }
  for (int i = tid; i < S; i += blockDim.x) {
    const bool v = i < K;
    out[i] = v ? (int32_t)col[i] + offset : pad_id;
    mk[i] = v ? 1 : 0;
  }
  if (tid == 0 && lengths) lengths[b] = K;
}

}  // namespace esm

using namespace esm;

extern "C" int esm_rank_encode(const int64_t* indptr, const int64_t* cols, const float* vals, const float* medians,
                               int64_t n_genes, const int64_t* rows, int n_rows, int max_len, int S, int32_t* ids,
                               int32_t* am, int32_t* lengths, int32_t* status, int max_nnz, esm_stream_t stream) {
  ESM_CHECK_ARG(indptr && medians && ids && am && status && n_rows >= 0 && max_len >= 0 && S > 0 && n_genes > 0 &&
                    n_genes < 0xFFFFFFFFll,
                "esm_rank_encode: bad args");
  ESM_CHECK_ARG(max_nnz >= 0, "esm_rank_encode: max_nnz >= 0");
  if (n_rows == 0) return 0;
  int P = 1;  // staging capacity: next power of two >= the longest row, at most 16384 (192 KB of shared memory)
  while (P < max_nnz && P < 16384) P <<= 1;
  const size_t smem = (size_t)P * (sizeof(uint64_t) + sizeof(uint32_t));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rank_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_last_error("esm_rank_encode: %s", cudaGetErrorString(e));
      return (int)e;
    }
  }
  const int threads = P >= 1024 ? 1024 : (P < 64 ? 64 : P);
  rank_encode_kernel<<<n_rows, threads, smem, S_rank(stream)>>>(indptr, cols, vals, medians, n_genes, rows, max_len,
                                                                 S, 0, 2, ids, am, lengths, status, P);
  ESM_LAUNCH_RET();
}

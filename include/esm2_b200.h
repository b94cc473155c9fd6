/*
 * esm2_b200.h -- C ABI of the B200-native (sm_100a) ESM-2 MLM train-step kernels.
 *
 * Boundary
 * --------
 * The reference (/root/reference, the `densefeed` data toolkit) has no model,
 * kernel or FFI for this path: there is no
 * reference C interface to replace.  Each entry point below replaces one
 * operator of the Hugging Face EsmForMaskedLM forward/backward that the
 * reference's training loop would call (third-party semantics, transformers
 * 5.5.0 `models/esm/modeling_esm.py`, "HF:" below), and the whole step is
 * invoked through the reference seam `densefeed.sizing.collect_peak_alloc(
 * samples, workload, feature_fn, meter)` (pkg/src/densefeed/sizing.py:76-100)
 * by the Python host layer (paper_2411_10548_b200.seams).
 *
 * Conventions
 * ---------------------------
 *  - plain device pointers + sizes; no torch types; the caller owns all memory
 *    (kernels never allocate); every call is asynchronous on `stream`.
 *  - every call returns 0 on success, an ESM_E* code on bad arguments, or the
 *    cudaError_t of a failed launch; esm_last_error() describes the failure.
 *  - `dtype` selects the activation type: ESM_F32 (fp32 parity mode, SIMT
 *    kernels) or ESM_BF16 (production: tcgen05/TMEM/TMA GEMMs and flash
 *    attention, vectorised warp-shuffle epilogues).  Parameters are fp32 masters with
 *    a bf16 shadow for GEMM operands; gradients are always fp32.
 *  - activations are token-major: row t = b*S + s of a [T, width] matrix.
 *  - the step's bf16 kernels are launched with programmatic dependent launch: a kernel may be scheduled while
 *    its stream predecessor drains, but waits (griddepcontrol.wait) for the predecessor's completion before
 *    touching memory, so stream-order semantics are unchanged (environment ESM_PDL=0 disables it).
 */
#ifndef ESM2_B200_H
#define ESM2_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* esm_stream_t; /* a cudaStream_t */

enum { ESM_F32 = 0, ESM_BF16 = 1, ESM_I32 = 2 /* collectives only */ };
enum { ESM_OK = 0, ESM_EINVAL = 1001, ESM_ENOTSUP = 1002, ESM_EDRIVER = 1003, ESM_ENCCL_BASE = 2000 /* + ncclResult_t */ };

/* GEMM epilogues (applied to acc = A·Bᵀ, fp32) */
enum {
  ESM_EPI_STORE = 0,      /* C = acc (+ bias[n])                         act dtype    HF nn.Linear          */
  ESM_EPI_GELU = 1,       /* Z = acc + bias; C = gelu(Z)  (Z -> aux_out)  act dtype    HF:406-414, 57-61     */
  ESM_EPI_RESID = 2,      /* C = acc + bias + R           (R = aux_in)    act dtype    HF:365-375, 417-427   */
  ESM_EPI_DGELU = 3,      /* C = acc * gelu'(Z) (Z = aux_in); colsum(C) -> col_sum     backward of HF:411-414 */
  ESM_EPI_F32_ACC = 4,    /* C(fp32) += acc  (weight gradients; split-K safe)                               */
  ESM_EPI_QKV_ROPE = 5,   /* acc + bias -> q*scale, RoPE(q), RoPE(k), v scattered to [B,nh,S,dh]  HF:318-344 (bf16) */
  ESM_EPI_STORE_LN = 6,   /* C = acc = dy of a LayerNorm; col_sum += colsum(dy) (dbeta), col_sum2 += colsum(dy * xhat)
                             (dgamma) with xhat = (X - row_mean) * row_rstd, X = aux_in (the LN input)  (bf16)   */
  ESM_EPI_GELU_GRADAUX = 7, /* Z = acc + bias; C = gelu(Z), aux_out = gelu'(Z)  (bf16: the FC1 forward keeps the
                               derivative its backward needs, computed from the same exp/erfc evaluation)        */
  ESM_EPI_MUL_AUX = 8,      /* C = acc * G (G = aux_in, e.g. gelu'(Z) from GELU_GRADAUX); colsum(C) -> col_sum (bf16) */
  ESM_EPI_DELTA = 9         /* C = acc = dO (attention output gradient, token-major [M = B*seq_len, N = n_heads*head_dim]);
                               row_dot[b, h, s] = sum_{c in head h} bf16(C[t, c]) * O[t, c]  (O = aux_in, t = b*seq_len+s):
                               the attention backward's Delta = rowsum(dO o O) (HF:257-282 backward); replaces a
                               separate pass over dO and O (bf16, B N-major dgrad only)                            */
};

/* Hidden dropout (HF EsmSelfOutput / EsmOutput, HF:modeling_esm.py:369-375, 421-427): counter-based keep mask,
 * regenerated in the backward instead of stored.  For element (row r, column c) of a call site:
 *   k0 = lo32(seed) ^ h(2*site+1),  k1 = hi32(seed) ^ h(2*site+2),  h = lowbias32
 *   u  = h(h(r * 0x9E3779B1 ^ k0) ^ ((c >> 1) + k1));  bits = c odd ? u >> 16 : u & 0xFFFF
 *   keep = bits >= threshold   (threshold = round(p * 65536));  kept values are scaled by `scale` = 1/(1-p).
 * Bit-exact with oracle/esm2_oracle.py:dropout_keep. */
typedef struct esm_dropout {
  const uint64_t* seed; /* device pointer, per-step seed (read at run time: CUDA-graph safe); NULL = off */
  uint32_t site;        /* call site: 2*layer + 0 (attention output) / 1 (FFN output) */
  uint32_t threshold;   /* 0 = off */
  float scale;
} esm_dropout;

typedef struct esm_gemm_args {
  int dtype;                 /* ESM_F32 / ESM_BF16: dtype of A, B and activation outputs        */
  int M, N, K;               /* C[M,N] = A[M,K] · B[N,K]ᵀ                                        */
  const void* A; int64_t lda; int a_mn_major; /* 0: A[m*lda+k]   1: A[k*lda+m]                   */
  const void* B; int64_t ldb; int b_mn_major; /* 0: B[n*ldb+k]   1: B[k*ldb+n]                   */
  void* C; int64_t ldc;
  int epilogue;
  const float* bias;         /* [N] fp32 or NULL                                                   */
  const void* aux_in; int64_t ld_aux_in;    /* residual R or pre-activation Z                      */
  void* aux_out; int64_t ld_aux_out;        /* GELU pre-activation Z output                        */
  float* col_sum;            /* [N] fp32 accumulated column sums (bias grad) or NULL               */
  int split_k;               /* ESM_EPI_F32_ACC only; 0 = auto                                     */
  /* ESM_EPI_QKV_ROPE only: N = 3*n_heads*head_dim, rows t = b*seq_len + s */
  const float* rope_cos;     /* [seq_len, head_dim/2] fp32 */
  const float* rope_sin;
  void* q_out; void* k_out; void* v_out;   /* [B, n_heads, seq_len, head_dim] */
  int seq_len, n_heads, head_dim;
  float q_scale;
  /* ESM_EPI_STORE_LN only */
  const float* row_mean;     /* [M] */
  const float* row_rstd;     /* [M] */
  float* col_sum2;           /* [N] */
  /* ESM_EPI_RESID only: C = R + dropout(acc + bias) */
  esm_dropout drop;
  /* ESM_EPI_DELTA only: [B, n_heads, seq_len] fp32 per-head row dot products (zeroed, then reduced into, by the
     callee on `stream`) */
  float* row_dot;
} esm_gemm_args;

/* ---------------- library ---------------- */
int esm_version(void);
const char* esm_last_error(void);
int esm_device_sm_count(int device);

/* ---------------- data path ---------------- */
/* Host: ESM-2 alphabet tokenizer.  out = <cls> ids <eos>; returns #ids (or -needed if max_out small). */
int esm_tokenize(const char* seq, int len, int32_t* out, int max_out);
/* Device: 15% / 80-10-10 MLM masking (splitmix64 counter RNG, integer thresholds;
 * bit-exact with oracle/esm2_oracle.py:mlm_mask).  Also counts labelled tokens into *n_labels (int32, accumulated). */
int esm_mlm_mask(const int32_t* ids, int32_t* input_ids, int32_t* labels, int32_t* n_labels, int64_t n,
                 uint64_t seed, uint64_t stream_id, esm_stream_t stream);
/* Same draws, vocabulary given explicitly (Geneformer: eligible [2, V-1], <mask>=1, random from [2, V-1];
 * reference pkg/src/densefeed/tokenizer.py:16-18 PAD_ID/MASK_ID/TOKEN_OFFSET).  Selected ids in
 * [elig_lo, elig_hi]; 80% -> mask_id, 10% -> rand_lo + (r % rand_n), 10% kept. */
int esm_mlm_mask_ex(const int32_t* ids, int32_t* input_ids, int32_t* labels, int32_t* n_labels, int64_t n,
                    uint64_t seed, uint64_t stream_id, int elig_lo, int elig_hi, int mask_id, int rand_lo,
                    int rand_n, esm_stream_t stream);

/* Device: Geneformer rank-value tokenisation of CSR expression rows (replaces the reference's
 * rank_encode, pkg/src/densefeed/tokenizer.py:68-83, applied per row as in corpus.py / bindings __getitem__).
 * For output row b (source row rows[b], or b when rows == NULL): score = (double)vals / (double)medians[col],
 * order = descending score, ties by ascending col, truncate to min(max_len, S), id = col + 2 (TOKEN_OFFSET),
 * PAD = 0 past the length; am[b, i] = i < length.  lengths[b] (optional) = tokens written.
 * *status (caller zeroes): 1 = a col >= n_genes (the reference's ValidationError), 2 = a row has more
 * than max_nnz entries (<= 16384, staged in shared memory). */
int esm_rank_encode(const int64_t* indptr, const int64_t* cols, const float* vals, const float* medians,
                    int64_t n_genes, const int64_t* rows, int n_rows, int max_len, int S, int32_t* ids, int32_t* am,
                    int32_t* lengths, int32_t* status, int max_nnz, esm_stream_t stream);

/* ---------------- embeddings (HF:modeling_esm.py:189-236) ---------------- */
/* x[t,:] = E[ids[t]] * (ids!=mask) * row_scale[b] * am[t];  row_scale = 0.88/(1 - n_mask/len) (token_dropout). */
int esm_embed_fwd(int dtype, const int32_t* ids, const int32_t* am, const void* E, void* x, float* row_scale,
                  int B, int S, int H, int token_dropout, int mask_id, esm_stream_t stream);
/* dE[v,:] += sum_{t: ids[t]=v, v!=pad, v!=mask_id} dx[t,:] * row_scale[b] * am[t]   (fp32).  mask_id = the
 * token-dropout mask id (its rows were zeroed in the forward), or -1 without token dropout.  V <= 128:
 * shared-memory column accumulators; larger V (Geneformer): per-row vector fp32 atomics. */
int esm_embed_bwd(int dtype, const int32_t* ids, const int32_t* am, const float* row_scale, const void* dx,
                  float* dE, int B, int S, int H, int V, int mask_id, int pad_id, esm_stream_t stream);

/* ---------------- LayerNorm (nn.LayerNorm, eps) ---------------- */
int esm_layernorm_fwd(int dtype, const void* x, const float* gamma, const float* beta, void* y, float* mean,
                      float* rstd, int rows, int H, float eps, esm_stream_t stream);
/* dx = LNᵀ(dy) [+ dres]; optional: dx *= gelu'(gelu_z) (LM head), dgamma/dbeta += , col_sum += colsum(dx).
 * With drop (threshold > 0) and dx_drop: dx_drop = dx * keep * scale -- the gradient of the dropped-out branch
 * whose output fed this LayerNorm's input residual sum -- and col_sum accumulates colsum(dx_drop) (that branch's
 * bias gradient). */
int esm_layernorm_bwd(int dtype, const void* dy, const void* x, const float* gamma, const float* mean,
                      const float* rstd, const void* dres, const void* gelu_z, void* dx, float* dgamma,
                      float* dbeta, float* col_sum, int rows, int H, const esm_dropout* drop, void* dx_drop,
                      esm_stream_t stream);
/* out[r * cols + c] = keep(r, c) (uint8) -- the dropout mask of a call site, for tests. */
int esm_dropout_mask(const esm_dropout* drop, int64_t rows, int cols, uint8_t* out, esm_stream_t stream);

/* ---------------- linear layers ---------------- */
int esm_gemm(const esm_gemm_args* args, esm_stream_t stream);

/* ---------------- rotary + head layout (HF:modeling_esm.py:318-344) ---------------- */
/* qkv[T,3H] (bias already added) -> q,k,v [B,nh,S,dh]; q *= q_scale, then RoPE(q), RoPE(k). cos/sin: [S, dh/2] fp32. */
int esm_qkv_rope_fwd(int dtype, const void* qkv, void* q, void* k, void* v, const float* cos_t, const float* sin_t,
                     int B, int S, int nh, int dh, float q_scale, esm_stream_t stream);
/* dq (fp32 [B,nh,S,dh]), dk, dv ([B,nh,S,dh] act dtype) -> dqkv[T,3H] with RoPEᵀ and q_scale; col_sum[3H] += bias grads. */
int esm_qkv_rope_bwd(int dtype, const float* dq, const void* dk, const void* dv, void* dqkv, float* col_sum,
                     const float* cos_t, const float* sin_t, int B, int S, int nh, int dh, float q_scale,
                     esm_stream_t stream);

/* ---------------- attention (HF:modeling_esm.py:257-282; scaling = 1) ---------------- */
/* The bf16 attention kernels are persistent (one or two CTAs per SM looping over (head, tile) work claimed from
 * a counter).  Their scheduling state lives in a caller-owned workspace `sched` (int32[ESM_ATTN_SCHED_WORDS(B)],
 * no global mutable state): esm_attn_prepare records each batch row's valid-key count / prefix flag from
 * key_mask and zeroes the work counters; every fwd / bwd kernel leaves the counters at zero when it finishes,
 * so one prepared buffer serves all layers of a step while key_mask is unchanged.  Attention calls that may
 * run concurrently (different streams) need distinct `sched` buffers.  fp32 calls ignore `sched` (may be NULL). */
#define ESM_ATTN_SCHED_WORDS(B) (16 + 2 * (int64_t)(B))
int esm_attn_prepare(const int32_t* key_mask, int32_t* sched, int B, int S, esm_stream_t stream);
/* q,k,v [B,nh,S,dh]; key_mask [B,S] int32 (0 = padded key); o [T, nh*dh]; lse [B,nh,S] fp32 holds each row's
 * log-normaliser in the form the backward consumes, -log2(sum_k exp(s_k)) = -LSE * log2(e).
 * bf16: S % 4 == 0 (the collate step pads to a multiple of 8). */
int esm_attn_fwd(int dtype, const void* q, const void* k, const void* v, const int32_t* key_mask, int32_t* sched,
                 void* o, float* lse, int B, int nh, int S, int dh, esm_stream_t stream);
/* dO [T, nh*dh]; outputs dq (fp32 accum, zeroed by callee), dk, dv [B,nh,S,dh]; delta workspace [2,B,nh,S] fp32.
 * o == NULL (bf16): delta[0:B*nh*S] already holds Delta = rowsum(dO o O) per (b, h, s) -- e.g. accumulated by the
 * ESM_EPI_DELTA epilogue of the GEMM that produced dO -- and the separate Delta pass is skipped. */
int esm_attn_bwd(int dtype, const void* q, const void* k, const void* v, const void* o, const void* dout,
                 const float* lse, const int32_t* key_mask, int32_t* sched, float* delta, float* dq, void* dk,
                 void* dv, int B, int nh, int S, int dh, esm_stream_t stream);

/* Fused backward for the ESM layer (bf16, S % 4 == 0): writes dqkv[T, 3H] = [dq, dk, dv] with RoPEᵀ (and
 * q_scale on dq) applied -- the layout the QKV dgrad / wgrad GEMMs consume -- and col_sum[3H] += the q/k/v
 * bias gradients.  dq_ws: fp32 [T, H] workspace (zeroed by callee); delta: [2, B, nh, S] fp32 workspace
 * (o == NULL: precomputed Delta, as for esm_attn_bwd). */
int esm_attn_bwd_qkv(const void* q, const void* k, const void* v, const void* o, const void* dout,
                     const float* lse, const int32_t* key_mask, int32_t* sched, float* delta, float* dq_ws, void* dqkv,
                     float* col_sum, const float* cos_t, const float* sin_t, float q_scale, int B, int nh, int S,
                     int dh, esm_stream_t stream);

/* Attention-probability dropout (HF EsmSelfAttention: context = dropout(softmax(S)) @ V, HF:modeling_esm.py:
 * 257-282, attention_probs_dropout_prob): the same three calls with an esm_dropout (NULL or threshold 0 = off).
 * keep(b, h, q, k) is the esm_dropout bit of row (b*nh + h)*S + q, column k; the softmax normaliser keeps every
 * probability, P.V uses keep * P / (1 - p); the backward regenerates the mask (dV = (Z o P)^T dO,
 * dS = P o (Z o dP - Delta)); bf16 (tcgen05) and fp32 (parity) kernels. */
int esm_attn_fwd_dropout(int dtype, const void* q, const void* k, const void* v, const int32_t* key_mask,
                         int32_t* sched, void* o, float* lse, int B, int nh, int S, int dh, const esm_dropout* drop,
                         esm_stream_t stream);
int esm_attn_bwd_dropout(int dtype, const void* q, const void* k, const void* v, const void* o, const void* dout,
                         const float* lse, const int32_t* key_mask, int32_t* sched, float* delta, float* dq, void* dk,
                         void* dv, int B, int nh, int S, int dh, const esm_dropout* drop, esm_stream_t stream);
int esm_attn_bwd_qkv_dropout(const void* q, const void* k, const void* v, const void* o, const void* dout,
                             const float* lse, const int32_t* key_mask, int32_t* sched, float* delta, float* dq_ws,
                             void* dqkv, float* col_sum, const float* cos_t, const float* sin_t, float q_scale, int B,
                             int nh, int S, int dh, const esm_dropout* drop, esm_stream_t stream);

/* ---------------- LM head decoder + masked cross-entropy (HF:modeling_esm.py:777-815) ---------------- */
/* logits = n·Eᵀ + bias for labelled rows; loss_sum += Σ nll * inv_denom[0]; dlogits -> dn (= dlogits·E),
 * dE += dlogitsᵀ·n, dbias += Σ dlogits.  Unlabelled rows get dn = 0. */
int esm_lmhead_xent(int dtype, const void* n, const void* E, const float* bias, const int32_t* labels,
                    const float* inv_denom, float* loss_sum, float* dlogits_ws, void* dn, float* dE, float* dbias,
                    int T, int H, int V, esm_stream_t stream);
/* Large-vocabulary head (V > 40, Geneformer V = 25426): the decoder runs only on labelled rows.
 * esm_label_compact: idx[0..cap) = ascending indices of rows with labels >= 0 (then -1), lab = their labels
 * (then -100), *count = total labelled rows (may exceed cap: the caller sizes cap, rows past cap are dropped). */
int esm_label_compact(const int32_t* labels, int64_t T, int32_t* idx, int32_t* lab, int32_t* count, int cap,
                      esm_stream_t stream);
/* dst[i,:] = src[idx[i],:] (0 where idx[i] < 0); H % 8 == 0. */
int esm_gather_rows(int dtype, const void* src, const int32_t* idx, void* dst, int cap, int H, esm_stream_t stream);
/* dst[T,H] = 0; dst[idx[i],:] = src[i,:] for idx[i] >= 0. */
int esm_scatter_rows(int dtype, const void* src, const int32_t* idx, void* dst, int cap, int H, int64_t T,
                     esm_stream_t stream);
/* Per row r < rows with lab[r] >= 0: loss_sum += (logsumexp(x[r,:V]) - x[r,lab]) * inv_denom[0];
 * x[r,:] <- (softmax - onehot) * inv_denom[0] in place (columns V..ld zeroed; rows with lab < 0 zeroed). */
int esm_xent_rows(int dtype, void* logits, const int32_t* lab, int rows, int V, int64_t ld, const float* inv_denom,
                  float* loss_sum, esm_stream_t stream);
/* out[c] += sum_r x[r,c], c < V (fp32 accumulate) -- the decoder-bias gradient. */
int esm_colsum_rows(int dtype, const void* x, int rows, int V, int64_t ld, float* out, esm_stream_t stream);
/* inv_denom[0] = 1 / max(1, n_labels[0]) (fp32) -- the loss normaliser, device-side (graph-safe). */
int esm_inv_count(const int32_t* n_labels, float* inv_denom, esm_stream_t stream);

/* ---------------- optimizer ---------------- */
/* Fused multi-tensor AdamW over one flat fp32 buffer (torch.optim.AdamW semantics, decoupled decay).
 * hyper (device fp32[8]): {lr, beta1, beta2, eps, weight_decay, step, grad_scale, unused}.
 * decay_chunk[i] (uint8) = 1 if elements [i*256, (i+1)*256) are weight-decayed.  p16 = bf16 shadow (or NULL). */
int esm_adamw(float* p, const float* g, float* m, float* v, void* p16, const uint8_t* decay_chunk, int64_t n,
              const float* hyper, esm_stream_t stream);
/* Same update with bf16 gradients g (data-parallel buckets reduced in bf16). */
int esm_adamw_bf16g(float* p, const void* g, float* m, float* v, void* p16, const uint8_t* decay_chunk, int64_t n,
                    const float* hyper, esm_stream_t stream);
/* fp32 -> bf16 copy (shadow refresh, bf16 gradient buckets); src 16-byte, dst 8-byte aligned. */
int esm_cast_f32_bf16(const float* src, void* dst, int64_t n, esm_stream_t stream);
/* bf16 -> fp32 copy. */
int esm_cast_bf16_f32(const void* src, float* dst, int64_t n, esm_stream_t stream);

/* ---------------- data-parallel collectives (NCCL over NVLink / NVSwitch; SURVEY.md §8b "Comms") ----------------
 * NCCL is resolved at run time (the libnccl.so.2 already loaded in the process, i.e. torch.distributed's, else
 * the system one).  Rendezvous: rank 0 calls esm_comm_unique_id and the host layer broadcasts the 128 bytes
 * (torch.distributed); every rank then calls esm_comm_init.  Collectives are in place, SUM, enqueued on
 * `stream` (CUDA-graph capturable).  Errors: ESM_ENCCL_BASE + ncclResult_t. */
#define ESM_COMM_ID_BYTES 128
typedef struct esm_comm* esm_comm_t;
int esm_comm_version(void); /* NCCL version code, 0 if NCCL cannot be loaded */
int esm_comm_unique_id(uint8_t* out /* ESM_COMM_ID_BYTES */);
int esm_comm_init(const uint8_t* id, int rank, int world, esm_comm_t* out);
int esm_comm_destroy(esm_comm_t comm);
/* buf[0..count) = sum over ranks (ESM_F32 / ESM_BF16 / ESM_I32) -- the gradient-bucket all-reduce. */
int esm_comm_allreduce(esm_comm_t comm, void* buf, int64_t count, int dtype, esm_stream_t stream);
/* count % world == 0; slice r = buf[r*count/world, (r+1)*count/world) of rank r receives the sum of that slice. */
int esm_comm_reduce_scatter(esm_comm_t comm, void* buf, int64_t count, int dtype, esm_stream_t stream);
/* count % world == 0; every rank receives every rank's slice r of buf (the sharded-optimizer parameter gather). */
int esm_comm_allgather(esm_comm_t comm, void* buf, int64_t count, int dtype, esm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* ESM2_B200_H */
